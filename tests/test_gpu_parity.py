"""GPU parity: the B200 engine against the oracle, through the C ABI.

Bar: bit-exact lists -- same indices, same distance bits -- as the reference's
brute_force_knn (oracle: the C restatement, pinned in test_oracle_pin.py, and
the golden fixtures made by the compiled reference).  Every arithmetic policy
must meet it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

from tests.helpers import assert_lists_bit_equal, golden_input

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
ARITHS = ["exact", "tensor", "tensor+capture"]


@pytest.fixture(autouse=True)
def _capture_mode(request, monkeypatch):
    """'tensor+capture' runs the TENSOR policy with every row forced through
    the second, band-capture pass (KNN_B200_FORCE_CAPTURE)."""
    arith = request.node.callspec.params.get("arith") if hasattr(request.node, "callspec") else None
    if arith == "tensor+capture":
        monkeypatch.setenv("KNN_B200_FORCE_CAPTURE", "1")
    else:
        monkeypatch.delenv("KNN_B200_FORCE_CAPTURE", raising=False)


@pytest.fixture(scope="module")
def ctx():
    from paper_0906_0231_b200 import Context
    c = Context(0)
    yield c
    c.close()


def metric_obj(name):
    from paper_0906_0231_b200 import distance_by_name
    return distance_by_name(name)


def arith_id(name):
    from paper_0906_0231_b200 import _lib
    return _lib.ARITH_NAMES[name.split("+")[0]]


@pytest.mark.parametrize("arith", ARITHS)
def test_golden_fixtures(ctx, golden, c_oracle, arith):
    z, meta = golden
    for case in meta:
        x = golden_input(c_oracle.generate, case)
        idx, dist, st = ctx.solve(x, case["k"], metric_obj(case["metric"]), arith_id(arith))
        assert_lists_bit_equal(idx, dist, z[case["name"] + "__index"],
                               z[case["name"] + "__dist_bits"].view(np.float32), f"{case['name']} [{arith}]")
        assert st["pair_evaluations"] == case["pairs"]


@pytest.mark.parametrize("arith", ARITHS)
def test_random_instances_vs_oracle(ctx, c_oracle, arith):
    """The acceptance sampler's shape mix (acceptance.cpp:66-96): n in
    [10, 2000], d <= 128, k <= 200, both built-in metrics, plus cosine."""
    rng = np.random.default_rng(0xACCE97ED)
    from oracle import normalize_rows
    for trial in range(36):
        if trial < 24:
            n, dmax = int(rng.integers(10, 311)), 48
        elif trial < 32:
            n, dmax = int(rng.integers(311, 1001)), 64
        else:
            n, dmax = int(rng.integers(1500, 2001)), 128
        d = int(rng.integers(1, dmax + 1))
        k = int(rng.integers(1, min(200, n - 1) + 1))
        m = ("hellinger", "sqeuclidean", "cosine")[trial % 3]
        x = c_oracle.generate(n, d, int(rng.integers(0, 2**63)))
        if m == "cosine":
            x = normalize_rows(x)
        ri, rd, _ = c_oracle.brute_force(x, k, m)
        idx, dist, _ = ctx.solve(x, k, metric_obj(m), arith_id(arith))
        assert_lists_bit_equal(idx, dist, ri, rd, f"trial {trial} n={n} d={d} k={k} {m} [{arith}]")


@pytest.mark.parametrize("arith", ARITHS)
def test_edge_shapes(ctx, c_oracle, arith):
    cases = [
        (np.array([[1, 0], [0, 1]], np.float32), 1, "hellinger"),          # test_oracle.cpp:45-53
        (np.array([[0], [1], [2], [4], [8]], np.float32), 2, "sqeuclidean"),  # :55-66
        (np.array([[0, 1], [1, 0], [0.25, 0.25]], np.float32), 2, "hellinger"),  # test_engine.cpp:30-41
        (c_oracle.generate(12, 4, 5), 500, "hellinger"),                    # k > n-1
        (c_oracle.generate(2, 1, 3), 1, "sqeuclidean"),                     # n = 2, d = 1
        (np.zeros((70, 3), np.float32), 5, "sqeuclidean"),                  # all distances tie at 0
        (np.floor(c_oracle.generate(300, 2, 4) * 3), 40, "sqeuclidean"),    # heavy ties
        (c_oracle.generate(129, 1000, 6), 7, "sqeuclidean"),                # d not a chunk multiple
        (c_oracle.generate(257, 31, 6), 256, "hellinger"),                  # klist = 256 (max)
        (-c_oracle.generate(100, 9, 2), 3, "sqeuclidean"),                  # negative coordinates
        # subnormal terms and sums (the packed FADD2/FMUL2 fold terms must not flush them)
        (c_oracle.generate(200, 16, 7) * np.float32(1e-19), 5, "sqeuclidean"),
        (c_oracle.generate(150, 40, 8) * np.float32(3e-20), 9, "sqeuclidean"),
    ]
    for x, k, m in cases:
        x = np.ascontiguousarray(x, np.float32)
        ri, rd, _ = c_oracle.brute_force(x, k, m)
        idx, dist, _ = ctx.solve(x, k, metric_obj(m), arith_id(arith))
        assert_lists_bit_equal(idx, dist, ri, rd, f"shape {x.shape} k={k} {m} [{arith}]")


def test_device_validation_errors(ctx):
    from paper_0906_0231_b200 import EngineError, ValidationError
    x = np.ones((5, 3), np.float32)
    x[3, 2] = np.inf
    with pytest.raises(ValidationError, match="non-finite coordinate 2 in vector 3"):
        ctx.solve(x, 2, metric_obj("sqeuclidean"))
    x = np.ones((5, 3), np.float32)
    x[1, 0] = -0.5
    x[4, 1] = -2.0
    with pytest.raises(ValidationError, match="coordinate 0 of vector 1 .* outside the domain of hellinger"):
        ctx.solve(x, 2, metric_obj("hellinger"))
    idx, _, _ = ctx.solve(x, 2, metric_obj("sqeuclidean"))  # no domain for sqeuclidean
    assert idx.shape == (5, 2)


def test_python_mirror_solve_knn_lanes(c_oracle):
    """solve_knn (the Python mirror) with n_lanes > devices still equals the
    oracle bit for bit (engine.hpp:33-36)."""
    from paper_0906_0231_b200 import Dataset, EngineOptions, hellinger, solve_knn
    x = c_oracle.generate(337, 19, 777)
    ri, rd, _ = c_oracle.brute_force(x, 25, "hellinger")
    for lanes in (1, 2, 7):
        r = solve_knn(Dataset.from_array(x), hellinger(), EngineOptions(k=25, n_lanes=lanes, gsize=64, bsize=16))
        assert_lists_bit_equal(r.index, r.distance, ri, rd, f"lanes={lanes}")
        assert r.pair_evaluations == 337 * 336 // 2
        assert r.select_stats.offered == 2 * r.pair_evaluations
        assert r.lists[0].query == 0 and len(r.lists[0].neighbors) == 25


def test_row_shards_device_api(ctx, c_oracle):
    """Query-row shards through the device API concatenate to the full answer
    (the multi-GPU decomposition)."""
    import torch
    from paper_0906_0231_b200 import solve_rows_torch, squared_euclidean
    x = c_oracle.generate(1000, 40, 13)
    ri, rd, _ = c_oracle.brute_force(x, 9, "sqeuclidean")
    xt = torch.from_numpy(x).cuda()
    parts = []
    bounds = [0, 1, 333, 334, 999, 1000]
    for a, b in zip(bounds[:-1], bounds[1:]):
        i, dd, _ = solve_rows_torch(ctx, xt, 9, squared_euclidean(), a, b)
        parts.append((i.cpu().numpy().view(np.uint32), dd.cpu().numpy()))
    idx = np.concatenate([p[0] for p in parts])
    dist = np.concatenate([p[1] for p in parts])
    assert_lists_bit_equal(idx, dist, ri, rd, "shards")


@pytest.mark.parametrize("arith", ARITHS)
def test_c1_sampled_rows(ctx, c_oracle, arith):
    """Config C1 (n=16384, d=64, k=10, Euclidean, seed 42) in full on the GPU,
    checked on 1024 sampled rows by the exact sampled-row oracle."""
    x = c_oracle.generate(16384, 64, 42)
    idx, dist, st = ctx.solve(x, 10, metric_obj("sqeuclidean"), arith_id(arith))
    rows = np.random.default_rng(1).choice(16384, 1024, replace=False).astype(np.uint32)
    ri, rd = c_oracle.rows_topk(x, 10, "sqeuclidean", rows)
    assert_lists_bit_equal(idx[rows], dist[rows], ri, rd, f"C1 sampled rows [{arith}]")
    assert st["pair_evaluations"] == 16384 * 16383 // 2


def _run_binary(path: Path, args, arith: str, timeout=900):
    if not path.exists():
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    env = dict(os.environ, KNN_B200_ARITH=arith.split("+")[0])
    if arith.endswith("+capture"):
        env["KNN_B200_FORCE_CAPTURE"] = "1"
    p = subprocess.run([str(path), *args], capture_output=True, text=True, timeout=timeout, env=env)
    return p


@pytest.mark.parametrize("arith", ARITHS)
def test_reference_engine_tests_on_dropin(arith):
    """test_engine.cpp's cases, linked against the unmodified reference
    library with engine.cpp replaced by the B200 drop-in."""
    p = _run_binary(ROOT / "build" / "test_engine_b200", [], arith)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout


@pytest.mark.parametrize("arith", ARITHS)
def test_reference_acceptance_gate_on_dropin(arith):
    """The reference's own acceptance.cpp, criteria 1,2,3,6,7 (4 measures CPU
    lane scaling, 5 needs the CLI), with solve_knn = the B200 drop-in."""
    p = _run_binary(ROOT / "oracle" / "_ref" / "acceptance_b200", ["--skip", "4", "--skip", "5"], arith)
    assert p.returncode == 0, p.stdout + p.stderr
    assert p.stdout.count("PASS") == 5, p.stdout


@pytest.mark.parametrize("arith", ["tensor", "tensor+capture", "tensor+rect"])
def test_full_size_c2_sampled_rows(ctx, c_oracle, arith, monkeypatch):
    """Config C2 (n=1M, d=256, k=10, Euclidean, seed 1) at full size on the
    GPU (inputs from the device generator, bit-identical to
    generate_dataset), checked on 96 sampled rows by the exact oracle."""
    import torch
    from paper_0906_0231_b200 import euclidean, generate_torch, solve_rows_torch
    if arith == "tensor+rect":  # the rectangular (both-direction) sweep instead of the triangle
        monkeypatch.setenv("KNN_B200_TRI", "0")
    n, d, k = 1_000_000, 256, 10
    x = generate_torch(ctx, n, d, 1)
    idx, dist, st = solve_rows_torch(ctx, x, k, euclidean(), 0, n, arith_id(arith), want_stats=True)
    xh = x.cpu().numpy()
    assert np.array_equal(xh[:3], c_oracle.generate(3, d, 1))  # device generator == SplitMix64 stream
    rows = np.random.default_rng(7).choice(n, 96, replace=False).astype(np.uint32)
    ri, rd = c_oracle.rows_topk(xh, k, "sqeuclidean", rows)
    gi = idx.cpu().numpy().view(np.uint32)[rows]
    gd = dist.cpu().numpy()[rows]
    assert_lists_bit_equal(gi, gd, ri, np.sqrt(rd), f"C2 sampled [{arith}]")
    assert st["arith_used"] == 2
    if arith != "tensor+capture":
        # ~0.1-0.3% of rows lack a completeness proof and take the band-capture
        # pass (still bit-exact); more would mean a broken bound
        assert st["fallback_rows"] < n // 100


@pytest.mark.parametrize("n,d,k,m", [(400000, 48, 7, "sqeuclidean"), (393216, 32, 1, "hellinger"),
                                     (450001, 100, 10, "euclidean"), (420000, 33, 3, "sqeuclidean")])
def test_triangle_sweep_sampled_rows(ctx, c_oracle, n, d, k, m):
    """The triangle sweep (each unordered pair once; the default from n =
    393216 with k <= 11, d <= 256) on sampled rows against the exact oracle,
    including the first and last rows of the norm order's extremes."""
    from paper_0906_0231_b200 import generate_torch, solve_rows_torch
    x = generate_torch(ctx, n, d, 77 + n)
    idx, dist, st = solve_rows_torch(ctx, x, k, metric_obj(m), 0, n, arith_id("tensor"), want_stats=True)
    xh = x.cpu().numpy()
    norms = ((xh - xh.mean(0)) ** 2).sum(1)
    rows = np.unique(np.concatenate([np.random.default_rng(n).choice(n, 40, replace=False),
                                     np.argsort(norms)[:4], np.argsort(norms)[-4:], [0, n - 1]])).astype(np.uint32)
    om = "sqeuclidean" if m == "euclidean" else m
    ri, rd = c_oracle.rows_topk(xh, k, om, rows)
    if m == "euclidean":
        rd = np.sqrt(rd)
    assert_lists_bit_equal(idx.cpu().numpy().view(np.uint32)[rows], dist.cpu().numpy()[rows], ri, rd,
                           f"triangle n={n} d={d} k={k} {m}")
    assert st["fallback_rows"] < n // 100


def test_triangle_sample_precision_does_not_change_results(ctx, c_oracle, monkeypatch):
    """The sample pass only sets thresholds: its E4M3 (default) and fp16
    (KNN_B200_TRI_E4M3=0) forms must give the same bits on every row."""
    import torch
    from paper_0906_0231_b200 import generate_torch, solve_rows_torch
    n, d, k = 400000, 200, 10
    x = generate_torch(ctx, n, d, 31)
    idx8, dist8, _ = solve_rows_torch(ctx, x, k, metric_obj("euclidean"), 0, n, arith_id("tensor"))
    monkeypatch.setenv("KNN_B200_TRI_E4M3", "0")
    idx16, dist16, _ = solve_rows_torch(ctx, x, k, metric_obj("euclidean"), 0, n, arith_id("tensor"))
    assert (idx8 == idx16).all().item()
    assert (dist8.view(torch.int32) == dist16.view(torch.int32)).all().item()
    rows = np.random.default_rng(2).choice(n, 16, replace=False).astype(np.uint32)
    ri, rd = c_oracle.rows_topk(x.cpu().numpy(), k, "sqeuclidean", rows)
    assert_lists_bit_equal(idx8.cpu().numpy().view(np.uint32)[rows], dist8.cpu().numpy()[rows], ri, np.sqrt(rd),
                           "triangle e4m3 sample")


def test_triangle_log_overflow_falls_back(ctx, c_oracle, monkeypatch):
    """A triangle sweep whose column-side append logs overflow must redo the
    call with the rectangular sweep: same bits (KNN_B200_TRI_LOGCAP forces it)."""
    from paper_0906_0231_b200 import generate_torch, solve_rows_torch
    n, d, k = 400000, 40, 5
    x = generate_torch(ctx, n, d, 5)
    monkeypatch.setenv("KNN_B200_TRI_LOGCAP", "64")
    idx, dist, _ = solve_rows_torch(ctx, x, k, metric_obj("sqeuclidean"), 0, n, arith_id("tensor"))
    rows = np.random.default_rng(3).choice(n, 32, replace=False).astype(np.uint32)
    ri, rd = c_oracle.rows_topk(x.cpu().numpy(), k, "sqeuclidean", rows)
    assert_lists_bit_equal(idx.cpu().numpy().view(np.uint32)[rows], dist.cpu().numpy()[rows], ri, rd,
                           "triangle overflow fallback")


def test_triangle_heavy_ties_sampled_rows(ctx, c_oracle):
    """Triangle-size input with massive ties (256 distinct points): the
    column side overflows and the call falls back; ties resolve by index."""
    import torch
    from paper_0906_0231_b200 import solve_rows_torch
    n, d, k = 400000, 8, 10
    xh = np.floor(c_oracle.generate(n, d, 9) * 2).astype(np.float32)
    x = torch.from_numpy(xh).cuda()
    idx, dist, _ = solve_rows_torch(ctx, x, k, metric_obj("sqeuclidean"), 0, n, arith_id("tensor"))
    rows = np.random.default_rng(4).choice(n, 24, replace=False).astype(np.uint32)
    ri, rd = c_oracle.rows_topk(xh, k, "sqeuclidean", rows)
    assert_lists_bit_equal(idx.cpu().numpy().view(np.uint32)[rows], dist.cpu().numpy()[rows], ri, rd,
                           "triangle heavy ties")


@pytest.mark.gpu
def test_staged_host_copies_match_device_path(ctx):
    """Pageable host buffers of 16 MB and more go through the pinned staging
    lanes (api.cu host_copy) in both directions: the results must equal the
    device-resident path's bit for bit, for pageable and pinned inputs."""
    import torch
    from paper_0906_0231_b200 import generate_torch, solve_rows_torch
    n, d, k = 70000, 64, 64  # 17.9 MB in, 17.9 MB per output array
    xt = generate_torch(ctx, n, d, 5)
    di, dd, _ = solve_rows_torch(ctx, xt, k, metric_obj("euclidean"), 0, n)
    di = di.cpu().numpy().view(np.uint32)
    dd = dd.cpu().numpy()
    x_pageable = xt.cpu().numpy()
    xp = xt.cpu().pin_memory()
    x_pinned = xp.numpy()
    for x in (x_pageable, x_pinned):
        idx, dist, st = ctx.solve(x, k, metric_obj("euclidean"))
        assert np.array_equal(idx, di)
        assert np.array_equal(dist.view(np.uint32), dd.view(np.uint32))
        assert st["h2d_ms"] > 0 and st["d2h_ms"] > 0


def test_solve_into_caller_owned_pinned_outputs(ctx, c_oracle):
    """Context.solve(out=...) writes into caller-owned (here pinned) arrays,
    the ABI's direct-DMA path, with the same bits as its own outputs."""
    import torch
    from paper_0906_0231_b200 import ConfigError
    x = c_oracle.generate(3000, 40, 21)
    m = metric_obj("sqeuclidean")
    idx_pin = torch.empty((3000, 10), dtype=torch.int32, pin_memory=True)
    dist_pin = torch.empty((3000, 10), dtype=torch.float32, pin_memory=True)
    out = (idx_pin.numpy().view(np.uint32), dist_pin.numpy())
    i1, d1, _ = ctx.solve(x, 10, m, arith_id("tensor"), out=out)
    assert i1 is out[0] and d1 is out[1]
    i0, d0, _ = ctx.solve(x, 10, m, arith_id("tensor"))
    assert np.array_equal(i0, i1) and np.array_equal(d0.view(np.uint32), d1.view(np.uint32))
    with pytest.raises(ConfigError):
        ctx.solve(x, 10, m, arith_id("tensor"), out=(out[0][:, :5], out[1]))


@pytest.mark.parametrize("n,d,k,m", [(5000, 40, 1000, "sqeuclidean"), (1300, 17, 5000, "hellinger"),
                                     (3000, 64, 300, "cosine"), (2500, 33, 257, "euclidean")])
def test_long_lists_beyond_256(ctx, c_oracle, n, d, k, m):
    """min(k, n-1) > 256: the reference keeps any k (heap.cpp:66-70); here the
    sort-based EXACT path (exact_bigk.cu) -- same bits as brute_force_knn."""
    from oracle import normalize_rows
    x = c_oracle.generate(n, d, n + k)
    if m == "cosine":
        x = normalize_rows(x)
    om = "sqeuclidean" if m == "euclidean" else m
    ri, rd, _ = c_oracle.brute_force(x, k, om)
    if m == "euclidean":
        rd = np.sqrt(rd)
    for arith in ("auto", "tensor"):
        idx, dist, st = ctx.solve(x, k, metric_obj(m), arith_id(arith))
        assert_lists_bit_equal(idx, dist, ri, rd, f"long lists n={n} k={k} {m} [{arith}]")
        assert st["arith_used"] == 1


def test_long_lists_heavy_ties_and_f64(ctx, c_oracle):
    """Tie-heavy data (16 distinct points) with k = 400: ties break by index;
    and the KNN_DOUBLE_ACCUM build's long lists (double keys, stable sort)."""
    x = np.floor(c_oracle.generate(2000, 2, 12) * 4).astype(np.float32)
    ri, rd, _ = c_oracle.brute_force(x, 400, "sqeuclidean")
    idx, dist, _ = ctx.solve(x, 400, metric_obj("sqeuclidean"))
    assert_lists_bit_equal(idx, dist, ri, rd, "long lists, heavy ties")
    for xx, k, m in ((x, 400, "sqeuclidean"), (c_oracle.generate(1500, 30, 5), 600, "hellinger")):
        ri, rd = c_oracle.brute_force_f64(xx, k, m)
        idx, dist, _ = ctx.solve_f64(xx, k, metric_obj(m))
        assert np.array_equal(idx, ri), f"f64 long lists {m}: indices"
        assert np.array_equal(dist.view(np.uint64), rd.view(np.uint64)), f"f64 long lists {m}: distance bits"


def test_device_api_empty_shard_and_stream_switch(ctx, c_oracle):
    """An empty row range is a valid (empty) shard; consecutive calls on
    different streams reuse the workspace safely (the context orders each
    call after the previous one)."""
    import torch
    from paper_0906_0231_b200 import ConfigError, solve_rows_torch, squared_euclidean
    x = c_oracle.generate(6000, 24, 3)
    ri, rd, _ = c_oracle.brute_force(x, 8, "sqeuclidean")
    xt = torch.from_numpy(x).cuda()
    i0, d0, _ = solve_rows_torch(ctx, xt, 8, squared_euclidean(), 300, 300)
    assert i0.shape == (0, 8)
    outs = []
    for rep in range(3):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            outs.append(solve_rows_torch(ctx, xt, 8, squared_euclidean(), 0, 6000, arith_id("tensor")))
    torch.cuda.synchronize()
    for i, dd, _ in outs:
        assert_lists_bit_equal(i.cpu().numpy().view(np.uint32), dd.cpu().numpy(), ri, rd, "stream switch")
    bad = torch.empty((10, 8), dtype=torch.int32, device="cuda")
    with pytest.raises(ConfigError):
        solve_rows_torch(ctx, xt, 8, squared_euclidean(), 0, 6000, out=(bad, bad.float()))


@pytest.mark.parametrize("n,d,k,m", [(20000, 48, 30, "sqeuclidean"), (9000, 300, 100, "euclidean"),
                                     (12000, 64, 20, "cosine"), (5000, 20, 64, "hellinger"),
                                     (3000, 1024, 11, "sqeuclidean"), (6000, 37, 24, "sqeuclidean")])
def test_threshold_triangle_forced_all_rows(ctx, c_oracle, monkeypatch, n, d, k, m):
    """The threshold triangle (k > 10: each pair once, both endpoints against
    fixed thresholds, capture rescore; KNN_B200_TCAP=force below its size
    gate), every row against the oracle -- resident (d <= 256) and streamed
    query rows (d > 256), cosine without the norm order; the band rescore's
    cp.async ring with whole and partial 32-coordinate chunks (d % 4 == 0)
    and its register-staged fold (d = 37)."""
    import torch
    from oracle import normalize_rows
    from paper_0906_0231_b200 import solve_rows_torch
    monkeypatch.setenv("KNN_B200_TCAP", "force")
    xh = c_oracle.generate(n, d, n + k)
    if m == "cosine":
        xh = normalize_rows(xh)
    om = "sqeuclidean" if m == "euclidean" else m
    ri, rd = c_oracle.rows_topk(xh, k, om, np.arange(n, dtype=np.uint32))
    if m == "euclidean":
        rd = np.sqrt(rd)
    x = torch.from_numpy(np.ascontiguousarray(xh)).cuda()
    idx, dist, st = solve_rows_torch(ctx, x, k, metric_obj(m), 0, n, arith_id("tensor"), want_stats=True)
    assert_lists_bit_equal(idx.cpu().numpy().view(np.uint32), dist.cpu().numpy(), ri, rd,
                           f"threshold triangle n={n} d={d} k={k} {m}")
    assert st["fallback_rows"] < n  # most rows proven by the first pass


@pytest.mark.parametrize("ew", ["8", "16"])
def test_threshold_triangle_epilogue_widths(ctx, c_oracle, monkeypatch, ew):
    """The threshold triangle with 8 and 16 epilogue warps (KNN_B200_TCAP_EW;
    16 is the default for resident query rows): the same bits."""
    import torch
    from paper_0906_0231_b200 import solve_rows_torch
    monkeypatch.setenv("KNN_B200_TCAP", "force")
    monkeypatch.setenv("KNN_B200_TCAP_EW", ew)
    n, d, k = 12000, 96, 24
    xh = c_oracle.generate(n, d, 91)
    ri, rd = c_oracle.rows_topk(xh, k, "sqeuclidean", np.arange(n, dtype=np.uint32))
    idx, dist, _ = solve_rows_torch(ctx, torch.from_numpy(xh).cuda(), k, metric_obj("sqeuclidean"), 0, n,
                                    arith_id("tensor"), want_stats=True)
    assert_lists_bit_equal(idx.cpu().numpy().view(np.uint32), dist.cpu().numpy(), ri, rd, f"TCAP_EW={ew}")


@pytest.mark.parametrize("dyn", ["0", "1"])
def test_threshold_triangle_walks_streamed_rows(ctx, c_oracle, monkeypatch, dyn):
    """Streamed query rows (d > 256) under the static walk and the unit
    queue (KNN_B200_TRI_DYN; the queue is the default): the same bits."""
    import torch
    from paper_0906_0231_b200 import solve_rows_torch
    monkeypatch.setenv("KNN_B200_TCAP", "force")
    monkeypatch.setenv("KNN_B200_TRI_DYN", dyn)
    n, d, k = 7000, 320, 40
    xh = c_oracle.generate(n, d, 93)
    ri, rd = c_oracle.rows_topk(xh, k, "sqeuclidean", np.arange(n, dtype=np.uint32))
    idx, dist, _ = solve_rows_torch(ctx, torch.from_numpy(xh).cuda(), k, metric_obj("sqeuclidean"), 0, n,
                                    arith_id("tensor"), want_stats=True)
    assert_lists_bit_equal(idx.cpu().numpy().view(np.uint32), dist.cpu().numpy(), ri, rd, f"TRI_DYN={dyn}")


def test_threshold_triangle_retry_and_overflow_paths(ctx, c_oracle, monkeypatch):
    """Thresholds forced far too low (every row retried through the second
    capture pass) and a pool forced to overflow (the rectangular sweep redoes
    the call): the same bits either way."""
    import torch
    from paper_0906_0231_b200 import solve_rows_torch
    monkeypatch.setenv("KNN_B200_TCAP", "force")
    n, d, k = 8000, 40, 25
    xh = c_oracle.generate(n, d, 77)
    ri, rd = c_oracle.rows_topk(xh, k, "sqeuclidean", np.arange(n, dtype=np.uint32))
    x = torch.from_numpy(xh).cuda()
    for env, val in (("KNN_B200_TCAP_RANK", "1"), ("KNN_B200_TRI_LOGCAP", "4096")):
        monkeypatch.setenv(env, val)
        idx, dist, st = solve_rows_torch(ctx, x, k, metric_obj("sqeuclidean"), 0, n, arith_id("tensor"),
                                         want_stats=True)
        assert_lists_bit_equal(idx.cpu().numpy().view(np.uint32), dist.cpu().numpy(), ri, rd, f"{env}={val}")
        monkeypatch.delenv(env)


@pytest.mark.parametrize("m", ["manhattan", "root_of_squares"])
def test_custom_functor_folds(ctx, c_oracle, m):
    """The reference suite's own custom functors (test_distance.cpp:134-145
    manhattan, :166-178 sqeuclidean finalized by sqrt) run on the device
    (EXACT, whatever the policy asked), bit for bit, float and double builds,
    short and long lists, tie-heavy data."""
    cases = [(c_oracle.generate(1500, 24, 3), 12), (c_oracle.generate(700, 5, 4), 300),
             (np.floor(c_oracle.generate(600, 3, 5) * 7) * np.float32(0.37), 30)]
    for x, k in cases:
        x = np.ascontiguousarray(x, np.float32)
        ri, rd, _ = c_oracle.brute_force(x, k, m)
        for arith in ("auto", "tensor"):
            idx, dist, st = ctx.solve(x, k, metric_obj(m), arith_id(arith))
            assert_lists_bit_equal(idx, dist, ri, rd, f"{m} n={x.shape[0]} k={k} [{arith}]")
            assert st["arith_used"] == 1
        ri64, rd64 = c_oracle.brute_force_f64(x, k, m)
        i64, d64, _ = ctx.solve_f64(x, k, metric_obj(m))
        assert np.array_equal(i64, ri64) and np.array_equal(d64.view(np.uint64), rd64.view(np.uint64)), f"{m} f64"

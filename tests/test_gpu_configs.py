"""Full-size BASELINE configs and adversarial inputs on the GPU.

Every BASELINE.json config runs at its full size through the device API
(`solve_rows_torch`, the path bench.py times), with inputs from the device
generator (bit-identical to generate_dataset, io.cpp:57-62).  Each is checked
bit for bit against the exact sampled-row oracle (the
reference's fold and heap for a subset of query rows, oracle.cpp:22-32) on
128 random rows plus the extremes of the norm order the sweep sorts by.

The adversarial cases stress the TENSOR policy's fp16 filter and its
completeness proof: clusters with near-duplicates, a wide
dynamic range plus one outlier row, engineered near-ties at the k-th
distance at d = 1024 / k = 100, and all-equal norms.  The bar does not move:
identical indices and distance bits.
"""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import assert_lists_bit_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_0906_0231_b200 import Context
    c = Context(0)
    yield c
    c.close()


def _metric(name):
    from paper_0906_0231_b200 import distance_by_name
    return distance_by_name(name)


def _norm_extremes(x, count=4):
    """Rows at both ends of the order the sweep sorts its columns by
    (||x - mu||^2, mu = column mean), computed on the device in chunks."""
    import torch
    mu = x.double().mean(0) if x.shape[0] * x.shape[1] <= (1 << 28) else _chunked_mean(x)
    mu = mu.float()
    norms = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    step = 1 << 20
    for a in range(0, x.shape[0], step):
        norms[a:a + step] = ((x[a:a + step] - mu) ** 2).sum(1)
    order = torch.argsort(norms)
    return torch.cat([order[:count], order[-count:]]).cpu().numpy()


def _chunked_mean(x):
    import torch
    acc = torch.zeros(x.shape[1], dtype=torch.float64, device=x.device)
    step = 1 << 20
    for a in range(0, x.shape[0], step):
        acc += x[a:a + step].double().sum(0)
    return acc / x.shape[0]


def _check_rows(c_oracle, x_host, idx, dist, rows, k, metric, what):
    om = "sqeuclidean" if metric == "euclidean" else metric
    ri, rd = c_oracle.rows_topk(x_host, k, om, rows)
    if metric == "euclidean":
        rd = np.sqrt(rd)
    gi = idx[rows].cpu().numpy().view(np.uint32)
    gd = dist[rows].cpu().numpy()
    assert_lists_bit_equal(gi, gd, ri, rd, what)


def _run_config(ctx, c_oracle, n, d, k, metric, seed, nrows=128, normalize=False):
    import torch
    from paper_0906_0231_b200 import _lib, generate_torch, solve_rows_torch
    x = generate_torch(ctx, n, d, seed)
    if normalize:  # cosine rows L2-normalised in double, stored f32
        from oracle import normalize_rows
        x = torch.from_numpy(normalize_rows(x.cpu().numpy())).to(x.device)
    idx, dist, st = solve_rows_torch(ctx, x, k, _metric(metric), 0, n, _lib.ARITH_AUTO, want_stats=True)
    torch.cuda.synchronize()
    rows = np.random.default_rng(seed).choice(n, nrows, replace=False)
    extremes = np.array([0, n - 1]) if normalize else _norm_extremes(x)
    rows = np.unique(np.concatenate([rows, extremes])).astype(np.uint32)
    x_host = x.cpu().numpy()
    del x
    torch.cuda.empty_cache()
    _check_rows(c_oracle, x_host, idx, dist, rows, k, metric, f"n={n} d={d} k={k} {metric} seed={seed}")
    print(f"\n[config n={n} d={d} k={k} {metric}] sweep {st['sweep_ms']:.1f} ms, kernels {st['kernel_ms']:.1f} ms, "
          f"capture rows {st['fallback_rows']}, exact rows {st['exact_rows']}, policy {st['arith_used']}")
    return st


def test_c1_all_rows(ctx, c_oracle):
    """C1 (n=16384, d=64, k=10, Euclidean, seed 42): every row."""
    from paper_0906_0231_b200 import _lib
    x = c_oracle.generate(16384, 64, 42)
    idx, dist, st = ctx.solve(x, 10, _metric("euclidean"), _lib.ARITH_AUTO)
    ri, rd = c_oracle.rows_topk(x, 10, "sqeuclidean", np.arange(16384, dtype=np.uint32))
    assert_lists_bit_equal(idx, dist, ri, np.sqrt(rd), "C1 all rows")


def test_c3_full_size(ctx, c_oracle):
    """C3: n=1M, d=1024, k=100, Euclidean, seed 2 (large-d chunking, k=100)."""
    st = _run_config(ctx, c_oracle, 1_000_000, 1024, 100, "euclidean", 2)
    assert st["arith_used"] == 2


def test_c4_full_size(ctx, c_oracle):
    """C4: n=4M, d=128, k=32, cosine on L2-normalised rows, seed 3."""
    st = _run_config(ctx, c_oracle, 4_000_000, 128, 32, "cosine", 3, normalize=True)
    assert st["arith_used"] == 2


def test_c5_full_size_one_gpu(c_oracle):
    """C5: n=16M, d=256, k=10, Euclidean, seed 4 -- the 8-GPU scaling config,
    here whole on one B200 (4.1e9 input elements: 64-bit offsets).  Its own
    context, closed afterwards: the workspace is large."""
    import torch
    from paper_0906_0231_b200 import Context
    c = Context(0)
    try:
        st = _run_config(c, c_oracle, 16_000_000, 256, 10, "euclidean", 4)
    finally:
        c.close()
        torch.cuda.empty_cache()
    assert st["arith_used"] == 2
    assert st["exact_rows"] == 0


def test_device_generator_past_2_32(ctx, c_oracle):
    """The device generator at element and byte offsets past 2^31 and 2^32
    against the oracle's Weyl-jumped stream (rng.hpp:13-23)."""
    import torch
    from paper_0906_0231_b200 import _lib
    from paper_0906_0231_b200.engine import raise_for_status
    count = (1 << 32) + 4096  # 17.2 GB: element indices past 2^32
    x = torch.empty(count, dtype=torch.float32, device="cuda:0")
    stream = torch.cuda.current_stream().cuda_stream
    raise_for_status(_lib.load().knn_b200_generate_device(ctx._h, x.data_ptr(), count, 4, stream))
    torch.cuda.synchronize()
    probes = [0, (1 << 29) - 8, (1 << 30) - 8, (1 << 31) - 8, (1 << 31) + 12345, (1 << 32) - 8,
              16_000_000 * 256 - 64, count - 64]
    for first in probes:
        got = x[first:first + 64].cpu().numpy()
        want = c_oracle.generate_at(4, first, 64)
        assert np.array_equal(got, want), f"generator mismatch at element {first}"
    del x
    torch.cuda.empty_cache()


# --------------------------------------------------------------------------
# adversarial inputs for the fp16 filter's proof


def _solve_and_check(ctx, c_oracle, xh, k, metric, what, nrows=64, extra_rows=()):
    import torch
    from paper_0906_0231_b200 import _lib, solve_rows_torch
    n = xh.shape[0]
    x = torch.from_numpy(np.ascontiguousarray(xh, np.float32)).cuda()
    idx, dist, st = solve_rows_torch(ctx, x, k, _metric(metric), 0, n, _lib.ARITH_TENSOR, want_stats=True)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([np.random.default_rng(n + k).choice(n, nrows, replace=False),
                                     np.asarray(extra_rows, dtype=np.int64), [0, n - 1]])).astype(np.uint32)
    _check_rows(c_oracle, xh, idx, dist, rows, k, metric, what)
    print(f"\n[{what}] capture rows {st['fallback_rows']}, exact rows {st['exact_rows']}")
    return st


def _clusters(n, d, centers, spread, seed):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal((centers, d)).astype(np.float32)
    lab = rng.integers(0, centers, n)
    x = c[lab] + spread * rng.standard_normal((n, d)).astype(np.float32)
    # exact duplicates and 1-ulp near-duplicates of random rows
    src = rng.choice(n, n // 50, replace=False)
    dst = rng.choice(n, n // 50, replace=False)
    x[dst] = x[src]
    near = dst[: dst.size // 2]
    x[near, 0] = np.nextafter(x[near, 0], np.float32(np.inf))
    return np.ascontiguousarray(x, np.float32)


@pytest.mark.parametrize("n,d,k", [(400_000, 64, 10), (50_000, 128, 32), (20_000, 48, 100)])
def test_gaussian_clusters_with_near_duplicates(ctx, c_oracle, n, d, k):
    xh = _clusters(n, d, 1000, 0.05, 11 + k)
    _solve_and_check(ctx, c_oracle, xh, k, "sqeuclidean", f"clusters n={n} d={d} k={k}")


@pytest.mark.parametrize("n,d,k", [(400_000, 32, 10), (60_000, 96, 32)])
def test_wide_dynamic_range_with_outlier(ctx, c_oracle, n, d, k):
    """Row magnitudes spanning 1e-3..1e3 plus one row 1e4 times the largest:
    the proof's dataset-wide maxima widen every row's band."""
    rng = np.random.default_rng(5)
    xh = rng.standard_normal((n, d)).astype(np.float32)
    xh *= (10.0 ** rng.uniform(-3, 3, (n, 1))).astype(np.float32)
    out = int(rng.integers(n))
    xh[out] = 1e7 * np.abs(xh[out]) / np.abs(xh[out]).max()
    small = np.argsort(np.abs(xh).max(1))[:8]
    _solve_and_check(ctx, c_oracle, xh, k, "sqeuclidean", f"dynamic range n={n} d={d} k={k}",
                     extra_rows=[out, *small])


def test_near_ties_at_kth_d1024_k100(ctx, c_oracle):
    """d=1024, k=100: clusters of 150 points c + r(1 + m 2^-22) e_j on random
    axes, so each member's ~149 cluster neighbours are all near-tied and the
    100th/101st distances differ in the last bits."""
    rng = np.random.default_rng(21)
    d, per, ncl = 1024, 150, 200
    n = per * ncl
    c = rng.uniform(0, 1, (ncl, d)).astype(np.float32)
    xh = np.repeat(c, per, axis=0)
    axes = rng.integers(0, d, n)
    r = (0.25 * (1.0 + rng.integers(0, 8, n) * 2.0 ** -22)).astype(np.float32)
    xh[np.arange(n), axes] += r
    xh = np.ascontiguousarray(xh, np.float32)
    _solve_and_check(ctx, c_oracle, xh, 100, "euclidean", "near ties d=1024 k=100")


@pytest.mark.parametrize("n,d,k,metric", [(400_000, 64, 10, "sqeuclidean"), (40_000, 256, 50, "sqeuclidean"),
                                          (100_000, 64, 16, "cosine")])
def test_all_equal_norms(ctx, c_oracle, n, d, k, metric):
    """Every row on the unit sphere: the norm sort orders nothing and the
    chunk bounds rest on the thresholds alone."""
    from oracle import normalize_rows
    rng = np.random.default_rng(n + d)
    xh = normalize_rows(rng.standard_normal((n, d)).astype(np.float32))
    _solve_and_check(ctx, c_oracle, xh, k, metric, f"equal norms n={n} d={d} k={k} {metric}")

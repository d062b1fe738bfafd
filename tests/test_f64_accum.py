"""The reference's KNN_DOUBLE_ACCUM build (include/knn/types.hpp:9-13,
proj/CMakeLists.txt:11): dist_t = double.

CPU: the C restatement's double fold and brute force (oracle/knn_oracle.c,
ko_brute_force_f64) pinned against the reference library compiled with
-DKNN_DOUBLE_ACCUM (oracle/_ref/f64/), and the KAT test_oracle.cpp:55-66 in
double.
GPU (marked): knn_b200_solve_f64 bit-exact against that oracle, and the
reference's own acceptance.cpp / test_engine.cpp cases linked against the
double build of the drop-in.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import REF_F64_CAPI_PATH, ReferenceF64
from tests.test_gpu_parity import _run_binary, ROOT

CASES = [  # n, d, k, metric, seed
    (2, 1, 1, "sqeuclidean", 1),
    (3, 4, 5, "hellinger", 2),
    (17, 5, 3, "cosine", 3),
    (64, 33, 10, "sqeuclidean", 4),
    (130, 7, 40, "hellinger", 5),
    (97, 64, 300, "sqeuclidean", 6),
    (150, 3, 140, "cosine", 7),
]


def _instance(n, d, seed, ties=False):
    rng = np.random.default_rng(seed)
    if ties:  # integer grid: many equal distances, index tie-breaks decide
        return rng.integers(0, 3, size=(n, d)).astype(np.float32)
    return rng.random((n, d), dtype=np.float32)


def _assert_f64_equal(i0, d0, i1, d1, what):
    assert i0.shape == i1.shape, what
    assert np.array_equal(i0, i1), f"{what}: index mismatch"
    assert np.array_equal(d0.view(np.uint64), d1.view(np.uint64)), f"{what}: distance bits differ"


def test_five_points_on_a_line_f64(c_oracle):
    # test_oracle.cpp:55-66 restated in the double build
    x = np.array([[0.0], [1.0], [2.0], [4.0], [8.0]], dtype=np.float32)
    idx, dist = c_oracle.brute_force_f64(x, 2, "sqeuclidean")
    assert idx.tolist() == [[1, 2], [0, 2], [1, 0], [2, 1], [3, 2]]
    assert dist.dtype == np.float64
    assert dist.tolist() == [[1, 4], [1, 1], [1, 4], [4, 9], [16, 36]]


def test_f64_fold_differs_from_f32_fold(c_oracle):
    # the double build must actually accumulate in double: a long fold of
    # small steps loses bits in float that double keeps
    u = np.full(4096, 0.1, dtype=np.float32)
    v = np.zeros(4096, dtype=np.float32)
    f32 = c_oracle.fold("sqeuclidean", u, v)
    f64 = c_oracle.lib.ko_fold_f64(1, u.ctypes.data_as(c_oracle.lib.ko_fold.argtypes[1]),
                                   v.ctypes.data_as(c_oracle.lib.ko_fold.argtypes[2]), 4096)
    t = np.float64(np.float32(0.1))
    assert f64 == pytest.approx(4096 * t * t, rel=1e-12)
    assert float(f32) != f64


@pytest.mark.skipif(not REF_F64_CAPI_PATH.exists(), reason="oracle/_ref/f64 not built")
@pytest.mark.parametrize("case", CASES + [(60, 4, 9, "sqeuclidean", 8, True)])
def test_f64_restatement_matches_compiled_reference(c_oracle, case):
    n, d, k, metric, seed, *ties = case
    x = _instance(n, d, seed, bool(ties))
    ri, rd = ReferenceF64().brute_force(x, k, metric)
    oi, od = c_oracle.brute_force_f64(x, k, metric)
    _assert_f64_equal(oi, od, ri, rd, f"f64 oracle vs reference {case}")


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES + [(60, 4, 9, "sqeuclidean", 8, True), (1000, 96, 256, "hellinger", 9),
                                          (700, 256, 100, "euclidean", 10)])
def test_solve_f64_bit_exact(c_oracle, case):
    from paper_0906_0231_b200 import Context, distance_by_name
    n, d, k, metric, seed, *ties = case
    x = _instance(n, d, seed, bool(ties))
    ctx = Context(0)
    try:
        gi, gd, st = ctx.solve_f64(x, k, distance_by_name(metric))
    finally:
        ctx.close()
    fold = "sqeuclidean" if metric == "euclidean" else metric
    oi, od = c_oracle.brute_force_f64(x, k, fold)
    if metric == "euclidean":
        od = np.sqrt(od)
    assert gd.dtype == np.float64
    _assert_f64_equal(gi, gd, oi, od, f"solve_f64 vs oracle {case}")
    assert st["pair_evaluations"] == n * (n - 1) // 2


def test_f64_rows_topk_equals_brute_force(c_oracle):
    x = _instance(90, 7, 12)
    rows = np.array([0, 5, 44, 89], dtype=np.uint32)
    bi, bd = c_oracle.brute_force_f64(x, 9, "hellinger")
    ri, rd = c_oracle.rows_topk_f64(x, 9, "hellinger", rows)
    _assert_f64_equal(ri, rd, bi[rows], bd[rows], "rows_topk_f64 vs brute_force_f64")


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,k,metric", [(65536, 64, 50, "sqeuclidean"), (40000, 300, 129, "cosine")])
def test_solve_f64_large_sampled_rows(c_oracle, n, d, k, metric):
    """Many column tiles and list merges per CTA: sampled rows against the
    double oracle, bit for bit."""
    from paper_0906_0231_b200 import Context, distance_by_name
    x = _instance(n, d, 13)
    if metric == "cosine":
        x /= np.linalg.norm(x.astype(np.float64), axis=1, keepdims=True).astype(np.float32)
    ctx = Context(0)
    try:
        gi, gd, _ = ctx.solve_f64(x, k, distance_by_name(metric))
    finally:
        ctx.close()
    rows = np.unique(np.concatenate([np.random.default_rng(3).choice(n, 48, replace=False), [0, n - 1]]))
    oi, od = c_oracle.rows_topk_f64(x, k, metric, rows.astype(np.uint32))
    _assert_f64_equal(gi[rows], gd[rows], oi, od, f"solve_f64 sampled rows n={n} d={d} k={k} {metric}")


@pytest.mark.gpu
def test_solve_f64_validation_errors():
    from paper_0906_0231_b200 import Context, ValidationError, ConfigError, distance_by_name
    ctx = Context(0)
    try:
        x = np.ones((4, 3), dtype=np.float32)
        x[2, 1] = -1.0
        with pytest.raises(ValidationError):
            ctx.solve_f64(x, 2, distance_by_name("hellinger"))
        x[2, 1] = np.nan
        with pytest.raises(ValidationError):
            ctx.solve_f64(x, 2, distance_by_name("sqeuclidean"))
        with pytest.raises(ConfigError):
            ctx.solve_f64(np.ones((4, 3), dtype=np.float32), 0, distance_by_name("sqeuclidean"))
    finally:
        ctx.close()


@pytest.mark.gpu
def test_reference_engine_tests_on_dropin_f64():
    p = _run_binary(ROOT / "build" / "test_engine_b200_f64", [], "exact")
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout


@pytest.mark.gpu
def test_reference_acceptance_gate_on_dropin_f64():
    """acceptance.cpp compiled with -DKNN_DOUBLE_ACCUM, criteria 1,2,3,6,7,
    with solve_knn = the double build of the B200 drop-in."""
    p = _run_binary(ROOT / "oracle" / "_ref" / "acceptance_b200_f64", ["--skip", "4", "--skip", "5"], "exact")
    assert p.returncode == 0, p.stdout + p.stderr
    assert p.stdout.count("PASS") == 5, p.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("lanes", [1, 2, 8])
def test_solve_multi_f64_lanes(c_oracle, lanes):
    """knn_b200_solve_multi_f64 (the double build's n_lanes): min(lanes,
    devices) row shards, lists independent of the lane count."""
    import ctypes
    from paper_0906_0231_b200 import _lib
    n, d, k = 300, 24, 12
    x = _instance(n, d, 11)
    idx = np.empty((n, k), dtype=np.uint32)
    dist = np.empty((n, k), dtype=np.float64)
    st = _lib.Stats()
    rc = _lib.load().knn_b200_solve_multi_f64(x.ctypes.data, n, d, k, 1, lanes, idx.ctypes.data,
                                               dist.ctypes.data, ctypes.byref(st))
    assert rc == 0, _lib.last_error()
    oi, od = c_oracle.brute_force_f64(x, k, "sqeuclidean")
    _assert_f64_equal(idx, dist, oi, od, f"solve_multi_f64 lanes={lanes}")
    assert st.pair_evaluations == n * (n - 1) // 2

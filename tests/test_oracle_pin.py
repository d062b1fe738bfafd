"""Pin the CPU oracle before trusting it (CPU only).

The C restatement (oracle/knn_oracle.c) is checked against
  * the reference's own known-answer tests, restated with their values
    (test_io.cpp:44-64, test_oracle.cpp:45-66, test_distance.cpp, test_heap.cpp),
  * the golden fixtures produced by the compiled reference (tests/golden/),
  * and, when oracle/_ref was built here, the reference library itself.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import Reference, reference
from tests.helpers import assert_lists_bit_equal, golden_input


def test_splitmix64_kat(c_oracle):
    # test_io.cpp:44-50
    assert c_oracle.splitmix64(0, 4) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                         0x06C45D188009454F, 0xF88BB8A8724C81EC]


def test_unit_float_kat(c_oracle):
    # test_io.cpp:52-64
    got = c_oracle.unit_floats(1234567, 4)
    want = np.array([0.3500795364379883, 0.1736440658569336, 0.5322072505950928, 0.24900764226913452],
                    dtype=np.float32)
    assert np.array_equal(np.array(got, dtype=np.float32), want)
    xs = np.array(c_oracle.unit_floats(99, 1000), dtype=np.float32)
    assert (xs >= 0).all() and (xs < 1).all()


def test_generate_is_row_major_stream(c_oracle):
    # io.cpp:57-62: one stream, row-major
    x = c_oracle.generate(3, 5, 77)
    assert np.array_equal(x.reshape(-1), np.array(c_oracle.unit_floats(77, 15), dtype=np.float32))
    assert np.array_equal(c_oracle.generate(50, 9, 2024), c_oracle.generate(50, 9, 2024))
    assert not np.array_equal(c_oracle.generate(50, 9, 2024), c_oracle.generate(50, 9, 2025))


def test_generate_at_jumps_the_same_stream(c_oracle):
    """generate_at (the Weyl jump the large-offset generator checks use)
    reproduces slices of the sequential stream: start, middle, end of a
    20M-element stream, and the reference's own stream when it was built."""
    full = c_oracle.generate(20_000, 1000, 4).reshape(-1)
    for first, count in ((0, 1000), (123_457, 5000), (19_999_000, 1000), (7, 1)):
        assert np.array_equal(c_oracle.generate_at(4, first, count), full[first:first + count])
    import oracle
    ref = oracle.reference()
    if ref is not None:
        assert np.array_equal(ref.generate(300, 7, 99).reshape(-1), c_oracle.generate_at(99, 0, 2100))


def test_distance_kats(c_oracle):
    # test_distance.cpp / SPEC examples
    f = c_oracle.fold
    assert f("hellinger", np.array([1, 0]), np.array([0, 1])) == np.float32(2.0)
    assert f("sqeuclidean", np.array([3, 0]), np.array([0, 4])) == np.float32(25.0)
    u = np.array([0.25, 0.75], np.float32)
    v = np.array([0.5, 0.5], np.float32)
    want = sum((np.sqrt(np.float64(a)) - np.sqrt(np.float64(b))) ** 2 for a, b in zip(u, v))
    assert abs(float(f("hellinger", u, v)) - want) < 1e-6
    rng = np.random.default_rng(0)
    for _ in range(20):
        a = rng.random(37, dtype=np.float32)
        b = rng.random(37, dtype=np.float32)
        for m in ("hellinger", "sqeuclidean", "cosine"):
            assert f(m, a, b).tobytes() == f(m, b, a).tobytes()  # bitwise symmetry


def test_two_vectors_hellinger(c_oracle):
    # test_oracle.cpp:45-53
    idx, dist, pairs = c_oracle.brute_force(np.array([[1, 0], [0, 1]], np.float32), 1, "hellinger")
    assert idx.tolist() == [[1], [0]] and dist.tolist() == [[2.0], [2.0]] and pairs == 1


def test_five_points_on_a_line(c_oracle):
    # test_oracle.cpp:55-66
    x = np.array([[0], [1], [2], [4], [8]], np.float32)
    idx, dist, pairs = c_oracle.brute_force(x, 2, "sqeuclidean")
    assert idx.tolist() == [[1, 2], [0, 2], [1, 0], [2, 1], [3, 2]]
    assert dist.tolist() == [[1, 4], [1, 1], [1, 4], [4, 9], [16, 36]]
    assert pairs == 10


def test_k_beyond_n(c_oracle):
    # test_oracle.cpp:88-93
    idx, _, _ = c_oracle.brute_force(c_oracle.generate(6, 3, 52), 100, "hellinger")
    assert idx.shape == (6, 5)


def test_flat_sort_reference(c_oracle):
    # test_oracle.cpp:68-86: oracle == sort of all pairs, via numpy
    rng = np.random.default_rng(51)
    for trial in range(12):
        n = int(rng.integers(2, 62))
        d = int(rng.integers(1, 11))
        k = int(rng.integers(1, n + 5))
        x = rng.random((n, d), dtype=np.float32)
        m = "hellinger" if trial % 2 == 0 else "sqeuclidean"
        idx, dist, pairs = c_oracle.brute_force(x, k, m)
        assert pairs == n * (n - 1) // 2
        for i in range(n):
            cand = sorted((float(c_oracle.fold(m, x[max(i, j)], x[min(i, j)])), j) for j in range(n) if j != i)
            cand = cand[:min(k, n - 1)]
            assert [c[1] for c in cand] == idx[i].tolist()
            assert np.array_equal(np.array([c[0] for c in cand], np.float32), dist[i])


def test_heap_stream_matches_sort(c_oracle):
    # test_heap.cpp:92-109 / acceptance criterion 6: bounded heap == sort oracle
    rng = np.random.default_rng(6)
    for _ in range(200):
        cnt = int(rng.integers(0, 300))
        cap = int(rng.integers(1, 40))
        dist = rng.integers(0, 20, cnt).astype(np.float32)  # many ties
        index = rng.permutation(cnt).astype(np.uint32)
        oi, od = c_oracle.heap_stream(cap, dist, index)
        order = sorted(zip(dist.tolist(), index.tolist()))[:cap]
        assert oi.tolist() == [o[1] for o in order]
        assert od.tolist() == [o[0] for o in order]


def test_rows_topk_equals_brute_force(c_oracle):
    x = c_oracle.generate(500, 20, 8)
    for m in ("hellinger", "sqeuclidean"):
        idx, dist, _ = c_oracle.brute_force(x, 15, m)
        rows = np.array([0, 1, 250, 499], np.uint32)
        ri, rd = c_oracle.rows_topk(x, 15, m, rows, threads=3)
        assert_lists_bit_equal(ri, rd, idx[rows], dist[rows], m)


def test_oracle_matches_golden_fixtures(c_oracle, golden):
    z, meta = golden
    for case in meta:
        x = golden_input(c_oracle.generate, case)
        idx, dist, pairs = c_oracle.brute_force(x, case["k"], case["metric"])
        assert pairs == case["pairs"]
        assert_lists_bit_equal(idx, dist, z[case["name"] + "__index"],
                               z[case["name"] + "__dist_bits"].view(np.float32), case["name"])


@pytest.mark.skipif(reference() is None, reason="oracle/_ref not built (no /root/reference at build time)")
def test_restatement_matches_compiled_reference(c_oracle):
    ref: Reference = reference()
    rng = np.random.default_rng(1234)
    for trial in range(16):
        n = int(rng.integers(2, 400))
        d = int(rng.integers(1, 70))
        k = int(rng.integers(1, 80))
        seed = int(rng.integers(0, 2**63))
        x = ref.generate(n, d, seed)
        assert np.array_equal(x, c_oracle.generate(n, d, seed))
        m = ("hellinger", "sqeuclidean", "cosine")[trial % 3]
        if m == "cosine":
            from oracle import normalize_rows
            x = normalize_rows(x)
        ci, cd, cp = c_oracle.brute_force(x, k, m)
        ri, rd, rp, _ = ref.brute_force(x, k, m)
        assert cp == rp
        assert_lists_bit_equal(ci, cd, ri, rd, f"trial {trial} {m}")
        # and the reference's own multi-lane engine agrees (engine.hpp:33-36)
        ei, ed, ep, _ = ref.solve_knn(x, k, m, n_lanes=1 + trial % 3)
        assert_lists_bit_equal(ei, ed, ri, rd, f"engine trial {trial} {m}")


def test_custom_functor_folds_pinned_to_the_reference(c_oracle):
    """The oracle's restatements of the reference suite's custom functors
    equal the compiled reference running the same functors through its own
    registry (oracle/ref_capi.cpp), float and double builds."""
    import oracle
    ref = oracle.reference()
    if ref is None:
        pytest.skip("reference not built")
    for m in ("manhattan", "root_of_squares"):
        for n, d, k, seed in ((90, 7, 5, 1), (300, 3, 40, 2)):
            x = c_oracle.generate(n, d, seed)
            ri, rd, _, _ = ref.brute_force(x, k, m)
            oi, od, _ = c_oracle.brute_force(x, k, m)
            assert np.array_equal(ri, oi) and np.array_equal(rd.view(np.uint32), od.view(np.uint32)), m
            if oracle.REF_F64_CAPI_PATH.exists():
                ri64, rd64 = oracle.ReferenceF64().brute_force(x, k, m)
                oi64, od64 = c_oracle.brute_force_f64(x, k, m)
                assert np.array_equal(ri64, oi64) and np.array_equal(rd64.view(np.uint64), od64.view(np.uint64)), m

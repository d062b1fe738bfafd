"""Shared helpers for the parity tests."""
from __future__ import annotations

import numpy as np


def golden_input(gen, case) -> np.ndarray:
    """Rebuild a golden case's input (see tests/golden/make_golden.py)."""
    from oracle import normalize_rows

    x = gen(case["n"], case["d"], case["seed"])
    if case["transform"] == "normalize":
        x = normalize_rows(x)
    elif case["transform"] == "quantize":
        x = np.floor(x * 4.0).astype(np.float32)
    return np.ascontiguousarray(x, dtype=np.float32)


def assert_lists_bit_equal(idx, dist, ref_idx, ref_dist, what=""):
    """The reference's lists_equal (test_engine.cpp:18-26): same indices and
    identical distance bits, row by row."""
    idx = np.asarray(idx).astype(np.uint32)
    ref_idx = np.asarray(ref_idx).astype(np.uint32)
    assert idx.shape == ref_idx.shape, f"{what}: shape {idx.shape} != {ref_idx.shape}"
    bad_i = np.nonzero((idx != ref_idx).any(axis=1))[0]
    db = np.asarray(dist, dtype=np.float32).view(np.uint32)
    rb = np.asarray(ref_dist, dtype=np.float32).view(np.uint32)
    bad_d = np.nonzero((db != rb).any(axis=1))[0]
    if bad_i.size or bad_d.size:
        r = int(bad_i[0] if bad_i.size else bad_d[0])
        raise AssertionError(
            f"{what}: {bad_i.size} rows differ in indices, {bad_d.size} in distance bits; "
            f"first row {r}: got {idx[r][:8]} / {np.asarray(dist)[r][:8]}, "
            f"want {ref_idx[r][:8]} / {np.asarray(ref_dist)[r][:8]}")


def tolerance_check(idx, dist, ref_idx, ref_dist, ref_next, rtol=1e-5):
    """north_star's rule: index sets equal per row except where the oracle's
    k-th and (k+1)-th distances are within rtol; distances within rtol.
    Returns (unexplained_rows, exempt_rows, max_rel_err)."""
    unexplained = exempt = 0
    max_rel = 0.0
    for r in range(idx.shape[0]):
        rel = np.abs(dist[r].astype(np.float64) - ref_dist[r]) / np.maximum(np.abs(ref_dist[r]), 1e-30)
        max_rel = max(max_rel, float(rel.max(initial=0.0)))
        if set(idx[r].tolist()) != set(ref_idx[r].tolist()):
            kth, nxt = float(ref_dist[r][-1]), float(ref_next[r])
            if abs(nxt - kth) <= rtol * max(abs(kth), 1e-30):
                exempt += 1
            else:
                unexplained += 1
    return unexplained, exempt, max_rel

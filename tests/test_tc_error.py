"""The tensor core's accumulation error against the proof's allowance.

The TENSOR policy's completeness proof assumes
|dot_tc - dot| <= c d 2^-23 ||a|| ||b|| with c = kTcSafety = 4.  Measured with
the sweep's own instruction on adversarial fp16 inputs
(tools/tc_error_margin.py), the largest ratio must stay within c -- the
assumption the bit-exactness rests on (profiles/r02_tc_error_margin.txt has
the full table).
"""
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))


def test_tensor_core_error_within_the_proofs_allowance():
    from tc_error_margin import measure

    from paper_0906_0231_b200 import Context
    ctx = Context(0)
    try:
        res = measure(ctx, rows=256, dims=(64, 1024, 4096))
    finally:
        ctx.close()
    worst = max(r["max_ratio"] for r in res)
    print(f"\nworst |dot_tc - dot| / (d 2^-23 |a||b|) = {worst:.3e} (allowance c = 4)")
    assert worst <= 4.0
    # and within the textbook bound of sequential fp32 accumulation, d 2^-23
    # sum|a_k b_k| (measured: about d / 20 -- one rounding per 16-wide MMA step)
    assert all(r["max_rel_to_mass"] <= r["d"] for r in res)

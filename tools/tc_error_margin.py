"""How much of the proof's tensor-core allowance the hardware uses.

DESIGN.md §4 bounds the tensor core's FP32 accumulation of exact fp16
products by  |dot_tc - dot| <= c d 2^-23 ||a|| ||b||  with c = kTcSafety = 4
(tensor_path.cu).  This measures, with the sweep's own instruction
(knn_b200_debug_tc_dots: tcgen05.mma kind::f16, M=128 N=256, FP32 in TMEM),
the largest observed

    ratio = |dot_tc - dot_exact| / (d 2^-23 ||a|| ||b||)      (the proof uses ratio <= c)
    rel   = |dot_tc - dot_exact| / (2^-23 sum_k |a_k b_k|)    (error per unit of |partial sum| mass)

over adversarial fp16 inputs; dot_exact is the fp64 sum of the exact
products (fp16 x fp16 is exact in fp64; the fp64 sum's own error is
< d 2^-53 sum|ab|, negligible here).

    python tools/tc_error_margin.py [--rows 1024]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_0906_0231_b200 import Context, _lib  # noqa: E402
from paper_0906_0231_b200.engine import raise_for_status  # noqa: E402


def tc_dots(ctx, a, b):
    m, d = a.shape
    n = b.shape[0]
    out = torch.empty((m, n), dtype=torch.float32, device=a.device)
    raise_for_status(_lib.load().knn_b200_debug_tc_dots(ctx._h, a.data_ptr(), m, b.data_ptr(), n, d, out.data_ptr(),
                                                        torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return out


def inputs(kind, m, n, d, g):
    def f16(x):
        return x.clamp(-65504, 65504).half()
    if kind == "uniform_centered":      # what prep feeds the sweep: (x - mu) * 2^e, |.| <= 65504
        return f16((torch.rand(m, d, generator=g) - 0.5) * 131000), f16((torch.rand(n, d, generator=g) - 0.5) * 131000)
    if kind == "gaussian":
        return f16(torch.randn(m, d, generator=g) * 12000), f16(torch.randn(n, d, generator=g) * 12000)
    if kind == "mixed_exponents":       # full mantissas, magnitudes 2^-8 .. 2^15
        def mk(r):
            mant = 1 + torch.rand(r, d, generator=g)
            ex = torch.randint(-8, 15, (r, d), generator=g).float()
            sg = torch.randint(0, 2, (r, d), generator=g).float() * 2 - 1
            return f16(sg * mant * torch.exp2(ex))
        return mk(m), mk(n)
    if kind == "cancellation":          # partial sums grow to sum|ab|/2, then cancel to ~0
        a = f16((torch.rand(m, d, generator=g) + 0.5) * 30000)
        s = torch.ones(d)
        s[d // 2:] = -1
        b = f16(a[torch.randint(0, m, (n,), generator=g)].float() * s *
                (1 + 1e-3 * torch.randn(n, d, generator=g)))
        return a, b
    if kind == "same_sign_large":       # all products positive and large: partial sums maximal
        return f16((torch.rand(m, d, generator=g) * 0.5 + 0.5) * 60000), \
            f16((torch.rand(n, d, generator=g) * 0.5 + 0.5) * 60000)
    raise ValueError(kind)


KINDS = ["uniform_centered", "gaussian", "mixed_exponents", "cancellation", "same_sign_large"]


def measure(ctx, rows=512, dims=(64, 256, 1024, 4096), seed=7):
    g = torch.Generator().manual_seed(seed)
    out = []
    for d in dims:
        for kind in KINDS:
            a, b = inputs(kind, rows, 256, d, g)
            a, b = a.cuda().contiguous(), b.cuda().contiguous()
            tc = tc_dots(ctx, a, b).double()
            ex = a.double() @ b.double().T
            err = (tc - ex).abs()
            bound = d * 2.0 ** -23 * a.double().norm(dim=1)[:, None] * b.double().norm(dim=1)[None, :]
            mass = 2.0 ** -23 * (a.double().abs() @ b.double().abs().T)
            out.append({"d": d, "inputs": kind, "max_ratio": float((err / bound).max()),
                        "max_rel_to_mass": float((err / mass.clamp_min(1e-300)).max()),
                        "dots": int(err.numel())})
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1024)
    a = ap.parse_args()
    ctx = Context(0)
    res = measure(ctx, a.rows)
    worst = max(r["max_ratio"] for r in res)
    for r in res:
        print(json.dumps(r))
    print(json.dumps({"worst_ratio": worst, "kTcSafety": 4.0, "fraction_of_allowance_used": worst / 4.0}))

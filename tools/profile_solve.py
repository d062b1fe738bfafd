"""Run N device-resident solves of a synthetic config (dev/profiling tool)."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_0906_0231_b200 import Context, _lib, distance_by_name, generate_torch, solve_rows_torch

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=131072)
ap.add_argument("--d", type=int, default=256)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--metric", default="euclidean")
ap.add_argument("--arith", default="tensor")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
ctx = Context(0)
x = generate_torch(ctx, a.n, a.d, a.seed)
if a.metric == "cosine":  # rows L2-normalised in double, stored f32
    xd = x.double()
    x = (xd / xd.norm(dim=1, keepdim=True)).float().contiguous()
    del xd
for _ in range(a.reps):
    _, _, st = solve_rows_torch(ctx, x, a.k, distance_by_name(a.metric), 0, a.n, _lib.ARITH_NAMES[a.arith], want_stats=True)
    print({k: st[k] for k in ("sweep_ms", "kernel_ms", "fallback_rows", "rescored", "kernel_launches")}, flush=True)

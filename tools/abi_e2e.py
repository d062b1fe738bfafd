"""Time the C-ABI host path (knn_b200_solve: pageable numpy in, numpy out) at
a config and print its h2d / kernel / d2h split (dev tool)."""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_0906_0231_b200 import Context, distance_by_name, generate_torch

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1000000); ap.add_argument("--d", type=int, default=256)
ap.add_argument("--k", type=int, default=10); ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
ctx = Context(0)
x = generate_torch(ctx, a.n, a.d, 1).cpu().numpy()  # pageable host copy
m = distance_by_name("euclidean")
for _ in range(a.reps):
    t0 = time.perf_counter()
    idx, dist, st = ctx.solve(x, a.k, m)
    wall = (time.perf_counter() - t0) * 1e3
    print({"wall_ms": round(wall, 1), **{k: round(st[k], 2) for k in ("h2d_ms", "kernel_ms", "d2h_ms")}}, flush=True)

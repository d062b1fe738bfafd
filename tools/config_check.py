"""Full-size config run on the GPU + sampled-row parity against the oracle
(dev tool; the committed tests are tests/test_gpu_configs.py::test_c1_all_rows,
test_c3_full_size, test_c4_full_size and test_c5_full_size_one_gpu)."""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import oracle
from paper_0906_0231_b200 import Context, _lib, distance_by_name, generate_torch, solve_rows_torch

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int); ap.add_argument("--d", type=int); ap.add_argument("--k", type=int)
ap.add_argument("--metric", default="euclidean"); ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--rows", type=int, default=128); ap.add_argument("--arith", default="auto")
a = ap.parse_args()
ctx = Context(0)
x = generate_torch(ctx, a.n, a.d, a.seed)
if a.metric == "cosine":
    xd = x.double(); x = (xd / xd.norm(dim=1, keepdim=True)).float().contiguous(); del xd
m = distance_by_name(a.metric)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.time()
    idx, dist, st = solve_rows_torch(ctx, x, a.k, m, 0, a.n, _lib.ARITH_NAMES[a.arith], want_stats=True)
    torch.cuda.synchronize()
    print(f"rep {rep}: {time.time()-t0:.3f}s", {k: st[k] for k in ("sweep_ms", "kernel_ms", "fallback_rows", "exact_rows", "arith_used")}, flush=True)
xh = x.cpu().numpy()
rows = np.random.default_rng(0).choice(a.n, a.rows, replace=False).astype(np.uint32)
om = "sqeuclidean" if a.metric == "euclidean" else a.metric
t0 = time.time()
ri, rd = oracle.c_oracle().rows_topk(xh, a.k, om, rows)
if a.metric == "euclidean":
    rd = np.sqrt(rd)
gi = idx.cpu().numpy().view(np.uint32)[rows]; gd = dist.cpu().numpy()[rows]
print(f"oracle {a.rows} rows {time.time()-t0:.1f}s; idx equal rows {int((gi == ri).all(1).sum())}/{a.rows}; "
      f"dist bit-equal rows {int((gd.view(np.uint32) == rd.view(np.uint32)).all(1).sum())}/{a.rows}", flush=True)

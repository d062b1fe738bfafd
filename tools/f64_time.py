"""Dev tool: time knn_b200_solve_f64 (KNN_DOUBLE_ACCUM policy) at a config."""
import argparse, json, sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_0906_0231_b200 import Context, distance_by_name

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--metric", default="euclidean")
a = ap.parse_args()
rng = np.random.default_rng(42)
x = rng.random((a.n, a.d), dtype=np.float32)
ctx = Context(0)
ctx.solve_f64(x, a.k, distance_by_name(a.metric))
best = None
for _ in range(3):
    _, _, st = ctx.solve_f64(x, a.k, distance_by_name(a.metric))
    best = st if best is None or st["sweep_ms"] < best["sweep_ms"] else best
pairs = a.n * (a.n - 1) / 2
ordered = a.n * a.n
print(json.dumps({"n": a.n, "d": a.d, "k": a.k, "metric": a.metric, "sweep_ms": best["sweep_ms"],
                  "seconds": best["seconds"], "pairs_per_s": pairs / (best["sweep_ms"] / 1e3),
                  "dfma_tflops": 2 * ordered * a.d / (best["sweep_ms"] / 1e3) / 1e12}))
ctx.close()

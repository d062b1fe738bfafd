"""GPU probe of the CTA-pair sweep (KNN_B200_PAIR=1) against the oracle (dev tool)."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle
from paper_0906_0231_b200 import Context, _lib, distance_by_name

co = oracle.c_oracle()
ctx = Context(0)
cases = [(4096, 64, 10, "sqeuclidean"), (1100, 33, 1, "sqeuclidean"), (2048, 64, 10, "hellinger"),
         (4096, 256, 10, "euclidean"), (5000, 100, 5, "cosine"), (3000, 17, 3, "sqeuclidean"),
         (20000, 256, 10, "euclidean"), (2000, 128, 14, "sqeuclidean")]
for n, d, k, m in cases:
    x = co.generate(n, d, 11)
    if m == "cosine":
        x = oracle.normalize_rows(x)
    om = "sqeuclidean" if m == "euclidean" else m
    ri, rd, _ = co.brute_force(x, k, om)
    if m == "euclidean":
        rd = np.sqrt(rd)
    for pair in ("0", "1"):
        os.environ["KNN_B200_PAIR"] = pair
        idx, dist, st = ctx.solve(x, k, distance_by_name(m), _lib.ARITH_TENSOR)
        ok_i = (idx == ri).all(axis=1)
        ok_d = (dist.view(np.uint32) == rd.view(np.uint32)).all(axis=1)
        print(f"pair={pair} n={n} d={d} k={k} {m}: idx_rows_bad={int((~ok_i).sum())} "
              f"dist_rows_bad={int((~ok_d).sum())} fallback={st['fallback_rows']} sweep_ms={st['sweep_ms']:.3f}",
              flush=True)

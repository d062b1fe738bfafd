"""GPU probe of an opt-in sweep variant against the oracle (dev tool).
usage: sym_probe.py [ENV_VAR]   (default KNN_B200_SYM; e.g. KNN_B200_TRI)"""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle
from paper_0906_0231_b200 import Context, _lib, distance_by_name

KNOB = sys.argv[1] if len(sys.argv) > 1 else "KNN_B200_SYM"
co = oracle.c_oracle()
ctx = Context(0)
cases = [(1100, 33, 1, "sqeuclidean"), (2048, 64, 10, "sqeuclidean"), (2048, 64, 10, "hellinger"),
         (4096, 256, 10, "euclidean"), (5000, 100, 5, "cosine"), (3000, 17, 3, "sqeuclidean"),
         (20000, 256, 10, "euclidean"), (70000, 64, 10, "sqeuclidean"), (9000, 200, 7, "hellinger")]
for n, d, k, m in cases:
    x = co.generate(n, d, 11)
    if m == "cosine":
        x = oracle.normalize_rows(x)
    om = "sqeuclidean" if m == "euclidean" else m
    ri, rd, _ = co.brute_force(x, k, om)
    if m == "euclidean":
        rd = np.sqrt(rd)
    for sym in ("0", "1"):
        os.environ[KNOB] = sym
        t0 = time.time()
        idx, dist, st = ctx.solve(x, k, distance_by_name(m), _lib.ARITH_TENSOR)
        dt = time.time() - t0
        ok_i = (idx == ri).all(axis=1)
        ok_d = (dist.view(np.uint32) == rd.view(np.uint32)).all(axis=1)
        print(f"sym={sym} n={n} d={d} k={k} {m}: idx_rows_bad={int((~ok_i).sum())} "
              f"dist_rows_bad={int((~ok_d).sum())} fallback={st['fallback_rows']} exact_rows={st['exact_rows']} "
              f"rescored={st['rescored']} launches={st['kernel_launches']} sweep_ms={st['sweep_ms']:.3f} t={dt:.3f}s",
              flush=True)
        if (~ok_i).any():
            r = int(np.argmin(ok_i))
            print("  row", r, idx[r][:6], ri[r][:6], dist[r][:4], rd[r][:4])

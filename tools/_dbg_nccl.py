import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_0906_0231_b200 import (Context, _lib, comm_init, comm_unique_id, distance_by_name, solve_rows_torch,
                                  solve_sharded_torch)
co = oracle.c_oracle()
m = distance_by_name("euclidean")
step = sys.argv[1]
n, d, k = 400_000, 96, 10
x = torch.from_numpy(co.generate(n, d, n)).cuda()
c = Context(0)
def run(tag, f):
    try:
        f(); torch.cuda.synchronize(); print(tag, "ok", flush=True)
    except Exception as e:
        print(tag, "FAIL", e, flush=True); raise SystemExit(1)
run("rows1", lambda: solve_rows_torch(c, x, k, m, 0, n, _lib.ARITH_AUTO))
if step in ("init", "solve", "solve2"):
    run("comm_init", lambda: comm_init(c, comm_unique_id(), 0, 1))
if step in ("solve", "solve2"):
    run("sharded", lambda: solve_sharded_torch(c, x, k, m, _lib.ARITH_AUTO, 0, 1, want_stats=True))
if step == "solve2":
    run("sharded2", lambda: solve_sharded_torch(c, x, k, m, _lib.ARITH_AUTO, 0, 1, want_stats=True))
run("rows2", lambda: solve_rows_torch(c, x, k, m, 0, n, _lib.ARITH_AUTO))
c2 = Context(0)
run("rows_newctx", lambda: solve_rows_torch(c2, x, k, m, 0, n, _lib.ARITH_AUTO))

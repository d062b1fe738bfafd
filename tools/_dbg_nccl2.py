import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_0906_0231_b200 import (Context, _lib, comm_broadcast_torch, comm_init, comm_unique_id, distance_by_name,
                                  solve_rows_torch, solve_sharded_torch)
co = oracle.c_oracle()
m = distance_by_name("euclidean")
c = Context(0)
comm_init(c, comm_unique_id(), 0, 1)
skip_bcast = "nobcast" in sys.argv
for n, d, k, force in ((400_000, 96, 10, False), (30_000, 33, 6, True), (5000, 20, 40, False)):
    if force: os.environ["KNN_B200_TRI"] = "force"
    else: os.environ.pop("KNN_B200_TRI", None)
    x = torch.from_numpy(co.generate(n, d, n)).cuda()
    if not skip_bcast:
        comm_broadcast_torch(c, x, 0); torch.cuda.synchronize(); print(n, "bcast ok", flush=True)
    try:
        i1, d1, st = solve_sharded_torch(c, x, k, m, _lib.ARITH_AUTO, 0, 1, want_stats=True); torch.cuda.synchronize()
        print(n, "sharded ok", flush=True)
        i0, d0, _ = solve_rows_torch(c, x, k, m, 0, n, _lib.ARITH_AUTO); torch.cuda.synchronize()
        print(n, "rows ok", bool((i0 == i1).all().item()), flush=True)
    except Exception as e:
        print(n, "FAIL", e, flush=True); raise SystemExit(1)

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KNN_B200_TRI"] = "force"
import numpy as np, torch
import oracle
from paper_0906_0231_b200 import Context, _lib, distance_by_name, solve_rows_torch
co = oracle.c_oracle()
m = distance_by_name("euclidean")
for n, d, k in [(30000, 33, 6), (20000, 48, 7), (9000, 40, 9), (3000, 200, 4), (1500, 17, 1), (30000, 96, 10), (100000, 33, 6)]:
    c = Context(0)
    x = torch.from_numpy(co.generate(n, d, n)).cuda()
    try:
        i, dd, st = solve_rows_torch(c, x, k, m, 0, n, _lib.ARITH_TENSOR, want_stats=True)
        torch.cuda.synchronize()
        ri, rd = co.rows_topk(x.cpu().numpy(), k, "sqeuclidean", np.arange(n, dtype=np.uint32))
        ok = np.array_equal(i.cpu().numpy().view(np.uint32), ri)
        print(n, d, k, "ok" if ok else "MISMATCH", st["fallback_rows"], flush=True)
    except Exception as e:
        print(n, d, k, "FAIL", e, flush=True)
        raise SystemExit(1)
    c.close()

"""Small solves through every tcgen05 kernel, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize_tri.py
    compute-sanitizer --tool synccheck python tools/sanitize_tri.py
    compute-sanitizer --tool memcheck  python tools/sanitize_tri.py

KNN_B200_TRI=force runs the triangle sweep (CTA pairs, cluster mbarriers with
relaxed remote arrives, the column-side pool) at n = 8192; then the E4M3
sample pass, the rectangular pair and single-CTA sweeps, the capture pass,
the sharded loopback (world 2) and the EXACT kernels -- each checked against
the oracle so a sanitizer-clean run is also a correct one.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["KNN_B200_TRI"] = "force"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_0906_0231_b200 import (Context, _lib, distance_by_name, solve_rows_torch,  # noqa: E402
                                  solve_sharded_loopback_torch)

co = oracle.c_oracle()
ctx = Context(0)
n, d, k = int(os.environ.get("SAN_N", "8192")), 64, 10
xh = co.generate(n, d, 3)
x = torch.from_numpy(xh).cuda()
ri, rd, _ = co.brute_force(xh, k, "sqeuclidean")
m = distance_by_name("sqeuclidean")


def check(i, dd, what):
    ok = np.array_equal(i.cpu().numpy().view(np.uint32), ri) and \
        np.array_equal(dd.cpu().numpy().view(np.uint32), rd.view(np.uint32))
    print(f"{what}: {'bit-exact' if ok else 'MISMATCH'}", flush=True)
    return ok


good = True
i, dd, st = solve_rows_torch(ctx, x, k, m, 0, n, _lib.ARITH_TENSOR, want_stats=True)
good &= check(i, dd, f"triangle sweep (capture rows {st['fallback_rows']})")
os.environ["KNN_B200_FORCE_CAPTURE"] = "1"
i, dd, st = solve_rows_torch(ctx, x, k, m, 0, n, _lib.ARITH_TENSOR, want_stats=True)
good &= check(i, dd, f"triangle sweep, every row through the capture pass ({st['fallback_rows']})")
del os.environ["KNN_B200_FORCE_CAPTURE"]
os.environ["KNN_B200_TRI"] = "0"
i, dd, _ = solve_rows_torch(ctx, x, k, m, 0, n, _lib.ARITH_TENSOR)
good &= check(i, dd, "rectangular pair sweep")
i, dd, _ = solve_rows_torch(ctx, x, k, m, 1000, 3000, _lib.ARITH_TENSOR)
ok = np.array_equal(i.cpu().numpy().view(np.uint32), ri[1000:3000])
print(f"row shard (single-CTA sweep): {'bit-exact' if ok else 'MISMATCH'}", flush=True)
good &= ok
os.environ["KNN_B200_TRI"] = "force"
i, dd, _, _, _ = solve_sharded_loopback_torch(ctx, x, k, m, 2)
good &= check(i, dd, "sharded triangle, loopback world 2")
i, dd, _ = solve_rows_torch(ctx, x, k, m, 0, n, _lib.ARITH_EXACT)
good &= check(i, dd, "EXACT kernel")
ctx.close()
print("ALL BIT-EXACT" if good else "FAILURES", flush=True)
sys.exit(0 if good else 1)

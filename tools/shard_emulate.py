"""Per-rank time of the sharded triangle at world W, emulated on one B200.

Runs every rank program of knn_b200_debug_solve_sharded_loopback on the one
device (one after another) and reports, per rank, the CUDA-event time of its
phases: replicated prep (+ second order), its sample slice, its triangle
sweep + binning, its merge + rescore (+ capture).  The slowest rank's sum is
what an 8-GPU box would wait for, less the exchanges, which are estimated
from the bytes each rank sends (column-side candidates, 12 B each; the
thresholds all-gather and the result reduce-scatter are added as bytes too)
at a conservative 300 GB/s per GPU over NVLink 5.  T1 is the single-GPU solve
(solve_rows_torch, the bench path) of the same problem.

    python tools/shard_emulate.py [--n 1000000 --d 256 --k 10 --seed 1 --worlds 1,2,4,8]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0906_0231_b200 import (Context, _lib, distance_by_name, generate_torch,  # noqa: E402
                                  solve_rows_torch, solve_sharded_loopback_torch)

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=256)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--nvlink-gbs", type=float, default=300.0)
ap.add_argument("--metric", default="euclidean")
a = ap.parse_args()
ctx = Context(0)
x = generate_torch(ctx, a.n, a.d, a.seed)
if a.metric == "cosine":  # rows L2-normalised in double, stored f32
    xd = x.double()
    x = (xd / xd.norm(dim=1, keepdim=True)).float().contiguous()
    del xd
m = distance_by_name(a.metric)
klist = min(a.k, a.n - 1)
# the sharded runs first, on their own context (its workspace is freed
# before the single-GPU solve allocates its own: C5 needs both to fit)
rows = []
outs = {}
for w in [int(v) for v in a.worlds.split(",")]:
    # each rank program is deterministic; run-to-run spread on one device is
    # clock noise, so every phase of every rank takes its minimum over reps
    best = None
    for _ in range(a.reps + 1):
        iw, dw, st, rank_ms, xb = solve_sharded_loopback_torch(ctx, x, a.k, m, w)
        if best is None:
            best = (None, rank_ms.copy(), xb.copy(), st)
        else:
            best = (None, np.minimum(best[1], rank_ms), xb.copy(), st)
    best = (best[1].sum(1), best[1], best[2], best[3])
    outs[w] = (iw.cpu(), dw.cpu())
    del iw, dw
    rows.append((w, best))
ctx.close()
torch.cuda.empty_cache()
ctx = Context(0)
t1 = []
for _ in range(a.reps + 1):
    ref_i, ref_d, st = solve_rows_torch(ctx, x, a.k, m, 0, a.n, _lib.ARITH_TENSOR, want_stats=True)
    t1.append(st["kernel_ms"])
T1 = float(np.median(t1[1:])) if len(t1) > 1 else t1[0]
print(json.dumps({"n": a.n, "d": a.d, "k": a.k, "T1_ms": T1, "T1_runs": t1}), flush=True)
ref_i, ref_d = ref_i.cpu(), ref_d.cpu()
for w, (tot, rank_ms, xb, st) in rows:
    iw, dw = outs[w]
    same = bool((iw == ref_i).all().item() and (dw.view(torch.int32) == ref_d.view(torch.int32)).all().item())
    # exchanges: column-side all-to-all (measured bytes), thresholds
    # all-gather (8 B/row), rows reduce-scatter (8 B x klist per row, x2 for
    # the reduction's read+write)
    xchg_bytes = xb.max() + 8 * a.n * (w - 1) / w + 2 * 8 * klist * a.n * (w - 1) / w if w > 1 else 0
    xchg_ms = xchg_bytes / (a.nvlink_gbs * 1e9) * 1e3
    slowest = float(tot.max()) + xchg_ms
    print(json.dumps({
        "world": w, "bit_identical_to_single_gpu": same, "overflow": st["reserved"],
        "rank_ms_phases[prep,sample,sweep+bin,merge]": np.round(rank_ms, 2).tolist(),
        "rank_ms_total": np.round(tot, 2).tolist(), "max_rank_ms": float(tot.max()),
        "sent_MB": np.round(xb / 1e6, 1).tolist(), "exchange_ms_est": round(xchg_ms, 2),
        "slowest_with_exchange_ms": round(slowest, 2), "T1_over_w_ms": round(T1 / w, 2),
        "ratio_to_T1_over_w": round(slowest / (T1 / w), 3), "est_speedup": round(T1 / slowest, 2),
        "capture_rows": st["fallback_rows"]}), flush=True)

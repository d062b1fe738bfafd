"""Kernel timeline of one device-resident solve (dev tool): torch.profiler
(CUPTI) records every kernel and memcpy of the solve; prints the busy time,
the wall time between the first start and the last end, and the largest idle
gaps between consecutive GPU activities with their neighbours.

    python tools/timeline.py [--n 1000000 --d 256 --k 10 --metric euclidean --seed 1]
"""
import argparse, json, sys, tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_0906_0231_b200 import Context, _lib, distance_by_name, generate_torch, solve_rows_torch

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=256)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--metric", default="euclidean")
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
ctx = Context(0)
x = generate_torch(ctx, a.n, a.d, a.seed)
if a.metric == "cosine":
    xd = x.double()
    x = (xd / xd.norm(dim=1, keepdim=True)).float().contiguous()
    del xd
m = distance_by_name(a.metric)
for _ in range(2):
    solve_rows_torch(ctx, x, a.k, m, 0, a.n, _lib.ARITH_AUTO)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    solve_rows_torch(ctx, x, a.k, m, 0, a.n, _lib.ARITH_AUTO)
    torch.cuda.synchronize()
tmp = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(tmp)
ev = json.load(open(tmp))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
if not gpu:
    print("no GPU events recorded"); sys.exit(1)
t0, t1 = gpu[0]["ts"], max(e["ts"] + e["dur"] for e in gpu)
busy = 0.0
gaps = []
end = gpu[0]["ts"]
prev = None
for e in gpu:
    if e["ts"] > end:
        gaps.append((e["ts"] - end, prev["name"][:60] if prev else "", e["name"][:60]))
    if e["ts"] + e["dur"] > end:
        busy += e["ts"] + e["dur"] - max(end, e["ts"])
        end = e["ts"] + e["dur"]
        prev = e
print(json.dumps({"wall_ms": (t1 - t0) / 1e3, "busy_ms": busy / 1e3, "idle_ms": (t1 - t0 - busy) / 1e3,
                  "gpu_events": len(gpu), "gaps_over_20us": sum(1 for g in gaps if g[0] > 20)}))
for g in sorted(gaps, reverse=True)[:a.top]:
    print(f"{g[0] / 1e3:8.3f} ms  after {g[1]!r}  before {g[2]!r}")

#!/usr/bin/env python
"""bench.py -- all-pairs k-NN throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--arith auto]
    python bench.py --impl reference ...          # the reference CPU path

A "step" is one complete exact all-pairs k-NN solve of the configured
synthetic dataset (every query row against every vector, Phase 1 + Phase 2).
The unit of work is one unordered pair {x, y} (reference counter
pair_evaluations, engine.hpp:28), so

    value = n (n-1) / 2 * K / (max-over-ranks time of K steps)   [pairs/s]

Inputs are SplitMix64 generate_dataset(n, d, seed) (src/io.cpp:57-62), made on
the device by knn_b200_generate_device (bit-identical to the host stream).
Multi-GPU (torchrun, one rank per GPU): rank 0 generates, the reference set is
replicated by an NCCL broadcast over the engine's own communicator, and the
ranks solve the whole problem together -- the sharded triangle computes each
unordered pair once across the ranks and exchanges column-side candidates
(NCCL all-to-all); each rank ends with a contiguous shard of rows.  n is
fixed as N grows: "strong" scaling.

`value` is device-resident (inputs already in HBM); `e2e` is the same metric
through the public API with the host copy of the inputs and the device->host
copy of every rank's result lists inside the timed region: one GPU, the C
ABI's own call on pageable host buffers; N GPUs, every rank's row slice from
its pinned host memory over its own PCIe link, replicated by an NCCL
all-gather over NVLink.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: n, d, k, metric, seed  (SURVEY §8(d) seeds C1=42 ... C5=4)
    "c1": dict(n=16384, d=64, k=10, metric="euclidean", seed=42, label="n=16384 d=64 k=10 Euclidean"),
    "c2": dict(n=1_000_000, d=256, k=10, metric="euclidean", seed=1, label="n=1M d=256 k=10 Euclidean"),
    "c3": dict(n=1_000_000, d=1024, k=100, metric="euclidean", seed=2, label="n=1M d=1024 k=100 Euclidean"),
    "c4": dict(n=4_000_000, d=128, k=32, metric="cosine", seed=3, label="n=4M d=128 k=32 cosine"),
    "c5": dict(n=16_000_000, d=256, k=10, metric="euclidean", seed=4, label="n=16M d=256 k=10 Euclidean"),
}
DEFAULT_CONFIG = "c2"   # BASELINE.json configs[1]: the metric's 1-GPU configuration
METRIC = "all-pairs k-NN distance-evals/s (unordered pairs)"
UNIT = "pairs/s"


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._pump, daemon=True)
        self.thread.start()

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# --------------------------------------------------------------------------
# CPU reference arm / cpu_baseline (the ONLY places bench.py runs oracle/)

# The CPU sample: a prefix of n' rows of the same stream (SURVEY §8(d) CPU
# baseline (ii): n' in {32768, 65536}).  One fixed size per config, used by
# BOTH the cpu_baseline leg and the --impl reference arm, so the two report
# the same measurement.
CPU_SAMPLE_N = {"c1": 16384, "c2": 65536, "c3": 32768, "c4": 65536, "c5": 65536}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_sample(cfg, nn: int):
    """Time the reference's own solve_knn (oracle/_ref, unmodified library,
    all host cores as lanes) once on the prefix of nn rows, or the C
    restatement when the reference was not compiled.  Returns
    (pairs_per_s, seconds, cores, kind, sample_desc, nn)."""
    import numpy as np

    import oracle
    cores = os.cpu_count() or 1
    ref = oracle.reference()
    co = oracle.c_oracle()
    metric = {"euclidean": "sqeuclidean"}.get(cfg["metric"], cfg["metric"])
    d, k = cfg["d"], cfg["k"]

    def run(nn):
        x = co.generate(nn, d, cfg["seed"])  # prefix rows of the same stream
        if metric == "cosine":
            x = oracle.normalize_rows(x)
        if ref is not None:
            # every lane gets >= 2 grid rows (SURVEY §8(d) CPU baseline (ii))
            gsize = 64 * max(1, math.ceil(nn / (2 * cores * 64)))
            t0 = time.perf_counter()
            ref.solve_knn(x, k, metric, n_lanes=cores, gsize=gsize, want_lists=False)
            return time.perf_counter() - t0, "reference", f"reference solve_knn, {cores} lanes, gsize {gsize}"
        rows = np.arange(nn, dtype=np.uint32)
        t0 = time.perf_counter()
        co.rows_topk(x, k, metric, rows, threads=cores)
        # rows_topk evaluates every ordered pair: report unordered-pair rate
        return 2 * (time.perf_counter() - t0), "port", f"C restatement rows_topk, {cores} threads (x2: no symmetry)"

    nn = min(nn, cfg["n"])
    t, kind, desc = run(nn)
    pairs = nn * (nn - 1) / 2
    sample = (f"prefix n'={nn} of {cfg['label']} (same seed/metric), {desc}; "
              f"pairs/s = n'(n'-1)/2 / time; host {cpu_model()}, nproc {cores}")
    return pairs / t, t, cores, kind, sample, nn


def run_reference_arm(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    cores = os.cpu_count() or 1
    nn = min(CPU_SAMPLE_N.get(args.config, 65536), cfg["n"])
    kind = "reference" if oracle.reference() is not None else "port"
    ref = oracle.reference()
    co = oracle.c_oracle()
    metric = {"euclidean": "sqeuclidean"}.get(cfg["metric"], cfg["metric"])
    x = co.generate(nn, cfg["d"], cfg["seed"])
    if metric == "cosine":
        x = oracle.normalize_rows(x)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if ref is not None:
            gsize = 64 * max(1, math.ceil(nn / (2 * cores * 64)))
            ref.solve_knn(x, cfg["k"], metric, n_lanes=cores, gsize=gsize, want_lists=False)
            dt = time.perf_counter() - t0
        else:
            co.rows_topk(x, cfg["k"], metric, np.arange(nn, dtype=np.uint32), threads=cores)
            dt = 2 * (time.perf_counter() - t0)
        if i >= args.warmup:
            times.append(dt)
    pairs = nn * (nn - 1) / 2
    total = sum(times)
    value = pairs * len(times) / total
    desc = (f"reference solve_knn, {cores} lanes, gsize {64 * max(1, math.ceil(nn / (2 * cores * 64)))}"
            if ref is not None else f"C restatement rows_topk, {cores} threads (x2: no symmetry)")
    sample = (f"prefix n'={nn} of {cfg['label']} (same seed/metric), {desc}; pairs/s = n'(n'-1)/2 / time; "
              f"host {cpu_model()}, nproc {cores}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SplitMix64 generate_dataset)",
        "config": {"workload": cfg["label"], "sample": sample, "metric_fold": metric},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# B200 arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=None, help="override n (smoke/profiling only)")
    ap.add_argument("--arith", default="auto", choices=["auto", "exact", "tensor"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-n", type=int, default=None, help="CPU sample rows (default CPU_SAMPLE_N)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.n:
        cfg["n"] = args.n
        cfg["label"] += f" [n overridden to {args.n}]"
    if args.impl == "reference":
        return run_reference_arm(args, cfg)

    import torch
    import torch.distributed as dist

    from paper_0906_0231_b200 import (Context, _lib, comm_broadcast_torch, comm_init, comm_unique_id,
                                      distance_by_name, generate_torch, shard_rows, solve_sharded_torch)

    rank, world, local = dist_env()
    launched = "RANK" in os.environ and "MASTER_ADDR" in os.environ  # torchrun (any world size)
    torch.cuda.set_device(local if launched else 0)
    if launched:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local if launched else 0}")
    ctx = Context(dev.index)
    n, d, k = cfg["n"], cfg["d"], cfg["k"]
    metric = distance_by_name(cfg["metric"])
    arith = _lib.ARITH_NAMES[args.arith]
    klist = min(k, n - 1)
    r0, r1 = shard_rows(n, rank, world)
    stream = torch.cuda.current_stream(dev)
    if launched:
        # the engine's own NCCL communicator (one rank per GPU): rank 0 makes
        # the id, torch.distributed ships it
        box = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        comm_init(ctx, box[0], rank, world)

    # ---- inputs: generated on rank 0's device, replicated by NCCL broadcast
    x = generate_torch(ctx, n, d, cfg["seed"], dev) if rank == 0 else torch.empty((n, d), dtype=torch.float32,
                                                                                  device=dev)
    if cfg["metric"] == "cosine" and rank == 0:
        xd = x.double()
        x = (xd / xd.norm(dim=1, keepdim=True).clamp_min(1e-300)).float().contiguous()
        del xd
    if launched:
        comm_broadcast_torch(ctx, x, 0)  # NCCL broadcast of the reference set
    torch.cuda.synchronize()

    def barrier():
        if launched:
            dist.barrier(device_ids=[dev.index])
        torch.cuda.synchronize()

    def device_step(xx=None, want_stats=True):
        # one whole solve across the ranks: each rank gets its row shard
        # (the sharded triangle where eligible)
        i, dd, st = solve_sharded_torch(ctx, x if xx is None else xx, k, metric, arith, rank, world,
                                        want_stats=want_stats)
        return i, dd, st

    # ---- warm-up (W >= 3 full steps)
    for _ in range(max(args.warmup, 0)):
        device_step()
    barrier()

    # ---- timed device-resident region
    clocks = ClockSampler(dev.index)
    clocks.start()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    sweep_ms, stats = [], []
    for _ in range(args.steps):
        _, _, st = device_step()
        launches += st["kernel_launches"]
        sweep_ms.append(st["sweep_ms"])
        stats.append(st)
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if launched:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    pairs = n * (n - 1) / 2
    value = pairs * args.steps / (ms_max / 1e3)

    # ---- e2e through the public API.  One GPU: the drop-in's own call,
    #      knn_b200_solve (C ABI) with PAGEABLE host buffers as the reference's
    #      Dataset / NeighborList vectors are (staged H2D, solve, staged D2H;
    #      synchronous, so timed by the host clock around each call).
    #      N GPUs: pinned host input -> H2D (rank 0) -> NCCL broadcast ->
    #      shard solve -> D2H of the shard's lists, timed by CUDA events.
    e2e_path = None
    e2e_pinned_ms = None
    if not launched:
        import numpy as np

        x_np = x.cpu().numpy()  # pageable
        ctx.solve(x_np, k, metric, arith)  # staging buffers allocated outside the timed region
        torch.cuda.synchronize()
        t_e2e = time.perf_counter()
        for _ in range(args.steps):
            ctx.solve(x_np, k, metric, arith)
        e2e_ms = (time.perf_counter() - t_e2e) * 1e3
        e2e_path = "knn_b200_solve (C ABI), pageable host buffers in and out, host clock"
        del x_np
        # The same call with pinned host buffers (the ABI then DMAs directly):
        # reported beside the pageable headline, not instead of it.
        x_pin = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
        x_pin.copy_(x)
        idx_pin = torch.empty((n, klist), dtype=torch.int32, pin_memory=True)
        dist_pin = torch.empty((n, klist), dtype=torch.float32, pin_memory=True)
        pin_out = (idx_pin.numpy().view(np.uint32), dist_pin.numpy())
        ctx.solve(x_pin.numpy(), k, metric, arith, out=pin_out)
        torch.cuda.synchronize()
        t_pin = time.perf_counter()
        for _ in range(args.steps):
            ctx.solve(x_pin.numpy(), k, metric, arith, out=pin_out)
        e2e_pinned_ms = (time.perf_counter() - t_pin) * 1e3 / args.steps
        del x_pin, idx_pin, dist_pin, pin_out
        # The C++ drop-in itself (knn::solve_knn from the reference's header,
        # engine_b200.cpp): pageable Dataset in, EngineResult.lists (one
        # std::vector per row) out -- what a reference user's call costs.
        dropin = ROOT / "build" / "bench_dropin"
        dropin_ms = None
        if dropin.exists() and not args.n:
            try:
                out = subprocess.run([str(dropin), str(n), str(d), str(k), str(cfg["seed"]), str(args.steps), "1"],
                                     capture_output=True, text=True, timeout=600, check=True).stdout
                dropin_ms = json.loads(out.strip().splitlines()[-1])["ms_per_step"]
            except Exception as e:  # reported, never substituted
                dropin_ms = f"unavailable: {e}"
    if launched:
        # Each process holds its own row slice of the input in pinned host
        # memory (as a job reading its shard of the file would) and copies it
        # over its own PCIe link; the slices are replicated by one NCCL
        # all-gather over NVLink (world 1: rank 0 copies the whole set).
        R = -(-n // world)
        x_e2e = torch.empty((world * R, d), dtype=torch.float32, device=dev)
        host_slice = torch.empty((r1 - r0, d), dtype=torch.float32, pin_memory=True)
        host_slice.copy_(x[r0:r1])
        idx_host = torch.empty((r1 - r0, klist), dtype=torch.int32, pin_memory=True)
        dist_host = torch.empty((r1 - r0, klist), dtype=torch.float32, pin_memory=True)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            x_e2e[r0:r1].copy_(host_slice, non_blocking=True)
            if world > 1:
                dist.all_gather_into_tensor(x_e2e, x_e2e[rank * R:(rank + 1) * R])
            out_idx, out_dist, _ = device_step(x_e2e[:n], want_stats=False)
            idx_host.copy_(out_idx, non_blocking=True)
            dist_host.copy_(out_dist, non_blocking=True)
        e1.record(stream)
        barrier()
        t2 = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        e2e_ms = float(t2.item())
        e2e_path = ("each rank's row slice from its own pinned host memory over its own PCIe link, NCCL all-gather "
                    "over NVLink, sharded solve, D2H of each rank's rows; CUDA events, max over ranks")
    e2e_value = pairs * args.steps / (e2e_ms / 1e3)

    # ---- roofline of the dominant kernel (the fused distance + top-k sweep)
    peaks = load_peaks()
    last = stats[-1]
    tensor = last["arith_used"] == _lib.ARITH_TENSOR
    # algorithmic work per launch: 2*d flop per unordered pair;
    # each of the world ranks covers (about) 1/world of the n(n-1)/2 pairs
    alg_flop = n * (n - 1) / 2 / world * 2 * d
    sweep_avg_s = statistics.mean(sweep_ms) / 1e3
    achieved = alg_flop / sweep_avg_s / 1e12
    if tensor:
        # A sweep that runs for >100 ms sits under the 1 kW power cap: compare
        # against the measured SUSTAINED cuBLAS rate (B200_PROFILING.md).
        long_kernel = statistics.mean(sweep_ms) > 100.0
        key = "bf16_tflops_sustained" if long_kernel else "bf16_tflops"
        peak = peaks.get(key, 1400.0 if long_kernel else 1590.0)
        peak_src = (f"measured bf16 dense {'sustained' if long_kernel else 'burst'} ({key}, MEASURED_PEAKS.json; "
                    "fp16 runs at the bf16 rate)") if peaks else "fallback (B200_PROFILING.md)"
        bound = "tensor"
    else:
        sm = peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * 2 * sm * 1e6 / 1e12
        peak_src = f"FP32 SIMT nominal 148 SM x 128 lanes x 2 flop x {sm:.0f} MHz (no measured FP32 peak)"
        bound = "fp32"

    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists() and not args.n:
        entry = json.loads(tfile.read_text()).get(args.config)
        if entry and tensor:
            traffic = entry["dram_bytes_per_launch"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if not tensor else "f16->f32 filter, f32 exact rescore",
        "data": "synthetic (SplitMix64 generate_dataset on device)",
        "config": {"workload": cfg["label"], "n": n, "d": d, "k": k, "metric": cfg["metric"],
                   "seed": cfg["seed"], "arith": args.arith,
                   "parallelism": f"sharded triangle x{world} (each pair once across ranks; NCCL all-to-all of "
                                  f"column-side candidates)" if world > 1 else "one GPU, triangle sweep",
                   "l2": f"inputs {n * d * 4 / 1e9:.2f} GB > 126 MB L2 (no flush needed)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms / args.steps,
                "h2d_bytes_per_step": n * d * 4,  # whole job: every rank's input slice
                "d2h_bytes_per_step": n * klist * 8,  # whole job: every rank's result rows
                "path": e2e_path,
                "pinned_ms_per_step": e2e_pinned_ms,
                "dropin_ms_per_step": dropin_ms if not launched else None,
                "dropin_path": "build/bench_dropin: C++ knn::solve_knn (reference header, B200 drop-in), "
                               "pageable Dataset in, EngineResult.lists out, sqeuclidean fold, host clock"},
        "gpu_launches": launches,
        "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes/launch (DRAM, ncu)",
                     "peak_source": peak_src,
                     "kernel_ms": statistics.mean(sweep_ms),
                     "kernel": "tensor sweep phase, CUDA events on the solve stream: for whole problems with "
                               "n >= 393216, k <= 11, d <= 256 the 1/16 sample pass + the triangle sweep (each "
                               "unordered pair once), else the rectangular sweep",
                     "alg_flop_per_launch": alg_flop},
        "clocks": clk,
        "gpu_stats": {kk: last[kk] for kk in ("distance_evals", "rescored", "fallback_rows", "arith_used")},
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            nn = args.cpu_sample_n or CPU_SAMPLE_N.get(args.config, 65536)
            rate, t_cpu, cores, kind, sample, _ = cpu_reference_sample(cfg, nn)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                                    "seconds": t_cpu, "cpu_model": cpu_model()}
        except Exception as e:  # reported, never substituted
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if launched:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

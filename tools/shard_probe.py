"""Time row shards of C2 on one GPU (what each rank of a multi-GPU run does) (dev tool)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_0906_0231_b200 import Context, _lib, distance_by_name, generate_torch, solve_rows_torch
ctx = Context(0)
n, d, k = 1_000_000, 256, 10
x = generate_torch(ctx, n, d, 1)
m = distance_by_name("euclidean")
for parts in (1, 2, 8):
    r0, r1 = 0, n // parts
    for _ in range(2):
        _, _, st = solve_rows_torch(ctx, x, k, m, r0, r1, _lib.ARITH_TENSOR, want_stats=True)
    print(f"shard 1/{parts}: rows [{r0},{r1}) kernel_ms={st['kernel_ms']:.1f} sweep_ms={st['sweep_ms']:.1f} "
          f"fallback={st['fallback_rows']} x{parts} = {st['kernel_ms'] * parts:.1f} ms", flush=True)

"""Multi-GPU driver: query-row shards over torch.distributed.

The path shards by query rows: a row's neighbor list depends only on the
replicated reference set, so ranks exchange nothing on the data path.  The
one real exchange is the replication itself -- an NCCL broadcast of the
n x d reference set from rank 0 (the paper's per-GPU full copy, PAPER.md
§IV) -- and, when the caller wants every list in one place, a gather of the
shards' results (the reference's merge_all has nothing to do here: each row
has exactly one owner).

Backend-agnostic: the host logic is exercised with gloo on CPU in
tests/test_parallel.py; on B200s the same calls run over NCCL.
"""
from __future__ import annotations


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced query-row shard [begin, end) of `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    return n * rank // world, n * (rank + 1) // world


def shard_pairs(n: int, begin: int, end: int) -> int:
    """Unordered pairs {x, y} with at least one endpoint in [begin, end)."""
    rows = end - begin
    return rows * (n - 1) - rows * (rows - 1) // 2


def tri_unit_plan(units: int, world: int, pairs_max: int = 74) -> list[list[int]]:
    """The sharded triangle's unit ownership, from the product's host planner
    (knn_b200_tri_unit_plan): per rank, its 256-row units in launch order."""
    import ctypes

    import numpy as np

    from . import _lib
    from .engine import raise_for_status

    out = np.zeros(max(units, 1), dtype=np.uint32)
    counts = np.zeros(world, dtype=np.uint32)
    raise_for_status(_lib.load().knn_b200_tri_unit_plan(units, world, pairs_max, out.ctypes.data,
                                                        counts.ctypes.data))
    at, plan = 0, []
    for c in counts.tolist():
        plan.append(out[at:at + c].tolist())
        at += c
    return plan


def replicate(x, src: int = 0):
    """Broadcast the reference set from `src` to every rank (in place)."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(x, src=src)
    return x


def gather_lists(index, dist_, n: int, klist: int):
    """All-gather every rank's (rows x klist) shard into full n x klist
    tensors on every rank (shards are contiguous, ranks in order)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return index, dist_
    world = dist.get_world_size()
    spans = [shard_bounds(n, world, r) for r in range(world)]
    width = max(e - b for b, e in spans)  # collectives want equal sizes: pad, gather, trim

    def padded(t):
        if t.shape[0] == width:
            return t.contiguous()
        pad = torch.zeros((width - t.shape[0], klist), dtype=t.dtype, device=t.device)
        return torch.cat([t, pad])

    out_i = [torch.empty((width, klist), dtype=index.dtype, device=index.device) for _ in spans]
    out_d = [torch.empty((width, klist), dtype=dist_.dtype, device=dist_.device) for _ in spans]
    dist.all_gather(out_i, padded(index))
    dist.all_gather(out_d, padded(dist_))
    return (torch.cat([t[: e - b] for t, (b, e) in zip(out_i, spans)]),
            torch.cat([t[: e - b] for t, (b, e) in zip(out_d, spans)]))


def solve_sharded(ctx, x, k: int, metric, arith: int = 0, gather: bool = False):
    """Replicate `x` (valid on rank 0), solve this rank's shard on its GPU and
    optionally all-gather the full lists."""
    import torch.distributed as dist

    from .engine import solve_rows_torch

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    replicate(x)
    n = x.shape[0]
    b, e = shard_bounds(n, world, rank)
    idx, dd, _ = solve_rows_torch(ctx, x, k, metric, b, e, arith)
    if gather:
        return gather_lists(idx, dd, n, min(k, n - 1))
    return idx, dd

"""Multi-GPU host logic on CPU: world_size-2 gloo runs of the query-row
sharding, the reference-set broadcast and the result gather
(paper_0906_0231_b200/parallel.py).  The per-shard compute is the oracle's
sampled-row solver standing in for the GPU kernel (CPU test only); the
assembled lists must equal the single-process brute force bit for bit."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0906_0231_b200.parallel import shard_bounds, shard_pairs


def test_shard_bounds_cover_rows_once():
    for n in (2, 3, 7, 1000, 1_000_003):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_shard_pairs_sum_to_all_pairs_once_counted_per_owner():
    # pairs with >= 1 endpoint in a shard; summed over shards every pair is
    # counted once or twice -- and n(n-1)/2 when one shard owns everything
    n = 1001
    assert shard_pairs(n, 0, n) == n * (n - 1) // 2
    tot = sum(shard_pairs(n, *shard_bounds(n, 4, r)) for r in range(4))
    assert n * (n - 1) // 2 <= tot <= n * (n - 1)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, d, k, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import c_oracle
    from paper_0906_0231_b200.parallel import gather_lists, replicate

    co = c_oracle()
    # rank 0 owns the data; the others receive it through the broadcast
    x = torch.from_numpy(co.generate(n, d, 99)) if rank == 0 else torch.zeros((n, d), dtype=torch.float32)
    replicate(x)
    b, e = shard_bounds(n, world, rank)
    idx, dd = co.rows_topk(x.numpy(), k, "sqeuclidean", np.arange(b, e, dtype=np.uint32), threads=1)
    gi, gd = gather_lists(torch.from_numpy(idx.view(np.int32)), torch.from_numpy(dd), n, min(k, n - 1))
    np.save(os.path.join(out_dir, f"idx{rank}.npy"), gi.numpy())
    np.save(os.path.join(out_dir, f"dist{rank}.npy"), gd.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_shards_assemble_the_full_answer(tmp_path, world):
    n, d, k = 301, 12, 7
    mp.spawn(_worker, args=(world, _free_port(), n, d, k, str(tmp_path)), nprocs=world, join=True)
    from oracle import c_oracle

    co = c_oracle()
    ri, rd, _ = co.brute_force(co.generate(n, d, 99), k, "sqeuclidean")
    for r in range(world):
        gi = np.load(tmp_path / f"idx{r}.npy").view(np.uint32)
        gd = np.load(tmp_path / f"dist{r}.npy")
        assert np.array_equal(gi, ri)
        assert np.array_equal(gd.view(np.uint32), rd.view(np.uint32))

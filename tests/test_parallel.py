"""Multi-GPU host logic on CPU: world_size-2 gloo runs of the query-row
sharding, the reference-set broadcast and the result gather
(paper_0906_0231_b200/parallel.py).  The per-shard compute is the oracle's
sampled-row solver standing in for the GPU kernel (CPU test only); the
assembled lists must equal the single-process brute force bit for bit."""
from __future__ import annotations

import math
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


def _unit_cost(u, units):
    """tri_unit_cost (tri_shard.cuh): tiles, weighted up for low-norm units."""
    tau = max(1.0, 0.004 * units)
    return (units - u) * (1.0 + 0.9 * math.exp(-u / tau))


def test_tri_unit_plan_is_boustrophedon_and_balanced():
    """The product's host planner (knn_b200_tri_unit_plan): unit u belongs to
    lane_of_row(u) (schedule.cpp:40-44) rotated by one rank per block of
    2 * world units, every unit exactly once, and the
    per-rank work (sum of U - u) balanced like the reference's lanes
    (test_schedule.cpp:169-185).  The list triangle's static walk deals each
    rank's units to its CTA pairs (pair p: positions p, p + P, ...) by
    estimated cost, equal unit counts per round: each pair's cost within 2% of
    the mean with >= 40 units per pair.  At C2's 8-rank shape (6.6 per pair) the
    heaviest hub unit alone is over half a pair's share; the measured per-pair
    times are within 1.5 ms of 25 (profiles/r02au_cta_lpt.txt)."""
    from paper_0906_0231_b200.parallel import tri_unit_plan
    for units, world, pairs in ((3907, 8, 74), (1563, 2, 74), (38, 3, 2), (5, 8, 74), (62500, 8, 74), (3907, 1, 74),
                                (3907, 2, 74), (3907, 4, 74)):
        plan = tri_unit_plan(units, world, pairs)
        flat = sorted(u for r in plan for u in r)
        assert flat == list(range(units))
        for r, lst in enumerate(plan):
            for u in lst:
                m = u % (2 * world)
                assert ((m if m < world else 2 * world - 1 - m) + u // (2 * world)) % world == r
        if units >= 2 * world * 8:
            work = [sum(units - u for u in lst) for lst in plan]
            assert max(work) / min(work) < 1.01
        for lst in plan:
            if not lst:
                continue
            p = min(len(lst), pairs)
            counts = [len(lst[i::p]) for i in range(p)]
            assert max(counts) - min(counts) <= 1 and counts == sorted(counts, reverse=True)
            per = [sum(_unit_cost(u, units) for u in lst[i::p]) for i in range(p)]
            if len(lst) >= 40 * p:
                assert max(per) / (sum(per) / p) < 1.02
            elif len(lst) >= 3 * p:  # a hub unit is over half a pair's share here: counts stay equal
                assert max(per) / (sum(per) / p) < 1.20


def test_tri_unit_plan_queue_is_ascending(monkeypatch):
    """KNN_B200_TRI_DYN=1 (the dynamic unit queue): each rank's units stay
    ascending -- claimed heaviest first, and a column group's units with work
    are a prefix."""
    from paper_0906_0231_b200.parallel import tri_unit_plan
    monkeypatch.setenv("KNN_B200_TRI_DYN", "1")
    for units, world, pairs in ((3907, 8, 74), (1563, 2, 74)):
        plan = tri_unit_plan(units, world, pairs)
        assert sorted(u for r in plan for u in r) == list(range(units))
        for lst in plan:
            assert lst == sorted(lst)


def _tri_worker(rank, world, port, n, d, k, unit, out_dir):
    """One rank of the sharded triangle's protocol, on CPU (gloo): own units
    from the product planner; each unordered pair of the own rows' triangle
    computed once (oracle fold standing in for the GPU tile); row-side
    candidates kept, column-side candidates all-to-all'ed to the rows' owners
    and merged there -- the reference's lane heaps + merge_row
    (engine.cpp:27-59, merge.cpp:10-57) with GPUs as lanes."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import c_oracle
    from paper_0906_0231_b200.parallel import tri_unit_plan

    co = c_oracle()
    x = co.generate(n, d, 123)
    units = -(-n // unit)
    plan = tri_unit_plan(units, world, 3)
    owner = {u: r for r, lst in enumerate(plan) for u in lst}
    rows = lambda u: range(u * unit, min((u + 1) * unit, n))  # noqa: E731
    fold = lambda i, j: float(co.fold("sqeuclidean", x[max(i, j)], x[min(i, j)]))  # noqa: E731
    cand = {i: [] for u in plan[rank] for i in rows(u)}
    send = [[] for _ in range(world)]
    for u in plan[rank]:
        for i in rows(u):
            for t in range(u, units):
                for j in rows(t):
                    if j == i:
                        continue
                    dv = fold(i, j)
                    cand[i].append((dv, j))                   # row side
                    if t > u:
                        send[owner[t]].append((j, dv, i))     # column side -> row j's owner
    # all-to-all: counts, then (row, dist, index) triples as float64 (exact)
    sc = torch.tensor([len(s) for s in send], dtype=torch.int64)
    rcnt = torch.empty(world, dtype=torch.int64)
    dist.all_to_all_single(rcnt, sc)
    flat = torch.tensor([v for s in send for e in s for v in e], dtype=torch.float64).reshape(-1)
    recv = torch.empty(int(rcnt.sum()) * 3, dtype=torch.float64)
    dist.all_to_all_single(recv, flat, [int(c) * 3 for c in rcnt], [int(c) * 3 for c in sc])
    for j, dv, i in recv.reshape(-1, 3).tolist():
        cand[int(j)].append((dv, int(i)))
    out = {}
    for i, lst in cand.items():
        idx = [j for _, j in lst]
        assert len(idx) == len(set(idx)) == n - 1, f"row {i}: pair coverage broken"  # merge.cpp:22-35
        best = sorted(lst)[: min(k, n - 1)]
        out[i] = best
    np.save(os.path.join(out_dir, f"tri{rank}.npy"),
            np.array([[i, *[j for _, j in out[i]]] for i in sorted(out)], dtype=np.int64))
    np.save(os.path.join(out_dir, f"trid{rank}.npy"),
            np.array([[dv for dv, _ in out[i]] for i in sorted(out)], dtype=np.float32))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_sharded_triangle_protocol(tmp_path):
    n, d, k, unit, world = 150, 6, 5, 8, 2
    mp.spawn(_tri_worker, args=(world, _free_port(), n, d, k, unit, str(tmp_path)), nprocs=world, join=True)
    from oracle import c_oracle

    co = c_oracle()
    ri, rd, _ = co.brute_force(co.generate(n, d, 123), k, "sqeuclidean")
    seen = set()
    for r in range(world):
        a = np.load(tmp_path / f"tri{r}.npy")
        dd = np.load(tmp_path / f"trid{r}.npy")
        for row, dist_row in zip(a, dd):
            i = int(row[0])
            seen.add(i)
            assert np.array_equal(row[1:].astype(np.uint32), ri[i])
            assert np.array_equal(dist_row.view(np.uint32), rd[i].view(np.uint32))
    assert seen == set(range(n))

"""The sharded triangle (tri_shard.cuh) on one B200.

Every rank program of a world-W sharded solve runs on the one device, one
after another, with the exchanges as device copies
(knn_b200_debug_solve_sharded_loopback): boustrophedon unit ownership
(schedule.cpp:40-44), each unordered pair computed once across the ranks,
column-side candidates exchanged to the rows' owners and merged there
(merge.cpp:10-57).  The assembled lists must equal the oracle's bit for bit,
and the single-GPU solve's, for every world size.  The NCCL driver of the
same phases runs at world 1 on the box's one GPU (a communicator of one rank:
the collectives degenerate but execute).
"""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import assert_lists_bit_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_0906_0231_b200 import Context
    c = Context(0)
    yield c
    c.close()


def _metric(name):
    from paper_0906_0231_b200 import distance_by_name
    return distance_by_name(name)


def _oracle_rows(c_oracle, xh, k, metric, rows):
    om = "sqeuclidean" if metric == "euclidean" else metric
    ri, rd = c_oracle.rows_topk(xh, k, om, rows)
    return ri, (np.sqrt(rd) if metric == "euclidean" else rd)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_loopback_shards_equal_single_gpu_and_oracle(ctx, c_oracle, world):
    """n = 400000 (the triangle's default range): every row equals the
    single-GPU solve bit for bit; sampled rows equal the oracle."""
    import torch
    from paper_0906_0231_b200 import _lib, generate_torch, solve_rows_torch, solve_sharded_loopback_torch
    n, d, k = 400_000, 64, 10
    x = generate_torch(ctx, n, d, 606)
    m = _metric("euclidean")
    i1, d1, _ = solve_rows_torch(ctx, x, k, m, 0, n, _lib.ARITH_TENSOR)
    iw, dw, st, rank_ms, xbytes = solve_sharded_loopback_torch(ctx, x, k, m, world)
    torch.cuda.synchronize()
    assert st["reserved"] == 0  # no log overflow
    assert (iw == i1).all().item(), f"world {world}: indices differ from the single-GPU solve"
    assert (dw.view(torch.int32) == d1.view(torch.int32)).all().item(), f"world {world}: distance bits differ"
    rows = np.unique(np.concatenate([np.random.default_rng(world).choice(n, 48, replace=False), [0, n - 1]]))
    rows = rows.astype(np.uint32)
    ri, rd = _oracle_rows(c_oracle, x.cpu().numpy(), k, "euclidean", rows)
    assert_lists_bit_equal(iw.cpu().numpy().view(np.uint32)[rows], dw.cpu().numpy()[rows], ri, rd,
                           f"loopback world {world}")
    assert (rank_ms > 0).all() or world > 1
    if world > 1:
        assert (xbytes > 0).all()
    print(f"\n[world {world}] per-rank ms (prep, sample, sweep+bin, merge): {np.round(rank_ms, 2).tolist()}; "
          f"sent MB {np.round(xbytes / 1e6, 1).tolist()}; capture rows {st['fallback_rows']}")


@pytest.mark.parametrize("world,n,d,k,metric", [(2, 20000, 48, 7, "sqeuclidean"), (5, 9000, 40, 9, "hellinger"),
                                                (4, 3000, 200, 4, "euclidean"), (8, 1500, 17, 1, "sqeuclidean")])
def test_loopback_small_forced_all_rows(ctx, c_oracle, monkeypatch, world, n, d, k, metric):
    """KNN_B200_TRI=force: the sharded triangle at small n (ranks with few or
    no units), every row against the oracle."""
    import torch
    from paper_0906_0231_b200 import solve_sharded_loopback_torch
    monkeypatch.setenv("KNN_B200_TRI", "force")
    xh = c_oracle.generate(n, d, n + world)
    x = torch.from_numpy(xh).cuda()
    iw, dw, st, _, _ = solve_sharded_loopback_torch(ctx, x, k, _metric(metric), world)
    ri, rd = _oracle_rows(c_oracle, xh, k, metric, np.arange(n, dtype=np.uint32))
    assert_lists_bit_equal(iw.cpu().numpy().view(np.uint32), dw.cpu().numpy(), ri, rd,
                           f"forced loopback world={world} n={n} {metric}")


def test_loopback_log_overflow_falls_back(ctx, c_oracle, monkeypatch):
    """Column-side logs that overflow on any rank: the solve redoes itself
    with the rectangular sweep -- same bits."""
    import torch
    from paper_0906_0231_b200 import solve_sharded_loopback_torch
    monkeypatch.setenv("KNN_B200_TRI", "force")
    monkeypatch.setenv("KNN_B200_TRI_LOGCAP", "16")
    n, d, k = 6000, 24, 5
    xh = c_oracle.generate(n, d, 8)
    iw, dw, st, _, _ = solve_sharded_loopback_torch(ctx, torch.from_numpy(xh).cuda(), k, _metric("sqeuclidean"), 4)
    assert st["reserved"] == 1
    ri, rd = _oracle_rows(c_oracle, xh, k, "sqeuclidean", np.arange(n, dtype=np.uint32))
    assert_lists_bit_equal(iw.cpu().numpy().view(np.uint32), dw.cpu().numpy(), ri, rd, "overflow fallback")


def test_nccl_driver_world_one(c_oracle, monkeypatch):
    """The NCCL driver (run_tri_nccl: all-gather, grouped send/recv,
    reduce-scatter) on a communicator of one rank, through the public
    collective entry point knn_b200_solve_sharded_device."""
    import torch
    from paper_0906_0231_b200 import (Context, _lib, comm_broadcast_torch, comm_init, comm_unique_id,
                                      solve_rows_torch, solve_sharded_torch)
    c = Context(0)
    try:
        comm_init(c, comm_unique_id(), 0, 1)
        for n, d, k, force in ((400_000, 96, 10, False), (30_000, 33, 6, True), (5000, 20, 40, False)):
            if force:
                monkeypatch.setenv("KNN_B200_TRI", "force")
            else:
                monkeypatch.delenv("KNN_B200_TRI", raising=False)
            xh = c_oracle.generate(n, d, n)
            x = torch.from_numpy(xh).cuda()
            comm_broadcast_torch(c, x, 0)
            i1, d1, st = solve_sharded_torch(c, x, k, _metric("euclidean"), _lib.ARITH_AUTO, 0, 1, want_stats=True)
            i0, d0, _ = solve_rows_torch(c, x, k, _metric("euclidean"), 0, n, _lib.ARITH_AUTO)
            assert (i0 == i1).all().item() and (d0.view(torch.int32) == d1.view(torch.int32)).all().item()
            rows = np.unique(np.concatenate([np.random.default_rng(n).choice(n, 32, replace=False), [0, n - 1]]))
            ri, rd = _oracle_rows(c_oracle, xh, k, "euclidean", rows.astype(np.uint32))
            assert_lists_bit_equal(i1.cpu().numpy().view(np.uint32)[rows], d1.cpu().numpy()[rows], ri, rd,
                                   f"nccl world 1 n={n}")
    finally:
        c.close()


def test_solve_multi_nccl_path_one_gpu(c_oracle):
    """knn_b200_solve_multi (the drop-in's n_lanes) with the broadcast path;
    on one GPU every lane count maps to one device."""
    from paper_0906_0231_b200 import Dataset, EngineOptions, solve_knn, squared_euclidean
    x = c_oracle.generate(400_000, 16, 3)
    rows = np.random.default_rng(3).choice(400_000, 24, replace=False).astype(np.uint32)
    ri, rd = c_oracle.rows_topk(x, 10, "sqeuclidean", rows)
    for lanes in (1, 4):
        r = solve_knn(Dataset.from_array(x), squared_euclidean(), EngineOptions(k=10, n_lanes=lanes))
        assert_lists_bit_equal(r.index[rows], r.distance[rows], ri, rd, f"solve_knn lanes={lanes}")


@pytest.mark.parametrize("world,n,d,k,metric", [(2, 20000, 48, 30, "sqeuclidean"), (3, 9000, 300, 100, "euclidean"),
                                                (8, 12000, 64, 20, "cosine"), (5, 4000, 20, 64, "hellinger")])
def test_loopback_threshold_triangle_all_rows(ctx, c_oracle, monkeypatch, world, n, d, k, metric):
    """The threshold triangle (10 < k <= 128) sharded the same way: every
    pair once across the ranks, both endpoints' candidates binned by owner,
    the capture rescore at the owner -- every row against the oracle."""
    import torch
    from oracle import normalize_rows
    from paper_0906_0231_b200 import solve_sharded_loopback_torch
    monkeypatch.setenv("KNN_B200_TCAP", "force")
    xh = c_oracle.generate(n, d, n + world)
    if metric == "cosine":
        xh = normalize_rows(xh)
    x = torch.from_numpy(np.ascontiguousarray(xh)).cuda()
    iw, dw, st, rank_ms, xbytes = solve_sharded_loopback_torch(ctx, x, k, _metric(metric), world)
    assert st["reserved"] == 0
    ri, rd = _oracle_rows(c_oracle, xh, k, metric, np.arange(n, dtype=np.uint32))
    assert_lists_bit_equal(iw.cpu().numpy().view(np.uint32), dw.cpu().numpy(), ri, rd,
                           f"threshold-triangle loopback world={world} n={n} {metric}")

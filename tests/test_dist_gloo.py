"""Multi-rank path on CPU: world_size 2 over gloo.  Each rank owns a contiguous
shard; the merged top-k (all_gather + (d2, id) merge) must equal the exact
top-k over the union, computed by the oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1610_07328_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, payload, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids, d2, ncand, cnt, k = payload[rank]
        mi, md, nc, cc = D.merge_across_ranks(torch.from_numpy(ids), torch.from_numpy(d2),
                                              torch.from_numpy(ncand), torch.from_numpy(cnt), k)
        if rank == 0:
            out_q.put((mi.numpy(), md.numpy(), nc.numpy(), cc.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for N, W in [(10, 3), (1_000_000, 8), (7, 8), (64_000_000, 8)]:
        rs = [D.shard_range(N, r, W) for r in range(W)]
        assert rs[0][0] == 0 and rs[-1][1] == N
        assert all(rs[i][1] == rs[i + 1][0] for i in range(W - 1))
        assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_merge_local_matches_lexsort():
    rng = np.random.default_rng(0)
    ids = rng.integers(0, 50, size=(6, 30)).astype(np.int64)
    d2 = rng.integers(0, 5, size=(6, 30)).astype(np.float64)  # many exact ties
    ids[:, -3:] = -1
    d2[:, -3:] = np.inf
    mi, md, n = D.merge_topk_local(torch.from_numpy(ids), torch.from_numpy(d2), 10)
    ri, rd = D.merge_numpy([(ids, d2)], 10)
    assert np.array_equal(mi.numpy(), ri) and np.array_equal(md.numpy(), rd)


def test_two_rank_merge_equals_global_topk():
    """Shard a cascade problem over 2 gloo ranks and check against the oracle."""
    from fixture_data import case_data
    from oracle import oracle as O

    X, Q, _, band = case_data("rw512")
    N, m = X.shape
    r = O.radius(band, m)
    k = 10
    rng = np.random.default_rng(1)
    payload = []
    full_cand = []
    per_rank = []
    for rank in range(2):
        lo, hi = D.shard_range(N, rank, 2)
        ids_r = np.full((len(Q), k), -1, np.int64)
        d2_r = np.full((len(Q), k), np.inf)
        nc = np.zeros(len(Q), np.int64)
        for qi, q in enumerate(Q):
            cand = np.sort(rng.choice(np.arange(lo, hi), size=120, replace=False))
            full_cand.append((qi, cand))
            bi, bd = O.brute_force_topk_over(X, cand, q, r, k)
            ids_r[qi, :len(bi)] = bi
            d2_r[qi, :len(bd)] = bd
            nc[qi] = len(cand)
        cnt = np.tile(np.arange(5, dtype=np.int64), (len(Q), 1)) * (rank + 1)
        payload.append((ids_r, d2_r, nc, cnt, k))
        per_rank.append((ids_r, d2_r))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, 2, port, payload, q)) for rk in range(2)]
    for p in procs:
        p.start()
    mi, md, nc, cc = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for qi, qv in enumerate(Q):
        cand = np.concatenate([c for (qq, c) in full_cand if qq == qi])
        gi, gd = O.brute_force_topk_over(X, cand, qv, r, k)
        assert mi[qi].tolist() == gi.tolist()
        assert md[qi].tolist() == gd.tolist()
        assert nc[qi] == len(cand)
    assert cc[0].tolist() == (np.arange(5) * 3).tolist()

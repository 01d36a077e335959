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


def _sharded_worker(rank, world, port, fallback, out_q):
    """One rank of a 2-shard index (oracle shard indexes as the per-rank
    engine): sharded_query must equal the single-index answer."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from fixture_data import case_data
        from oracle import oracle as O

        X, Q, _, band = case_data("rw512")
        X = X[:1200]
        Qs = _mixed_queries(X, Q)
        N, m = X.shape
        lo, hi = D.shard_range(N, rank, world)
        oidx = O.build_index(X[lo:hi], 80, 3, 15, 20, 4, 0, band)
        r = O.radius(band, m)

        def local(Qt, k):
            res = O.query_batch(oidx, Qt.numpy(), k)
            ids = np.where(res["ids"] >= 0, res["ids"] + lo, -1)
            st = (res["n_cand"] == 0).astype(np.int32)
            return (torch.from_numpy(ids), torch.from_numpy(res["d2"]), torch.from_numpy(res["n"]),
                    torch.from_numpy(res["n_cand"]), torch.from_numpy(res["counters"]), torch.from_numpy(st))

        def exact(Qt, k):
            nq = Qt.shape[0]
            ids = np.full((nq, k), -1, np.int64)
            d2 = np.full((nq, k), np.inf)
            for i, qv in enumerate(Qt.numpy()):
                bi, bd = O.brute_force_topk_over(X, np.arange(lo, hi), qv, r, k)
                ids[i, :len(bi)] = bi
                d2[i, :len(bd)] = bd
            nc = np.full(nq, hi - lo, np.int64)
            return (torch.from_numpy(ids), torch.from_numpy(d2), torch.from_numpy((ids >= 0).sum(1).astype(np.int32)),
                    torch.from_numpy(nc), torch.zeros((nq, 5), dtype=torch.int64),
                    torch.full((nq,), 2, dtype=torch.int32))

        out = D.sharded_query(torch.from_numpy(Qs), 10, local, exact, fallback_on_empty=fallback)
        if rank == 0:
            out_q.put(tuple(t.numpy() for t in out))
    finally:
        dist.destroy_process_group()


def _mixed_queries(X, Q):
    """Warped queries (non-empty R) plus white-noise series (R empty on both
    shards) and one database row (R non-empty)."""
    rng = np.random.default_rng(9)
    noise = rng.standard_normal((3, X.shape[1]))
    noise = ((noise - noise.mean(1, keepdims=True)) / noise.std(1, keepdims=True)).astype(np.float32)
    return np.ascontiguousarray(np.concatenate([Q[:4], noise, X[7:8]]), dtype=np.float32)


@pytest.mark.parametrize("fallback", [False, True])
def test_sharded_query_statuses_equal_single_index(fallback):
    """Global semantics over R = U_g R_g (index.py:233-243): no-candidates only
    when every shard's R_g is empty; fallback searches all shards exactly."""
    from fixture_data import case_data
    from oracle import oracle as O

    X, Q, _, band = case_data("rw512")
    X = X[:1200]
    Qs = _mixed_queries(X, Q)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(rk, 2, port, fallback, q)) for rk in range(2)]
    for p in procs:
        p.start()
    ids, d2, n_out, n_cand, _, status = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = O.query_batch(O.build_index(X, 80, 3, 15, 20, 4, 0, band), Qs, 10)
    r = O.radius(band, X.shape[1])
    saw_empty = False
    for i, qv in enumerate(Qs):
        if full["n_cand"][i] == 0:
            saw_empty = True
            if fallback:
                bi, bd = O.brute_force_topk_over(X, np.arange(X.shape[0]), qv, r, 10)
                assert status[i] == 2 and ids[i].tolist() == bi.tolist() and d2[i].tolist() == bd.tolist()
                assert n_cand[i] == X.shape[0]
            else:
                assert status[i] == 1 and n_out[i] == 0 and n_cand[i] == 0
        else:
            n = int(full["n"][i])
            assert status[i] == 0 and n_cand[i] == full["n_cand"][i]
            assert ids[i][:n].tolist() == full["ids"][i][:n].tolist()
            assert d2[i][:n].tolist() == full["d2"][i][:n].tolist()
    assert saw_empty

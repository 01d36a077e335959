"""Sharded index over the GPUs of one node (one process per GPU).

The database shards by series id (contiguous ranges): every
rank builds its own bucket tables over its rows with global ids, so the
build needs no collective.  Queries are replicated; each rank answers the
batch over its shard (R_g, exact local top-k by (d2, id)), and the global
answer is the (d2, id) merge of the per-rank lists, which equals the exact
top-k of R = U_g R_g.  The exchange is one all_gather of the per-rank top-k
(d2 f64, id i64) and one all_reduce(sum) of |R_g| and the cascade counters,
all batched over the whole query batch.

Statuses follow the reference over the union R (index.py:233-243): a query
is "no-candidates" only when every R_g is empty (|R| = sum of |R_g| is
all-reduced first), and with fallback_on_empty such queries run the exact
search over every shard (SSH_QUERY_EXACT) and merge the same way
(`sharded_query`), so the global answer equals the single-index one.
"""

from __future__ import annotations

import os

import numpy as np


def _torch():
    import torch

    return torch


def init_from_env(backend: str = "nccl"):
    """Initialise torch.distributed from RANK/WORLD_SIZE/MASTER_* if present."""
    torch = _torch()
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def shard_range(N: int, rank: int, world: int):
    """Contiguous id range [lo, hi) of `rank` (balanced to within one row)."""
    base, extra = divmod(N, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def merge_topk_local(ids, d2, k: int):
    """(d2, id)-lexicographic top-k of concatenated candidate lists.

    ids/d2: (nq, C) tensors, id -1 / d2 inf for empty slots.  Returns
    (ids (nq, k), d2 (nq, k), n (nq,))."""
    torch = _torch()
    big = torch.iinfo(torch.int64).max
    idk = torch.where(ids < 0, torch.full_like(ids, big), ids)
    o1 = torch.argsort(idk, dim=1, stable=True)
    d2s = torch.gather(d2, 1, o1)
    ids1 = torch.gather(ids, 1, o1)
    o2 = torch.argsort(d2s, dim=1, stable=True)
    d2o = torch.gather(d2s, 1, o2)[:, :k]
    ido = torch.gather(ids1, 1, o2)[:, :k]
    n = (ido >= 0).sum(dim=1).to(torch.int32)
    return ido, d2o, n


def merge_topk_device(g_ids, g_d2, lists: int, nq: int, k: int):
    """ssh_merge_topk on the device: g_ids / g_d2 (lists * nq, k_in) in the
    all_gather layout (rank-major) -> (ids (nq, k), d2 (nq, k), n (nq,))."""
    torch = _torch()
    from . import _native as nat

    k_in = int(g_ids.shape[1])
    dev = g_ids.device
    ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
    d2 = torch.empty((nq, k), dtype=torch.float64, device=dev)
    n = torch.empty(nq, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    nat.check(nat.lib().ssh_merge_topk(nat.ptr(g_ids.contiguous()), nat.ptr(g_d2.contiguous()), nq, lists, k_in, k,
                                       nat.ptr(ids), nat.ptr(d2), nat.ptr(n), __import__("ctypes").c_void_p(stream)),
              "ssh_merge_topk")
    return ids, d2, n


def merge_across_ranks(ids, d2, n_cand, counters, k: int, group=None):
    """All-gather per-rank top-k and merge; all-reduce |R_g| and counters.

    ids (nq, k) int64 global ids (-1 pad), d2 (nq, k) f64 (inf pad),
    n_cand (nq,) int64, counters (nq, 5) int64 — all on the rank's device
    (CPU tensors under gloo)."""
    torch = _torch()
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if world == 1:
        return ids, d2, n_cand, counters
    nq = ids.shape[0]
    if ids.is_cuda and dist.get_backend(group) == "gloo":
        # gloo collectives run on host tensors (functional tests of the sharded
        # path on one GPU); the merge itself still runs on the device
        dev = ids.device
        g_ids = torch.empty((world * nq, k), dtype=ids.dtype)
        g_d2 = torch.empty((world * nq, k), dtype=d2.dtype)
        dist.all_gather_into_tensor(g_ids, ids.cpu().contiguous(), group=group)
        dist.all_gather_into_tensor(g_d2, d2.cpu().contiguous(), group=group)
        red = torch.cat([n_cand.view(nq, 1), counters], dim=1).cpu().contiguous()
        dist.all_reduce(red, op=dist.ReduceOp.SUM, group=group)
        mids, md2, _ = merge_topk_device(g_ids.to(dev), g_d2.to(dev), world, nq, k)
        red = red.to(dev)
        return mids, md2, red[:, 0].contiguous(), red[:, 1:].contiguous()
    g_ids = torch.empty((world * nq, k), dtype=ids.dtype, device=ids.device)
    g_d2 = torch.empty((world * nq, k), dtype=d2.dtype, device=d2.device)
    dist.all_gather_into_tensor(g_ids, ids.contiguous(), group=group)
    dist.all_gather_into_tensor(g_d2, d2.contiguous(), group=group)
    red = torch.cat([n_cand.view(nq, 1), counters], dim=1).contiguous()
    dist.all_reduce(red, op=dist.ReduceOp.SUM, group=group)
    if g_ids.is_cuda:
        mids, md2, _ = merge_topk_device(g_ids, g_d2, world, nq, k)
    else:  # host tensors (gloo tests of the merge logic without a GPU)
        cat_ids = g_ids.view(world, nq, k).permute(1, 0, 2).reshape(nq, world * k)
        cat_d2 = g_d2.view(world, nq, k).permute(1, 0, 2).reshape(nq, world * k)
        mids, md2, _ = merge_topk_local(cat_ids, cat_d2, k)
    return mids, md2, red[:, 0].contiguous(), red[:, 1:].contiguous()


def merge_numpy(parts, k: int):
    """Reference merge for tests: parts = [(ids, d2)] per rank -> (ids, d2)."""
    ids = np.concatenate([p[0] for p in parts], axis=1)
    d2 = np.concatenate([p[1] for p in parts], axis=1)
    out_i = np.full((ids.shape[0], k), -1, dtype=np.int64)
    out_d = np.full((ids.shape[0], k), np.inf)
    for q in range(ids.shape[0]):
        sel = ids[q] >= 0
        order = np.lexsort((ids[q][sel], d2[q][sel]))[:k]
        out_i[q, :order.shape[0]] = ids[q][sel][order]
        out_d[q, :order.shape[0]] = d2[q][sel][order]
    return out_i, out_d


def sharded_query(Q, k: int, local, exact=None, fallback_on_empty: bool = False, group=None):
    """query_index_batch over a series-sharded index (index.py:204-273).

    local(Q, k) -> (ids, d2, n_out, n_cand, counters, status) of this rank's
    shard, run WITHOUT the empty-R fallback; exact(Qsub, k) -> the same tuple
    for an exact search of Qsub over the rank's shard (dtw.py:293-326).
    Returns the merged tuple (identical on every rank): ids/d2 the exact
    (d2, id) top-k of R = U_g R_g, n_cand = |R|, counters summed, status 0 ok,
    1 no-candidates (every R_g empty), 2 fallback (exact over all shards)."""
    torch = _torch()
    ids, d2, _, n_cand, counters, _ = local(Q, k)
    mids, md2, nc, cnt = merge_across_ranks(ids, d2, n_cand, counters, k, group=group)
    empty = nc == 0
    status = torch.zeros(nc.shape, dtype=torch.int32, device=nc.device)
    if bool(empty.any()):  # same decision on every rank (nc is all-reduced)
        if fallback_on_empty and exact is not None:
            sub = torch.nonzero(empty).flatten()
            eids, ed2, _, enc, ecnt, _ = exact(Q[sub.to(Q.device)].contiguous(), k)
            fi, fd, fnc, fc = merge_across_ranks(eids, ed2, enc, ecnt, k, group=group)
            sub = sub.to(mids.device)
            mids[sub] = fi.to(mids.device)
            md2[sub] = fd.to(md2.device)
            nc[sub] = fnc.to(nc.device)
            cnt[sub] = fc.to(cnt.device)
            status[sub] = 2
        else:
            status[empty] = 1
    n_out = (mids >= 0).sum(dim=1).to(torch.int32)
    return mids, md2, n_out, nc, cnt, status


def index_query_fns(index):
    """(local, exact) callables of sharded_query for a device SshIndex shard."""
    from .index import query_batch_device

    def local(Q, k):
        return query_batch_device(index, Q, k, False)

    def exact(Q, k):
        return query_batch_device(index, Q, k, False, exact=True)

    return local, exact


def _pad_k(t, k: int, fill):
    torch = _torch()
    if t.shape[1] == k:
        return t
    pad = torch.full((t.shape[0], k - t.shape[1]), fill, dtype=t.dtype, device=t.device)
    return torch.cat([t, pad], dim=1)


def query_index_batch_sharded(index, Q, k: int, fallback_on_empty: bool = False, group=None) -> list:
    """query_index_batch (index.py:204-273) over a series-sharded index: every
    rank of `group` calls it with its own shard (an SshIndex built with
    id_base = the shard's first global id) and the same queries, and every
    rank gets the same list of QueryResult — the exact top-k of the union
    R = U_g R_g, |R| summed, statuses and the empty-R fallback decided over
    R (sharded_query).  k is clamped to the total series count, with the
    reference's warning."""
    import time

    import torch.distributed as dist

    from .index import _prepare_queries, _results_from_arrays, _to_host

    torch = _torch()
    Qd = _prepare_queries(index, Q)
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    gloo = dist.get_backend(group) == "gloo"
    n_tot = torch.tensor([index.n_series], dtype=torch.int64, device="cpu" if gloo else Qd.device)
    dist.all_reduce(n_tot, op=dist.ReduceOp.SUM, group=group)
    N = int(n_tot.item())
    warning = None
    if k > N:
        warning = f"k={k} exceeds index size {N}; returning at most {N} series"
        k = N
    kl = min(k, index.n_series)
    local_fn, exact_fn = index_query_fns(index)

    def local(Qs, _k):
        ids, d2, n_out, nc, cnt, st = local_fn(Qs, kl)
        return _pad_k(ids, k, -1), _pad_k(d2, k, float("inf")), n_out, nc, cnt, st

    def exact(Qs, _k):
        ids, d2, n_out, nc, cnt, st = exact_fn(Qs, kl)
        return _pad_k(ids, k, -1), _pad_k(d2, k, float("inf")), n_out, nc, cnt, st

    t0 = time.perf_counter()
    with index.context().use():
        dev = sharded_query(Qd, k, local, exact, fallback_on_empty, group=group)
        ids, d2, n_out, n_cand, counters, status = _to_host(dev, index.device)
    dt = time.perf_counter() - t0
    return _results_from_arrays(ids, d2, n_out, n_cand, counters, status, N, dt, warning)

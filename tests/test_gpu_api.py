"""Device parity of the reference-facing surface beyond the index hot path:
the public DTW utilities (dtw.py:239-284), the wide-band warp-wavefront DTW
(any radius), concurrent queries on one index, the reference's timing keys,
sharded indexes (id_base) merged across shards, and shard persistence."""

import concurrent.futures as cf

import numpy as np
import pytest

from fixture_data import case_data
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _params(band=0.05, K=4, **kw):
    import paper_1610_07328_b200 as ssh

    d = dict(W=80, delta=3, n=15, d=20, seed=0, band=band, K=K)
    d.update(kw)
    return ssh.SshParams(**d)


def test_dtw_utilities_golden(cuda, golden):
    """dtw_distance / build_envelope / lb_keogh / lb_keogh2 / lb_kim on the
    reference-generated float64 pairs: bit-identical to sshts.dtw."""
    import paper_1610_07328_b200 as ssh

    for p in golden["dtw"]["pairs"]:
        x, y = np.array(p["x"]), np.array(p["y"])
        wp = ssh.WarpingParams(band=p["band"])
        assert ssh.dtw_distance(x, y, wp) == float(np.sqrt(p["d2"]))
        env = ssh.build_envelope(y, wp)
        assert env.upper.tolist() == p["upper"] and env.lower.tolist() == p["lower"]
        assert ssh.lb_keogh(env, x) == float(np.sqrt(p["lb_keogh_sq"]))
        assert ssh.lb_keogh2(x, y, wp) == float(np.sqrt(p["lb_keogh_sq"]))
        d0, dm = x[0] - y[0], x[-1] - y[-1]
        assert ssh.lb_kim(x, y) == float(np.sqrt(d0 * d0 + dm * dm))
    one = ssh.dtw_distance(np.array([1.0, 2, 3]), np.array([2.0, 3, 4]), ssh.WarpingParams(band=1.0))
    assert one == golden["dtw"]["spec_sqrt2"]
    with pytest.raises(ValueError, match="length mismatch"):
        ssh.dtw_distance(np.zeros(3), np.zeros(4))


@pytest.mark.parametrize("m,r", [(700, 0), (700, 5), (700, 31), (700, 32), (700, 100), (2048, 205), (900, 600)])
def test_dtw_pairs_any_radius(cuda, m, r):
    """The band-chunked warp wavefront (C = ceil((2r+1)/32) cells per lane,
    2 <= C <= 32) and the row kernel beyond it: bit-identical to the oracle's
    reference recurrence, with and without the row-minimum abandon."""
    import paper_1610_07328_b200 as ssh

    rng = np.random.default_rng(r + m)
    X = np.cumsum(rng.standard_normal((12, m)), axis=1)
    Y = np.cumsum(rng.standard_normal((12, m)), axis=1)
    wp = ssh.WarpingParams(band=r / m)
    assert wp.radius(m) == r
    got = ssh.dtw_pairs(X, Y, wp)
    want = np.sqrt([O.dtw_sq(X[i], Y[i], r) for i in range(12)])
    assert got.tolist() == want.tolist()
    ab = float(np.median(want))
    got_ab = ssh.dtw_pairs(X, Y, wp, abandon_above=ab)
    want_ab = np.sqrt([O.dtw_sq(X[i], Y[i], r, ab * ab) for i in range(12)])
    assert got_ab.tolist() == want_ab.tolist()


@pytest.mark.parametrize("band", [0.12, 0.2, 0.45])
def test_query_wide_band_vs_oracle(cuda, band):
    """Radii 61 / 102 / 230 at m = 512 take the wide-band wavefront DTW in the
    query waves (and the band-chunked f64 rescoring): ids, |R| and squared
    distances identical to the oracle cascade."""
    import paper_1610_07328_b200 as ssh

    X, Q, _, _ = case_data("rw512")
    p = _params(band, K=4)
    idx = ssh.build_index(ssh.Dataset(X), p)
    oidx = O.build_index(X, 80, 3, 15, 20, 4, 0, band)
    ores = O.query_batch(oidx, Q, 10)
    for i, r in enumerate(ssh.query_index_batch(idx, Q, 10)):
        n = int(ores["n"][i])
        assert r.stats.candidates == int(ores["n_cand"][i]), i
        assert r.ids == ores["ids"][i][:n].tolist(), i
        assert r.distances == np.sqrt(ores["d2"][i][:n]).tolist(), i


def test_concurrent_queries_threadpool(cuda):
    """SPEC.md:424 / bench.py:129-133: query_index from 8 threads on one index
    (each thread on its own CUDA stream) equals serial calls."""
    import torch

    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data("rw1024")
    idx = ssh.build_index(ssh.Dataset(X), _params(band))
    serial = [ssh.query_index(idx, q, 10) for q in Q]

    def work(i):
        with torch.cuda.stream(torch.cuda.Stream()):
            return ssh.query_index(idx, Q[i], 10)

    for _ in range(2):
        with cf.ThreadPoolExecutor(8) as ex:
            par = list(ex.map(work, range(len(Q))))
        for a, b in zip(serial, par):
            assert (a.ids, a.distances, a.status, a.stats) == (b.ids, b.distances, b.status, b.stats)


def test_timings_keys_cli_style(cuda, golden):
    """QueryResult.timings carries the reference's "hash"/"probe"/"rerank"
    seconds, so the reference CLI's report loop (cli.py:172-186) runs
    unchanged against the drop-in."""
    import io

    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data("rw512")
    idx = ssh.build_index(ssh.Dataset(X), _params(band))
    out, err = io.StringIO(), io.StringIO()
    for qi in range(3):
        q = ssh.z_normalize(ssh.TimeSeries(np.asarray(Q[qi], dtype=np.float64))) if idx.normalized else Q[qi]
        res = ssh.query_index(idx, q, 10, fallback_on_empty=False)
        s = res.stats
        print(f"# query {qi}: status={res.status} candidates={s.candidates} "
              f"hash_pruned={s.hash_pruned_fraction:.6f} total_pruned={s.total_pruned_fraction:.6f}", file=out)
        for rank, (sid, dist) in enumerate(zip(res.ids, res.distances), start=1):
            print(f"{rank},{sid},{dist:.10g}", file=out)
        print(f"timings: hash={res.timings['hash']:.4f}s probe={res.timings['probe']:.4f}s "
              f"rerank={res.timings['rerank']:.4f}s", file=err)
        assert all(res.timings[key] >= 0.0 for key in ("hash", "probe", "rerank"))
        assert res.timings["hash"] + res.timings["probe"] + res.timings["rerank"] > 0.0
    assert out.getvalue().count("# query") == 3


def test_id_base_shards_merge_equals_single_index(cuda):
    """3 id_base shards of one dataset on one GPU, merged by
    (d2, id) with summed |R_g|, equal the single index and the oracle; a query
    with R empty on every shard is "no-candidates" (and exact under fallback)."""
    import torch

    import paper_1610_07328_b200 as ssh
    from paper_1610_07328_b200 import dist as D
    from paper_1610_07328_b200.index import query_batch_device

    X, Q, _, band = case_data("rw1024")
    rng = np.random.default_rng(9)
    noise = rng.standard_normal((2, X.shape[1]))
    noise = ((noise - noise.mean(1, keepdims=True)) / noise.std(1, keepdims=True)).astype(np.float32)
    Qs = np.ascontiguousarray(np.concatenate([Q, noise]), dtype=np.float32)
    p = _params(band)
    Xd = torch.from_numpy(X).cuda()
    Qd = torch.from_numpy(Qs).cuda()
    N = X.shape[0]
    single = ssh.query_index_batch(ssh.build_index(ssh.Dataset(Xd), p), Qs, 10, fallback_on_empty=True)
    parts = []
    for g in range(3):
        lo, hi = D.shard_range(N, g, 3)
        idx = ssh.build_index(ssh.Dataset(Xd[lo:hi]), p, id_base=lo)
        parts.append((idx, query_batch_device(idx, Qd, 10)))
    ids = torch.cat([o[0] for _, o in parts], dim=1)
    d2 = torch.cat([o[1] for _, o in parts], dim=1)
    mi, md, n = D.merge_topk_local(ids, d2, 10)
    ncand = sum(o[3] for _, o in parts)
    oidx = O.build_index(X, 80, 3, 15, 20, 4, 0, band)
    ores = O.query_batch(oidx, Qs, 10)
    r = O.radius(band, X.shape[1])
    empty = 0
    for i in range(Qs.shape[0]):
        k_i = int(ores["n"][i])
        assert int(ncand[i]) == int(ores["n_cand"][i]) == single[i].stats.candidates or single[i].status == "fallback"
        if ores["n_cand"][i] == 0:
            empty += 1
            assert int(n[i]) == 0
            bi, bd = O.brute_force_topk_over(X, np.arange(N), Qs[i], r, 10)
            assert single[i].status == "fallback" and single[i].ids == bi.tolist()
            # the sharded exact fallback: every shard searched exactly, merged
            ex = [query_batch_device(idx, Qd[i:i + 1], 10, exact=True) for idx, _ in parts]
            ei, ed, _ = D.merge_topk_local(torch.cat([e[0] for e in ex], 1), torch.cat([e[1] for e in ex], 1), 10)
            assert ei[0].tolist() == bi.tolist() and ed[0].tolist() == bd.tolist()
            continue
        assert mi[i][:k_i].tolist() == ores["ids"][i][:k_i].tolist() == single[i].ids
        assert md[i][:k_i].tolist() == ores["d2"][i][:k_i].tolist()
    assert empty >= 1


def test_shard_save_load_round_trip(cuda, tmp_path):
    """save_index of an id_base shard writes local ids (the file describes its
    own rows); load_index(id_base=...) restores the global numbering."""
    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data("rw512")
    p = _params(band, K=1)
    lo = X.shape[0] // 2
    idx = ssh.build_index(ssh.Dataset(X[lo:]), p, id_base=lo)
    ssh.save_index(idx, tmp_path / "s.sshi")
    back = ssh.load_index(tmp_path / "s.sshi", id_base=lo)
    a = ssh.query_index_batch(idx, Q[:4], 10)
    b = ssh.query_index_batch(back, Q[:4], 10)
    assert [r.ids for r in a] == [r.ids for r in b] and all(min(r.ids) >= lo for r in a if r.ids)
    assert [r.distances for r in a] == [r.distances for r in b]


def _sharded_worker(rank, world, port, band, out_path):
    """One rank of test_query_index_batch_sharded_two_processes (gloo, cuda:0)."""
    import os
    import pickle

    import torch
    import torch.distributed as dist

    import paper_1610_07328_b200 as ssh
    from fixture_data import case_data as cd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    X, Q, _, _ = cd("rw1024")
    rng = np.random.default_rng(9)
    noise = rng.standard_normal((2, X.shape[1]))
    noise = ((noise - noise.mean(1, keepdims=True)) / noise.std(1, keepdims=True)).astype(np.float32)
    Qs = np.ascontiguousarray(np.concatenate([Q, noise]), dtype=np.float32)
    lo, hi = ssh.shard_range(X.shape[0], rank, world)
    idx = ssh.build_index(ssh.Dataset(torch.from_numpy(X[lo:hi]).cuda()), _params(band), id_base=lo)
    got = {}
    for fb in (False, True):
        res = ssh.query_index_batch_sharded(idx, Qs, 10, fallback_on_empty=fb)
        got[fb] = [(r.ids, r.distances, r.status, r.stats.candidates, r.stats.n_indexed) for r in res]
    big = ssh.query_index_batch_sharded(idx, Qs[:2], X.shape[0] + 5)
    got["big"] = [(r.ids, r.warning) for r in big]
    if rank == 0:
        with open(out_path, "wb") as f:
            pickle.dump(got, f)
    dist.barrier()
    dist.destroy_process_group()


def test_query_index_batch_sharded_two_processes(cuda, tmp_path):
    """The public sharded API with two real ranks (two processes on cuda:0
    over gloo; functional, not a performance claim): every status, id list,
    distance and |R| equals the single-index query_index_batch, with and
    without the empty-R fallback, and k > N_total clamps with the warning."""
    import pickle
    import socket

    import torch
    import torch.multiprocessing as mp

    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data("rw1024")
    rng = np.random.default_rng(9)
    noise = rng.standard_normal((2, X.shape[1]))
    noise = ((noise - noise.mean(1, keepdims=True)) / noise.std(1, keepdims=True)).astype(np.float32)
    Qs = np.ascontiguousarray(np.concatenate([Q, noise]), dtype=np.float32)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "sharded.pkl"
    mp.spawn(_sharded_worker, args=(2, port, band, str(out)), nprocs=2, join=True)
    got = pickle.loads(out.read_bytes())
    idx = ssh.build_index(ssh.Dataset(torch.from_numpy(X).cuda()), _params(band))
    for fb in (False, True):
        want = [(r.ids, r.distances, r.status, r.stats.candidates, r.stats.n_indexed)
                for r in ssh.query_index_batch(idx, Qs, 10, fallback_on_empty=fb)]
        assert got[fb] == want
    assert any(w[2] == "no-candidates" for w in got[False]) and any(w[2] == "fallback" for w in got[True])
    big = ssh.query_index_batch(idx, Qs[:2], X.shape[0] + 5)
    assert got["big"] == [(r.ids, r.warning) for r in big]


@pytest.mark.parametrize("lists,k_in,k_out", [(2, 10, 10), (8, 10, 10), (3, 64, 20), (8, 2048, 2048), (5, 7, 40)])
def test_merge_topk_kernel_matches_lexsort(cuda, lists, k_in, k_out):
    """ssh_merge_topk (the cross-shard merge) against a numpy lexsort of the
    concatenated per-shard lists: exact d2 ties broken by id, inf distances
    before padding, short lists padded with id -1 / +inf."""
    import torch

    from paper_1610_07328_b200 import dist as D

    rng = np.random.default_rng(lists * 1000 + k_in)
    nq = 37
    parts = []
    for g in range(lists):
        ids = np.full((nq, k_in), -1, dtype=np.int64)
        d2 = np.full((nq, k_in), np.inf)
        for q in range(nq):
            n = int(rng.integers(0, k_in + 1))
            cand_ids = rng.choice(10 * k_in + 10, size=n, replace=False) * lists + g  # disjoint across shards
            vals = np.round(rng.random(n) * 4) / 4  # many exact ties
            vals[rng.random(n) < 0.05] = np.inf
            o = np.lexsort((cand_ids, vals))
            ids[q, :n] = cand_ids[o]
            d2[q, :n] = vals[o]
        parts.append((ids, d2))
    g_ids = torch.from_numpy(np.concatenate([p[0] for p in parts])).cuda()
    g_d2 = torch.from_numpy(np.concatenate([p[1] for p in parts])).cuda()
    mi, md, n = D.merge_topk_device(g_ids, g_d2, lists, nq, k_out)
    want_i, want_d = D.merge_numpy(parts, k_out)
    assert np.array_equal(mi.cpu().numpy(), want_i)
    assert np.array_equal(md.cpu().numpy(), want_d)
    assert np.array_equal(n.cpu().numpy(), (want_i >= 0).sum(1))


@pytest.mark.parametrize("m,bits,f64", [(512, 64, False), (512, 100, True), (301, 16, False), (1024, 256, True),
                                         (96, 300, False)])
def test_srp_tensor_cores_vs_f64(cuda, m, bits, f64):
    """srp_matrix on the tensor cores (tcgen05 TF32 screen + f64 recheck; bits
    > 256 take the SIMT fp32 path) equals the SIMT kernel and numpy's f64
    product signs (index.py:420-423) wherever the f64 value is not within a
    few ulps of zero; float64 inputs are rechecked in float64."""
    import paper_1610_07328_b200 as ssh

    rng = np.random.default_rng(m + bits)
    X = np.cumsum(rng.standard_normal((3000, m)), axis=1)
    X = (X - X.mean(1, keepdims=True)) / X.std(1, keepdims=True)
    X[5] = 0.0  # all-zero row: every projection is 0 -> +1
    Xin = X if f64 else X.astype(np.float32)
    st = {}
    got = ssh.srp_matrix(Xin, bits, 7, stats=st)
    simt = ssh.srp_matrix(Xin, bits, 7, tensor_cores=False)
    proj = np.asarray(Xin, dtype=np.float64) @ ssh.srp_vectors(m, bits, 7).T
    want = np.where(proj >= 0.0, 1, -1).astype(np.int8)
    safe = np.abs(proj) > 1e-9 * np.sqrt(m) * 10
    assert np.array_equal(got[safe], want[safe]) and np.array_equal(simt[safe], want[safe])
    assert np.array_equal(got, simt)
    assert (got[5] == 1).all()
    assert st["rechecked"] < 0.2 * got.size

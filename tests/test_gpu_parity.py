"""Device parity: every stage of the CUDA path against the CPU oracle (itself
pinned to the reference's golden vectors) and the golden digests.

Bit-exact: sketch bits, shingle sets, CWS slot keys, signatures, bucket
tables (CSR), candidate sets R.  Top-k: identical ids, squared distances
bit-identical to the reference's f64 DTW (the device rescoring is exact)."""

import ctypes
import hashlib
import warnings

import numpy as np
import pytest

from fixture_data import CASES, case_data
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def csr_digest(tables):
    h = hashlib.sha256()
    for keys, offsets, ids in tables:
        for b, key in enumerate(keys):
            h.update(np.uint64(key).tobytes())
            h.update(np.ascontiguousarray(ids[offsets[b]:offsets[b + 1]], dtype=np.int64).tobytes())
        h.update(b"|")
    return h.hexdigest()


def params(band=0.05, K=4, **kw):
    import paper_1610_07328_b200 as ssh

    d = dict(W=80, delta=3, n=15, d=20, seed=0, band=band, K=K)
    d.update(kw)
    return ssh.SshParams(**d)


def unpack_bits(words, nb):
    b = np.unpackbits(words.view(np.uint8), axis=1, bitorder="little")[:, :nb]
    return np.where(b > 0, 1, -1).astype(np.int8)


def _stage_ctx(p, m):
    from paper_1610_07328_b200.index import get_context

    return get_context(0, p, m)


@pytest.mark.parametrize("name", list(CASES))
def test_sketch_bits_golden(cuda, golden, name):
    import torch

    from paper_1610_07328_b200 import _native as nat
    from paper_1610_07328_b200.index import _stream_ptr

    X, _, _, band = case_data(name)
    p = params(band)
    ctx = _stage_ctx(p, X.shape[1])
    Xd = torch.from_numpy(X).cuda()
    bits = torch.zeros((X.shape[0], ctx.words), dtype=torch.int64, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    nat.check(nat.lib().ssh_sketch(ctx.handle, nat.ptr(Xd), X.shape[0], X.shape[1], nat.ptr(bits),
                                   nat.ptr(stats), _stream_ptr(0)))
    got = unpack_bits(bits.cpu().numpy().view(np.uint64), ctx.nb)
    assert sha(got) == golden["cases"][name]["bits_sha"]
    assert int(stats[1]) == golden["cases"][name]["n_dot_below_1e9"]


def test_sketch_recheck_near_zero(cuda):
    """Windows whose dot is exactly 0 (sign(0) = +1) and tiny: the f32 screen
    must defer to the exact f64 sequence."""
    import torch

    from paper_1610_07328_b200 import _native as nat
    from paper_1610_07328_b200.index import _stream_ptr

    p = params(0.05)
    m = 512
    ctx = _stage_ctx(p, m)
    rng = np.random.default_rng(4)
    X = np.zeros((64, m), dtype=np.float32)
    X[1:20] = rng.standard_normal((19, m)).astype(np.float32) * 1e-3
    X[20:40] = rng.standard_normal((20, m)).astype(np.float32)
    X[40:] = (rng.integers(-2, 3, size=(24, m))).astype(np.float32)  # small integers: exact cancellations
    Xd = torch.from_numpy(X).cuda()
    bits = torch.zeros((64, ctx.words), dtype=torch.int64, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    nat.check(nat.lib().ssh_sketch(ctx.handle, nat.ptr(Xd), 64, m, nat.ptr(bits), nat.ptr(stats), _stream_ptr(0)))
    got = unpack_bits(bits.cpu().numpy().view(np.uint64), ctx.nb)
    want, dots = O.sketch_matrix(X, O.make_filter(80, 0), 3, return_dots=True)
    assert np.array_equal(got, want)
    assert got[0].tolist() == [1] * ctx.nb  # all-zero series: every dot is 0 -> +1
    assert int(stats[1]) == int((np.abs(dots) < 1e-9).sum())


@pytest.mark.parametrize("host", [False, True])
def test_build_index_reports_near_zero_ties(cuda, host):
    """The product build (device and host-input paths) counts the windows it
    re-evaluated in f64 and the near-zero sign ties |dot| < 1e-9 among them
    (BASELINE.json north star: 'counted and reported')."""
    import torch

    import paper_1610_07328_b200 as ssh

    m = 512
    rng = np.random.default_rng(5)
    X = np.zeros((300, m), dtype=np.float32)
    X[1:100] = rng.standard_normal((99, m)).astype(np.float32)
    X[100:] = rng.integers(-2, 3, size=(200, m)).astype(np.float32)
    vals = X if host else torch.from_numpy(X).cuda()
    index = ssh.build_index(ssh.Dataset(vals), params(0.05))
    _, dots = O.sketch_matrix(X, O.make_filter(80, 0), 3, return_dots=True)
    st = index.sketch_stats
    assert st["near_zero"] == int((np.abs(dots) < 1e-9).sum()) > 0
    assert st["rechecked"] >= st["near_zero"]


@pytest.mark.parametrize("m", [512, 1024, 2048])
def test_sketch_stream_ring_partial_tile(cuda, m):
    """TMA-staged sketch kernel: enough series that every CTA wraps its stage
    ring several times, a partial last tile, and rows with NaN / inf / huge
    values (the screen must defer to the exact f64 sequence there)."""
    import torch

    from paper_1610_07328_b200 import _native as nat
    from paper_1610_07328_b200.index import _stream_ptr

    p = params(0.05)
    ctx = _stage_ctx(p, m)
    N = 16 * 148 * 9 + 5
    rng = np.random.default_rng(11 + m)
    X = np.cumsum(rng.standard_normal((N, m)), axis=1).astype(np.float32)
    X[7, 100] = np.nan
    X[N - 2, 3] = np.inf
    X[N - 1, m - 1] = -np.inf
    X[N // 2] *= np.float32(1e30)
    Xd = torch.from_numpy(X).cuda()
    bits = torch.zeros((N, ctx.words), dtype=torch.int64, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    nat.check(nat.lib().ssh_sketch(ctx.handle, nat.ptr(Xd), N, m, nat.ptr(bits), nat.ptr(stats), _stream_ptr(0)))
    got = unpack_bits(bits.cpu().numpy().view(np.uint64), ctx.nb)
    rows = np.unique(np.concatenate([np.arange(16), np.arange(N - 40, N), [N // 2],
                                     rng.choice(N, 400, replace=False)]))
    with np.errstate(invalid="ignore", over="ignore"):
        want = O.sketch_matrix(X[rows], O.make_filter(80, 0), 3)
    assert np.array_equal(got[rows], want)


@pytest.mark.parametrize("name", ["rw512", "rw2048"])
def test_shingle_and_cws_stages(cuda, name):
    import torch

    from paper_1610_07328_b200 import _native as nat
    from paper_1610_07328_b200.index import _stream_ptr

    X, _, _, band = case_data(name)
    p = params(band)
    N, m = X.shape
    ctx = _stage_ctx(p, m)
    L = nat.lib()
    st = _stream_ptr(0)
    Xd = torch.from_numpy(X).cuda()
    bits = torch.zeros((N, ctx.words), dtype=torch.int64, device="cuda")
    nat.check(L.ssh_sketch(ctx.handle, nat.ptr(Xd), N, m, nat.ptr(bits), None, st))
    T = ctx.T
    tok = torch.zeros((N, T), dtype=torch.int32, device="cuda")
    cnt = torch.zeros((N, T), dtype=torch.int16, device="cuda")
    ln = torch.zeros(N, dtype=torch.int32, device="cuda")
    nat.check(L.ssh_shingle(ctx.handle, nat.ptr(bits), N, nat.ptr(tok), nat.ptr(cnt), nat.ptr(ln), st))
    S = p.K * p.d
    keys = torch.zeros((N, S), dtype=torch.int64, device="cuda")
    sig = torch.zeros((N, p.d), dtype=torch.int64, device="cuda")
    nat.check(L.ssh_cws(ctx.handle, nat.ptr(tok), nat.ptr(cnt), nat.ptr(ln), N, nat.ptr(keys), nat.ptr(sig), st))
    torch.cuda.synchronize()
    obits = O.sketch_matrix(X, O.make_filter(80, 0), 3)
    tabs = O.get_tables(15, S, 0, T)
    tokh, cnth, lnh = tok.cpu().numpy().view(np.uint32), cnt.cpu().numpy().view(np.uint16), ln.cpu().numpy()
    keysh = keys.cpu().numpy().view(np.uint64)
    for i in range(0, N, max(1, N // 40)):
        ot, oc = O.shingle(obits[i], 15)
        D = int(lnh[i])
        assert tokh[i, :D].tolist() == ot.tolist() and cnth[i, :D].tolist() == oc.tolist()
        assert keysh[i].tolist() == O.cws_keys_tab(ot, oc, S, tabs).tolist()
    osig = O.signatures(X, 80, 3, 15, 20, 4, 0, threads=8)
    assert np.array_equal(sig.cpu().numpy().view(np.uint64), osig)


def test_cws_large_counts(cuda, golden):
    """Synthetic weighted sets with counts up to 699 through ssh_cws (count>1 path)."""
    import torch

    from paper_1610_07328_b200 import _native as nat
    from paper_1610_07328_b200.index import _stream_ptr

    p = params(0.10)
    ctx = _stage_ctx(p, 2048)  # T = 643 slots per row
    T = ctx.T
    sets = [cw for cw in golden["cws"] if cw["seed"] == 0 and max(cw["counts"]) <= T and len(cw["tokens"]) <= T]
    N = len(sets)
    tok = np.zeros((N, T), dtype=np.uint32)
    cnt = np.zeros((N, T), dtype=np.uint16)
    ln = np.zeros(N, dtype=np.int32)
    for i, cw in enumerate(sets):
        D = len(cw["tokens"])
        tok[i, :D] = cw["tokens"]
        cnt[i, :D] = cw["counts"]
        ln[i] = D
    td, cd, ld = (torch.from_numpy(a.view(v)).cuda() for a, v in ((tok, np.int32), (cnt, np.int16), (ln, np.int32)))
    keys = torch.zeros((N, 80), dtype=torch.int64, device="cuda")
    sig = torch.zeros((N, 20), dtype=torch.int64, device="cuda")
    nat.check(nat.lib().ssh_cws(ctx.handle, nat.ptr(td), nat.ptr(cd), nat.ptr(ld), N, nat.ptr(keys),
                                nat.ptr(sig), _stream_ptr(0)))
    got = keys.cpu().numpy().view(np.uint64)
    for i, cw in enumerate(sets):
        assert got[i].tolist() == cw["keys"]


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("K", [1, 4])
def test_build_index_golden(cuda, golden, name, K):
    import paper_1610_07328_b200 as ssh

    X, _, _, band = case_data(name)
    c = golden["cases"][name]
    idx = ssh.build_index(ssh.Dataset(X), params(band, K=K))
    assert sha(idx.signatures) == c[f"sig_k{K}_sha"]
    assert csr_digest([idx.table_csr(j) for j in range(20)]) == c[f"tables_k{K}_sha"]
    assert [len(t) for t in idx.tables] == c[f"tables_k{K}_nbuckets"]


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("K", [1, 4])
def test_query_golden(cuda, golden, name, K):
    """ids and distances bit-identical to the reference's query_index."""
    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data(name)
    c = golden["cases"][name]
    idx = ssh.build_index(ssh.Dataset(X), params(band, K=K))
    res = ssh.query_index_batch(idx, Q, 10)
    for qi, (r, g) in enumerate(zip(res, c[f"queries_k{K}"])):
        assert r.status == g["status"]
        assert r.stats.candidates == g["candidates"], qi
        assert r.ids == g["ids"], qi
        assert r.distances == g["distances"], qi
        assert ssh.query_signature(idx, Q[qi]).tolist() == c[f"qsig_k{K}"][qi]


def test_probe_candidates_exact(cuda):
    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data("rw512")
    idx = ssh.build_index(ssh.Dataset(X), params(band, K=4))
    oidx = O.build_index(X, 80, 3, 15, 20, 4, 0, band)
    for q in Q[:6]:
        qs = ssh.query_signature(idx, q)
        got = ssh.probe_candidates(idx, qs)
        want = []
        for j, (ukeys, offsets, ids) in enumerate(oidx.csr):
            b = np.searchsorted(ukeys, qs[j])
            if b < len(ukeys) and ukeys[b] == qs[j]:
                want.append(ids[offsets[b]:offsets[b + 1]])
        want = np.unique(np.concatenate(want)) if want else np.empty(0, np.int64)
        assert np.array_equal(got, want)


def test_no_candidates_and_fallback(cuda, golden):
    import paper_1610_07328_b200 as ssh

    X, _, _, band = case_data("rw512")
    idx = ssh.build_index(ssh.Dataset(X[:200]), params(band, K=1))
    q = np.array(golden["empty"]["query"])
    r0 = ssh.query_index(idx, q, 10)
    assert r0.status == "no-candidates" and r0.ids == [] and r0.stats.candidates == 0
    r1 = ssh.query_index(idx, q, 10, fallback_on_empty=True)
    assert r1.status == "fallback"
    assert r1.ids == golden["empty"]["fallback_ids"]
    # the golden query is float64; the device path indexes/queries float32 values
    np.testing.assert_allclose(r1.distances, golden["empty"]["fallback_distances"], rtol=1e-6)
    q32 = q.astype(np.float32)
    ids, d2 = O.brute_force_topk_over(X[:200], np.arange(200), q32, O.radius(band, 512), 10)
    assert r1.ids == ids.tolist() and r1.distances == np.sqrt(d2).tolist()


def test_k_larger_than_n_and_validation(cuda):
    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data("rw512")
    idx = ssh.build_index(ssh.Dataset(X[:30]), params(band, K=1))
    r = ssh.query_index(idx, X[3], 50)
    assert r.warning and "exceeds index size 30" in r.warning
    assert len(r.ids) == r.stats.candidates <= 30
    assert r.ids[0] == 3 and r.distances[0] == 0.0  # self-retrieval
    with pytest.raises(ValueError, match="does not match indexed length"):
        ssh.query_index(idx, X[0, :100], 5)
    with pytest.raises(ValueError, match="k must be >= 1"):
        ssh.query_index(idx, X[0], 0)


def test_duplicates_tie_break_by_id(cuda):
    """Identical series -> identical distances; ties break toward the lower id."""
    import paper_1610_07328_b200 as ssh

    X, _, _, band = case_data("rw512")
    base = X[:50].copy()
    Xd = np.concatenate([base, base, base])  # ids i, i+50, i+100 identical
    idx = ssh.build_index(ssh.Dataset(Xd), params(band, K=1))
    oidx = O.build_index(Xd, 80, 3, 15, 20, 1, 0, band)
    Q = np.stack([base[7], base[20] + 0.01])
    res = ssh.query_index_batch(idx, Q, 10)
    ores = O.query_batch(oidx, Q, 10)
    for i, r in enumerate(res):
        n = int(ores["n"][i])
        assert r.ids == ores["ids"][i][:n].tolist()
        assert r.distances == np.sqrt(ores["d2"][i][:n]).tolist()
    assert res[0].ids[:3] == [7, 57, 107]


@pytest.mark.parametrize("m,band,N", [(514, 0.05, 700), (1022, 0.05, 300), (600, 0.085, 500), (2050, 0.1, 90),
                                      (777, 0.033, 400), (1500, 0.02, 150)])
def test_odd_shapes_vs_oracle(cuda, m, band, N):
    """Row lengths that are not multiples of 4, odd and even radii on the
    long-row (single buffer) and short-row summaries forms, rows longer than
    512 with few series: signatures, |R|, ids and squared distances equal to
    the oracle's."""
    import paper_1610_07328_b200 as ssh
    from fixture_data import perturbed_queries, random_walks

    X = random_walks(N, m, 4000 + m)
    Q, _ = perturbed_queries(X, 5, 77 + m)
    p = params(band, K=2)
    idx = ssh.build_index(ssh.Dataset(X), p)
    oidx = O.build_index(X, 80, 3, 15, 20, 2, 0, band)
    assert np.array_equal(idx.signatures, oidx.sig)
    ores = O.query_batch(oidx, Q, 7)
    for i, r in enumerate(ssh.query_index_batch(idx, Q, 7)):
        n = int(ores["n"][i])
        assert r.stats.candidates == int(ores["n_cand"][i]), i
        assert r.ids == ores["ids"][i][:n].tolist(), i
        assert r.distances == np.sqrt(ores["d2"][i][:n]).tolist(), i
    # exact search (R = the whole shard) exercises every summary row
    xres = ssh.exact_search_batch(ssh.Dataset(X), Q, 7, ssh.WarpingParams(band=band))
    for q, r in zip(Q, xres):
        oi, od = O.brute_force_topk_over(X, np.arange(N), q, O.radius(band, m), 7)
        assert r.ids == oi.tolist() and r.distances == np.sqrt(od).tolist()


def test_massive_ties_beyond_rescoring_lists(cuda):
    """6,000 copies of one series: every copy ties at distance 0 with the query,
    far more than the rescoring lists (4096 + 4k) hold.  The reference cascade
    (dtw.py:171-236) always answers; the device path grows the lists and
    searches the slice again instead of failing: ids 0..k-1 (ties by id),
    distances 0, |R| equal to the oracle's, also next to an ordinary query."""
    import paper_1610_07328_b200 as ssh

    X, _, _, band = case_data("rw512")
    Xd = np.concatenate([np.repeat(X[3:4], 6000, axis=0), X[:200]]).astype(np.float32)
    idx = ssh.build_index(ssh.Dataset(Xd), params(band, K=4))
    oidx = O.build_index(Xd, 80, 3, 15, 20, 4, 0, band)
    Q = np.stack([X[3], X[150] + 0.01, X[3] + 1e-4])
    for k in (10, 50):
        res = ssh.query_index_batch(idx, Q, k)
        ores = O.query_batch(oidx, Q, k)
        for i, r in enumerate(res):
            n = int(ores["n"][i])
            assert r.stats.candidates == int(ores["n_cand"][i]), (k, i)
            assert r.ids == ores["ids"][i][:n].tolist(), (k, i)
            assert r.distances == np.sqrt(ores["d2"][i][:n]).tolist(), (k, i)
        assert res[0].ids == list(range(k)) and set(res[0].distances) == {0.0}
    # the per-query counters still add up to |R| after the rerun
    st = res[0].stats.cascade
    assert (st.kim_pruned + st.keogh_pruned + st.keogh2_pruned + st.dtw_computed) == res[0].stats.candidates


def test_constant_and_edge_shapes(cuda):
    """Flat (z-normalised to zero) series, N=1, and m == W (one sketch bit, n=1)."""
    import paper_1610_07328_b200 as ssh

    rng = np.random.default_rng(8)
    X = rng.standard_normal((40, 128)).astype(np.float32)
    X[5] = 0.0
    X[6] = 0.0
    idx = ssh.build_index(ssh.Dataset(X), ssh.SshParams(W=16, delta=2, n=6, d=6, band=0.1, K=2))
    oidx = O.build_index(X, 16, 2, 6, 6, 2, 0, 0.1)
    assert np.array_equal(idx.signatures, oidx.sig)
    r = ssh.query_index(idx, X[5], 3)
    assert r.ids[:2] == [5, 6] and r.distances[:2] == [0.0, 0.0]
    one = ssh.build_index(ssh.Dataset(X[:1]), ssh.SshParams(W=16, delta=2, n=6, d=6, band=0.1))
    assert ssh.query_index(one, X[0], 5).ids == [0]
    # m == W: N_B = 1, n must be 1
    Y = rng.standard_normal((20, 30)).astype(np.float32)
    p = ssh.SshParams(W=30, delta=5, n=1, d=4, band=0.2, K=1)
    idy = ssh.build_index(ssh.Dataset(Y), p)
    oy = O.build_index(Y, 30, 5, 1, 4, 1, 0, 0.2)
    assert np.array_equal(idy.signatures, oy.sig)
    ores = O.query_batch(oy, Y[:3], 4)
    for i, r in enumerate(ssh.query_index_batch(idy, Y[:3], 4)):
        n = int(ores["n"][i])
        assert r.ids == ores["ids"][i][:n].tolist()


@pytest.mark.parametrize("W,delta,n,band,K,d", [(30, 5, 15, 0.05, 1, 20), (30, 2, 10, 0.1, 2, 8),
                                                 (17, 1, 12, 0.03, 3, 5)])
def test_other_parameters_vs_oracle(cuda, W, delta, n, band, K, d):
    """Non-default (W, delta) exercise the generic sketch kernel and other radii."""
    import paper_1610_07328_b200 as ssh

    X, Q, _, _ = case_data("rw512")
    X, Q = X[:400], Q[:5]
    idx = ssh.build_index(ssh.Dataset(X), ssh.SshParams(W=W, delta=delta, n=n, d=d, band=band, K=K))
    oidx = O.build_index(X, W, delta, n, d, K, 0, band)
    assert np.array_equal(idx.signatures, oidx.sig)
    ores = O.query_batch(oidx, Q, 10)
    for i, r in enumerate(ssh.query_index_batch(idx, Q, 10)):
        nn = int(ores["n"][i])
        assert r.stats.candidates == int(ores["n_cand"][i])
        assert r.ids == ores["ids"][i][:nn].tolist()
        assert r.distances == np.sqrt(ores["d2"][i][:nn]).tolist()


def test_dtw_exact_pairs(cuda, golden):
    """ssh_dtw_exact == reference _dtw_band_sq bits (FMA-free f64)."""
    import paper_1610_07328_b200 as ssh
    from paper_1610_07328_b200.index import dtw_exact_pairs

    X, Q, _, band = case_data("rw1024")
    idx = ssh.build_index(ssh.Dataset(X), params(band, K=4))
    rng = np.random.default_rng(2)
    qrow = rng.integers(0, Q.shape[0], 64)
    xrow = rng.integers(0, X.shape[0], 64)
    got = dtw_exact_pairs(idx, Q, qrow, xrow)
    r = O.radius(band, X.shape[1])
    want = np.array([O.dtw_sq(X[b], Q[a], r) for a, b in zip(qrow, xrow)])
    assert np.array_equal(got, want)


def test_config0_full_parity(cuda):
    """SURVEY §8c scale plan, configs[0] in full: every signature, all 20
    bucket tables and all 100 warped queries (ids, distances, |R|, statuses)
    against an oracle index built independently from the same f32 series."""
    import paper_1610_07328_b200 as ssh
    from paper_1610_07328_b200 import datagen

    X, Q, src, p = datagen.workload(0, device="cuda")
    assert X.shape == (10_000, 512) and Q.shape == (100, 512)
    params_ = ssh.SshParams(**p)
    idx = ssh.build_index(ssh.Dataset(X), params_)
    res = ssh.query_index_batch(idx, Q, 10)
    Xh = X.cpu().numpy()
    oidx = O.build_index(Xh, 80, 3, 15, 20, 4, 0, p["band"], threads=16)
    assert np.array_equal(idx.signatures, oidx.sig)
    for j in range(20):
        k, o, i = idx.table_csr(j)
        assert np.array_equal(k, oidx.csr[j][0]) and np.array_equal(o, oidx.csr[j][1]) \
            and np.array_equal(i, oidx.csr[j][2]), j
    ores = O.query_batch(oidx, Q, 10, threads=16)
    for i, r in enumerate(res):
        n = int(ores["n"][i])
        assert r.status == "ok" and r.stats.candidates == int(ores["n_cand"][i]) > 0, i
        assert r.ids == ores["ids"][i][:n].tolist(), i
        assert r.distances == np.sqrt(ores["d2"][i][:n]).tolist(), i
    assert idx.sketch_stats["near_zero"] == 0


def _full_size_vs_oracle(cfg, nq, sig_rows):
    """Full-size configs[cfg]: signatures of `sig_rows` sampled rows against the
    oracle's, all 20 device tables against the reference table construction
    over the device signatures, and `nq` queries' |R|, top-10 ids and
    distances against the oracle cascade (index.py:204-273) over the same
    tables (A2-A6 sampled, tables exact, >= 20 queries)."""
    import paper_1610_07328_b200 as ssh
    from paper_1610_07328_b200 import datagen

    X, Q, src, p = datagen.workload(cfg, device="cuda", nq=nq)
    assert X.shape[0] == datagen.CONFIGS[cfg]["N"]
    params_ = ssh.SshParams(**p)
    idx = ssh.build_index(ssh.Dataset(X), params_)
    res = ssh.query_index_batch(idx, Q, 10)
    Xh = X.cpu().numpy()
    del X
    sig = idx.signatures
    rows = np.random.default_rng(cfg).choice(Xh.shape[0], sig_rows, replace=False)
    assert np.array_equal(sig[rows], O.signatures(Xh[rows], 80, 3, 15, 20, 4, 0, threads=16))
    ocsr = O.tables_from_signatures(sig)
    for j in range(20):
        k, o, i = idx.table_csr(j)
        assert np.array_equal(k, ocsr[j][0]) and np.array_equal(o, ocsr[j][1]) \
            and np.array_equal(i, ocsr[j][2]), j
    oidx = O.OracleIndex(Xh, 80, 3, 15, 20, 4, 0, p["band"], O.make_filter(80, 0), sig, ocsr)
    ores = O.query_batch(oidx, Q, 10, threads=16)
    for i, r in enumerate(res):
        n = int(ores["n"][i])
        assert r.stats.candidates == int(ores["n_cand"][i]), i
        assert r.ids == ores["ids"][i][:n].tolist(), i
        assert r.distances == np.sqrt(ores["d2"][i][:n]).tolist(), i


@pytest.mark.slow
def test_full_scale_cfg1_vs_oracle(cuda):
    """configs[1] (N=1,000,000, m=512, band 5%): 10k sampled signatures, all
    tables, 24 queries against the oracle."""
    _full_size_vs_oracle(1, 24, 10_000)


def _adversarial_sets():
    rng = np.random.default_rng(11)
    m = 256
    ints = np.cumsum(rng.integers(-2, 3, size=(1500, m)), axis=1).astype(np.float32)  # grid-aligned values
    steps = np.repeat(rng.integers(-3, 4, size=(1500, m // 32)), 32, axis=1).astype(np.float32)  # flat segments
    offset = (np.cumsum(rng.standard_normal((1500, m)), axis=1) * 1e-2 + 4e3).astype(np.float32)  # tiny range, big offset
    mixed = np.cumsum(rng.standard_normal((1500, m)), axis=1).astype(np.float32)
    mixed[::7] *= 1e3
    mixed[3::7] = 0.0
    mixed[5::7, : m // 2] = 2.5
    return {"ints": ints, "steps": steps, "offset": offset, "mixed": mixed}


@pytest.mark.parametrize("kind", ["ints", "steps", "offset", "mixed"])
def test_cascade_bounds_adversarial(cuda, kind):
    """The u8-coded rerank summaries (LB_PAA / LB_Keogh / LB_Keogh2 over
    bracketing codes) never prune a true top-k member: values on the code grid,
    flat segments (PAA means on grid points), a range tiny against the offset,
    mixed scales and constant rows; few tables and short shingles make R large
    (most of the shard), queries include exact copies and near-duplicates."""
    import paper_1610_07328_b200 as ssh

    X = _adversarial_sets()[kind]
    rng = np.random.default_rng(12)
    src = rng.integers(0, X.shape[0], 12)
    Q = X[src].copy()
    Q[6:] += rng.standard_normal((6, X.shape[1])).astype(np.float32) * np.float32(0.3 * (np.abs(X[src[6:]]).max() + 1e-3))
    p = ssh.SshParams(W=16, delta=2, n=4, d=3, band=0.08, K=1)
    idx = ssh.build_index(ssh.Dataset(X), p)
    oidx = O.build_index(X, 16, 2, 4, 3, 1, 0, 0.08)
    ores = O.query_batch(oidx, Q, 10)
    res = ssh.query_index_batch(idx, Q, 10, fallback_on_empty=True)
    for i, r in enumerate(res):
        n = int(ores["n"][i])
        if n == 0:
            continue
        assert r.ids == ores["ids"][i][:n].tolist(), (kind, i)
        assert r.distances == np.sqrt(ores["d2"][i][:n]).tolist(), (kind, i)


def test_query_member_budget_split(cuda, golden, monkeypatch):
    """A tiny member budget splits the batch into many sub-ranges (each with
    its own member lists and wave loop); results stay identical."""
    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data("rw512")
    c = golden["cases"]["rw512"]
    idx = ssh.build_index(ssh.Dataset(X), params(band, K=1))
    monkeypatch.setenv("SSH_DEBUG_MEMBER_BUDGET", "300")
    res = ssh.query_index_batch(idx, Q, 10)
    for qi, (r, g) in enumerate(zip(res, c["queries_k1"])):
        assert r.stats.candidates == g["candidates"], qi
        assert r.ids == g["ids"], qi
        assert r.distances == g["distances"], qi


@pytest.mark.parametrize("target", ["8", "64"])
def test_query_overflow_round(cuda, golden, monkeypatch, target):
    """A tiny round-0 member target cuts every query's list far below its
    threshold, so the overflow round must supply the rest; results stay
    identical to the reference."""
    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data("rw1024")
    c = golden["cases"]["rw1024"]
    idx = ssh.build_index(ssh.Dataset(X), params(band, K=4))
    monkeypatch.setenv("SSH_DEBUG_MEMBER_TARGET", target)
    res = ssh.query_index_batch(idx, Q, 10)
    for qi, (r, g) in enumerate(zip(res, c["queries_k4"])):
        assert r.stats.candidates == g["candidates"], qi
        assert r.ids == g["ids"], qi
        assert r.distances == g["distances"], qi


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [2, 3])
def test_full_scale_cfg2_cfg3_vs_oracle(cuda, cfg):
    """configs[2] (2M ECG windows, m=1024, band 5%: radius 51, pooled register
    band) and configs[3] (4M random walks, m=2048, band 10%: radius 205, warp
    wavefront) at FULL size: 4k sampled signatures, all tables, 20 queries'
    top-10 ids and distances identical to the oracle cascade."""
    _full_size_vs_oracle(cfg, 20, 4000)


@pytest.mark.slow
def test_config3_full_size_properties(cuda):
    """configs[3] at full size (N=4,000,000, m=2048): self-queries return their
    own row first at distance 0, distances ascend, and every reported distance
    equals the exact f64 DTW of that pair (ssh_dtw_exact)."""
    import torch

    import paper_1610_07328_b200 as ssh
    from paper_1610_07328_b200 import datagen
    from paper_1610_07328_b200.index import dtw_exact_pairs

    X, _, _, p = datagen.workload(3, device="cuda", nq=0)
    idx = ssh.build_index(ssh.Dataset(X), ssh.SshParams(**p))
    rows = np.random.default_rng(5).choice(X.shape[0], 12, replace=False)
    Q = X[torch.from_numpy(rows).cuda()].cpu().numpy()
    res = ssh.query_index_batch(idx, Q, 10)
    for i, r in enumerate(res):
        assert r.ids[0] == int(rows[i]) and r.distances[0] == 0.0
        assert r.distances == sorted(r.distances)
        d2 = dtw_exact_pairs(idx, Q, np.full(len(r.ids), i), np.asarray(r.ids))
        assert np.sqrt(d2).tolist() == r.distances


def _device_tables(sig_u64):
    """ssh_index_build over a given signature matrix -> host CSR per table."""
    import torch

    from paper_1610_07328_b200 import _native as nat
    from paper_1610_07328_b200.index import _stream_ptr

    N, L = sig_u64.shape
    ctx = _stage_ctx(params(), 512)
    lib = nat.lib()
    sig = torch.from_numpy(np.ascontiguousarray(sig_u64).view(np.int64)).cuda()
    h = ctypes.c_void_p()
    nat.check(lib.ssh_index_build(ctx.handle, nat.ptr(sig), N, 0, ctypes.byref(h), _stream_ptr(0)))
    out = []
    try:
        for j in range(L):
            nb = ctypes.c_int64()
            nat.check(lib.ssh_index_num_buckets(h, j, ctypes.byref(nb)))
            keys = np.empty(nb.value, dtype=np.uint64)
            offsets = np.empty(nb.value + 1, dtype=np.int64)
            ids = np.empty(N, dtype=np.int64)
            nat.check(lib.ssh_index_export(h, j, nat.ptr(keys), nat.ptr(offsets), nat.ptr(ids), _stream_ptr(0)))
            out.append((keys, offsets, ids))
    finally:
        lib.ssh_index_destroy(h)
    return out


@pytest.mark.parametrize("kind", ["few_hi_long_runs", "pair_runs_over_capacity", "random"])
def test_tables_high_half_collisions(cuda, kind):
    """The bucket tables sort on the high 32 key bits and fix up runs whose keys
    share a high half: crafted signatures with long colliding runs, more
    colliding runs than the fix-up list holds (full-key fallback), and random
    keys all give the reference's tables (stable argsort, index.py:141-156)."""
    rng = np.random.default_rng(21)
    N, L = 40_000, 20
    if kind == "few_hi_long_runs":
        hi = rng.integers(0, 3, size=(N, L)).astype(np.uint64)
        lo = rng.integers(0, 5, size=(N, L)).astype(np.uint64) * np.uint64(0x9E3779B1)
    elif kind == "pair_runs_over_capacity":
        hi = (np.arange(N, dtype=np.uint64) // np.uint64(2))[:, None].repeat(L, 1)
        lo = rng.integers(0, 2, size=(N, L)).astype(np.uint64)
    else:
        hi = rng.integers(0, 2**32, size=(N, L), dtype=np.uint64)
        lo = rng.integers(0, 2**32, size=(N, L), dtype=np.uint64)
    sig = (hi << np.uint64(32)) | lo
    got = _device_tables(sig)
    want = O.tables_from_signatures(sig)
    for j in range(L):
        for a, b in zip(got[j], want[j]):
            assert np.array_equal(a, b), (kind, j)


def test_save_index_bytes_and_round_trip(cuda, golden, tmp_path):
    """save_index from the device CSR is byte-identical to the reference's file
    (K=1); load_index rebuilds an index with the same signatures, tables and
    query results; K=4 round-trips through version 2."""
    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data("rw512")
    X200 = X[:200].astype(np.float64)
    idx = ssh.build_index(ssh.Dataset(X200), params(band, K=1))
    ssh.save_index(idx, tmp_path / "idx.sshi")
    data = (tmp_path / "idx.sshi").read_bytes()
    assert hashlib.sha256(data).hexdigest() == golden["persist"]["index_sha256"]
    back = ssh.load_index(tmp_path / "idx.sshi")
    assert np.array_equal(back.signatures, idx.signatures)
    for j in (0, 7, 19):
        for a, b in zip(back.table_csr(j), idx.table_csr(j)):
            assert np.array_equal(a, b)
    r1 = ssh.query_index_batch(idx, Q, 10)
    r2 = ssh.query_index_batch(back, Q, 10)
    assert [r.ids for r in r1] == [r.ids for r in r2]
    assert [r.distances for r in r1] == [r.distances for r in r2]
    idx4 = ssh.build_index(ssh.Dataset(X200), params(band, K=4))
    ssh.save_index(idx4, tmp_path / "k4.sshi")
    back4 = ssh.load_index(tmp_path / "k4.sshi")
    assert back4.params.K == 4 and np.array_equal(back4.signatures, idx4.signatures)
    assert [r.ids for r in ssh.query_index_batch(back4, Q, 10)] == [r.ids for r in ssh.query_index_batch(idx4, Q, 10)]


@pytest.mark.parametrize("name", ["rw512", "rw1024"])
def test_exact_search_vs_oracle(cuda, name):
    """exact_search (dtw.py:293-326) on the device == the oracle's brute-force
    (d2, id) top-k over every series (bench.py:45-60)."""
    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data(name)
    X = X[:600]
    res = ssh.exact_search_batch(ssh.Dataset(X), Q[:6], 10, ssh.WarpingParams(band))
    r = O.radius(band, X.shape[1])
    for i, rr in enumerate(res):
        ids, d2 = O.brute_force_topk_over(X, np.arange(X.shape[0]), Q[i], r, 10)
        assert rr.ids == ids.tolist(), i
        assert rr.distances == np.sqrt(d2).tolist(), i
        assert rr.stats.candidates == X.shape[0]
    one = ssh.exact_search(ssh.Dataset(X[:5]), Q[0], 9, ssh.WarpingParams(band))
    assert one.warning and len(one.ids) == 5


@pytest.mark.parametrize("key", ["rw20000_t128", "rw6000_t1000"])
def test_make_dataset_device_matches_reference(cuda, golden, key):
    """Windowing + per-window z-normalisation on the device (ssh_windows) is
    bit-identical to the reference's make_dataset (core.py:162-169), float64;
    the float32 output is its rounding."""
    import paper_1610_07328_b200 as ssh

    g = golden["windows"][key]
    rec = np.cumsum(np.random.default_rng(g["seed"]).standard_normal(g["length"]))  # generate_random_walk
    d64 = ssh.make_dataset(ssh.TimeSeries(values=rec), g["t"], dtype="float64")
    v = d64.values.cpu().numpy()
    assert v.shape == (g["count"], g["t"])
    assert sha(v) == g["sha256"]
    d32 = ssh.make_dataset(ssh.TimeSeries(values=rec), g["t"])
    assert np.array_equal(d32.values.cpu().numpy(), v.astype(np.float32))
    raw = ssh.make_dataset(ssh.TimeSeries(values=rec), g["t"], normalize=False, stride=7, dtype="float64")
    assert np.array_equal(raw.values.cpu().numpy(), np.lib.stride_tricks.sliding_window_view(rec, g["t"])[::7])


@pytest.mark.parametrize("bits,seed", [(64, 3), (100, 11)])
def test_srp_matrix_matches_reference(cuda, golden, bits, seed):
    """srp_matrix (index.py:420-423) on the device == the reference's int8 signs."""
    import paper_1610_07328_b200 as ssh

    X, _, _, _ = case_data("rw512")
    got = ssh.srp_matrix(X[:300], bits, seed)
    assert got.dtype == np.int8 and got.shape == (300, bits)
    assert sha(got) == golden["srp"][f"b{bits}_s{seed}"]
    assert np.array_equal(ssh.srp_signature(X[7], bits, seed), got[7])


@pytest.mark.parametrize("band", [0.0605, 0.0625, 0.0])
def test_dtw_exact_band_edges(cuda, band):
    """The exact f64 DTW (warp wavefront for 2r+1 <= 64, other kernels above):
    radii 31 / 32 / 0 around the wavefront limit, bit-identical to the oracle's
    reference recurrence."""
    import paper_1610_07328_b200 as ssh
    from paper_1610_07328_b200.index import dtw_exact_pairs

    X, Q, _, _ = case_data("rw512")
    idx = ssh.build_index(ssh.Dataset(X[:300]), params(band, K=1))
    rng = np.random.default_rng(4)
    qrow = rng.integers(0, Q.shape[0], 40)
    xrow = rng.integers(0, 300, 40)
    got = dtw_exact_pairs(idx, Q, qrow, xrow)
    r = O.radius(band, X.shape[1])
    want = np.array([O.dtw_sq(X[b], Q[a], r) for a, b in zip(qrow, xrow)])
    assert np.array_equal(got, want)


def test_large_k_vs_oracle(cuda):
    """k = 700 (top-k sort and rescoring sets far beyond the usual 10) against
    the oracle cascade; results sorted by (distance, id)."""
    import paper_1610_07328_b200 as ssh

    X, Q, _, band = case_data("rw512")
    p = ssh.SshParams(W=16, delta=2, n=4, d=3, band=band, K=1)  # short shingles: R is most of the shard
    idx = ssh.build_index(ssh.Dataset(X), p)
    oidx = O.build_index(X, 16, 2, 4, 3, 1, 0, band)
    ores = O.query_batch(oidx, Q[:4], 700)
    for i, r in enumerate(ssh.query_index_batch(idx, Q[:4], 700)):
        n = int(ores["n"][i])
        assert r.ids == ores["ids"][i][:n].tolist(), i
        assert r.distances == np.sqrt(ores["d2"][i][:n]).tolist(), i


def test_k_beyond_2048_vs_oracle(cuda):
    """k = 3000 of a 4,000-series shard (the round-1 device limit was 2048; the
    reference accepts any k, index.py:204-232) and k = 16384 clamped to N."""
    import paper_1610_07328_b200 as ssh
    from fixture_data import perturbed_queries, random_walks

    X = random_walks(4000, 256, 99)
    Q, _ = perturbed_queries(X, 3, 17)
    p = ssh.SshParams(W=16, delta=2, n=4, d=3, band=0.05, K=1)  # short shingles: R is most of the shard
    idx = ssh.build_index(ssh.Dataset(X), p)
    oidx = O.build_index(X, 16, 2, 4, 3, 1, 0, 0.05)
    for k in (3000, 16384):
        kk = min(k, 4000)
        ores = O.query_batch(oidx, Q, kk)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = ssh.query_index_batch(idx, Q, k)
        for i, r in enumerate(res):
            n = int(ores["n"][i])
            assert n > 2048 and len(r.ids) == n, (k, i, n)
            assert r.ids == ores["ids"][i][:n].tolist(), (k, i)
            assert r.distances == np.sqrt(ores["d2"][i][:n]).tolist(), (k, i)


def _dec32(c, sc, lo):
    """fmaf(c, sc, lo) in f32 (c * sc is exact in long double; one rounding)."""
    return (c.astype(np.longdouble) * np.longdouble(sc) + np.longdouble(lo)).astype(np.float32)


@pytest.mark.parametrize("m,band", [(512, 0.05), (1024, 0.05), (2048, 0.10), (301, 0.1), (5000, 0.01)])
def test_summaries_codes_exact(cuda, m, band):
    """Rerank summaries read back from the device: every sample code brackets
    its value with the decoder's own fp32 arithmetic, PAA codes bracket the
    f64 segment means (rows not flagged ambiguous), and the envelope codes are
    exactly max/min of the sample codes over the Sakoe-Chiba window
    [i - r, i + r] (dtw.py:124-151), U8 = max + 1 and L8 = min (the
    byte/u16-packed doubling must reproduce the plain running max/min)."""
    import paper_1610_07328_b200 as ssh

    rng = np.random.default_rng(m)
    n = 300
    X = np.cumsum(rng.standard_normal((n, m)), axis=1).astype(np.float32)
    X[7] = 0.0
    X[11, : m // 3] = 3.5
    X[13] = np.round(X[13])
    p = ssh.SshParams(W=16, delta=2, n=4, d=3, band=band, K=1)
    idx = ssh.build_index(ssh.Dataset(X), p)
    rec, codes, mp = idx.summaries()
    r = p.warping().radius(m)
    assert codes.shape == (n, 3 * mp)
    f = rec[:, :16].copy().view(np.float32)
    lo, sc = f[:, 0], f[:, 1]
    x8 = codes[:, :m].astype(np.int64)
    ul = codes[:, mp:mp + 2 * m].reshape(n, m, 2).astype(np.int64)
    seg = (m + 47) // 48
    nseg = (m + seg - 1) // seg
    for i in range(n):
        scale = abs(sc[i])
        if not np.isfinite(scale):
            continue
        assert f[i, 2] == X[i, 0] and f[i, 3] == X[i, -1], i
        assert (_dec32(x8[i], scale, lo[i]) <= X[i]).all(), i
        assert (_dec32(x8[i] + 1, scale, lo[i]) >= X[i]).all(), i
        pad_hi = np.concatenate([np.full(r, -1), x8[i], np.full(r, -1)])
        pad_lo = np.concatenate([np.full(r, 1 << 20), x8[i], np.full(r, 1 << 20)])
        win = np.lib.stride_tricks.sliding_window_view
        assert np.array_equal(ul[i, :, 0], win(pad_hi, 2 * r + 1).max(1) + 1), i
        assert np.array_equal(ul[i, :, 1], win(pad_lo, 2 * r + 1).min(1)), i
        if sc[i] > 0:
            pc = rec[i, 16:16 + nseg].astype(np.int64)
            means = np.array([X[i, s * seg:min(m, s * seg + seg)].astype(np.float64).mean() for s in range(nseg)])
            assert (_dec32(pc, scale, lo[i]).astype(np.float64) <= means).all(), i
            assert (_dec32(pc + 1, scale, lo[i]).astype(np.float64) >= means).all(), i

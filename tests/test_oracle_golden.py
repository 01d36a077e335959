"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py imports /root/reference).  CPU only."""

import hashlib

import numpy as np
import pytest

from fixture_data import CASES, case_data
from oracle import oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def csr_digest(csr):
    h = hashlib.sha256()
    for ukeys, offsets, ids in csr:
        for b, key in enumerate(ukeys):
            h.update(np.uint64(key).tobytes())
            h.update(np.ascontiguousarray(ids[offsets[b]:offsets[b + 1]], dtype=np.int64).tobytes())
        h.update(b"|")
    return h.hexdigest()


def test_spec_worked_examples(golden):
    # X=(1,2,4,1), r=(0.1,-0.1), delta=2 -> (-1,+1)
    bits = O.sketch_matrix(np.array([[1.0, 2, 4, 1]]), np.array([0.1, -0.1]), 2)
    assert bits[0].tolist() == [-1, 1] == golden["spec"]["sketch"]
    # shingles of (+1,+1,-1,-1,+1,+1), n=2
    tok, cnt = O.shingle(np.array([1, 1, -1, -1, 1, 1], dtype=np.int8), 2)
    assert {int(t): int(c) for t, c in zip(tok, cnt)} == {int(k): v for k, v in golden["spec"]["shingle"].items()}
    # DTW((1,2,3),(2,3,4), band 1) = sqrt(2)
    assert np.sqrt(O.dtw_sq(np.array([1.0, 2, 3]), np.array([2.0, 3, 4]), 3)) == golden["dtw"]["spec_sqrt2"]
    assert O.make_filter(80, 0).tolist() == golden["spec"]["filter80"]


@pytest.mark.parametrize("name", list(CASES))
def test_sketch_and_shingle(golden, name):
    c = golden["cases"][name]
    X, _, _, _ = case_data(name)
    bits = O.sketch_matrix(X, O.make_filter(80, 0), 3)
    assert sha(bits) == c["bits_sha"]
    for i, s in enumerate(c["shingle_sets"]):
        tok, cnt = O.shingle(bits[i], 15)
        assert tok.tolist() == s["tokens"] and cnt.tolist() == s["counts"]


@pytest.mark.parametrize("name", list(CASES))
def test_signatures_and_tables(golden, name):
    c = golden["cases"][name]
    X, _, _, _ = case_data(name)
    sig1 = O.signatures(X, 80, 3, 15, 20, 1, 0, threads=4)
    assert sha(sig1) == c["sig_k1_sha"]
    sig4 = O.signatures(X, 80, 3, 15, 20, 4, 0, threads=4)
    assert sha(sig4) == c["sig_k4_sha"]
    csr1 = O.tables_from_signatures(sig1)
    csr4 = O.tables_from_signatures(sig4)
    assert csr_digest(csr1) == c["tables_k1_sha"]
    assert csr_digest(csr4) == c["tables_k4_sha"]
    assert [len(t[0]) for t in csr4] == c["tables_k4_nbuckets"]


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("K", [1, 4])
def test_queries(golden, name, K):
    c = golden["cases"][name]
    X, Q, _, band = case_data(name)
    idx = O.build_index(X, 80, 3, 15, 20, K, 0, band, threads=4)
    res = O.query_batch(idx, Q, 10, threads=4)
    for qi, q in enumerate(c[f"queries_k{K}"]):
        n = int(res["n"][qi])
        assert res["ids"][qi][:n].tolist() == q["ids"]
        assert np.sqrt(res["d2"][qi][:n]).tolist() == q["distances"]
        assert int(res["n_cand"][qi]) == q["candidates"]
        assert res["counters"][qi].tolist() == q["counters"]
        assert res["qsig"][qi].tolist() == c[f"qsig_k{K}"][qi]


def test_cws_keys(golden):
    for cw in golden["cws"]:
        tokens = np.array(cw["tokens"], dtype=np.uint64)
        counts = np.array(cw["counts"], dtype=np.int64)
        assert O.cws_keys_numpy(tokens, counts, np.arange(80, dtype=np.uint64), 0).tolist() == cw["keys"]
        tabs = O.get_tables(15, 80, cw["seed"], 700)
        want = cw["keys_seed"] if cw["seed"] else cw["keys"]
        assert O.cws_keys_tab(tokens, counts, 80, tabs).tolist() == want


def test_dtw_envelope_lb(golden):
    for p in golden["dtw"]["pairs"]:
        x, y = np.array(p["x"]), np.array(p["y"])
        assert O.dtw_sq(x, y, p["r"]) == p["d2"]
        U, L = O.envelope(y, p["r"])
        assert U.tolist() == p["upper"] and L.tolist() == p["lower"]
        assert O.lb_keogh_sq(x, U, L) == p["lb_keogh_sq"]


def test_empty_candidates(golden):
    X, _, _, band = case_data("rw512")
    idx = O.build_index(X[:200], 80, 3, 15, 20, 1, 0, band)
    res = O.query_batch(idx, np.array([golden["empty"]["query"]]), 10)
    assert int(res["n_cand"][0]) == golden["empty"]["candidates"] == 0
    assert golden["empty"]["status"] == "no-candidates"
    # fallback == exact search over all rows (index.py:239-243)
    cand = np.arange(200)
    ids, d2 = O.brute_force_topk_over(X[:200], cand, np.array(golden["empty"]["query"]), O.radius(band, 512), 10)
    assert ids.tolist() == golden["empty"]["fallback_ids"]
    assert np.sqrt(d2).tolist() == golden["empty"]["fallback_distances"]


def test_table_cws_pins_numpy_restatement():
    """Table evaluation == direct np.log restatement on random sets (incl. large counts)."""
    rng = np.random.default_rng(5)
    tabs = O.get_tables(15, 80, 0, 700)
    for _ in range(30):
        D = int(rng.integers(1, 150))
        tokens = np.sort(rng.choice(1 << 15, size=D, replace=False)).astype(np.uint64)
        counts = rng.integers(1, 700, size=D).astype(np.int64)
        a = O.cws_keys_tab(tokens, counts, 80, tabs)
        b = O.cws_keys_numpy(tokens, counts, np.arange(80, dtype=np.uint64), 0)
        assert np.array_equal(a, b)


def test_cascade_equals_brute_force_over_R():
    """The cascade result is the exact top-k of R by (d2, id) — the property the
    device rerank relies on."""
    X, Q, _, band = case_data("rw512")
    r = O.radius(band, X.shape[1])
    rng = np.random.default_rng(3)
    for q in Q[:4]:
        cand = np.sort(rng.choice(X.shape[0], size=300, replace=False))
        U, L = O.envelope(q.astype(np.float64), r)
        order = rng.permutation(cand)
        ids, d2, _ = O.cascade_search(X, order, q, U, L, r, 10)
        bids, bd2 = O.brute_force_topk_over(X, cand, q, r, 10)
        assert ids.tolist() == bids.tolist() and d2.tolist() == bd2.tolist()

"""CPU oracle for the SSH hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or the timed
CPU baseline.  The product package (paper_1610_07328_b200) never imports it.

Contents
--------
* numpy restatements of the reference's stateless randomness
  (wmh.py:26-49: salts, mix64, _unit_interval) and of `_cws_keys`
  (wmh.py:52-81) that evaluates np.log on the fly exactly like the
  reference — this pins the table-based evaluation below;
* `cws_tables` — the per-(token, slot) variates r, ln_c, beta over the whole
  2^n token universe, built with the reference's own op sequence
  (wmh.py:60-72) so every entry is bit-identical to what `_cws_keys` computes
  for that (token, slot);
* ctypes bindings to ssh_oracle.c (sketch, shingle, CWS from tables, DTW,
  envelope, LB_Keogh, cascade, K-aware query_index);
* `tables_from_signatures` — restatement of index.py:141-156 (stable argsort
  per table, ids ascending within a bucket) returned as CSR arrays.

Parity pins: tests/golden/*.npz were produced by importing the reference
package itself (tests/golden/make_golden.py); tests/test_oracle_golden.py
checks this oracle against them.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_BUILD = _HERE / "_build"
_LIB_PATH = _BUILD / "libsshoracle.so"

# wmh.py:26-31
SALT_U1 = np.uint64(0xA0761D6478BD642F)
SALT_U2 = np.uint64(0xE7037ED1A0B428DB)
SALT_V1 = np.uint64(0x8EBC6AF09C88C6E3)
SALT_V2 = np.uint64(0x589965CC75374CC3)
SALT_BETA = np.uint64(0x1D8E4E27C47D124F)
SALT_KEY = np.uint64(0xEB44ACCAB455D165)
SLOT_MULT = np.uint64(0xD1B54A32D192ED03)
_MASK64 = (1 << 64) - 1


def mix64(x):
    """wmh.py:34-44 — splitmix64 finalizer on uint64 scalars/arrays."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def unit_interval(h):
    """wmh.py:47-49."""
    return ((h >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0**-53


def cws_keys_numpy(tokens, counts, slots, seed):
    """Direct restatement of wmh.py:52-81 (_cws_keys), np.log on the fly."""
    tokens = np.asarray(tokens, dtype=np.uint64)
    counts = np.asarray(counts, dtype=np.int64)
    slots = np.asarray(slots, dtype=np.uint64)
    if tokens.shape[0] == 0:
        raise ValueError("cannot hash an empty weighted set")
    with np.errstate(over="ignore"):
        tk = mix64(tokens ^ mix64(np.uint64(seed & _MASK64)))
        sl = mix64(slots * SLOT_MULT)
    base = mix64(tk[None, :] ^ sl[:, None])
    u1 = unit_interval(mix64(base ^ SALT_U1))
    u2 = unit_interval(mix64(base ^ SALT_U2))
    v1 = unit_interval(mix64(base ^ SALT_V1))
    v2 = unit_interval(mix64(base ^ SALT_V2))
    beta = unit_interval(mix64(base ^ SALT_BETA))
    r = -np.log(u1) - np.log(u2)
    ln_c = np.log(-np.log(v1) - np.log(v2))
    ln_w = np.log(counts.astype(np.float64))
    t = np.floor(ln_w[None, :] / r + beta)
    ln_y = r * (t - beta)
    ln_a = ln_c - ln_y - r
    j = np.argmin(ln_a, axis=1)
    rows = np.arange(slots.shape[0])
    t_star = t[rows, j].astype(np.int64).astype(np.uint64)
    return mix64(tokens[j] ^ mix64(t_star ^ SALT_KEY))


def signature_numpy(tokens, counts, L, seed, K=1):
    """wmh.py:107-125 (signature with concat=K) over cws_keys_numpy."""
    keys = cws_keys_numpy(tokens, counts, np.arange(L * K, dtype=np.uint64), seed)
    if K > 1:
        folded = keys.reshape(L, K)
        acc = folded[:, 0]
        for i in range(1, K):
            acc = mix64(acc ^ folded[:, i])
        keys = acc
    return keys


def cws_tables(n: int, S: int, seed: int):
    """Variates for every (token, slot) of the 2^n universe, layout [token][slot].

    Same op sequence as wmh.py:60-72, so each entry equals the value
    `_cws_keys` computes for that (token, slot) on this host's numpy.
    Returns (r, ln_c, beta) float64 arrays of shape (2^n, S).
    """
    tokens = np.arange(1 << n, dtype=np.uint64)
    slots = np.arange(S, dtype=np.uint64)
    with np.errstate(over="ignore"):
        tk = mix64(tokens ^ mix64(np.uint64(seed & _MASK64)))
        sl = mix64(slots * SLOT_MULT)
    base = mix64(tk[:, None] ^ sl[None, :])
    u1 = unit_interval(mix64(base ^ SALT_U1))
    u2 = unit_interval(mix64(base ^ SALT_U2))
    r = -np.log(u1) - np.log(u2)
    del u1, u2
    v1 = unit_interval(mix64(base ^ SALT_V1))
    v2 = unit_interval(mix64(base ^ SALT_V2))
    ln_c = np.log(-np.log(v1) - np.log(v2))
    del v1, v2
    beta = unit_interval(mix64(base ^ SALT_BETA))
    return np.ascontiguousarray(r), np.ascontiguousarray(ln_c), np.ascontiguousarray(beta)


def ln_counts(max_count: int):
    """np.log(counts.astype(float64)) of wmh.py:72 for counts 0..max_count
    (entry 0 unused)."""
    c = np.arange(max_count + 1, dtype=np.float64)
    c[0] = 1.0
    return np.log(c)


def make_filter(W: int, seed: int) -> np.ndarray:
    """sketch.py:36-43."""
    return np.random.default_rng(seed).standard_normal(W)


def radius(band: float, m: int) -> int:
    """dtw.py:38-39 (Python round: half to even)."""
    return int(round(band * m))


def num_sketch_bits(m: int, W: int, delta: int) -> int:
    """sketch.py:46-48."""
    return (m - W) // delta + 1


# ----------------------------------------------------------------- C side

_lib = None


def _compile():
    _BUILD.mkdir(parents=True, exist_ok=True)
    src = _HERE / "ssh_oracle.c"
    tmp = _LIB_PATH.with_suffix(".so.tmp%d" % os.getpid())
    subprocess.check_call(
        ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
         "-fno-fast-math", "-o", str(tmp), str(src), "-lm"]
    )
    os.replace(tmp, _LIB_PATH)


def build():
    """Compile ssh_oracle.c into oracle/_build/libsshoracle.so."""
    _compile()


def lib():
    global _lib
    if _lib is not None:
        return _lib
    src = _HERE / "ssh_oracle.c"
    if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        _compile()
    L = ctypes.CDLL(str(_LIB_PATH))
    P = ctypes.c_void_p
    i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.orc_sketch.argtypes = [P, i32, i64, i32, i64, P, i32, i32, P, P, i32]
    L.orc_signatures.argtypes = [P, i32, i64, i32, i64, P, i32, i32, i32, i32, i32, P, P, P, P, P, i32]
    L.orc_shingle.argtypes = [P, i32, i32, P, P, P]
    L.orc_shingle.restype = i32
    L.orc_cws_keys.argtypes = [P, P, i32, i32, P, P, P, P, P]
    L.orc_fold.argtypes = [P, i32, i32, P]
    L.orc_dtw.argtypes = [P, P, i32, i32, dbl]
    L.orc_dtw.restype = dbl
    L.orc_envelope.argtypes = [P, i32, i32, P, P, P]
    L.orc_lb_keogh_sq.argtypes = [P, P, P, i32, dbl]
    L.orc_lb_keogh_sq.restype = dbl
    L.orc_cascade_search.argtypes = [P, i32, i64, i32, P, i64, P, P, P, i32, i32, P, P, P]
    L.orc_cascade_search.restype = i32
    L.orc_query_batch.argtypes = [P, i32, i64, i32, i64, P, i32, P, i32, i32, i32, i32, i32,
                                  P, P, P, P, P, P, P, P, P, i32, i32, P, P, P, P, P, P, i32]
    L.orc_dtw_many.argtypes = [P, i32, i64, i32, P, i64, P, i32, P, i32]
    L.orc_mix64.argtypes = [ctypes.c_uint64]
    L.orc_mix64.restype = ctypes.c_uint64
    _lib = L
    return L


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _xarg(X):
    X = np.asarray(X)
    if X.dtype == np.float32:
        X = np.ascontiguousarray(X)
        return X, 1
    X = np.ascontiguousarray(X, dtype=np.float64)
    return X, 0


def _threads(threads):
    return threads if threads and threads > 0 else (len(os.sched_getaffinity(0)) or 1)


# ------------------------------------------------------- stage restatements

def sketch_matrix(X, w, delta, threads=1, return_dots=False):
    """sketch.py:69-89 -> (N, N_B) int8 in {+1,-1} (and the f64 dots)."""
    X, f32 = _xarg(X)
    N, m = X.shape
    w = np.ascontiguousarray(w, dtype=np.float64)
    nb = num_sketch_bits(m, w.shape[0], delta)
    bits = np.empty((N, nb), dtype=np.int8)
    dots = np.empty((N, nb), dtype=np.float64) if return_dots else None
    lib().orc_sketch(_p(X), f32, N, m, m, _p(w), w.shape[0], delta, _p(bits),
                     _p(dots) if dots is not None else None, _threads(threads))
    return (bits, dots) if return_dots else bits


def shingle(bits_row, n):
    """shingle.py:56-75 -> (tokens uint64 sorted, counts int64)."""
    bits_row = np.ascontiguousarray(bits_row, dtype=np.int8)
    nb = bits_row.shape[0]
    nt = nb - n + 1
    tok = np.empty(nt, dtype=np.uint64)
    cnt = np.empty(nt, dtype=np.int64)
    scr = np.empty(nt, dtype=np.uint64)
    D = lib().orc_shingle(_p(bits_row), nb, n, _p(tok), _p(cnt), _p(scr))
    return tok[:D].copy(), cnt[:D].copy()


@dataclass
class OracleTables:
    """CWS variates + ln(count) table for one (n, S, seed)."""
    n: int
    S: int
    seed: int
    r: np.ndarray
    ln_c: np.ndarray
    beta: np.ndarray
    ln_w: np.ndarray


_TAB_CACHE: dict = {}


def get_tables(n, S, seed, max_count):
    key = (n, S, seed)
    t = _TAB_CACHE.get(key)
    if t is None:
        r, lnc, beta = cws_tables(n, S, seed)
        t = OracleTables(n, S, seed, r, lnc, beta, ln_counts(max(max_count, 1)))
        _TAB_CACHE[key] = t
    if t.ln_w.shape[0] <= max_count:
        t.ln_w = ln_counts(max_count)
    return t


def cws_keys_tab(tokens, counts, S, tabs: OracleTables):
    tokens = np.ascontiguousarray(tokens, dtype=np.uint64)
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    keys = np.empty(S, dtype=np.uint64)
    lib().orc_cws_keys(_p(tokens), _p(counts), tokens.shape[0], S, _p(tabs.r), _p(tabs.ln_c),
                       _p(tabs.beta), _p(tabs.ln_w), _p(keys))
    return keys


def signatures(X, W, delta, n, L, K, seed, threads=1, w=None):
    """index.py:113-138 with the K-aware fold -> (N, L) uint64."""
    X, f32 = _xarg(X)
    N, m = X.shape
    if w is None:
        w = make_filter(W, seed)
    w = np.ascontiguousarray(w, dtype=np.float64)
    nb = num_sketch_bits(m, W, delta)
    tabs = get_tables(n, L * K, seed, nb - n + 1)
    sig = np.empty((N, L), dtype=np.uint64)
    lib().orc_signatures(_p(X), f32, N, m, m, _p(w), W, delta, n, L, K, _p(tabs.r),
                         _p(tabs.ln_c), _p(tabs.beta), _p(tabs.ln_w), _p(sig), _threads(threads))
    return sig


def tables_from_signatures(sig):
    """index.py:141-156 as CSR: per table j, (ukeys uint64[nb], offsets int64[nb+1],
    ids int64[N]); ids ascending within a bucket (stable argsort)."""
    N, L = sig.shape
    out = []
    for j in range(L):
        col = sig[:, j]
        order = np.argsort(col, kind="stable")
        sk = col[order]
        bnd = np.nonzero(np.diff(sk))[0] + 1
        starts = np.concatenate(([0], bnd)).astype(np.int64)
        ukeys = sk[starts].astype(np.uint64)
        offsets = np.concatenate((starts, [N])).astype(np.int64)
        out.append((ukeys, offsets, order.astype(np.int64)))
    return out


def tables_as_dicts(csr):
    """CSR -> the reference's list[dict[int, np.ndarray]] (index.py:151-155)."""
    res = []
    for ukeys, offsets, ids in csr:
        res.append({int(k): ids[offsets[b]:offsets[b + 1]] for b, k in enumerate(ukeys)})
    return res


def dtw_sq(x, y, r, abandon=-1.0):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return lib().orc_dtw(_p(x), _p(y), x.shape[0], r, abandon)


def envelope(x, r):
    x = np.ascontiguousarray(x, dtype=np.float64)
    m = x.shape[0]
    U = np.empty(m)
    Lo = np.empty(m)
    qb = np.empty(2 * m, dtype=np.int64)
    lib().orc_envelope(_p(x), m, r, _p(U), _p(Lo), _p(qb))
    return U, Lo


def lb_keogh_sq(c, U, Lo, abandon=-1.0):
    c = np.ascontiguousarray(c, dtype=np.float64)
    return lib().orc_lb_keogh_sq(_p(c), _p(np.ascontiguousarray(U)), _p(np.ascontiguousarray(Lo)),
                                 c.shape[0], abandon)


def cascade_search(X, cand, q, U, Lo, r, k):
    """dtw.py:171-236 -> (ids, d2, counters)."""
    X, f32 = _xarg(X)
    N, m = X.shape
    cand = np.ascontiguousarray(cand, dtype=np.int64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    size = min(k, cand.shape[0])
    ids = np.empty(max(size, 1), dtype=np.int64)
    d2 = np.empty(max(size, 1))
    cnt = np.zeros(5, dtype=np.int64)
    f = lib().orc_cascade_search(_p(X), f32, m, m, _p(cand), cand.shape[0], _p(q),
                                 _p(np.ascontiguousarray(U)), _p(np.ascontiguousarray(Lo)), r,
                                 k, _p(ids), _p(d2), _p(cnt))
    return ids[:f].copy(), d2[:f].copy(), cnt


@dataclass
class OracleIndex:
    X: np.ndarray
    W: int
    delta: int
    n: int
    L: int
    K: int
    seed: int
    band: float
    w: np.ndarray
    sig: np.ndarray
    csr: list


def build_index(X, W, delta, n, L, K, seed, band, threads=0):
    """build_index (index.py:159-172) with the K-aware signature."""
    X, _ = _xarg(X)
    w = make_filter(W, seed)
    sig = signatures(X, W, delta, n, L, K, seed, threads=threads, w=w)
    return OracleIndex(X, W, delta, n, L, K, seed, band, w, sig, tables_from_signatures(sig))


def query_batch(idx: OracleIndex, Q, k, threads=0):
    """query_index (index.py:204-273) for each row of Q, OpenMP over queries.
    Returns dict with ids (nq,k) int64 (-1 padded), d2 (nq,k), n (nq,),
    counters (nq,5), n_cand (nq,), qsig (nq,L)."""
    X, f32 = _xarg(idx.X)
    N, m = X.shape
    Q = np.ascontiguousarray(np.atleast_2d(Q), dtype=np.float64)
    nq = Q.shape[0]
    k = min(k, N)
    S = idx.L * idx.K
    nb = num_sketch_bits(m, idx.W, idx.delta)
    tabs = get_tables(idx.n, S, idx.seed, nb - idx.n + 1)
    ukeys = np.ascontiguousarray(np.concatenate([c[0] for c in idx.csr]))
    offsets = np.ascontiguousarray(np.concatenate([c[1] for c in idx.csr]))
    ids = np.ascontiguousarray(np.concatenate([c[2] for c in idx.csr]))
    tab_nb = np.array([c[0].shape[0] for c in idx.csr], dtype=np.int64)
    tab_kbase = np.concatenate(([0], np.cumsum(tab_nb)[:-1])).astype(np.int64)
    r = radius(idx.band, m)
    out_ids = np.full((nq, k), -1, dtype=np.int64)
    out_d2 = np.full((nq, k), np.inf)
    n_out = np.zeros(nq, dtype=np.int32)
    counters = np.zeros((nq, 5), dtype=np.int64)
    n_cand = np.zeros(nq, dtype=np.int64)
    qsig = np.zeros((nq, idx.L), dtype=np.uint64)
    w = np.ascontiguousarray(idx.w, dtype=np.float64)
    lib().orc_query_batch(_p(X), f32, N, m, m, _p(Q), nq, _p(w), idx.W, idx.delta, idx.n, idx.L,
                          idx.K, _p(tabs.r), _p(tabs.ln_c), _p(tabs.beta), _p(tabs.ln_w),
                          _p(ukeys), _p(offsets), _p(ids), _p(tab_nb), _p(tab_kbase), r, k,
                          _p(out_ids), _p(out_d2), _p(n_out), _p(counters), _p(n_cand), _p(qsig),
                          _threads(threads))
    return dict(ids=out_ids, d2=out_d2, n=n_out, counters=counters, n_cand=n_cand, qsig=qsig)


def dtw_many(X, ids, q, r, threads=0):
    """bench.py:37-42 over an id list -> d2 per id."""
    X, f32 = _xarg(X)
    N, m = X.shape
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    out = np.empty(ids.shape[0])
    lib().orc_dtw_many(_p(X), f32, m, m, _p(ids), ids.shape[0], _p(q), r, _p(out),
                       _threads(threads))
    return out


def brute_force_topk_over(X, cand, q, r, k, threads=0):
    """bench.py:45-60 restricted to `cand`: lexsort((ids, d2))[:k]."""
    cand = np.asarray(cand, dtype=np.int64)
    d2 = dtw_many(X, cand, q, r, threads)
    order = np.lexsort((cand, d2))[:k]
    return cand[order], d2[order]

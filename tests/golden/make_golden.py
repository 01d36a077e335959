"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The K=1 path is pinned by build_index / query_index directly
(index.py:159-273).  K>1 (BASELINE.json uses K=4) is pinned by
wmh.signature(concat=K) (wmh.py:107-125) per row + _tables_from_signatures
(index.py:141-156), and query_index with index.query_signature replaced by
the same K-aware composition.  Large arrays are stored
as SHA-256 digests plus an explicit head.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from fixture_data import CASES, SSH, case_data  # noqa: E402

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import sshts  # noqa: E402
from sshts import index as sidx  # noqa: E402
from sshts import wmh as swmh  # noqa: E402
from sshts import dtw as sdtw  # noqa: E402
from sshts.core import Dataset, TimeSeries  # noqa: E402
from sshts.shingle import tokenize_bits  # noqa: E402
from sshts.sketch import sketch_matrix, sketch_values  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def csr_digest(tables) -> str:
    h = hashlib.sha256()
    for t in tables:
        for key in sorted(t):
            h.update(np.uint64(key).tobytes())
            h.update(np.ascontiguousarray(t[key], dtype=np.int64).tobytes())
        h.update(b"|")
    return h.hexdigest()


def k_signatures(values, params, K):
    w = sshts.make_filter(params.W, params.seed).weights
    bits = sketch_matrix(values, w, params.delta)
    out = np.empty((values.shape[0], params.d), dtype=np.uint64)
    for i in range(values.shape[0]):
        stream = tokenize_bits(bits[i], params.n)
        tokens, counts = np.unique(stream, return_counts=True)
        ws = sshts.WeightedShingleSet(tokens=tokens, counts=counts.astype(np.int64), n=params.n)
        out[i] = swmh.signature(ws, params.d, params.seed, concat=K).values
    return out


def k_query_signature(K):
    def qs(index, q):
        values = q.values if isinstance(q, TimeSeries) else np.asarray(q, dtype=np.float64)
        bits = sketch_values(values, index.filter.weights, index.params.delta)
        stream = tokenize_bits(bits, index.params.n)
        tokens, counts = np.unique(stream, return_counts=True)
        ws = sshts.WeightedShingleSet(tokens=tokens, counts=counts.astype(np.int64), n=index.params.n)
        return swmh.signature(ws, index.params.d, index.params.seed, concat=K).values
    return qs


def run_queries(index, Q, k=10, fallback=False):
    res = []
    for q in Q:
        r = sidx.query_index(index, TimeSeries(values=q.astype(np.float64)), k, fallback_on_empty=fallback)
        c = r.stats.cascade
        res.append(dict(
            ids=r.ids, distances=r.distances, status=r.status, candidates=r.stats.candidates,
            counters=[c.kim_pruned, c.keogh_pruned, c.keogh2_pruned, c.dtw_computed, c.dtw_abandoned],
        ))
    return res


def case_fixture(name):
    X, Q, src, band = case_data(name)
    X64 = X.astype(np.float64)
    params = sidx.SshParams(band=band, **SSH)
    ds = Dataset(values=X64)
    w = sshts.make_filter(params.W, params.seed).weights
    bits = sketch_matrix(X64, w, params.delta)
    dots = np.lib.stride_tricks.sliding_window_view(X64, params.W, axis=1)[:, :: params.delta, :] @ w
    fx = dict(case=name, N=int(X.shape[0]), m=int(X.shape[1]), band=band,
              bits_sha=sha(bits), bits_head=bits[:8].tolist(),
              min_abs_dot=float(np.abs(dots).min()),
              n_dot_below_1e9=int((np.abs(dots) < 1e-9).sum()))
    # shingle sets of the first rows (shingle.py:56-75)
    sets = []
    for i in range(6):
        stream = tokenize_bits(bits[i], params.n)
        tok, cnt = np.unique(stream, return_counts=True)
        sets.append(dict(tokens=[int(t) for t in tok], counts=[int(c) for c in cnt]))
    fx["shingle_sets"] = sets
    # K = 1: the reference build_index / query_index path itself
    index1 = sidx.build_index(ds, params)
    fx["sig_k1_sha"] = sha(index1.signatures)
    fx["sig_k1_head"] = [[int(v) for v in row] for row in index1.signatures[:4]]
    fx["tables_k1_sha"] = csr_digest(index1.tables)
    fx["tables_k1_nbuckets"] = [len(t) for t in index1.tables]
    fx["queries_k1"] = run_queries(index1, Q)
    # K = 4 (BASELINE.json): wmh.signature(concat=4) + _tables_from_signatures
    sig4 = k_signatures(X64, params, 4)
    tables4 = sidx._tables_from_signatures(sig4)
    fx["sig_k4_sha"] = sha(sig4)
    fx["sig_k4_head"] = [[int(v) for v in row] for row in sig4[:4]]
    fx["tables_k4_sha"] = csr_digest(tables4)
    fx["tables_k4_nbuckets"] = [len(t) for t in tables4]
    index4 = sidx.SshIndex(params=params, filter=index1.filter, tables=tables4, dataset=ds,
                           signatures=sig4, normalized=True)
    orig = sidx.query_signature
    sidx.query_signature = k_query_signature(4)
    try:
        fx["queries_k4"] = run_queries(index4, Q)
        fx["qsig_k4"] = [[int(v) for v in sidx.query_signature(index4, q.astype(np.float64))] for q in Q]
    finally:
        sidx.query_signature = orig
    fx["qsig_k1"] = [[int(v) for v in sidx.query_signature(index1, q.astype(np.float64))] for q in Q]
    fx["query_src"] = [int(s) for s in src]
    return fx


def cws_fixture():
    """_cws_keys on synthetic weighted sets with large counts (count>1 path)."""
    rng = np.random.default_rng(77)
    out = []
    for trial in range(12):
        D = int(rng.integers(1, 200))
        tokens = np.sort(rng.choice(1 << 15, size=D, replace=False)).astype(np.uint64)
        if trial % 3 == 0:
            counts = rng.integers(1, 700, size=D)
        elif trial % 3 == 1:
            counts = np.ones(D, dtype=np.int64)
        else:
            counts = rng.geometric(0.5, size=D)
        counts = counts.astype(np.int64)
        keys = swmh._cws_keys(tokens, counts, np.arange(80, dtype=np.uint64), 0)
        seed = int(rng.integers(0, 1 << 40)) if trial >= 9 else 0
        keys_s = swmh._cws_keys(tokens, counts, np.arange(80, dtype=np.uint64), seed)
        out.append(dict(tokens=[int(t) for t in tokens], counts=[int(c) for c in counts],
                        keys=[int(k) for k in keys], seed=seed, keys_seed=[int(k) for k in keys_s]))
    return out


def dtw_fixture():
    rng = np.random.default_rng(99)
    pairs = []
    for trial in range(40):
        m = int(rng.choice([1, 2, 3, 8, 17, 64, 128]))
        band = float(rng.choice([0.0, 0.05, 0.1, 0.5, 1.0]))
        x = rng.standard_normal(m)
        y = rng.standard_normal(m)
        r = sdtw.WarpingParams(band=band).radius(m)
        d2 = float(sdtw._dtw_band_sq(x, y, r, -1.0))
        env = sdtw.build_envelope(y, sdtw.WarpingParams(band=band))
        lbk = float(sdtw._lb_keogh_sq(x, env.upper, env.lower, -1.0))
        pairs.append(dict(x=x.tolist(), y=y.tolist(), band=band, r=r, d2=d2, lb_keogh_sq=lbk,
                          upper=env.upper.tolist(), lower=env.lower.tolist()))
    spec = float(sdtw.dtw_distance(np.array([1.0, 2, 3]), np.array([2.0, 3, 4]), sdtw.WarpingParams(band=1.0)))
    return dict(pairs=pairs, spec_sqrt2=spec)


def spec_fixture():
    from sshts.sketch import BitSketch
    filt_bits = sketch_values(np.array([1.0, 2, 4, 1]), np.array([0.1, -0.1]), 2)
    sh = sshts.shingle_sketch(BitSketch(bits=np.array([1, 1, -1, -1, 1, 1], dtype=np.int8), delta=1,
                                        source_len=6), 2)
    return dict(sketch=[int(b) for b in filt_bits], shingle=sh.as_dict(),
                filter80=sshts.make_filter(80, 0).weights.tolist())


def empty_candidates_fixture():
    """A query that probes no bucket: status no-candidates / fallback."""
    X, _, _, band = case_data("rw512")
    X64 = X.astype(np.float64)
    params = sidx.SshParams(band=band, **SSH)
    ds = Dataset(values=X64[:200])
    index1 = sidx.build_index(ds, params)
    m = X.shape[1]
    t = np.arange(m)
    q = np.sin(2 * np.pi * t / 7.0) + 0.3 * np.sin(2 * np.pi * t / 3.1)
    q = (q - q.mean()) / q.std()
    r0 = sidx.query_index(index1, TimeSeries(values=q), 10)
    r1 = sidx.query_index(index1, TimeSeries(values=q), 10, fallback_on_empty=True)
    return dict(query=q.tolist(), status=r0.status, candidates=r0.stats.candidates,
                fallback_status=r1.status, fallback_ids=r1.ids, fallback_distances=r1.distances)


def persist_fixture():
    """save_index / save_dataset bytes of the reference (index.py:287-310,
    core.py:181-194): SHA-256 of the SSHI file and its f64le sidecar for a K=1
    index over rw512[:200] saved as 'idx.sshi', and of the CSV of 5 rows."""
    import tempfile

    from sshts.core import save_dataset

    X, Q, _, band = case_data("rw512")
    params = sidx.SshParams(band=band, **SSH)
    ds = Dataset(values=X[:200].astype(np.float64))
    index = sidx.build_index(ds, params)
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "idx.sshi"
        sidx.save_index(index, p)
        idx_sha = hashlib.sha256(p.read_bytes()).hexdigest()
        side_sha = hashlib.sha256((Path(td) / "idx.sshi.sshd").read_bytes()).hexdigest()
        idx_len = len(p.read_bytes())
        c = Path(td) / "five.csv"
        save_dataset(Dataset(values=X[:5].astype(np.float64)), c, fmt="csv")
        csv_sha = hashlib.sha256(c.read_bytes()).hexdigest()
    return dict(n=200, index_sha256=idx_sha, index_bytes=idx_len, sidecar_sha256=side_sha, csv5_sha256=csv_sha)


def windows_fixture():
    """make_dataset (core.py:162-169) of two seeded random-walk recordings:
    SHA-256 of the float64 window matrices (t=128 and t=1000; the latter
    exercises numpy's recursive pairwise split)."""
    from sshts.core import generate_random_walk, make_dataset

    out = {}
    for length, t, seed in ((20_000, 128, 7), (6_000, 1000, 8)):
        rec = generate_random_walk(length, seed)
        ds = make_dataset(rec, t, normalize=True)
        out[f"rw{length}_t{t}"] = dict(length=length, t=t, seed=seed, count=ds.n_series,
                                       sha256=sha(np.ascontiguousarray(ds.values, dtype=np.float64)))
    return out


def srp_fixture():
    """srp_matrix (index.py:420-423) over rw512[:300] (f64 of the f32 data),
    64 and 100 bits; precision_at_k / ndcg_at_k on fixed rankings."""
    from sshts import bench as sbench

    X, _, _, _ = case_data("rw512")
    V = X[:300].astype(np.float64)
    out = {}
    for bits, seed in ((64, 3), (100, 11)):
        out[f"b{bits}_s{seed}"] = sha(sidx.srp_matrix(V, bits, seed))
    retrieved = [5, 3, 9, 1, 7, 2, 8]
    gold = [3, 5, 1, 4, 9, 6, 0]
    out["metrics"] = {str(k): [sbench.precision_at_k(retrieved, gold, k), sbench.ndcg_at_k(retrieved, gold, k)]
                      for k in (1, 3, 5, 7)}
    return out


def main():
    out = dict(ssh=SSH, numpy=np.__version__, cases={})
    for name in CASES:
        print("case", name, flush=True)
        out["cases"][name] = case_fixture(name)
    out["cws"] = cws_fixture()
    out["dtw"] = dtw_fixture()
    out["spec"] = spec_fixture()
    out["empty"] = empty_candidates_fixture()
    out["persist"] = persist_fixture()
    out["windows"] = windows_fixture()
    out["srp"] = srp_fixture()
    (HERE / "golden.json").write_text(json.dumps(out, indent=None, separators=(",", ":")))
    print("wrote", HERE / "golden.json")


if __name__ == "__main__":
    main()

"""Drop-in device implementation of the reference index API (index.py:32-273).

Same names, dataclasses, validation messages and error types as the
reference `sshts.index`; `SshParams` gains `K` (the CWS concatenation order
of wmh.signature(concat=K), wmh.py:107-125; default 1 = reference
build_index behaviour).  Every stage runs in libsshgpu.so on an sm_100 GPU:

  build_index       -> ssh_signatures (K1-K3) + ssh_index_build (K4)
  query_signature   -> ssh_signatures on the query
  probe_candidates  -> ssh_probe (K6)
  query_index(_batch) -> ssh_query_batch (K5-K10)

PyTorch is used only for device memory and the current CUDA stream.
"""

from __future__ import annotations

import contextlib
import ctypes
import math
import threading
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import cws
from .core import ConfigError, Dataset, SshError, TimeSeries, _is_torch

MAX_SHINGLE_BITS = 64
DEVICE_MAX_SHINGLE_BITS = 20


def num_sketch_bits(m: int, W: int, delta: int) -> int:
    """floor((m - W) / delta) + 1 (sketch.py:46-48)."""
    return (m - W) // delta + 1


@dataclass(frozen=True)
class WarpingParams:
    """Sakoe-Chiba constraint |i - j| <= radius, radius = round(band * m) (dtw.py:28-39)."""

    band: float = 0.05

    def __post_init__(self):
        if not 0.0 <= self.band <= 1.0:
            raise ValueError(f"warping band must be in [0, 1], got {self.band}")

    def radius(self, m: int) -> int:
        return int(round(self.band * m))


@dataclass(frozen=True)
class SearchStats:
    """Cascade counters (dtw.py:50-72)."""

    candidates: int
    kim_pruned: int
    keogh_pruned: int
    keogh2_pruned: int
    dtw_computed: int
    dtw_abandoned: int

    @property
    def pruned(self) -> int:
        return self.kim_pruned + self.keogh_pruned + self.keogh2_pruned

    @property
    def pruned_fraction(self) -> float:
        return 0.0 if self.candidates == 0 else self.pruned / self.candidates

    def fraction(self, bound: str) -> float:
        return 0.0 if self.candidates == 0 else getattr(self, f"{bound}_pruned") / self.candidates


@dataclass(frozen=True)
class RandomFilter:
    weights: np.ndarray  # (W,) float64
    seed: int

    @property
    def W(self) -> int:
        return self.weights.shape[0]


def make_filter(W: int, seed: int) -> RandomFilter:
    """Deterministic filter: W standard normal draws from the given seed
    (sketch.py:36-43; same ValueError messages)."""
    return RandomFilter(weights=cws.filter_weights(W, seed), seed=seed)


@dataclass(frozen=True)
class SshParams:
    """W, delta, n, d (= L tables), seed, band (index.py:32-71) + K."""

    W: int = 30
    delta: int = 5
    n: int = 15
    d: int = 20
    seed: int = 0
    band: float = 0.05
    K: int = 1

    def __post_init__(self):
        if self.W < 1:
            raise ConfigError(f"filter length W must be >= 1, got {self.W}")
        if self.delta < 1:
            raise ConfigError(f"step size delta must be >= 1, got {self.delta}")
        if not 1 <= self.n <= MAX_SHINGLE_BITS:
            raise ConfigError(f"shingle length n must be in [1, {MAX_SHINGLE_BITS}], got {self.n}")
        if self.d < 1:
            raise ConfigError(f"table count d must be >= 1, got {self.d}")
        if self.seed < 0:
            raise ConfigError(f"seed must be non-negative, got {self.seed}")
        if not 0.0 <= self.band <= 1.0:
            raise ConfigError(f"warping band must be in [0, 1], got {self.band}")
        if self.K < 1:
            raise ConfigError(f"concat order K must be >= 1, got {self.K}")

    def validate_for_length(self, t: int) -> None:
        if t < self.W:
            raise ConfigError(f"series length t={t} violates t >= W (W={self.W})")
        nb = num_sketch_bits(t, self.W, self.delta)
        if nb < self.n:
            raise ConfigError(
                f"sketch length floor((t-W)/delta)+1 = {nb} violates >= n "
                f"(t={t}, W={self.W}, delta={self.delta}, n={self.n})"
            )
        if self.n > DEVICE_MAX_SHINGLE_BITS:
            raise ConfigError(
                f"shingle length n={self.n} exceeds the device limit {DEVICE_MAX_SHINGLE_BITS} "
                "(CWS variates are tabulated over the 2^n token universe)")

    def warping(self) -> WarpingParams:
        return WarpingParams(band=self.band)

    @property
    def L(self) -> int:
        return self.d


@dataclass(frozen=True)
class QueryStats:
    n_indexed: int
    candidates: int
    cascade: SearchStats

    @property
    def hash_pruned_fraction(self) -> float:
        return 1.0 - self.candidates / self.n_indexed

    @property
    def bound_pruned_fraction(self) -> float:
        return self.cascade.pruned / self.n_indexed

    @property
    def total_pruned_fraction(self) -> float:
        return 1.0 - self.cascade.dtw_computed / self.n_indexed


@dataclass(frozen=True)
class QueryResult:
    ids: list
    distances: list
    stats: QueryStats
    timings: dict
    status: str = "ok"  # "ok" | "no-candidates" | "fallback"
    warning: str | None = None


# ------------------------------------------------------------ device context

def _torch():
    import torch

    return torch


def _device_index(device) -> int:
    torch = _torch()
    if device is None:
        if not torch.cuda.is_available():
            raise SshError("no CUDA device available: the SSH device path needs an sm_100 GPU "
                           "(there is no CPU fallback)")
        return torch.cuda.current_device()
    return torch.device(device).index if not isinstance(device, int) else device


class DeviceContext:
    """One ssh_ctx per (device, parameters, series length).

    The ssh_ctx owns grow-only scratch slots that every build / query call
    reuses, so calls on one context must not overlap.  The
    reference's query_index is pure and callable from many threads at once
    (bench.py:129-133); `use()` makes the device path equally
    safe: it serialises the native calls on the context and orders each
    call's stream after the previous call's device work (an event), so two
    threads on different CUDA streams never share scratch in flight."""

    def __init__(self, device: int, params: SshParams, m: int):
        self.device = device
        self.params = params
        self.m = m
        self.lock = threading.RLock()
        self._last = None
        L = nat.lib()
        h = ctypes.c_void_p()
        nat.check(L.ssh_ctx_create(device, ctypes.byref(h)), "ssh_ctx_create")
        self.handle = h
        w = cws.filter_weights(params.W, params.seed)
        self.filter = RandomFilter(weights=w, seed=params.seed)
        S = params.K * params.d
        r, lnc, beta = cws.tables(params.n, S, params.seed)
        nb = num_sketch_bits(m, params.W, params.delta)
        max_count = nb - params.n + 1
        lnw = cws.ln_counts(max_count)
        p = nat.ssh_params(m=m, W=params.W, delta=params.delta, n=params.n, L=params.d, K=params.K,
                           seed=params.seed, radius=params.warping().radius(m), reserved=0)
        self.cparams = p
        nat.check(L.ssh_ctx_set_params(h, ctypes.byref(p), nat.ptr(np.ascontiguousarray(w)),
                                       nat.ptr(r), nat.ptr(lnc), nat.ptr(beta), nat.ptr(lnw),
                                       max_count), "ssh_ctx_set_params")
        self.nb = L.ssh_num_sketch_bits(h)
        self.words = L.ssh_sketch_words(h)
        self.T = L.ssh_tokens_per_series(h)

    @contextlib.contextmanager
    def use(self):
        """Exclusive, stream-ordered use of the context (see the class doc)."""
        with self.lock:
            torch = _torch()
            st = torch.cuda.current_stream(self.device)
            if self._last is not None:
                st.wait_event(self._last)
            try:
                yield st
            finally:
                ev = torch.cuda.Event()
                ev.record(st)
                self._last = ev

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                nat.lib().ssh_ctx_destroy(self.handle)
        except Exception:
            pass


_ctx_cache: dict = {}
_ctx_lock = threading.Lock()


def get_context(device: int, params: SshParams, m: int) -> DeviceContext:
    key = (device, params, m)
    with _ctx_lock:
        c = _ctx_cache.get(key)
        if c is None:
            if len(_ctx_cache) >= 4:
                _ctx_cache.pop(next(iter(_ctx_cache)))
            c = DeviceContext(device, params, m)
            _ctx_cache[key] = c
        return c


def _stream_ptr(device: int):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Float32RoundingWarning(UserWarning):
    """float64 input that float32 cannot represent exactly was rounded."""


def _warn_f32_rounding(values, what: str) -> None:
    """The device path computes on float32 series (BASELINE.json's workloads
    are float32; the oracle upcasts them exactly).  A float64 input whose
    values are not all float32-representable is rounded once, so sketch
    signs, signatures and distances can differ from the reference's float64
    evaluation of the unrounded values: say so (never silently)."""
    if _is_torch(values):
        torch = _torch()
        if values.dtype != torch.float64:
            return
        changed = bool((values.float().double() != values).any())
    else:
        v = np.asarray(values)
        if v.dtype != np.float64:
            return
        changed = bool(np.any(v.astype(np.float32).astype(np.float64) != v))
    if changed:
        warnings.warn(f"{what} values are float64 and not exactly representable in float32; the device "
                      "path rounds them to float32 once (results are the reference's for the rounded "
                      "values)", Float32RoundingWarning, stacklevel=3)


def _host_f32(values):
    """Contiguous f32 CPU tensor view of host series (None for device tensors)."""
    torch = _torch()
    if _is_torch(values):
        if values.is_cuda:
            return None
        t = values.to(dtype=torch.float32)
    else:
        t = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32))
    return t.contiguous()


def _as_device_f32(values, device: int):
    torch = _torch()
    if _is_torch(values):
        t = values.to(device=f"cuda:{device}", dtype=torch.float32)
    else:
        t = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).to(f"cuda:{device}")
    return t.contiguous()


# ------------------------------------------------------------------ index

class _TablesHandle:
    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            if self.handle:
                nat.lib().ssh_index_destroy(self.handle)
        except Exception:
            pass


@dataclass(eq=False)
class SshIndex:
    """params, filter, tables, dataset, signatures, normalized (index.py:103-110)
    plus the device state: X (f32 series), signature tensor, CSR tables."""

    params: SshParams
    filter: RandomFilter
    dataset: Dataset
    normalized: bool
    device: int
    X: object  # torch float32 (N, m) on device
    sig_dev: object  # torch int64 (N, L) on device (uint64 bit patterns)
    id_base: int = 0
    _tables: object = None
    _tables_host: list | None = field(default=None, repr=False)
    _sig_host: np.ndarray | None = field(default=None, repr=False)

    @property
    def n_series(self) -> int:
        return int(self.X.shape[0])

    @property
    def length(self) -> int:
        return int(self.X.shape[1])

    @property
    def signatures(self) -> np.ndarray:
        """(N, d) uint64 (index.py:109), copied from the device on first use."""
        if self._sig_host is None:
            self._sig_host = self.sig_dev.cpu().numpy().view(np.uint64)
        return self._sig_host

    def summaries(self, r0: int = 0, n: int | None = None):
        """Rerank summaries of rows [r0, r0 + n) copied to the host (inspection,
        tests): (rec u8[n][64], codes u8[n][cstride], mp) — rec = f32 {lo, sc,
        x0, x_last} + u8 PAA codes; codes = u8 sample codes x8[mp] followed by
        interleaved (U8, L8) envelope codes (layout in csrc/common.cuh)."""
        n = self.n_series - r0 if n is None else n
        L = nat.lib()
        mp = ctypes.c_int32()
        cs = ctypes.c_int64()
        nat.check(L.ssh_index_copy_summaries(self._tables.handle, 0, 0, None, None, ctypes.byref(mp),
                                             ctypes.byref(cs), _stream_ptr(self.device)))
        rec = np.empty((n, 64), dtype=np.uint8)
        codes = np.empty((n, cs.value), dtype=np.uint8)
        nat.check(L.ssh_index_copy_summaries(self._tables.handle, int(r0), int(n), nat.ptr(rec), nat.ptr(codes),
                                             None, None, _stream_ptr(self.device)), "ssh_index_copy_summaries")
        return rec, codes, mp.value

    def table_csr(self, j: int):
        """Table j as host CSR: (keys uint64[nb], offsets int64[nb+1], ids int64[N])."""
        L = nat.lib()
        nb = ctypes.c_int64()
        nat.check(L.ssh_index_num_buckets(self._tables.handle, j, ctypes.byref(nb)))
        keys = np.empty(nb.value, dtype=np.uint64)
        offsets = np.empty(nb.value + 1, dtype=np.int64)
        ids = np.empty(self.n_series, dtype=np.int64)
        nat.check(L.ssh_index_export(self._tables.handle, j, nat.ptr(keys), nat.ptr(offsets),
                                     nat.ptr(ids), _stream_ptr(self.device)), "ssh_index_export")
        return keys, offsets, ids

    @property
    def tables(self) -> list:
        """The reference's list[dict[key, ids ascending]] (index.py:141-156), materialised lazily."""
        if self._tables_host is None:
            out = []
            for j in range(self.params.d):
                keys, offsets, ids = self.table_csr(j)
                out.append({int(k): ids[offsets[b]:offsets[b + 1]] for b, k in enumerate(keys)})
            self._tables_host = out
        return self._tables_host

    def context(self) -> DeviceContext:
        return get_context(self.device, self.params, self.length)

    @property
    def sketch_stats(self) -> dict:
        """Sketch windows of this build whose f32 screen was undecided and that
        were re-evaluated with the reference's exact f64 dot ("rechecked"), and
        of those the near-zero sign ties |dot| < 1e-9 ("near_zero"; sign(0) is
        +1 as in sketch.py:60).  Zeros for an index built from signatures."""
        out = np.zeros(2, dtype=np.int64)
        nat.check(nat.lib().ssh_index_sketch_stats(self._tables.handle, nat.ptr(out), _stream_ptr(self.device)),
                  "ssh_index_sketch_stats")
        return {"rechecked": int(out[0]), "near_zero": int(out[1])}


def _check_params_length(params: SshParams, m: int):
    params.validate_for_length(m)


def compute_signatures_device(ctx: DeviceContext, X, stats=None):
    """(N, L) int64 device tensor of signatures (K1-K3 fused)."""
    torch = _torch()
    N = int(X.shape[0])
    sig = torch.empty((N, ctx.params.d), dtype=torch.int64, device=X.device)
    if N:
        with ctx.use():
            nat.check(nat.lib().ssh_signatures(ctx.handle, nat.ptr(X), N, int(X.stride(0)), nat.ptr(sig),
                                               nat.ptr(stats), _stream_ptr(ctx.device)), "ssh_signatures")
    return sig


def build_index(dataset, params: SshParams, normalized: bool = True, threads: int = 1,
                device=None, id_base: int = 0) -> SshIndex:
    """Hash every series into d tables (index.py:159-172).  `threads` is
    accepted for API compatibility; the device path is always parallel."""
    if not isinstance(dataset, Dataset):
        dataset = Dataset(values=dataset)
    params.validate_for_length(dataset.length)
    dev = _device_index(device)
    ctx = get_context(dev, params, dataset.length)
    torch = _torch()
    _warn_f32_rounding(dataset.values, "dataset")
    host = _host_f32(dataset.values)
    handle = ctypes.c_void_p()
    if host is not None:
        # host series: chunked copy into X overlapped with the per-chunk kernels
        N, m = host.shape
        X = torch.empty((N, m), dtype=torch.float32, device=f"cuda:{dev}")
        sig = torch.empty((N, params.d), dtype=torch.int64, device=X.device)
        with ctx.use():
            nat.check(nat.lib().ssh_build_index_host(ctx.handle, host.data_ptr(), N, m, int(id_base), nat.ptr(X),
                                                     nat.ptr(sig), ctypes.byref(handle), _stream_ptr(dev)),
                      "ssh_build_index_host")
    else:
        X = _as_device_f32(dataset.values, dev)
        sig = torch.empty((int(X.shape[0]), params.d), dtype=torch.int64, device=X.device)
        with ctx.use():
            nat.check(nat.lib().ssh_build_index(ctx.handle, nat.ptr(X), int(X.shape[0]), int(X.stride(0)),
                                                int(id_base), nat.ptr(sig), ctypes.byref(handle),
                                                _stream_ptr(dev)), "ssh_build_index")
    tables = _TablesHandle(handle)
    return SshIndex(params=params, filter=ctx.filter, dataset=dataset, normalized=normalized,
                    device=dev, X=X, sig_dev=sig, id_base=id_base, _tables=tables)


def index_from_signatures(dataset, params: SshParams, sig, normalized: bool = True, device=None,
                          id_base: int = 0, filter_weights=None, filter_seed=None) -> SshIndex:
    """An index over `dataset` whose (N, d) uint64 signatures are already known
    (load_index): device tables from the signatures (ssh_index_build) and the
    rerank summaries of the series (ssh_index_summarize)."""
    if not isinstance(dataset, Dataset):
        dataset = Dataset(values=dataset)
    params.validate_for_length(dataset.length)
    dev = _device_index(device)
    ctx = get_context(dev, params, dataset.length)
    if filter_weights is not None and not np.array_equal(np.asarray(filter_weights, dtype=np.float64),
                                                         ctx.filter.weights):
        raise ConfigError("index filter weights differ from make_filter(W, seed)")
    if filter_seed is not None and int(filter_seed) != ctx.filter.seed:
        raise ConfigError(f"index filter seed {filter_seed} differs from params.seed {ctx.filter.seed}")
    torch = _torch()
    _warn_f32_rounding(dataset.values, "dataset")
    X = _as_device_f32(dataset.values, dev)
    sig_h = np.ascontiguousarray(np.asarray(sig, dtype=np.uint64))
    if sig_h.shape != (X.shape[0], params.d):
        raise ConfigError(f"signatures shape {sig_h.shape} != ({X.shape[0]}, {params.d})")
    sig_d = torch.from_numpy(sig_h.view(np.int64)).to(X.device)
    handle = ctypes.c_void_p()
    L = nat.lib()
    with ctx.use():
        nat.check(L.ssh_index_build(ctx.handle, nat.ptr(sig_d), int(X.shape[0]), int(id_base),
                                    ctypes.byref(handle), _stream_ptr(dev)), "ssh_index_build")
        tables = _TablesHandle(handle)
        nat.check(L.ssh_index_summarize(ctx.handle, handle, nat.ptr(X), int(X.stride(0)), _stream_ptr(dev)),
                  "ssh_index_summarize")
    return SshIndex(params=params, filter=ctx.filter, dataset=dataset, normalized=normalized,
                    device=dev, X=X, sig_dev=sig_d, id_base=id_base, _tables=tables)


@dataclass
class SearchResult:
    """exact_search result (dtw.py:75-81)."""

    ids: list
    distances: list
    stats: SearchStats
    warning: str | None = None


def exact_search_batch(dataset, Q, k: int, params: WarpingParams = WarpingParams(), device=None) -> list:
    """exact_search (dtw.py:293-326) for every row of Q: the exact top-k by
    (DTW^2, id) over the whole dataset, on the device (an index without bucket
    tables; every query's candidate set is the full shard)."""
    if not isinstance(dataset, Dataset):
        dataset = Dataset(values=dataset)
    Qh = Q.detach().double().cpu().numpy() if _is_torch(Q) else np.asarray(Q, dtype=np.float64)
    if Qh.ndim == 1:
        Qh = Qh.reshape(1, -1)
    if dataset.length != Qh.shape[1]:
        raise ValueError(f"query length {Qh.shape[1]} does not match dataset length {dataset.length}")
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    _warn_f32_rounding(dataset.values, "dataset")
    _warn_f32_rounding(Qh, "query")
    warning = None
    if k > dataset.n_series:
        warning = f"k={k} exceeds dataset size {dataset.n_series}; returning all series"
        k = dataset.n_series
    sp = SshParams(W=min(30, dataset.length), delta=5, n=1, band=params.band)
    dev = _device_index(device)
    ctx = get_context(dev, sp, dataset.length)
    torch = _torch()
    X = _as_device_f32(dataset.values, dev)
    handle = ctypes.c_void_p()
    L = nat.lib()
    with ctx.use():
        nat.check(L.ssh_index_create_bare(ctx.handle, nat.ptr(X), int(X.shape[0]), int(X.stride(0)), 0,
                                          ctypes.byref(handle), _stream_ptr(dev)), "ssh_index_create_bare")
    bare = _TablesHandle(handle)
    Qd = _as_device_f32(Qh, dev)
    nq = int(Qd.shape[0])
    ids = torch.empty((nq, k), dtype=torch.int64, device=X.device)
    d2 = torch.empty((nq, k), dtype=torch.float64, device=X.device)
    n_out = torch.empty(nq, dtype=torch.int32, device=X.device)
    n_cand = torch.empty(nq, dtype=torch.int64, device=X.device)
    counters = torch.empty((nq, 5), dtype=torch.int64, device=X.device)
    status = torch.empty(nq, dtype=torch.int32, device=X.device)
    with ctx.use():
        nat.check(L.ssh_query_batch(ctx.handle, bare.handle, nat.ptr(X), nat.ptr(Qd), nq, k, nat.SSH_QUERY_EXACT,
                                    nat.ptr(ids), nat.ptr(d2), nat.ptr(n_out), nat.ptr(n_cand),
                                    nat.ptr(counters), nat.ptr(status), _stream_ptr(dev)), "ssh_query_batch")
    ids, d2, n_out, counters = ids.cpu().numpy(), d2.cpu().numpy(), n_out.cpu().numpy(), counters.cpu().numpy()
    del bare
    out = []
    for i in range(nq):
        n = int(n_out[i])
        c = counters[i]
        stats = SearchStats(candidates=dataset.n_series, kim_pruned=int(c[0]), keogh_pruned=int(c[1]),
                            keogh2_pruned=int(c[2]), dtw_computed=int(c[3]), dtw_abandoned=int(c[4]))
        out.append(SearchResult(ids=[int(v) for v in ids[i, :n]],
                                distances=[float(v) for v in np.sqrt(d2[i, :n])], stats=stats, warning=warning))
    return out


def exact_search(dataset, q, k: int, params: WarpingParams = WarpingParams(), device=None) -> SearchResult:
    """dtw.py:293-326 on the device."""
    qv = q.values if isinstance(q, TimeSeries) else q
    return exact_search_batch(dataset, qv, k, params, device)[0]


def compute_signatures(values, params: SshParams, weights=None, threads: int = 1, device=None):
    """(N, d) uint64 signature matrix (index.py:123-138, with the K fold)."""
    ds = values if isinstance(values, Dataset) else Dataset(values=values)
    params.validate_for_length(ds.length)
    dev = _device_index(device)
    ctx = get_context(dev, params, ds.length)
    if weights is not None and not np.array_equal(np.asarray(weights, dtype=np.float64),
                                                  ctx.filter.weights):
        raise ConfigError("custom filter weights are not supported on device; "
                          "the filter is make_filter(W, seed)")
    X = _as_device_f32(ds.values, dev)
    return compute_signatures_device(ctx, X).cpu().numpy().view(np.uint64)


def _query_values(q) -> np.ndarray:
    if isinstance(q, TimeSeries):
        return q.values
    if _is_torch(q):
        return q.detach().double().cpu().numpy()
    return np.asarray(q, dtype=np.float64)


def query_signature(index: SshIndex, q) -> np.ndarray:
    """(d,) uint64 signature of one query (index.py:175-181)."""
    qv = _query_values(q)
    torch = _torch()
    Q = _as_device_f32(qv.reshape(1, -1), index.device)
    sig = compute_signatures_device(index.context(), Q)
    return sig.cpu().numpy().view(np.uint64)[0]


def probe_candidates(index: SshIndex, qsig) -> np.ndarray:
    """Deduplicated union of the d probed buckets, ascending ids (index.py:184-190)."""
    torch = _torch()
    qs = torch.from_numpy(np.ascontiguousarray(np.asarray(qsig, dtype=np.uint64).view(np.int64))
                          .reshape(1, -1)).to(f"cuda:{index.device}")
    N = index.n_series
    NW = (N + 31) // 32
    bm = torch.empty((1, NW), dtype=torch.int32, device=qs.device)
    nc = torch.empty(1, dtype=torch.int64, device=qs.device)
    ctx = index.context()
    with ctx.use():
        nat.check(nat.lib().ssh_probe(ctx.handle, index._tables.handle, nat.ptr(qs), 1,
                                      nat.ptr(bm), nat.ptr(nc), _stream_ptr(index.device)), "ssh_probe")
    words = bm.cpu().numpy().view(np.uint32)[0]
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:N]
    return np.nonzero(bits)[0].astype(np.int64) + index.id_base


@dataclass
class BatchResult:
    """Raw device-batch output (host numpy)."""

    ids: np.ndarray       # (nq, k) int64, -1 padded
    d2: np.ndarray        # (nq, k) float64 squared DTW
    n_out: np.ndarray     # (nq,) int32
    n_cand: np.ndarray    # (nq,) int64
    counters: np.ndarray  # (nq, 5) int64
    seconds: float


def query_batch_device(index: SshIndex, Q, k: int, fallback_on_empty: bool = False, phase_ms: list | None = None,
                       exact: bool = False):
    """Run ssh_query_batch on a device tensor Q (nq, m) f32; returns device tensors."""
    torch = _torch()
    nq = int(Q.shape[0])
    dev = Q.device
    ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
    d2 = torch.empty((nq, k), dtype=torch.float64, device=dev)
    n_out = torch.empty(nq, dtype=torch.int32, device=dev)
    n_cand = torch.empty(nq, dtype=torch.int64, device=dev)
    counters = torch.empty((nq, 5), dtype=torch.int64, device=dev)
    status = torch.empty(nq, dtype=torch.int32, device=dev)
    flags = (nat.SSH_QUERY_FALLBACK_ON_EMPTY if fallback_on_empty else 0) | (nat.SSH_QUERY_EXACT if exact else 0)
    ctx = index.context()
    with ctx.use():
        nat.check(nat.lib().ssh_query_batch(
            ctx.handle, index._tables.handle, nat.ptr(index.X), nat.ptr(Q), nq, k, flags,
            nat.ptr(ids), nat.ptr(d2), nat.ptr(n_out), nat.ptr(n_cand), nat.ptr(counters),
            nat.ptr(status), _stream_ptr(index.device)), "ssh_query_batch")
        if phase_ms is not None:
            ph = (ctypes.c_double * 3)()
            nat.check(nat.lib().ssh_query_phase_ms(ctx.handle, ph), "ssh_query_phase_ms")
            phase_ms[:] = list(ph)
    return ids, d2, n_out, n_cand, counters, status


def _validate_k(index: SshIndex, k: int):
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    n = index.n_series
    warning = None
    if k > n:
        warning = f"k={k} exceeds index size {n}; returning at most {n} series"
        k = n
    return k, warning


def _results_from_arrays(ids, d2, n_out, n_cand, counters, status, N: int, dt: float, warning,
                         phase_ms=None) -> list:
    """QueryResult per query from the host copies of ssh_query_batch's outputs
    (ids/d2 (nq, k), n_out, n_cand, counters (nq, 5), status: 0 ok, 1 no-candidates,
    2 fallback); distances = sqrt(d2) (index.py:268).

    timings carries the reference's keys "hash", "probe" and "rerank"
    (index.py:235,265; read by cli.py:184-185), in seconds: each query's share
    of the batch's device time in that phase (phase_ms, ssh_query_phase_ms),
    plus "batch" (host wall time of the whole batch) and "per_query"."""
    nq = int(status.shape[0])
    # whole-batch conversions to Python scalars (tolist is exact: int64 -> int,
    # float64 -> float); the per-query loop only slices lists
    ids_l = ids.tolist()
    with np.errstate(invalid="ignore"):  # entries past n_out are unused
        dist_l = np.sqrt(d2).tolist()
    n_out_l = n_out.tolist()
    n_cand_l = n_cand.tolist()
    cnt_l = counters.tolist()
    status_l = status.tolist()
    per_q = dt / max(1, nq)
    ph = [0.0, 0.0, 0.0] if phase_ms is None else [v / 1e3 / max(1, nq) for v in phase_ms]
    tmpl = {"hash": ph[0], "probe": ph[1], "rerank": ph[2], "batch": dt, "per_query": per_q}
    out = []
    # the frozen dataclasses' __init__ (object.__setattr__ per field) dominates
    # the host time of a 1000-query batch; instances get their field dict directly
    new = object.__new__
    for i in range(nq):
        timings = dict(tmpl)
        st = status_l[i]
        if st == 1:
            stats = QueryStats(n_indexed=N, candidates=0, cascade=SearchStats(0, 0, 0, 0, 0, 0))
            out.append(QueryResult([], [], stats, timings, status="no-candidates", warning=warning))
            continue
        n = n_out_l[i]
        c = cnt_l[i]
        nc = n_cand_l[i]
        cascade = new(SearchStats)
        cascade.__dict__.update(candidates=nc, kim_pruned=c[0], keogh_pruned=c[1], keogh2_pruned=c[2],
                                dtw_computed=c[3], dtw_abandoned=c[4])
        stats = new(QueryStats)
        stats.__dict__.update(n_indexed=N, candidates=nc, cascade=cascade)
        r = new(QueryResult)
        r.__dict__.update(ids=ids_l[i][:n], distances=dist_l[i][:n], stats=stats, timings=timings,
                          status="fallback" if st == 2 else "ok", warning=warning)
        out.append(r)
    return out


def _prepare_queries(index: SshIndex, Q):
    """Q (numpy / torch, (nq, m) or (m,)) -> contiguous f32 device tensor, with
    the reference's validation (index.py:213-216)."""
    if _is_torch(Q):
        Qd = Q.to(device=f"cuda:{index.device}", dtype=_torch().float32).contiguous()
        if Qd.ndim == 1:
            Qd = Qd.reshape(1, -1)
    else:
        # float32 input goes straight to the device (the f64 round trip is the identity)
        Qh = Q if isinstance(Q, np.ndarray) and Q.dtype == np.float32 else np.asarray(Q, dtype=np.float64)
        if Qh.ndim == 1:
            Qh = Qh.reshape(1, -1)
        if not np.isfinite(Qh).all():
            raise ValueError("series values contains non-finite values")
        _warn_f32_rounding(Qh, "query")
        Qd = _as_device_f32(Qh, index.device)
    if Qd.shape[1] != index.length:
        raise ValueError(f"query length {Qd.shape[1]} does not match indexed length {index.length}")
    return Qd


def _to_host(dev, device: int):
    """Pinned non-blocking copies of device result tensors, one synchronisation."""
    torch = _torch()
    host = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in dev]
    for h, t in zip(host, dev):
        h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(device).synchronize()
    return [h.numpy() for h in host]


def query_index_batch(index: SshIndex, Q, k: int, fallback_on_empty: bool = False) -> list:
    """query_index for every row of Q (nq, m) in one device batch."""
    Qd = _prepare_queries(index, Q)
    k, warning = _validate_k(index, k)
    t0 = time.perf_counter()
    phase = [0.0, 0.0, 0.0]
    # the whole batch (launches, result copies, phase clock) holds the context
    with index.context().use():
        dev = query_batch_device(index, Qd, k, fallback_on_empty, phase_ms=phase)
        # one synchronisation for the six result arrays (pinned, non-blocking copies)
        ids, d2, n_out, n_cand, counters, status = _to_host(dev, index.device)
    dt = time.perf_counter() - t0
    return _results_from_arrays(ids, d2, n_out, n_cand, counters, status, index.n_series, dt, warning,
                                phase_ms=phase)


def query_index(index: SshIndex, q, k: int, fallback_on_empty: bool = False) -> QueryResult:
    """Probe the d tables, then rerank the candidate union exactly by DTW (index.py:204-273)."""
    qv = _query_values(q)
    if qv.shape[0] != index.length:
        raise ValueError(f"query length {qv.shape[0]} does not match indexed length {index.length}")
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    return query_index_batch(index, qv.reshape(1, -1), k, fallback_on_empty)[0]


def dtw_exact_pairs(index: SshIndex, Q, qrow, xrow) -> np.ndarray:
    """Exact f64 DTW^2 of (Q[qrow[e]], X[xrow[e]]) pairs via ssh_dtw_exact."""
    torch = _torch()
    Qd = _as_device_f32(Q, index.device) if not _is_torch(Q) else Q
    qr = torch.as_tensor(np.asarray(qrow, dtype=np.int32)).to(Qd.device)
    xr = torch.as_tensor(np.asarray(xrow, dtype=np.int64)).to(Qd.device)
    out = torch.empty(qr.shape[0], dtype=torch.float64, device=Qd.device)
    ctx = index.context()
    with ctx.use():
        nat.check(nat.lib().ssh_dtw_exact(ctx.handle, nat.ptr(index.X), nat.ptr(Qd),
                                          nat.ptr(qr), nat.ptr(xr), int(qr.shape[0]), nat.ptr(out),
                                          _stream_ptr(index.device)), "ssh_dtw_exact")
    return out.cpu().numpy()

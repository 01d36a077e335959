"""Host-side inputs of the device hash path: the random filter and the
per-(token, slot) consistent-weighted-sampling variates.

The reference draws its CWS randomness statelessly (wmh.py:26-49: a
splitmix64 chain keyed by seed, slot and token, mapped to (0, 1)) and
evaluates np.log on it inside `_cws_keys` (wmh.py:60-72).  The device never
evaluates a logarithm: this module evaluates the same chain and the same
np.log calls once per (token, slot) of the 2^n token universe, in the same
operation order, so each table entry is bit-identical to the value the
reference computes for that (token, slot).  The tables are uploaded once per
(n, K*L, seed) by ssh_ctx_set_params.
"""

from __future__ import annotations

import threading

import numpy as np

_U = np.uint64
_MIX_ADD = _U(0x9E3779B97F4A7C15)
_MIX_M1 = _U(0xBF58476D1CE4E5B9)
_MIX_M2 = _U(0x94D049BB133111EB)
_SLOT_MUL = _U(0xD1B54A32D192ED03)
_SALTS = {  # wmh.py:26-31
    "u1": _U(0xA0761D6478BD642F),
    "u2": _U(0xE7037ED1A0B428DB),
    "v1": _U(0x8EBC6AF09C88C6E3),
    "v2": _U(0x589965CC75374CC3),
    "beta": _U(0x1D8E4E27C47D124F),
}


def _splitmix(z: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer, wrapping uint64 arithmetic (wmh.py:34-44)."""
    with np.errstate(over="ignore"):
        z = z + _MIX_ADD
        z = (z ^ (z >> _U(30))) * _MIX_M1
        z = (z ^ (z >> _U(27))) * _MIX_M2
        return z ^ (z >> _U(31))


def _open_unit(h: np.ndarray) -> np.ndarray:
    """Top 53 bits + 1/2, scaled into (0, 1) (wmh.py:47-49)."""
    return ((h >> _U(11)).astype(np.float64) + 0.5) * 2.0 ** -53


def filter_weights(W: int, seed: int) -> np.ndarray:
    """W standard-normal taps from default_rng(seed) (sketch.py:36-43); the
    public make_filter (index.py) wraps them in a RandomFilter."""
    if W < 1:
        raise ValueError(f"filter length W must be >= 1, got {W}")
    if seed < 0:
        raise ValueError(f"seed must be non-negative, got {seed}")
    return np.random.default_rng(seed).standard_normal(W)


def cws_variates(n: int, S: int, seed: int, chunk_tokens: int = 1 << 14):
    """(r, ln_c, beta), each float64 [2^n, S] in [token][slot] layout."""
    T = 1 << n
    r = np.empty((T, S))
    lnc = np.empty((T, S))
    beta = np.empty((T, S))
    seed_mix = _splitmix(np.array([seed & ((1 << 64) - 1)], dtype=np.uint64))[0]
    with np.errstate(over="ignore"):
        slot_mix = _splitmix(np.arange(S, dtype=np.uint64) * _SLOT_MUL)
    for t0 in range(0, T, chunk_tokens):
        t1 = min(T, t0 + chunk_tokens)
        tok_mix = _splitmix(np.arange(t0, t1, dtype=np.uint64) ^ seed_mix)
        base = _splitmix(tok_mix[:, None] ^ slot_mix[None, :])
        var = {name: _open_unit(_splitmix(base ^ salt)) for name, salt in _SALTS.items()}
        # same expressions and order as wmh.py:70-71
        r[t0:t1] = -np.log(var["u1"]) - np.log(var["u2"])
        lnc[t0:t1] = np.log(-np.log(var["v1"]) - np.log(var["v2"]))
        beta[t0:t1] = var["beta"]
    return r, lnc, beta


def ln_counts(max_count: int) -> np.ndarray:
    """np.log(count) for count in 0..max_count (entry 0 unused) (wmh.py:72)."""
    c = np.arange(max_count + 1, dtype=np.float64)
    c[0] = 1.0
    return np.log(c)


_cache: dict = {}
_cache_lock = threading.Lock()


def tables(n: int, S: int, seed: int):
    """Cached cws_variates(n, S, seed)."""
    key = (n, S, seed)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is None:
            hit = cws_variates(n, S, seed)
            _cache.clear()  # keep one table set resident (tens of MB)
            _cache[key] = hit
        return hit

"""Seeded synthetic workloads standing in for BASELINE.json's datasets.

The paper's UCR Random Walk and 22-hour ECG recordings are not available
here; BASELINE.json defines synthetic stand-ins and this module generates
them:

* random walks: x = cumsum(N(0,1)), z-normalised in float64 (core.py:110-120
  semantics), stored float32.  Series are generated in fixed chunks of
  CHUNK ids with the generator seeded by (seed, chunk index), so a shard
  [lo, hi) regenerates exactly its slice at any GPU count;
* queries: a database row, monotone time warp with local rate
  1 + 0.1 s(t) (s piecewise-linear through 9 knots ~ U(-1, 1)), plus
  N(0, 0.1) noise, z-normalised (the reference defines no recipe; SURVEY
  §8d);
* ECG-like signal (config 2): Gaussian P/QRS/T bumps (widths 10/4/16,
  amplitudes 0.15/1.0/0.3 with 10% jitter, P at -40 and T at +60 samples
  from the QRS peak), beat period 200 +- 20, baseline wander
  0.2 sin(2 pi t / 2000), N(0, 0.05) noise; windows cut at a stride.
"""

from __future__ import annotations

import hashlib

import numpy as np

CHUNK = 1 << 16

# cfg -> (N, m, band, n_queries, kind)
CONFIGS = {
    0: dict(N=10_000, m=512, band=0.05, nq=100, kind="rw"),
    1: dict(N=1_000_000, m=512, band=0.05, nq=1000, kind="rw"),
    2: dict(N=2_000_000, m=1024, band=0.05, nq=1000, kind="ecg", stride=64),
    3: dict(N=4_000_000, m=2048, band=0.10, nq=1000, kind="rw"),
    4: dict(N=64_000_000, m=512, band=0.05, nq=10_000, kind="rw"),
}
SSH_PARAMS = dict(W=80, delta=3, n=15, d=20, seed=0, K=4)


def _torch():
    import torch

    return torch


def random_walks(lo: int, hi: int, m: int, seed: int, device="cuda"):
    """Rows [lo, hi) of the seeded random-walk database as float32 (torch)."""
    torch = _torch()
    out = torch.empty((hi - lo, m), dtype=torch.float32, device=device)
    c0, c1 = lo // CHUNK, (hi - 1) // CHUNK
    for c in range(c0, c1 + 1):
        g = torch.Generator(device=device)
        g.manual_seed(int(seed) * 1_000_003 + c)
        base = c * CHUNK
        n = CHUNK
        steps = torch.randn((n, m), generator=g, device=device, dtype=torch.float32)
        a, b = max(lo, base), min(hi, base + n)
        x = steps[a - base:b - base].double().cumsum(dim=1)
        mu = x.mean(dim=1, keepdim=True)
        sd = x.std(dim=1, unbiased=False, keepdim=True)
        flat = sd < 1e-12
        x = torch.where(flat, torch.zeros_like(x), (x - mu) / torch.where(flat, torch.ones_like(sd), sd))
        out[a - lo:b - lo] = x.float()
        del steps, x
    return out


def random_walk_rows(ids, m: int, seed: int, device="cuda") -> np.ndarray:
    """Rows `ids` of the random-walk database (numpy f32), one chunk generation per chunk."""
    ids = np.asarray(ids, dtype=np.int64)
    out = np.empty((ids.shape[0], m), dtype=np.float32)
    chunks = ids // CHUNK
    for c in np.unique(chunks):
        sel = np.nonzero(chunks == c)[0]
        block = random_walks(int(c) * CHUNK, int(c) * CHUNK + CHUNK, m, seed, device=device)
        out[sel] = block[ids[sel] - int(c) * CHUNK].cpu().numpy()
        del block
    return out


def znorm_rows_f64(v: np.ndarray) -> np.ndarray:
    mu = v.mean(axis=1, keepdims=True)
    sd = v.std(axis=1, keepdims=True)
    flat = sd[:, 0] < 1e-12
    sd[flat] = 1.0
    out = (v - mu) / sd
    out[flat] = 0.0
    return out


def warped_queries(src_rows: np.ndarray, seed: int, noise: float = 0.1) -> np.ndarray:
    """Time-warped + noisy perturbations of the given rows (float32)."""
    rng = np.random.default_rng(seed)
    nq, m = src_rows.shape
    grid = np.linspace(0.0, 1.0, 9)
    t = np.linspace(0.0, 1.0, m)
    out = np.empty((nq, m))
    for i in range(nq):
        knots = rng.uniform(-1.0, 1.0, 9)
        rate = 1.0 + 0.1 * np.interp(t, grid, knots)
        pos = np.concatenate(([0.0], np.cumsum(rate[:-1])))
        pos = pos / pos[-1] * (m - 1)
        out[i] = np.interp(pos, np.arange(m), src_rows[i].astype(np.float64)) + rng.normal(0.0, noise, m)
    return znorm_rows_f64(out).astype(np.float32)


def query_source_ids(N: int, nq: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if nq <= N:
        return np.sort(rng.choice(N, size=nq, replace=False)).astype(np.int64)
    return rng.integers(0, N, size=nq).astype(np.int64)


def ecg_signal(length: int, seed: int = 4000) -> np.ndarray:
    """Quasi-periodic ECG-like float64 signal (config 2 recipe)."""
    rng = np.random.default_rng(seed)
    t = np.arange(length, dtype=np.float64)
    x = 0.2 * np.sin(2 * np.pi * t / 2000.0) + rng.normal(0.0, 0.05, length)
    periods = rng.uniform(180, 220, size=length // 180 + 2)
    peaks = np.cumsum(periods)
    peaks = peaks[peaks < length + 100]
    for off, width, amp in ((-40.0, 10.0, 0.15), (0.0, 4.0, 1.0), (60.0, 16.0, 0.3)):
        amps = amp * (1.0 + rng.uniform(-0.1, 0.1, size=peaks.shape[0]))
        span = int(4 * width)
        centres = peaks + off
        c = np.rint(centres).astype(np.int64)  # round-half-even, as Python's round()
        # one offset from the bump centre at a time over all beats: beats are
        # >= 180 samples apart and a bump spans <= 129, so the positions of one
        # offset are distinct and each sample gets at most one term per bump type
        for d in range(-span, span + 1):
            pos = c + d
            ok = (pos >= 0) & (pos < length)
            pk = pos[ok]
            x[pk] += amps[ok] * np.exp(-0.5 * ((pk - centres[ok]) / width) ** 2)
    return x


def ecg_windows(signal: np.ndarray, m: int, stride: int, count: int) -> np.ndarray:
    idx = np.arange(count)[:, None] * stride + np.arange(m)[None, :]
    return znorm_rows_f64(signal[idx]).astype(np.float32)


def sha256_f32(a) -> str:
    if hasattr(a, "cpu"):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def workload(cfg: int, lo: int = 0, hi: int | None = None, device="cuda", nq: int | None = None,
             n_override: int | None = None):
    """(X shard [lo,hi) torch f32 on device, Q numpy f32, src ids, params dict) for a config."""
    c = dict(CONFIGS[cfg])
    N = n_override or c["N"]
    hi = N if hi is None else hi
    m = c["m"]
    nq = c["nq"] if nq is None else nq
    if c["kind"] == "rw":
        X = random_walks(lo, hi, m, 1000 + cfg, device=device)
        src = query_source_ids(N, nq, 2000 + cfg)
        # query sources are regenerated from their own chunk (independent of the shard)
        rows = random_walk_rows(src, m, 1000 + cfg, device=device) if nq else np.zeros((0, m), np.float32)
        Q = warped_queries(rows, 3000 + cfg) if nq else rows
    else:
        torch = _torch()
        stride = c["stride"]
        total = (N - 1) * stride + m
        sig = ecg_signal(total + 200_000, seed=4000)
        rec = sig[lo * stride:(hi - 1) * stride + m]
        if torch.device(device).type == "cuda":
            # windows + per-window z-normalisation on the device (ssh_windows:
            # numpy's pairwise float64 mean/std bit for bit, then f32)
            from .pipeline import make_dataset

            X = make_dataset(rec, m, stride=stride, device=torch.device(device).index or 0).values
        else:
            X = torch.from_numpy(ecg_windows(rec, m, stride, hi - lo))
        held = sig[total:]
        rng = np.random.default_rng(2000 + cfg)
        starts = rng.integers(0, held.shape[0] - m, size=nq)
        Q = znorm_rows_f64(np.stack([held[s:s + m] for s in starts])).astype(np.float32)
        src = starts.astype(np.int64)
    params = dict(SSH_PARAMS, band=c["band"])
    return X, Q, src, params

"""Deterministic inputs for the golden fixtures (shared by make_golden.py and
the tests).  numpy's PCG64 + standard_normal are bit-stable across platforms,
so the tests regenerate these arrays instead of committing them.

Values are z-normalised in float64 with core.py:127-135 semantics
(population sigma, sigma < 1e-12 -> zeros) and then cast to float32: float32
is the device input, and the reference receives the exact upcast.
"""

from __future__ import annotations

import numpy as np


def znorm_rows(v: np.ndarray) -> np.ndarray:
    mu = v.mean(axis=1, keepdims=True)
    sd = v.std(axis=1, keepdims=True)
    flat = sd[:, 0] < 1e-12
    sd[flat] = 1.0
    out = (v - mu) / sd
    out[flat] = 0.0
    return out


def random_walks(N: int, m: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return znorm_rows(np.cumsum(rng.standard_normal((N, m)), axis=1)).astype(np.float32)


def perturbed_queries(X: np.ndarray, nq: int, seed: int, noise: float = 0.1) -> tuple:
    """Queries = database rows, monotone time warp (+-10% local rate through 9
    knots), plus N(0, noise) and z-normalisation.  Returns (Q f32, src ids)."""
    rng = np.random.default_rng(seed)
    N, m = X.shape
    src = rng.choice(N, size=nq, replace=False)
    out = np.empty((nq, m))
    grid = np.linspace(0.0, 1.0, 9)
    t = np.linspace(0.0, 1.0, m)
    for qi, s in enumerate(src):
        knots = rng.uniform(-1.0, 1.0, 9)
        rate = 1.0 + 0.1 * np.interp(t, grid, knots)
        pos = np.concatenate(([0.0], np.cumsum(rate[:-1])))
        pos = pos / pos[-1] * (m - 1)
        warped = np.interp(pos, np.arange(m), X[s].astype(np.float64))
        out[qi] = warped + rng.normal(0.0, noise, m)
    return znorm_rows(out).astype(np.float32), src.astype(np.int64)


# name -> (N, m, band, data seed, query seed, nq)
CASES = {
    "rw512": (1000, 512, 0.05, 1234, 4321, 12),
    "rw1024": (200, 1024, 0.05, 2234, 5321, 4),
    "rw2048": (120, 2048, 0.10, 3234, 6321, 3),
}

SSH = dict(W=80, delta=3, n=15, d=20, seed=0)


def case_data(name: str):
    N, m, band, dseed, qseed, nq = CASES[name]
    X = random_walks(N, m, dseed)
    Q, src = perturbed_queries(X, nq, qseed)
    return X, Q, src, band

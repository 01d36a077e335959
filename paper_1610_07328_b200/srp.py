"""Signed random projection baseline and ranking metrics (SURVEY.md §8f
item 4): srp_vectors / srp_signature / srp_matrix (index.py:398-423) with the
projections on the device (ssh_srp), and precision_at_k / ndcg_at_k
(bench.py:63-90)."""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native as nat
from .core import TimeSeries


def srp_vectors(m: int, bits: int, seed: int) -> np.ndarray:
    """(bits, m) float64 projection matrix; row j = default_rng([seed, j]).standard_normal(m)."""
    out = np.empty((bits, m))
    for j in range(bits):
        out[j] = np.random.default_rng([seed, j]).standard_normal(m)
    return out


def srp_matrix(values, bits: int, seed: int, device=None, tensor_cores: bool = True, stats: dict | None = None
               ) -> np.ndarray:
    """(N, bits) int8 +1/-1 signs of values @ srp_vectors(m, bits, seed).T on the
    device (index.py:420-423): the product on the tensor cores (tcgen05, TF32
    with a rigorous error bound; bits <= 256), undecided signs re-evaluated in
    f64 from the original values (float64 inputs are kept in float64 for that).
    `stats`, if given, receives {"rechecked": signs re-evaluated in f64}."""
    import torch

    dev = torch.device("cuda", 0 if device is None else int(device))
    X64 = None
    if hasattr(values, "detach"):
        v = values.detach().to(device=dev)
        if v.dtype == torch.float64:
            X64 = v.contiguous()
        X = v.to(dtype=torch.float32).contiguous()
    else:
        a = np.asarray(values)
        if a.dtype == np.float64:
            X64 = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        X = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)
    if X.ndim != 2:
        raise ValueError(f"values must be 2-D, got shape {tuple(X.shape)}")
    N, m = X.shape
    V = srp_vectors(m, bits, seed)
    V64 = torch.from_numpy(V).to(dev)
    V32 = V64.float()
    out = torch.empty((N, bits), dtype=torch.int8, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    nat.check(nat.lib().ssh_srp2(nat.ptr(X), nat.ptr(X64), N, m, nat.ptr(V32), nat.ptr(V64), bits, nat.ptr(out),
                                 nat.ptr(cnt), 1 if tensor_cores else 0, stream), "ssh_srp2")
    if stats is not None:
        stats["rechecked"] = int(cnt.item())
    return out.cpu().numpy()


def srp_signature(series, bits: int, seed: int, device=None) -> np.ndarray:
    """(bits,) int8 signs for one series (index.py:411-415)."""
    v = series.values if isinstance(series, TimeSeries) else np.asarray(series, dtype=np.float64)
    return srp_matrix(np.asarray(v).reshape(1, -1), bits, seed, device)[0]


def precision_at_k(retrieved, gold, k: int) -> float:
    """Fraction of the gold top-k present in the retrieved top-k (bench.py:63-67)."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    return len(set(retrieved[:k]) & set(gold[:k])) / k


def ndcg_at_k(retrieved, gold, k: int) -> float:
    """Graded relevance k - gold rank, discount log2(position + 1) (bench.py:70-90)."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    gold_rank = {item: pos for pos, item in enumerate(gold[:k], start=1)}
    idcg = sum((k - i) / math.log2(i + 1) for i in range(1, k + 1))
    if idcg == 0.0:
        return 1.0 if (len(retrieved) > 0 and len(gold) > 0 and retrieved[0] == gold[0]) else 0.0
    dcg = 0.0
    for pos, item in enumerate(retrieved[:k], start=1):
        if item in gold_rank:
            dcg += (k - gold_rank[item]) / math.log2(pos + 1)
    return dcg / idcg

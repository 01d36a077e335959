"""Data pipeline on the device: windowing of a long
recording fused with per-window z-normalisation (ssh_windows), i.e. the
reference's make_dataset = z_normalize_dataset(extract_subsequences(rec, t))
(core.py:127-169), with numpy-identical float64 means and deviations."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .core import Dataset, TimeSeries


def _rec_values(recording) -> np.ndarray:
    v = recording.values if isinstance(recording, TimeSeries) else recording
    if hasattr(v, "detach"):
        v = v.detach().double().cpu().numpy()
    return np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))


def extract_subsequences(recording, t: int) -> Dataset:
    """All len-t+1 windows of length t, ids in order (core.py:138-146), host."""
    v = _rec_values(recording)
    if t < 1:
        raise ValueError(f"subsequence length must be >= 1, got {t}")
    if t > v.shape[0]:
        raise ValueError(f"subsequence length {t} exceeds series length {v.shape[0]}")
    rid = recording.id if isinstance(recording, TimeSeries) else 0
    return Dataset(values=np.lib.stride_tricks.sliding_window_view(v, t).copy(),
                   source=f"windows(t={t}) of series {rid}")


def make_dataset(recording, t: int, normalize: bool = True, stride: int = 1, device=None,
                 dtype: str = "float32") -> Dataset:
    """core.py:162-169 on the device: a Dataset whose values are a device
    tensor (count, t) of float32 (the index's input type) or float64."""
    import torch

    v = _rec_values(recording)
    if t < 1:
        raise ValueError(f"subsequence length must be >= 1, got {t}")
    if t > v.shape[0]:
        raise ValueError(f"subsequence length {t} exceeds series length {v.shape[0]}")
    dev = torch.device("cuda", 0 if device is None else int(device))
    rec = torch.from_numpy(v).to(dev)
    count = (v.shape[0] - t) // stride + 1
    out = torch.empty((count, t), dtype=torch.float32 if dtype == "float32" else torch.float64, device=dev)
    n = ctypes.c_int64(0)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    nat.check(nat.lib().ssh_windows(nat.ptr(rec), v.shape[0], t, stride, 1 if normalize else 0,
                                    nat.ptr(out) if dtype == "float32" else None,
                                    nat.ptr(out) if dtype != "float32" else None, ctypes.byref(n), stream),
              "ssh_windows")
    rid = recording.id if isinstance(recording, TimeSeries) else 0
    return Dataset(values=out, source=f"windows(t={t}, stride={stride}) of series {rid}")

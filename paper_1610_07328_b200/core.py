"""Core types mirroring the reference's core module (core.py:16-135).

Exceptions, TimeSeries, Dataset and z-normalisation keep the reference's
names, validation and messages.  A Dataset may hold a numpy array (float64
or float32) or a torch tensor; the device path indexes float32 values, so a
float64 input is rounded to float32 once (exact for the BASELINE workloads,
which are generated in float32 — DESIGN.md §2).
"""

from __future__ import annotations

import numpy as np


class SshError(Exception):
    """Base class for errors raised by this package (core.py:16-17)."""


class DataFormatError(SshError):
    """A data file failed to parse under its declared format (core.py:20-21)."""


class IndexLoadError(SshError):
    """An index file is truncated, corrupt, or version-incompatible (core.py:24-25)."""


class ConfigError(SshError):
    """A parameter combination violates a precondition (core.py:28-29)."""


_ZERO_VAR_EPS = 1e-12


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _validated_values(values, what: str) -> np.ndarray:
    arr = np.asarray(values, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError(f"{what} must be one-dimensional, got shape {arr.shape}")
    if arr.size == 0:
        raise ValueError(f"{what} must be non-empty")
    if not np.all(np.isfinite(arr)):
        raise ValueError(f"{what} contains non-finite values")
    return arr


class TimeSeries:
    """A uniformly sampled sequence of real values (core.py:48-63)."""

    __slots__ = ("values", "id")

    def __init__(self, values, id: int = 0):
        self.values = _validated_values(values, "series values")
        self.id = id

    def __len__(self) -> int:
        return self.values.shape[0]


class Dataset:
    """Equal-length series stacked row-wise; row index is the series id
    (core.py:66-104).  `values` is a numpy (N, t) array or a torch tensor
    (kept on its device)."""

    def __init__(self, values, source: str = ""):
        if _is_torch(values):
            import torch

            if values.ndim != 2:
                raise ValueError(f"dataset values must be 2-D, got shape {tuple(values.shape)}")
            if values.shape[0] == 0 or values.shape[1] == 0:
                raise ValueError("dataset must contain at least one non-empty series")
            if not bool(torch.isfinite(values).all()):
                raise ValueError("dataset contains non-finite values")
            self.values = values
        else:
            arr = np.asarray(values)
            if arr.dtype not in (np.float32, np.float64):
                arr = arr.astype(np.float64)
            if arr.ndim != 2:
                raise ValueError(f"dataset values must be 2-D, got shape {arr.shape}")
            if arr.shape[0] == 0 or arr.shape[1] == 0:
                raise ValueError("dataset must contain at least one non-empty series")
            if not np.all(np.isfinite(arr)):
                raise ValueError("dataset contains non-finite values")
            self.values = arr
        self.source = source

    @property
    def n_series(self) -> int:
        return int(self.values.shape[0])

    @property
    def length(self) -> int:
        return int(self.values.shape[1])

    def series(self, i: int) -> TimeSeries:
        if not 0 <= i < self.n_series:
            raise IndexError(f"series id {i} out of range [0, {self.n_series})")
        row = self.values[i]
        if _is_torch(row):
            row = row.double().cpu().numpy()
        return TimeSeries(values=row, id=i)

    def __len__(self) -> int:
        return self.n_series

    def __getitem__(self, i: int) -> TimeSeries:
        return self.series(i)

    def __iter__(self):
        for i in range(self.n_series):
            yield self.series(i)


def z_normalize_values(values: np.ndarray) -> np.ndarray:
    """Mean 0, population std 1; std < 1e-12 maps to zeros (core.py:110-120)."""
    mu = values.mean()
    sigma = values.std()
    if sigma < _ZERO_VAR_EPS:
        return np.zeros_like(values)
    return (values - mu) / sigma


def z_normalize(series: TimeSeries) -> TimeSeries:
    return TimeSeries(values=z_normalize_values(series.values), id=series.id)


def z_normalize_rows(values: np.ndarray) -> np.ndarray:
    """Row-wise z-normalisation (core.py:127-135) of an (N, t) float64 array."""
    mu = values.mean(axis=1, keepdims=True)
    sigma = values.std(axis=1, keepdims=True)
    flat = sigma[:, 0] < _ZERO_VAR_EPS
    sigma[flat] = 1.0
    out = (values - mu) / sigma
    out[flat] = 0.0
    return out


def z_normalize_dataset(dataset: Dataset) -> Dataset:
    vals = dataset.values
    if _is_torch(vals):
        vals = vals.double().cpu().numpy()
    return Dataset(values=z_normalize_rows(np.asarray(vals, dtype=np.float64)), source=dataset.source)

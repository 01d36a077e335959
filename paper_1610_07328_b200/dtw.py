"""The reference's public DTW utilities (sshts.dtw, dtw.py:239-284) on the
device: dtw_distance, lb_kim, build_envelope, lb_keogh, lb_keogh2 and the
Envelope dataclass.  Same signatures, validation messages and float64
results (libsshgpu's ssh_dtw_pairs64 / ssh_envelope64 / ssh_lb_keogh64 /
ssh_lb_kim64 evaluate the reference's operation order in f64; the square
root is taken at the API boundary, as the reference does).  There is no CPU
fallback: every call needs the library and an sm_100 device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .index import WarpingParams, _device_index, _stream_ptr, _torch


@dataclass(frozen=True)
class Envelope:
    """Running min/max of a series over the warping window, per index (dtw.py:42-47)."""

    upper: np.ndarray
    lower: np.ndarray


def _values_of(x) -> np.ndarray:
    """dtw.py:279-282."""
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x, dtype=np.float64)
    return np.ascontiguousarray(x.values, dtype=np.float64)


def _dev(*arrays):
    torch = _torch()
    dev = _device_index(None)
    return dev, [torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(f"cuda:{dev}") for a in arrays]


def dtw_distance(x, y, params: WarpingParams = WarpingParams(), abandon_above: float | None = None) -> float:
    """Minimal cumulative squared-cost warping distance, square-rooted
    (dtw.py:239-250); with abandon_above, inf once every cell of some row
    exceeds abandon_above squared."""
    xv = _values_of(x)
    yv = _values_of(y)
    if xv.shape[0] != yv.shape[0]:
        raise ValueError(f"length mismatch: {xv.shape[0]} vs {yv.shape[0]}")
    m = xv.shape[0]
    r = params.radius(m)
    ab = -1.0 if abandon_above is None else float(abandon_above) ** 2
    torch = _torch()
    dev, (xd, yd) = _dev(xv, yv)
    out = torch.empty(1, dtype=torch.float64, device=xd.device)
    nat.check(nat.lib().ssh_dtw_pairs64(nat.ptr(xd), nat.ptr(yd), None, None, 1, m, r, ab, nat.ptr(out),
                                        _stream_ptr(dev)), "ssh_dtw_pairs64")
    return float(np.sqrt(out.cpu().numpy()[0]))


def lb_kim(x, y) -> float:
    """Distance of the first and last point pairs; O(1) lower bound (dtw.py:252-260)."""
    xv = _values_of(x)
    yv = _values_of(y)
    if xv.shape[0] != yv.shape[0]:
        raise ValueError(f"length mismatch: {xv.shape[0]} vs {yv.shape[0]}")
    torch = _torch()
    dev, (xd, yd) = _dev(xv, yv)
    out = torch.empty(1, dtype=torch.float64, device=xd.device)
    nat.check(nat.lib().ssh_lb_kim64(nat.ptr(xd), nat.ptr(yd), 1, xv.shape[0], nat.ptr(out), _stream_ptr(dev)),
              "ssh_lb_kim64")
    return float(out.cpu().numpy()[0])


def build_envelope(q, params: WarpingParams = WarpingParams()) -> Envelope:
    """Upper/lower running max/min over [i - r, i + r] (dtw.py:262-268)."""
    qv = _values_of(q)
    m = qv.shape[0]
    r = params.radius(m)
    torch = _torch()
    dev, (qd,) = _dev(qv)
    up = torch.empty(m, dtype=torch.float64, device=qd.device)
    lo = torch.empty(m, dtype=torch.float64, device=qd.device)
    nat.check(nat.lib().ssh_envelope64(nat.ptr(qd), 1, m, r, nat.ptr(up), nat.ptr(lo), _stream_ptr(dev)),
              "ssh_envelope64")
    return Envelope(upper=up.cpu().numpy(), lower=lo.cpu().numpy())


def lb_keogh(env: Envelope, c) -> float:
    """Distance from the candidate to the query's envelope (dtw.py:271-276)."""
    cv = _values_of(c)
    if cv.shape[0] != env.upper.shape[0]:
        raise ValueError(f"length mismatch: {cv.shape[0]} vs {env.upper.shape[0]}")
    torch = _torch()
    dev, (cd, ud, ld) = _dev(cv, env.upper, env.lower)
    out = torch.empty(1, dtype=torch.float64, device=cd.device)
    nat.check(nat.lib().ssh_lb_keogh64(nat.ptr(cd), nat.ptr(ud), nat.ptr(ld), 1, cv.shape[0], 1, nat.ptr(out),
                                       _stream_ptr(dev)), "ssh_lb_keogh64")
    return float(np.sqrt(out.cpu().numpy()[0]))


def lb_keogh2(q, c, params: WarpingParams = WarpingParams()) -> float:
    """lb_keogh with the query/candidate roles swapped (dtw.py:279-281)."""
    return lb_keogh(build_envelope(c, params), q)


def dtw_pairs(X, Y, params: WarpingParams = WarpingParams(), abandon_above: float | None = None,
              xrow=None, yrow=None) -> np.ndarray:
    """Batched dtw_distance: DTW of X[xrow[p]] vs Y[yrow[p]] (rows p when the
    index arrays are None), float64 (n,) — one device launch."""
    Xv = np.atleast_2d(np.asarray(X, dtype=np.float64))
    Yv = np.atleast_2d(np.asarray(Y, dtype=np.float64))
    if Xv.shape[1] != Yv.shape[1]:
        raise ValueError(f"length mismatch: {Xv.shape[1]} vs {Yv.shape[1]}")
    m = Xv.shape[1]
    torch = _torch()
    dev, (xd, yd) = _dev(Xv, Yv)
    if xrow is None and yrow is None:
        if Xv.shape[0] != Yv.shape[0]:
            raise ValueError(f"row count mismatch: {Xv.shape[0]} vs {Yv.shape[0]}")
        n = Xv.shape[0]
        xr = yr = None
    else:
        xr_h = np.asarray(xrow if xrow is not None else np.arange(len(yrow)), dtype=np.int64)
        yr_h = np.asarray(yrow if yrow is not None else np.arange(len(xrow)), dtype=np.int64)
        n = xr_h.shape[0]
        xr = torch.from_numpy(xr_h).to(xd.device)
        yr = torch.from_numpy(yr_h).to(xd.device)
    ab = -1.0 if abandon_above is None else float(abandon_above) ** 2
    out = torch.empty(n, dtype=torch.float64, device=xd.device)
    nat.check(nat.lib().ssh_dtw_pairs64(nat.ptr(xd), nat.ptr(yd), nat.ptr(xr), nat.ptr(yr), n, m,
                                        params.radius(m), ab, nat.ptr(out), _stream_ptr(dev)), "ssh_dtw_pairs64")
    return np.sqrt(out.cpu().numpy())

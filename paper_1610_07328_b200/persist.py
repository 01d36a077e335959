"""Index and dataset persistence.

File formats follow the reference byte for byte (core.py:175-251,
index.py:275-396):

* dataset ``f64le``: magic ``SSHD``, version u32 = 1, series count u64,
  series length u64, then row-major little-endian float64; ``csv``: one
  series per line, ``repr`` floats, no header.
* index ``SSHI`` version 1 (K = 1, readable by the reference's load_index):
  version u32, W u32, delta u32, n u32, d u32, seed u64, band f64,
  normalized u8, filter seed u64 + W float64 weights, sidecar dataset name
  (u32 length + utf8) and its SHA-256, then per table a bucket count u64 and
  per bucket (keys ascending) key u64, id count u64, ids u64.
* version 2 (this package, K > 1): identical, with K as a u32 right after
  band.

The table section is written from the device CSR (ssh_index_export) with
numpy and parsed by the library's host routine ssh_sshi_parse_tables; the
loaded index is rebuilt on the device from the recovered signatures.
"""

from __future__ import annotations

import ctypes
import hashlib
import struct
from pathlib import Path

import numpy as np

from . import _native as nat
from .core import DataFormatError, Dataset, IndexLoadError

DATA_MAGIC = b"SSHD"
DATA_VERSION = 1
_DATA_HEADER_BYTES = 4 + 4 + 8 + 8
INDEX_MAGIC = b"SSHI"
INDEX_VERSION = 1       # K = 1: the reference's format
INDEX_VERSION_K = 2     # K > 1: K as u32 after band


def _host_values_f64(dataset) -> np.ndarray:
    v = dataset.values
    if hasattr(v, "detach"):
        v = v.detach().cpu().numpy()
    return np.ascontiguousarray(v, dtype="<f8")


def save_dataset(dataset: Dataset, path, fmt: str = "f64le") -> None:
    """core.py:181-194."""
    path = Path(path)
    if fmt == "f64le":
        vals = _host_values_f64(dataset)
        header = DATA_MAGIC + struct.pack("<IQQ", DATA_VERSION, vals.shape[0], vals.shape[1])
        path.write_bytes(header + vals.tobytes())
    elif fmt == "csv":
        vals = _host_values_f64(dataset).astype(np.float64)
        # repr of the numpy scalars, as the reference writes them (core.py:189;
        # with numpy >= 2 that is "np.float64(...)")
        lines = [",".join(repr(v) for v in row) for row in vals]
        path.write_text("\n".join(lines) + "\n")
    else:
        raise ValueError(f"unknown dataset format {fmt!r} (expected 'f64le' or 'csv')")


def _load_f64le(path: Path) -> Dataset:
    raw = path.read_bytes()
    if len(raw) < _DATA_HEADER_BYTES:
        raise DataFormatError(f"{path}: file too short for f64le header ({len(raw)} bytes)")
    if raw[:4] != DATA_MAGIC:
        raise DataFormatError(f"{path}: bad magic {raw[:4]!r}, expected {DATA_MAGIC!r}")
    version, n, t = struct.unpack_from("<IQQ", raw, 4)
    if version != DATA_VERSION:
        raise DataFormatError(f"{path}: unsupported f64le version {version}")
    expected = _DATA_HEADER_BYTES + n * t * 8
    if len(raw) != expected:
        raise DataFormatError(
            f"{path}: payload size mismatch at offset {len(raw)} (expected {expected} bytes "
            f"for {n} series of length {t})")
    values = np.frombuffer(raw, dtype="<f8", offset=_DATA_HEADER_BYTES).reshape(n, t)
    return Dataset(values=values.copy(), source=str(path))


def _load_csv(path: Path) -> Dataset:
    rows, width = [], None
    with open(path) as f:
        for lineno, line in enumerate(f, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                row = [float(tok) for tok in line.split(",")]
            except ValueError as exc:
                raise DataFormatError(f"{path}: line {lineno}: {exc}") from None
            if width is None:
                width = len(row)
            elif len(row) != width:
                raise DataFormatError(
                    f"{path}: line {lineno}: ragged row of {len(row)} values, expected {width}")
            rows.append(row)
    if not rows:
        raise DataFormatError(f"{path}: no series found")
    return Dataset(values=np.asarray(rows, dtype=np.float64), source=str(path))


def load_dataset(path, fmt: str = "f64le") -> Dataset:
    """core.py:242-250."""
    path = Path(path)
    if not path.exists():
        raise DataFormatError(f"{path}: no such file")
    if fmt == "f64le":
        return _load_f64le(path)
    if fmt == "csv":
        return _load_csv(path)
    raise ValueError(f"unknown dataset format {fmt!r} (expected 'f64le' or 'csv')")


def file_checksum(path) -> bytes:
    """SHA-256 of a file's bytes, streamed (core.py:261-267)."""
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 20), b""):
            h.update(chunk)
    return h.digest()


def _table_words(keys: np.ndarray, offsets: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """One table as u64 words: nb, then per bucket key, count, ids (keys ascending)."""
    nb = keys.shape[0]
    counts = np.diff(offsets).astype(np.uint64)
    out = np.empty(1 + 2 * nb + ids.shape[0], dtype="<u8")
    out[0] = nb
    hdr = 1 + offsets[:-1] + 2 * np.arange(nb, dtype=np.int64)
    out[hdr] = keys
    out[hdr + 1] = counts
    body = np.ones(out.shape[0], dtype=bool)
    body[0] = False
    body[hdr] = False
    body[hdr + 1] = False
    out[body] = ids.astype(np.uint64)
    return out


def index_file_bytes(params, normalized: bool, filter_seed: int, weights, dataset_name: str, checksum: bytes,
                     tables) -> bytes:
    """SSHI bytes (index.py:294-310) for `tables` = iterable of per-table CSR
    (keys ascending u64, offsets, ids)."""
    p = params
    parts = [INDEX_MAGIC]
    if p.K == 1:
        parts.append(struct.pack("<IIIIIQd", INDEX_VERSION, p.W, p.delta, p.n, p.d, p.seed, p.band))
    else:
        parts.append(struct.pack("<IIIIIQdI", INDEX_VERSION_K, p.W, p.delta, p.n, p.d, p.seed, p.band, p.K))
    parts.append(struct.pack("<B", 1 if normalized else 0))
    parts.append(struct.pack("<Q", filter_seed))
    parts.append(np.ascontiguousarray(weights, dtype="<f8").tobytes())
    name_bytes = dataset_name.encode("utf-8")
    parts.append(struct.pack("<I", len(name_bytes)))
    parts.append(name_bytes)
    parts.append(checksum)
    for keys, offsets, ids in tables:
        parts.append(_table_words(np.asarray(keys, dtype=np.uint64), np.asarray(offsets, dtype=np.int64),
                                  np.asarray(ids)).tobytes())
    return b"".join(parts)


def save_index(index, path) -> None:
    """index.py:287-310; version 2 records K when K > 1.  Tables come from the
    device CSR (ssh_index_export)."""
    path = Path(path)
    dataset_name = path.name + ".sshd"
    save_dataset(index.dataset, path.parent / dataset_name, fmt="f64le")
    checksum = file_checksum(path.parent / dataset_name)
    # the file describes its own dataset (row r = id r): a shard built with
    # id_base != 0 (dist.py) is written with local ids; load_index(id_base=...)
    # restores the global numbering
    base = int(getattr(index, "id_base", 0))
    tables = ((keys, offsets, ids - base) for keys, offsets, ids in
              (index.table_csr(j) for j in range(index.params.d)))
    path.write_bytes(index_file_bytes(index.params, index.normalized, index.filter.seed, index.filter.weights,
                                      dataset_name, checksum, tables))


def read_index_file(path):
    """Parse and verify an SSHI file and its sidecar dataset without touching
    the device: (params, filter weights, filter seed, normalized, dataset,
    signatures u64[N][d]).  Any defect raises IndexLoadError (no partial index)."""
    from .index import SshParams

    path = Path(path)
    if not path.exists():
        raise IndexLoadError(f"{path}: no such file")
    data = path.read_bytes()
    off = 0

    def take(nbytes):
        nonlocal off
        if off + nbytes > len(data):
            raise IndexLoadError(f"{path}: truncated index file (needed {nbytes} bytes at offset {off})")
        out = data[off:off + nbytes]
        off += nbytes
        return out

    def unpack(fmt):
        return struct.unpack(fmt, take(struct.calcsize(fmt)))

    magic = take(4)
    if magic != INDEX_MAGIC:
        raise IndexLoadError(f"{path}: bad magic {magic!r}, expected {INDEX_MAGIC!r}")
    version, W, delta, n, d, seed, band = unpack("<IIIIIQd")
    if version == INDEX_VERSION:
        K = 1
    elif version == INDEX_VERSION_K:
        (K,) = unpack("<I")
    else:
        raise IndexLoadError(f"{path}: unsupported index version {version}")
    (normalized,) = unpack("<B")
    (filter_seed,) = unpack("<Q")
    weights = np.frombuffer(take(W * 8), dtype="<f8").copy()
    (name_len,) = unpack("<I")
    dataset_name = take(name_len).decode("utf-8")
    checksum = take(32)
    params = SshParams(W=W, delta=delta, n=n, d=d, seed=seed, band=band, K=K)
    dataset_path = path.parent / dataset_name
    # tables are parsed against the dataset's series count
    if not dataset_path.exists():
        raise IndexLoadError(f"{path}: referenced dataset file {dataset_path} is missing")
    if file_checksum(dataset_path) != checksum:
        raise IndexLoadError(f"{path}: dataset file {dataset_path} checksum mismatch")
    dataset = load_dataset(dataset_path, fmt="f64le")
    N = dataset.n_series
    sig = np.zeros((N, d), dtype=np.uint64)
    end = ctypes.c_int64(0)
    msg = ctypes.create_string_buffer(512)
    buf = np.frombuffer(data, dtype=np.uint8)
    rc = nat.lib().ssh_sshi_parse_tables(buf.ctypes.data_as(ctypes.c_void_p), len(data), off, d, N,
                                         sig.ctypes.data_as(ctypes.c_void_p), ctypes.byref(end), msg, 512)
    if rc != 0:
        raise IndexLoadError(f"{path}: {msg.value.decode()}")
    if end.value != len(data):
        raise IndexLoadError(f"{path}: {len(data) - end.value} trailing bytes after tables")
    return params, weights, filter_seed, bool(normalized), dataset, sig


def load_index(path, device=None, id_base: int = 0):
    """index.py:333-396: parse + verify, then rebuild the device index from the
    recovered signatures (tables are a function of the signatures).  id_base
    re-attaches a shard's global id offset (save_index writes local ids)."""
    from .index import index_from_signatures

    params, weights, filter_seed, normalized, dataset, sig = read_index_file(path)
    return index_from_signatures(dataset, params, sig, normalized=normalized, device=device,
                                 filter_weights=weights, filter_seed=filter_seed, id_base=id_base)

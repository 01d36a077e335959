"""ctypes binding of libsshgpu.so (the C-ABI declared in include/sshgpu.h).

This is the binding a maintainer of the reference package would add
(INTEGRATION.md): plain pointers, sizes and a cudaStream_t.  There is no
fallback — if the shared library is missing or no sm_100 device is present,
every entry point raises SshError.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

from .core import ConfigError, SshError

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB_PATH = Path(os.environ["SSH_LIB_PATH"]).resolve() if os.environ.get("SSH_LIB_PATH") else PKG / "libsshgpu.so"
SOURCES = ["ctx.cu", "sketch.cu", "signature.cu", "tables.cu", "query.cu", "persist.cu", "windows.cu", "srp.cu", "pairs.cu",
           "merge.cu"]

NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared", "--cudart", "static",
]

SSH_OK = 0
SSH_ERR_INVALID = -1
SSH_ERR_CUDA = -2
SSH_ERR_OOM = -3
SSH_ERR_UNSUPPORTED = -4
SSH_ERR_STATE = -5
SSH_QUERY_FALLBACK_ON_EMPTY = 1
SSH_QUERY_EXACT = 2


class ssh_params(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int32), ("W", ctypes.c_int32), ("delta", ctypes.c_int32),
        ("n", ctypes.c_int32), ("L", ctypes.c_int32), ("K", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("radius", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def build_native(verbose: bool = False, force: bool = False) -> Path:
    """Compile csrc/*.cu for sm_100a into paper_1610_07328_b200/libsshgpu.so."""
    srcs = [CSRC / s for s in SOURCES]
    deps = srcs + [CSRC / "common.cuh", CSRC / "dtw_warp.cuh", INCLUDE / "sshgpu.h"]
    if (not force and LIB_PATH.exists()
            and LIB_PATH.stat().st_mtime >= max(p.stat().st_mtime for p in deps)):
        return LIB_PATH
    import concurrent.futures as cf
    import tempfile

    tmp = LIB_PATH.with_suffix(".so.tmp%d" % os.getpid())
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared", "--cudart", "static")]
    with tempfile.TemporaryDirectory() as td:
        objs = [str(Path(td) / (p.stem + ".o")) for p in srcs]
        cmds = [[nvcc(), *compile_flags, "-c", "-I", str(INCLUDE), "-o", o, str(p)] for p, o in zip(srcs, objs)]
        if verbose:
            for c in cmds:
                print(" ".join(c), flush=True)
        # one nvcc per translation unit, in parallel (query.cu dominates)
        with cf.ThreadPoolExecutor(len(cmds)) as ex:
            for f in [ex.submit(subprocess.check_call, c, cwd=str(CSRC)) for c in cmds]:
                f.result()
        link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "--cudart", "static",
                "-o", str(tmp), *objs]
        subprocess.check_call(link, cwd=str(CSRC))
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None
_lock = threading.Lock()


def lib():
    """Load libsshgpu.so (fails loudly; never falls back to a CPU path)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise SshError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        PP = ctypes.POINTER(ctypes.c_void_p)
        sigs = {
            "ssh_last_error": ([], ctypes.c_char_p),
            "ssh_abi_version": ([], ctypes.c_int),
            "ssh_launch_count": ([], i64),
            "ssh_ctx_set_profiling": ([P, ctypes.c_int], ctypes.c_int),
            "ssh_ctx_profile": ([P, P, ctypes.c_int], ctypes.c_int),
            "ssh_ctx_create": ([ctypes.c_int, PP], ctypes.c_int),
            "ssh_ctx_destroy": ([P], ctypes.c_int),
            "ssh_ctx_set_params": ([P, ctypes.POINTER(ssh_params), P, P, P, P, P, i32], ctypes.c_int),
            "ssh_num_sketch_bits": ([P], ctypes.c_int),
            "ssh_sketch_words": ([P], ctypes.c_int),
            "ssh_tokens_per_series": ([P], ctypes.c_int),
            "ssh_sketch": ([P, P, i64, i64, P, P, P], ctypes.c_int),
            "ssh_shingle": ([P, P, i64, P, P, P, P], ctypes.c_int),
            "ssh_cws": ([P, P, P, P, i64, P, P, P], ctypes.c_int),
            "ssh_signatures": ([P, P, i64, i64, P, P, P], ctypes.c_int),
            "ssh_index_build": ([P, P, i64, i64, PP, P], ctypes.c_int),
            "ssh_build_index": ([P, P, i64, i64, i64, P, PP, P], ctypes.c_int),
            "ssh_build_index_host": ([P, P, i64, i64, i64, P, P, PP, P], ctypes.c_int),
            "ssh_index_destroy": ([P], ctypes.c_int),
            "ssh_index_num_buckets": ([P, ctypes.c_int, ctypes.POINTER(i64)], ctypes.c_int),
            "ssh_index_size": ([P], i64),
            "ssh_index_sketch_stats": ([P, P, P], ctypes.c_int),
            "ssh_merge_topk": ([P, P, i32, i32, i32, i32, P, P, P, P], ctypes.c_int),
            "ssh_index_export": ([P, ctypes.c_int, P, P, P, P], ctypes.c_int),
            "ssh_probe": ([P, P, P, i32, P, P, P], ctypes.c_int),
            "ssh_index_summarize": ([P, P, P, i64, P], ctypes.c_int),
            "ssh_index_copy_summaries": ([P, i64, i64, P, P, ctypes.POINTER(i32), ctypes.POINTER(i64), P],
                                         ctypes.c_int),
            "ssh_query_batch": ([P, P, P, P, i32, i32, i32, P, P, P, P, P, P, P], ctypes.c_int),
            "ssh_dtw_exact": ([P, P, P, P, P, i64, P, P], ctypes.c_int),
            "ssh_query_phase_ms": ([P, P], ctypes.c_int),
            "ssh_dtw_pairs64": ([P, P, P, P, i64, i32, i32, ctypes.c_double, P, P], ctypes.c_int),
            "ssh_envelope64": ([P, i64, i32, i32, P, P, P], ctypes.c_int),
            "ssh_lb_keogh64": ([P, P, P, i64, i32, i32, P, P], ctypes.c_int),
            "ssh_lb_kim64": ([P, P, i64, i32, P, P], ctypes.c_int),
            "ssh_index_create_bare": ([P, P, i64, i64, i64, PP, P], ctypes.c_int),
            "ssh_windows": ([P, i64, i32, i64, i32, P, P, ctypes.POINTER(i64), P], ctypes.c_int),
            "ssh_srp": ([P, i64, i32, P, P, i32, P, P, P], ctypes.c_int),
            "ssh_srp2": ([P, P, i64, i32, P, P, i32, P, P, i32, P], ctypes.c_int),
            "ssh_sshi_parse_tables": ([P, i64, i64, i32, i64, P, ctypes.POINTER(i64), ctypes.c_char_p, i32],
                                      ctypes.c_int),
        }
        for name, (args, res) in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


EXPORTED = [
    "ssh_last_error", "ssh_abi_version", "ssh_launch_count", "ssh_ctx_set_profiling",
    "ssh_ctx_profile", "ssh_ctx_create", "ssh_ctx_destroy", "ssh_ctx_set_params",
    "ssh_num_sketch_bits", "ssh_sketch_words", "ssh_tokens_per_series", "ssh_sketch", "ssh_shingle",
    "ssh_cws", "ssh_signatures", "ssh_index_build", "ssh_build_index", "ssh_build_index_host", "ssh_index_destroy", "ssh_index_num_buckets",
    "ssh_index_size", "ssh_index_sketch_stats", "ssh_merge_topk", "ssh_index_export", "ssh_index_summarize", "ssh_index_copy_summaries", "ssh_probe", "ssh_query_batch", "ssh_dtw_exact",
    "ssh_query_phase_ms", "ssh_dtw_pairs64", "ssh_envelope64", "ssh_lb_keogh64", "ssh_lb_kim64",
    "ssh_index_create_bare", "ssh_sshi_parse_tables", "ssh_windows", "ssh_srp", "ssh_srp2",
]


def check(rc: int, what: str = "") -> None:
    if rc == SSH_OK:
        return
    msg = lib().ssh_last_error().decode(errors="replace")
    if rc in (SSH_ERR_INVALID, SSH_ERR_UNSUPPORTED):
        raise ConfigError(msg)
    raise SshError(f"{what}: {msg}" if what else msg)


def ptr(t) -> ctypes.c_void_p:
    """Raw device/host pointer of a torch tensor or numpy array."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return t.ctypes.data_as(ctypes.c_void_p)

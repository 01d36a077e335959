"""Dev tool: time each device stage at a config size with CUDA events.

python scripts/stage_timing.py --cfg 1 [--n N] [--nq Q]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1610_07328_b200 as ssh  # noqa: E402
from paper_1610_07328_b200 import _native as nat  # noqa: E402
from paper_1610_07328_b200 import datagen  # noqa: E402
from paper_1610_07328_b200.index import _stream_ptr, get_context  # noqa: E402


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=1)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--nq", type=int, default=None)
    a = ap.parse_args()
    t0 = time.time()
    X, Q, src, p = datagen.workload(a.cfg, device="cuda", nq=a.nq, n_override=a.n)
    torch.cuda.synchronize()
    print(f"datagen {time.time() - t0:.1f}s  X={tuple(X.shape)} Q={Q.shape}", flush=True)
    params = ssh.SshParams(**p)
    N, m = X.shape
    ctx = get_context(0, params, m)
    L = nat.lib()
    st = _stream_ptr(0)
    bits = torch.empty((N, ctx.words), dtype=torch.int64, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    res = {}
    ms, _ = timed(lambda: nat.check(L.ssh_sketch(ctx.handle, nat.ptr(X), N, m, nat.ptr(bits), nat.ptr(stats), st)))
    res["sketch_ms"] = ms
    res["sketch_GBps"] = N * (4 * m + 8 * ctx.words) / ms / 1e6
    T = ctx.T
    tok = torch.empty((N, T), dtype=torch.int32, device="cuda")
    cnt = torch.empty((N, T), dtype=torch.int16, device="cuda")
    ln = torch.empty(N, dtype=torch.int32, device="cuda")
    ms, _ = timed(lambda: nat.check(L.ssh_shingle(ctx.handle, nat.ptr(bits), N, nat.ptr(tok), nat.ptr(cnt), nat.ptr(ln), st)))
    res["shingle_ms"] = ms
    sig = torch.empty((N, params.d), dtype=torch.int64, device="cuda")
    ms, _ = timed(lambda: nat.check(L.ssh_cws(ctx.handle, nat.ptr(tok), nat.ptr(cnt), nat.ptr(ln), N, None, nat.ptr(sig), st)))
    res["cws_ms"] = ms
    res["mean_distinct"] = float(ln.float().mean())
    ms, _ = timed(lambda: nat.check(L.ssh_signatures(ctx.handle, nat.ptr(X), N, m, nat.ptr(sig), None, st)))
    res["signatures_fused_ms"] = ms
    def mk():
        h = ctypes.c_void_p()
        nat.check(L.ssh_index_build(ctx.handle, nat.ptr(sig), N, 0, ctypes.byref(h), st))
        return h
    ms, h = timed(mk)
    res["tables_ms"] = ms
    res["recheck_windows"] = int(stats[0]) // 3
    res["near_zero_windows"] = int(stats[1]) // 3
    t0 = time.time()
    index = ssh.build_index(ssh.Dataset(X), params)
    torch.cuda.synchronize()
    res["build_index_s"] = time.time() - t0
    Qd = torch.from_numpy(Q).cuda()
    ms, out = timed(lambda: ssh.index.query_batch_device(index, Qd, 10), reps=2)
    res["query_batch_ms"] = ms
    n_cand = out[3].cpu().numpy()
    cnt5 = out[4].cpu().numpy()
    res["mean_cand"] = float(n_cand.mean())
    res["mean_counters"] = cnt5.mean(axis=0).tolist()
    res["queries_per_s"] = Q.shape[0] / ms * 1e3
    res["series_per_s_build"] = N / (res["signatures_fused_ms"] + res["tables_ms"]) * 1e3
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

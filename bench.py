#!/usr/bin/env python
"""bench.py — SSH index build + query batch on B200 (driver contract).

A step = one pass of the hot path over one batch of synthetic input: build
the index over the rank's series (K1 sketch -> K2 shingle -> K3 CWS ->
K4 bucket tables) and answer the query batch (K5 hash -> K6 probe -> K7 LB
filter -> K8 DTW waves -> K10 exact rescoring -> K9 top-k, then the
cross-rank merge).

Workloads (BASELINE.json configs):
* the headline line: configs[1] (N=1,000,000 random walks, m=512, K=4, L=20,
  1,000 queries, band 5%, top-10) per GPU — weak scaling over N GPUs;
* at N=1 the same line carries "workloads" with configs[2] (2M ECG windows of
  1024) and configs[3] (4M x 2048 random walks, band 10%), each measured the
  same way (device events, per-stage rooflines);
* `--cfg 4`: configs[4], 64M series sharded across the N GPUs (strong
  scaling), 10,000 queries.

`--gpus N` without torchrun re-executes itself under torch.distributed.run
(one process per GPU, NCCL).  value = series indexed/s over the whole job
(build part of the timed steps, CUDA events, max over ranks); queries/s and
DTW cells/s are reported beside it.  `--impl reference` times the CPU oracle
port (oracle/ssh_oracle.c, all host threads) on bounded samples of the same
workload.
"""

from __future__ import annotations

import argparse
import ctypes
import gc
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "series indexed/s; queries/s (probe + DTW rerank, top-10); DTW cells/s"
UNIT = "series/s"
K_TOP = 10
PROFILE_ROUND = "r02"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm_gbs=float(d["hbm_gbs"]), sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)),
                    source="measured (MEASURED_PEAKS.json)")
    return dict(hbm_gbs=6650.0, sm_max_mhz=1965.0, source="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
                pw.append(float(r[3]))
            except ValueError:
                continue
            for n, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        # samples "under load": power above the idle floor of this run
        if pw:
            floor = min(pw) + 0.25 * (max(pw) - min(pw))
            load = [s for s, p in zip(sm, pw) if p >= floor] or sm
        else:
            load = sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` run directly: one rank per GPU under torch.distributed.run."""
    # the ranks get this command line through the environment: torchrun's own
    # parser would take abbreviations of its options (e.g. --n) after the script
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve())]
    env = dict(os.environ, SSH_BENCH_ARGV=json.dumps(sys.argv[1:]))
    print("relaunch: " + " ".join(cmd) + " (args " + " ".join(sys.argv[1:]) + ")", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


# ----------------------------------------------------------------- our arm

def _release_device_state():
    """Drop cached contexts (grow-only scratch) and pooled memory between workloads."""
    import torch

    from paper_1610_07328_b200 import index as I

    with I._ctx_lock:
        I._ctx_cache.clear()
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def measure(args, cfg, rank, world, local, steps, warmup, nq=None, n_per=None, strong=False,
            headline=False):
    """Time `steps` build+query steps of configs[cfg] on this rank's shard; returns
    the workload dict on rank 0 (None elsewhere)."""
    import numpy as np
    import torch
    import torch.distributed as tdist

    import paper_1610_07328_b200 as ssh
    from paper_1610_07328_b200 import _native as nat
    from paper_1610_07328_b200 import datagen
    from paper_1610_07328_b200 import dist as D
    from paper_1610_07328_b200.index import _stream_ptr, get_context, query_batch_device

    dev = torch.device(f"cuda:{local}")
    c = datagen.CONFIGS[cfg]
    m = c["m"]
    nq = c["nq"] if nq is None else nq
    if strong:
        N_total = n_per * world if n_per else c["N"]
        lo, hi = D.shard_range(N_total, rank, world)
    else:
        N = n_per or c["N"]
        N_total = N * world
        lo, hi = rank * N, (rank + 1) * N
    N = hi - lo
    t_gen = time.time()
    X, Q, src, p = datagen.workload(cfg, lo=lo, hi=hi, device=dev, nq=nq, n_override=N_total)
    torch.cuda.synchronize()
    t_gen = time.time() - t_gen
    params = ssh.SshParams(**p)
    ds = ssh.Dataset(X)
    Qd = torch.from_numpy(Q).to(dev)
    ctx = get_context(local, params, m)
    lib = nat.lib()
    # the previous step's index stays alive while the next one builds (steady
    # state of the stream-ordered pool) unless two indexes would not fit
    keep_prev = N * (4 * m + 3 * m + 300) * 2 < 0.6 * torch.cuda.get_device_properties(dev).total_memory
    local_fn = lambda index: (lambda Qs, k: query_batch_device(index, Qs, k, False))  # noqa: E731

    def step():
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record()
        index = ssh.build_index(ds, params, id_base=lo)
        e1.record()
        if world > 1:
            ids, d2, n_out, n_cand, counters, status = D.sharded_query(Qd, K_TOP, local_fn(index))
        else:
            ids, d2, n_out, n_cand, counters, status = query_batch_device(index, Qd, K_TOP)
        e2.record()
        return (e0, e1, e2), (index, ids, d2, n_cand, counters, status)

    last = None
    for _ in range(warmup):
        if not keep_prev:
            last = None
        _, last = step()
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = lib.ssh_launch_count()
    evs = []
    # the build synchronises with the host twice (bucket counts); a cyclic-GC
    # pause landing between those points would show up as device idle time
    gc.collect()
    gc.disable()
    for _ in range(steps):
        if not keep_prev:
            last = None
        ev, last = step()
        evs.append(ev)
    torch.cuda.synchronize()
    gc.enable()
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    launches = lib.ssh_launch_count() - launches0
    clocks = sampler.stop()
    build_each = [a.elapsed_time(b) for a, b, _ in evs]
    query_each = [b.elapsed_time(c2) for _, b, c2 in evs]
    t = torch.tensor([sum(build_each), sum(query_each), evs[0][0].elapsed_time(evs[-1][2])],
                     dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    build_ms, query_ms, total_ms = t.tolist()
    index, ids, d2, n_cand, counters, status = last
    ties = index.sketch_stats
    tie_t = torch.tensor([ties["rechecked"], ties["near_zero"]], dtype=torch.int64, device=dev)
    if world > 1:
        tdist.all_reduce(tie_t, op=tdist.ReduceOp.SUM)
    out = None
    if rank == 0:
        kind = "ECG windows" if c["kind"] == "ecg" else "random walk"
        out = {
            "value": N_total * steps / (build_ms / 1e3),
            "queries_per_s": nq * steps / (query_ms / 1e3),
            "ms_per_step": total_ms / steps,
            "build_ms_per_step": build_ms / steps,
            "query_ms_per_step": query_ms / steps,
            "build_ms_each": [round(v, 3) for v in build_each],
            "query_ms_each": [round(v, 3) for v in query_each],
            "steps": steps, "warmup": warmup,
            "config": {
                "workload": f"configs[{cfg}]: {kind} N={N_total} ({'sharded' if strong else 'per GPU'} "
                            f"x {world}) x m={m}, W=80 delta=3 n=15 K=4 L=20, {nq} queries, "
                            f"DTW band {c['band']}, top-{K_TOP}",
                "cfg": cfg, "N_per_gpu": N, "N_total": N_total, "m": m, "queries": nq, "K": 4, "L": 20,
                "band": c["band"], "radius": params.warping().radius(m), "k": K_TOP,
                "parallelism": (f"shard{world} (series-sharded, queries replicated, top-k all_gather + "
                                f"|R| all_reduce over NCCL)" if world > 1 else "single GPU"),
                "l2": "inputs larger than L2 (X = %.2f GB per GPU)" % (N * m * 4 / 1e9),
            },
            "mean_candidates": float(n_cand.double().mean()),
            "statuses": {s: int((status == v).sum()) for s, v in (("ok", 0), ("no-candidates", 1),
                                                                   ("fallback", 2))},
            "mean_counters": dict(zip(["kim_pruned", "keogh_pruned", "keogh2_pruned", "dtw_computed",
                                       "dtw_abandoned"], counters.double().mean(dim=0).tolist())),
            "sketch_ties": {"rechecked_f64": int(tie_t[0]), "near_zero_abs_dot_lt_1e-9": int(tie_t[1]),
                            "note": "windows of the last timed build (all ranks) whose f32 screen "
                                    "deferred to the exact f64 dot; |dot| < 1e-9 are sign ties"},
            "gpu_launches": int(launches),
            "gpu_launches_per_step": launches / steps,
            "clocks": clocks,
            "datagen_s": t_gen,
            "scaling": "strong" if strong else "weak",
        }
    if world > 1:
        tdist.barrier()
    if rank == 0:
        out["stages"] = stage_profile(ctx, X, Qd, index, params, lib, nat, _stream_ptr(local), query_batch_device,
                                      cfg, float(n_cand.double().sum()))
        out["dtw_cells_per_s"] = out["stages"].get("dtw_cells_per_s")
        # dominant kernel = the longest single-kernel stage with a roofline
        dom = max((s for s in out["stages"].values() if isinstance(s, dict) and s.get("roofline")),
                  key=lambda s: s["ms"])
        out["roofline"] = dom.get("roofline")
        out["dominant_stage"] = dom.get("name")
    del last, index
    if world > 1:
        tdist.barrier()
    if not args.no_e2e and (headline or args.e2e_all):
        e = e2e_run(X, Q, params, lo, nq, N_total, world)
        if rank == 0:
            out["e2e"] = e
    if rank == 0 and headline and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(X, Q, p, args, cfg)
    del X, Qd, ds
    return out


def run_ours(args):
    import torch
    import torch.distributed as tdist

    from paper_1610_07328_b200 import dist as D

    rank, world, local = D.init_from_env("nccl")
    torch.cuda.set_device(local)
    if args.gpus != world:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
    strong = args.cfg == 4 or args.strong
    if args.cfg == 4 and world == 1 and not args.n:
        # 64M x 512 f32 (128 GB) + codes/summaries/tables do not fit one GPU
        if rank == 0:
            print(json.dumps({"metric": METRIC, "unavailable": "configs[4] (64M series) needs >= 2 GPUs; "
                              "run with --gpus 2..8", "n_gpus": world}), flush=True)
        return
    w = measure(args, args.cfg, rank, world, local, args.steps, args.warmup, nq=args.nq, n_per=args.n,
                strong=strong, headline=True)
    extras = {}
    if world == 1 and args.cfg == 1 and not args.no_extra:
        for cfg in (2, 3):
            _release_device_state()
            try:
                extras[f"configs[{cfg}]"] = measure(args, cfg, rank, world, local, args.extra_steps,
                                                    args.extra_warmup, nq=args.extra_nq)
            except Exception as ex:  # report, never hide: the line says which workload failed
                extras[f"configs[{cfg}]"] = {"error": f"{type(ex).__name__}: {ex}"}
    if rank == 0:
        out = {
            "metric": METRIC,
            "value": w.pop("value"),
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": w.pop("ms_per_step"),
            "higher_is_better": True,
            "scaling": w.pop("scaling"),
            "vs_baseline": None,
            "dtype": "f32 screen + f64 exact (sign recheck, CWS, DTW rescoring); u64 keys",
            "data": "synthetic (BASELINE.json configs[%d] recipe, seeded; no public dataset)" % args.cfg,
        }
        out.update(w)
        if extras:
            for v in extras.values():
                if isinstance(v, dict):
                    v.pop("scaling", None)
            out["workloads"] = extras
        print(json.dumps(out), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def _time(fn, reps=5):
    import torch

    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def _profile_json(cfg):
    """The committed ncu summary of this workload (profiles/<round>/ncu_cfg<cfg>.json), or {}."""
    for rnd in (PROFILE_ROUND, "r01"):
        p = ROOT / "profiles" / rnd / f"ncu_cfg{cfg}.json"
        if p.exists():
            try:
                return json.loads(p.read_text())
            except Exception:
                return {}
    return {}


def _traffic(prof, kernel_prefix):
    """DRAM bytes (read + write) summed over the launches of kernels whose name
    starts with `kernel_prefix` (a string or a tuple of them) in one build +
    query batch (the committed ncu metrics capture)."""
    ks = prof.get("kernels", {})
    pre = kernel_prefix if isinstance(kernel_prefix, tuple) else (kernel_prefix,)
    tot = [v["dram_bytes"] for k, v in ks.items() if k.startswith(pre) and v.get("dram_bytes")]
    return float(sum(tot)) if tot else None


def stage_profile(ctx, X, Qd, index, params, lib, nat, st, query_batch_device, cfg, cand_total):
    import numpy as np
    import torch

    peaks = load_peaks()
    hbm = peaks["hbm_gbs"]
    prof_json = _profile_json(cfg)
    N, m = X.shape
    nq = Qd.shape[0]
    words = ctx.words
    bits = torch.empty((N, words), dtype=torch.int64, device=X.device)
    sig = torch.empty((N, params.d), dtype=torch.int64, device=X.device)
    res = {}
    ms = _time(lambda: nat.check(lib.ssh_sketch(ctx.handle, nat.ptr(X), N, m, nat.ptr(bits), None, st)))
    b = N * (4 * m + 8 * words)
    res["sketch"] = dict(name="sketch (K1)", ms=ms, bytes=b, roofline=dict(
        bound="hbm", achieved=b / ms / 1e6, peak=hbm, unit="GB/s", frac=b / ms / 1e6 / hbm,
        traffic=_traffic(prof_json, "sketch_"), kernel="sketch_stream_kernel",
        note="algorithmic bytes = N*(4m + 8*ceil(N_B/64)); peak = %s HBM copy; traffic = ncu dram bytes "
             "(profiles/%s/ncu_cfg%d.json)" % (peaks["source"], PROFILE_ROUND, cfg)))
    ms_sig = _time(lambda: nat.check(lib.ssh_signatures(ctx.handle, nat.ptr(X), N, m, nat.ptr(sig), None, st)))
    cws_ms = max(ms_sig - ms, 1e-6)
    # CWS work unit: S = K*L slot evaluations per distinct token per series
    # (SURVEY §8d); D = distinct tokens per series, counted on a sample
    ns = min(N, 16384)
    T = ctx.T
    tok = torch.empty((ns, T), dtype=torch.int32, device=X.device)
    cnt = torch.empty((ns, T), dtype=torch.int16, device=X.device)
    nset = torch.empty(ns, dtype=torch.int32, device=X.device)
    D_mean = None
    try:
        nat.check(lib.ssh_sketch(ctx.handle, nat.ptr(X), ns, m, nat.ptr(bits), None, st))
        nat.check(lib.ssh_shingle(ctx.handle, nat.ptr(bits), ns, nat.ptr(tok), nat.ptr(cnt), nat.ptr(nset), st))
        torch.cuda.synchronize()
        D_mean = float(nset.double().mean())
    except Exception:
        D_mean = None
    S = params.K * params.d
    ev = N * S * D_mean if D_mean else None
    cws_prof = prof_json.get("cws", {})
    res["shingle_cws"] = dict(
        name="shingle+CWS (K2+K3, fused)", ms=cws_ms, distinct_tokens_per_series=D_mean,
        evaluations=ev, evaluations_per_s=(ev / (cws_ms / 1e3)) if ev else None,
        l2_hit_rate=cws_prof.get("l2_hit_rate"), fp64_pipe_util=cws_prof.get("fp64_pipe_util"),
        issue_active=cws_prof.get("issue_active"),
        roofline=dict(
            bound="hbm", achieved=N * (8 * words + 8 * params.d) / cws_ms / 1e6, peak=hbm, unit="GB/s",
            frac=N * (8 * words + 8 * params.d) / cws_ms / 1e6 / hbm, traffic=_traffic(prof_json, "cws_"),
            kernel="cws_fast_kernel",
            note="HBM bytes in/out only (bits in, signatures out); the kernel is bound by dependent L2 "
                 "gathers of the CWS tables: see evaluations_per_s (S*D per series), l2_hit_rate, "
                 "fp64_pipe_util, issue_active (ncu --set full, profiles/%s)" % PROFILE_ROUND))
    res["signatures_fused"] = dict(name="K1-K3", ms_total=ms_sig)

    def mk():
        h = ctypes.c_void_p()
        nat.check(lib.ssh_index_build(ctx.handle, nat.ptr(sig), N, 0, ctypes.byref(h), st))
        lib.ssh_index_destroy(h)

    ms_t = _time(mk, reps=3)
    bt = N * params.d * 20
    tr = _traffic(prof_json, ("rs_", "rle_"))
    res["tables"] = dict(name="bucket tables (K4)", ms=ms_t, roofline=dict(
        bound="hbm", achieved=bt / ms_t / 1e6, peak=hbm, unit="GB/s", frac=bt / ms_t / 1e6 / hbm,
        traffic=tr, kernel="rs_*/rle_* (radix passes + run-length CSR)",
        note="algorithmic bytes = 20 B per (series, table): 8 B key in, 8 B key + 4 B id out; traffic = "
             "ncu dram bytes of every table kernel of one build"))
    # rerank summaries (part of every build, on the side stream beside K4):
    # standalone over the same rows
    def summ():
        nat.check(lib.ssh_index_summarize(ctx.handle, index._tables.handle, nat.ptr(X), m, st))

    ms_s = _time(summ, reps=3)
    mp = (m + 127) // 128 * 128
    bsum = N * (4 * m + 64 + 3 * mp)
    res["summaries"] = dict(name="rerank summaries (records + u8 sample/envelope codes)", ms=ms_s, roofline=dict(
        bound="hbm", achieved=bsum / ms_s / 1e6, peak=hbm, unit="GB/s", frac=bsum / ms_s / 1e6 / hbm,
        traffic=_traffic(prof_json, "summaries"), kernel="summaries_kernel",
        note="algorithmic bytes = N * (4m read + 64 B record + 3 m_p B codes written); runs on the build's side "
             "stream concurrently with K4; issue-bound on the envelope-code running max/min"))
    # query phases
    nat.check(lib.ssh_ctx_set_profiling(ctx.handle, 1))
    torch.cuda.synchronize()
    query_batch_device(index, Qd, K_TOP)
    torch.cuda.synchronize()
    prof = (ctypes.c_double * 24)()
    nat.check(lib.ssh_ctx_profile(ctx.handle, prof, 24))
    nat.check(lib.ssh_ctx_set_profiling(ctx.handle, 0))
    names = ["hash (K5)", "probe+bitmap (K6)", "member keys (sample, cutoff pass, overflow) + bin sort (K7)",
             "wave LB_Keogh2/LB_Keogh over u8 codes (K8a wave_lb_kernel)",
             "wave fp32 DTW (K8b)", "rescore+top-k (K9/K10)"]
    for i, n in enumerate(names):
        res[f"q{i}"] = dict(name=n, ms=prof[i])
    # K5: query sketch + CWS (K1-K3 on the batch): 4m B in + 8L B out per query
    bq = nq * (4 * m + 8 * params.d)
    if prof[0] > 0:
        res["q0"]["roofline"] = dict(
            bound="hbm", achieved=bq / prof[0] / 1e6, peak=hbm, unit="GB/s", frac=bq / prof[0] / 1e6 / hbm,
            traffic=None, kernel="sketch + cws_fast (query batch)",
            note="algorithmic bytes = nq (4m + 8L); a few launches over a small batch: launch/latency-bound")
    # K6: bitmap words written + bucket id lists read
    nw = (N + 31) // 32
    b6 = cand_total * 4 + nq * nw * 4 * 2
    if prof[1] > 0:
        res["q1"]["roofline"] = dict(
            bound="hbm", achieved=b6 / prof[1] / 1e6, peak=hbm, unit="GB/s", frac=b6 / prof[1] / 1e6 / hbm,
            traffic=_traffic(prof_json, ("probe", "bitmap", "count_kernel")), kernel="probe_kernel + bitmap_smem_kernel + count_kernel",
            note="algorithmic bytes = |R| x 4 B (member ids of the probed buckets, a lower bound: buckets of "
                 "different tables overlap) + the membership bitmap written and counted (2 x nq x N/8)")
    # K7: every member of R costs one 64-byte record read (L2/HBM) + its key
    # and bin written (8 B); the bitmap is read once per pass
    k7_bytes = cand_total * (64 + 8) + nq * nw * 4 * 2
    if prof[2] > 0:
        res["q2"]["roofline"] = dict(
            bound="hbm", achieved=k7_bytes / prof[2] / 1e6, peak=hbm, unit="GB/s",
            frac=k7_bytes / prof[2] / 1e6 / hbm, traffic=_traffic(prof_json, ("paa_members", "binsort", "bs_")),
            kernel="paa_members_kernel + binsort_kernel",
            note="algorithmic bytes = |R| x (64 B record + 8 B key/bin) + 2 bitmap passes; records are "
                 "L2-resident at configs[1] (64 MB)")
    cells = prof[6]
    dtw_ms = prof[4]
    res["dtw_cells"] = cells
    res["dtw_cells_per_s"] = cells / (dtw_ms / 1e3) if dtw_ms > 0 else None
    # a cell is FADD + FFMA + FMNMX3 (3 FP32-pipe instructions) at
    # 128 lanes/SM/clk -> 148 x 128 x f_max / 3 = 12.4 T cells/s at 1965 MHz
    peak_cells = 148 * 128 * peaks["sm_max_mhz"] * 1e6 / 3.0
    r = params.warping().radius(m)
    res["q4"]["roofline"] = dict(
        bound="fp32", achieved=(cells / (dtw_ms / 1e3)) / 1e12 if dtw_ms else 0,
        peak=peak_cells / 1e12, unit="Tcells/s",
        frac=(cells / (dtw_ms / 1e3)) / peak_cells if dtw_ms else 0,
        traffic=_traffic(prof_json, ("dtwp_", "dtw32")),
        kernel=("dtwp_first/dtwp_pass pooled register band" if r in (3, 6, 13, 26, 51)
                else "dtw32w_kernel (band-chunked warp wavefront)"),
        note="cells = in-band cells of the rows each fp32 DTW evaluated; peak = SURVEY §8d's 148 x 128 x "
             "f_max / 3 (FADD + FFMA + FMNMX3 per cell)")
    res["dtw_evaluated"] = prof[8]
    res["rescored"] = prof[9]
    # K10: exact f64 DTW of the rescoring set (the reference recurrence: DSUB, DMUL, DADD + 2 DMNMX per
    # cell on the FP64 pipe, 64 lanes/SM/clk) + the final (d64, id) top-k
    cells64 = prof[9] * m * (2 * r + 1)
    peak64 = 148 * 64 * peaks["sm_max_mhz"] * 1e6 / 5.0
    if prof[5] > 0:
        res["q5"]["roofline"] = dict(
            bound="fp64", achieved=cells64 / (prof[5] / 1e3) / 1e12, peak=peak64 / 1e12, unit="Tcells/s",
            frac=cells64 / (prof[5] / 1e3) / peak64, traffic=_traffic(prof_json, "dtw64"),
            kernel="dtw64r/dtw64band (exact rescoring) + select/topk",
            note="cells = rescored pairs x m x (2r+1) (upper bound); about k + a few pairs per query, so the "
                 "stage is latency-bound, not FP64-bound")
    lb_bytes = prof[7]
    lb_ms = prof[3]
    if lb_ms > 0:
        res["q3"]["roofline"] = dict(
            bound="hbm", achieved=lb_bytes / lb_ms / 1e6, peak=hbm, unit="GB/s",
            frac=lb_bytes / lb_ms / 1e6 / hbm, traffic=_traffic(prof_json, "wave_lb"), kernel="wave_lb_kernel",
            note="algorithmic bytes = u8 envelope-code and sample-code blocks the LB_Keogh2/LB_Keogh "
                 "cascade reads before abandoning (device counter, per query batch)")
    res["wave_lb_bytes"] = lb_bytes
    res["wave_lb_paa_skips"] = prof[10]
    res["wave_lb_keogh_prunes"] = prof[11]
    res["wave_members_visited"] = prof[12]
    res["dtw_cells_executed"] = prof[20]
    res["waves"] = prof[16]
    res["active_query_waves"] = prof[17]
    if prof[15] > 0:
        res["thr0_over_dk"] = prof[13] / prof[15]
        res["thr1_over_dk"] = prof[14] / prof[15]
    del bits, sig, tok, cnt, nset
    return res


def e2e_run(X, Q, params, lo, nq, N_total, world):
    """Public API with HOST buffers on every rank: build_index from pinned host
    memory and query_index_batch (query_index_batch_sharded at N > 1) from host
    numpy; H2D/D2H inside the timed region; wall time, max over ranks."""
    import torch
    import torch.distributed as tdist

    import paper_1610_07328_b200 as ssh

    Xh = X.cpu().pin_memory()
    dsh = ssh.Dataset.__new__(ssh.Dataset)
    dsh.values, dsh.source = Xh, "pinned host"
    N, m = Xh.shape
    reps = 2
    tb, tq = [], []
    for i in range(reps + 1):
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        index = ssh.build_index(dsh, params, id_base=lo)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if world > 1:
            res = ssh.query_index_batch_sharded(index, Q, K_TOP)
        else:
            res = ssh.query_index_batch(index, Q, K_TOP)
        t2 = time.perf_counter()
        if i:
            tb.append(t1 - t0)
            tq.append(t2 - t1)
        del index, res
    t = torch.tensor([statistics.median(tb), statistics.median(tq)], dtype=torch.float64,
                     device=X.device)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    tbm, tqm = t.tolist()
    h2d = N * m * 4 + Q.shape[0] * m * 4
    d2h = nq * K_TOP * 16 + nq * (4 + 8 + 40 + 4) + params.d * 8
    del Xh, dsh
    return {"value": N_total / tbm, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "queries_per_s": nq / tqm,
            "note": "build_index(Dataset(pinned host f32)) + query_index_batch(host numpy)"
                    + (" / query_index_batch_sharded" if world > 1 else "") +
                    " through the public API; wall clock with device sync, max over ranks; bytes per rank"}


# ----------------------------------------------------------- reference arm

def cpu_baseline(X, Q, p, args, cfg, reps=1):
    """The oracle port (oracle/ssh_oracle.c, OpenMP over all host threads) on a
    bounded sample of the same workload: build rate over the first
    --cpu-build-sample series; queries/s of --cpu-queries queries against an
    oracle index over the first --cpu-query-index series (1M = configs[1]'s
    full N, so queries/s is a same-N figure)."""
    from oracle import oracle as orc

    th = ncores()
    Xh = X.cpu().numpy() if hasattr(X, "cpu") else X
    n_build = min(Xh.shape[0], args.cpu_build_sample)
    orc.get_tables(p["n"], p["d"] * p["K"], p["seed"], Xh.shape[1])
    vals = []
    for _ in range(reps):
        t0 = time.perf_counter()
        sig = orc.signatures(Xh[:n_build], p["W"], p["delta"], p["n"], p["d"], p["K"], p["seed"], threads=th)
        orc.tables_from_signatures(sig)
        vals.append(n_build / (time.perf_counter() - t0))
    out = {"value": statistics.median(vals), "unit": UNIT, "cores": th, "kind": "port",
           "sample": f"build_index (K=4 signatures + stable-argsort tables) over the first {n_build} "
                     f"series of configs[{cfg}]"}
    n_idx = min(Xh.shape[0], args.cpu_query_index)
    t0 = time.perf_counter()
    idx = orc.build_index(Xh[:n_idx], p["W"], p["delta"], p["n"], p["d"], p["K"], p["seed"], p["band"],
                          threads=th)
    t_idx = time.perf_counter() - t0
    nq = min(Q.shape[0], args.cpu_queries)
    qv = []
    res = None
    for _ in range(reps):
        t0 = time.perf_counter()
        res = orc.query_batch(idx, Q[:nq], K_TOP, threads=th)
        qv.append(nq / (time.perf_counter() - t0))
    out["queries_per_s"] = statistics.median(qv)
    out["query_sample"] = (f"{nq} queries (query_index cascade, one per host thread) against an oracle "
                           f"index over the first {n_idx} series (mean |R|={float(res['n_cand'].mean()):.0f}; "
                           f"index build {t_idx:.1f} s = {n_idx / t_idx:.0f} series/s, untimed setup)")
    return out


def run_reference(args):
    """--impl reference: the CPU oracle port of the reference path on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1610_07328_b200 import datagen

    cfg = args.cfg if args.cfg != 4 else 1
    dev = "cuda" if _cuda_ok() else "cpu"
    c = datagen.CONFIGS[cfg]
    N = min(args.n or c["N"], max(args.cpu_build_sample, args.cpu_query_index))
    X, Q, src, p = datagen.workload(cfg, lo=0, hi=N, device=dev, nq=args.cpu_queries,
                                    n_override=(args.n or c["N"]))
    Xh = X.cpu().numpy()
    del X
    from oracle import oracle as orc

    th = ncores()
    orc.get_tables(p["n"], p["d"] * p["K"], p["seed"], Xh.shape[1])
    n_build = min(Xh.shape[0], args.cpu_build_sample)
    n_idx = min(Xh.shape[0], args.cpu_query_index)
    t0 = time.perf_counter()
    idx = orc.build_index(Xh[:n_idx], p["W"], p["delta"], p["n"], p["d"], p["K"], p["seed"], p["band"],
                          threads=th)
    t_idx = time.perf_counter() - t0
    nq = min(Q.shape[0], args.cpu_queries)
    vals, qps, cands = [], [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        sig = orc.signatures(Xh[:n_build], p["W"], p["delta"], p["n"], p["d"], p["K"], p["seed"], threads=th)
        orc.tables_from_signatures(sig)
        tb = time.perf_counter() - t0
        t0 = time.perf_counter()
        res = orc.query_batch(idx, Q[:nq], K_TOP, threads=th)
        tq = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(n_build / tb)
            qps.append(nq / tq)
            cands.append(float(res["n_cand"].mean()))
    v = statistics.median(vals)
    sample = (f"each step: build_index (K=4 signatures + stable-argsort tables) over the first {n_build} "
              f"series, then {nq} queries (query_index cascade, OpenMP over queries) against an oracle index "
              f"over the first {n_idx} series of configs[{cfg}] (mean |R|={statistics.mean(cands):.0f}; index "
              f"built once, {t_idx:.1f} s, untimed)")
    out = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic (BASELINE.json configs[%d] recipe, seeded)" % cfg,
        "config": {"workload": f"configs[{cfg}] (bounded CPU sample, see cpu_baseline.sample)",
                   "cfg": cfg, "N": args.n or c["N"], "m": c["m"], "K": 4, "L": 20, "k": K_TOP,
                   "queries": nq, "index_series": n_idx},
        "queries_per_s": statistics.median(qps),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": th, "kind": "port", "sample": sample,
                         "queries_per_s": statistics.median(qps)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "queries_per_s": statistics.median(qps)},
    }
    print(json.dumps(out), flush=True)


def _cuda_ok():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cfg", type=int, default=1)
    ap.add_argument("--strong", action="store_true", help="shard a fixed N_total (default for --cfg 4)")
    ap.add_argument("--n", type=int, default=None,
                    help="override N per GPU (weak) or N_total / GPUs (strong) (dev only)")
    ap.add_argument("--nq", type=int, default=None, help="override query count (dev only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-all", action="store_true", help="e2e for the extra workloads too")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the configs[2]/[3] workloads at N=1")
    ap.add_argument("--extra-steps", type=int, default=2)
    ap.add_argument("--extra-warmup", type=int, default=3)
    ap.add_argument("--extra-nq", type=int, default=None)
    ap.add_argument("--cpu-build-sample", type=int, default=100_000)
    ap.add_argument("--cpu-query-index", type=int, default=1_000_000)
    ap.add_argument("--cpu-queries", type=int, default=24)
    argv = json.loads(os.environ["SSH_BENCH_ARGV"]) if os.environ.get("SSH_BENCH_ARGV") else None
    args = ap.parse_args(argv)
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

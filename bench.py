#!/usr/bin/env python
"""bench.py — SSH index build + query batch on B200 (driver contract).

A step = one pass of the hot path over one batch of synthetic input: build
the index over the rank's series (K1 sketch -> K2 shingle -> K3 CWS ->
K4 bucket tables) and answer the query batch (K5 hash -> K6 probe -> K7 LB
filter -> K8 DTW waves -> K10 exact rescoring -> K9 top-k, then the
cross-rank merge).  Workload: BASELINE.json configs[1] (N=1,000,000 random
walks, m=512, K=4, L=20, 1,000 queries, top-10) per GPU (weak scaling).

value = series indexed/s over the whole job (build part of the timed steps,
CUDA events, max over ranks); queries/s and DTW cells/s are reported beside
it.  `--impl reference` times the CPU oracle port (oracle/ssh_oracle.c, all
host threads) on bounded samples of the same workload.
"""

from __future__ import annotations

import argparse
import gc
import ctypes
import json
import os
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


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm_gbs=float(d["hbm_gbs"]), sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)),
                    source="measured")
    return dict(hbm_gbs=6650.0, sm_max_mhz=1965.0, source="fallback")


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


# ----------------------------------------------------------------- our arm

def run_ours(args):
    import numpy as np
    import torch

    import paper_1610_07328_b200 as ssh
    from paper_1610_07328_b200 import _native as nat
    from paper_1610_07328_b200 import datagen
    from paper_1610_07328_b200 import dist as D
    from paper_1610_07328_b200.index import _stream_ptr, get_context, query_batch_device

    rank, world, local = D.init_from_env("nccl")
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    c = datagen.CONFIGS[args.cfg]
    N = args.n or c["N"]
    m = c["m"]
    nq = args.nq if args.nq is not None else c["nq"]
    N_total = N * world
    lo, hi = rank * N, (rank + 1) * N
    t_gen = time.time()
    X, Q, src, p = datagen.workload(args.cfg, lo=lo, hi=hi, device=dev, nq=nq, n_override=N_total)
    torch.cuda.synchronize()
    t_gen = time.time() - t_gen
    params = ssh.SshParams(**p)
    ds = ssh.Dataset(X)
    Qd = torch.from_numpy(Q).to(dev)
    ctx = get_context(local, params, m)
    lib = nat.lib()
    import torch.distributed as tdist

    def step():
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record()
        index = ssh.build_index(ds, params, id_base=lo)
        e1.record()
        ids, d2, n_out, n_cand, counters, status = query_batch_device(index, Qd, K_TOP)
        if world > 1:
            ids, d2, n_cand, counters = D.merge_across_ranks(ids, d2, n_cand, counters, K_TOP)
        e2.record()
        return (e0, e1, e2), (index, ids, d2, n_cand, counters)

    # warm-up mirrors the timed loop (the previous step's index stays alive while
    # the next one builds), so the stream-ordered memory pool reaches steady state
    last = None
    for _ in range(args.warmup):
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
    for _ in range(args.steps):
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
    build_ms = sum(build_each)
    query_ms = sum(query_each)
    total_ms = evs[0][0].elapsed_time(evs[-1][2])
    t = torch.tensor([build_ms, query_ms, total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    build_ms, query_ms, total_ms = t.tolist()
    index, ids, d2, n_cand, counters = last
    mean_cand = float(n_cand.double().mean())
    mean_cnt = counters.double().mean(dim=0).tolist()

    out = None
    if rank == 0:
        out = {
            "metric": METRIC,
            "value": N_total * args.steps / (build_ms / 1e3),
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32 screen + f64 exact (sign recheck, CWS, DTW rescoring); u64 keys",
            "data": "synthetic (BASELINE.json configs[%d] recipe, seeded; no public dataset)" % args.cfg,
            "config": {
                "workload": f"configs[{args.cfg}]: random walk N={N}/GPU x m={m}, W=80 delta=3 n=15 "
                            f"K=4 L=20, {nq} warped queries, DTW band {c['band']}, top-{K_TOP}",
                "N_per_gpu": N, "N_total": N_total, "m": m, "queries": nq, "K": 4, "L": 20,
                "band": c["band"], "k": K_TOP, "parallelism": f"shard{world} (series-sharded, "
                "queries replicated, top-k all_gather)",
                "l2": "inputs larger than L2 (X = %.2f GB per GPU)" % (N * m * 4 / 1e9),
            },
            "queries_per_s": nq * args.steps / (query_ms / 1e3),
            "build_ms_per_step": build_ms / args.steps,
            "build_ms_each": [round(v, 3) for v in build_each],
            "query_ms_each": [round(v, 3) for v in query_each],
            "query_ms_per_step": query_ms / args.steps,
            "mean_candidates": mean_cand,
            "mean_counters": dict(zip(["kim_pruned", "keogh_pruned", "keogh2_pruned", "dtw_computed",
                                       "dtw_abandoned"], mean_cnt)),
            "gpu_launches": int(launches),
            "gpu_launches_per_step": launches / args.steps,
            "clocks": clocks,
            "datagen_s": t_gen,
        }
    if world > 1:
        tdist.barrier()
    # ---- per-stage timing (outside the timed region) for the roofline
    if rank == 0:
        stages = stage_profile(ctx, X, Qd, index, params, lib, nat, _stream_ptr(local), query_batch_device)
        out["stages"] = stages
        out["dtw_cells_per_s"] = stages.get("dtw_cells_per_s")
        # dominant kernel = the longest stage that is a single kernel with a
        # roofline (grouped stages such as key+sort list their parts in "stages")
        dom = max((s for s in stages.values() if isinstance(s, dict) and s.get("roofline")),
                  key=lambda s: s["ms"])
        out["roofline"] = dom.get("roofline")
        out["dominant_stage"] = dom.get("name")
        if not args.no_e2e:
            out["e2e"] = e2e_run(args, ds, X, Q, params, lo, nq)
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(X, Q, p, args, with_queries=True)
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


def _ncu_traffic(kernel):
    """DRAM bytes (read + write) of all launches of `kernel` in one configs[1]
    build + 1000-query batch, from the committed ncu capture (profiles/), or None."""
    try:
        d = json.loads((Path(__file__).resolve().parent / "profiles" / "r01" / "traffic_cfg1.json").read_text())
        return d["kernels"][kernel]["dram_bytes"]
    except Exception:
        return None


def stage_profile(ctx, X, Qd, index, params, lib, nat, st, query_batch_device):
    import torch

    peaks = load_peaks()
    hbm = peaks["hbm_gbs"]
    N, m = X.shape
    words = ctx.words
    bits = torch.empty((N, words), dtype=torch.int64, device=X.device)
    sig = torch.empty((N, params.d), dtype=torch.int64, device=X.device)
    res = {}
    ms = _time(lambda: nat.check(lib.ssh_sketch(ctx.handle, nat.ptr(X), N, m, nat.ptr(bits), None, st)))
    b = N * (4 * m + 8 * words)
    res["sketch"] = dict(name="sketch (K1)", ms=ms, bytes=b, roofline=dict(
        bound="hbm", achieved=b / ms / 1e6, peak=hbm, unit="GB/s", frac=b / ms / 1e6 / hbm,
        traffic=_ncu_traffic("sketch_stream_kernel<80, 3, 20, 16>"), kernel="sketch_stream_kernel<80,3,20,16>",
        note="algorithmic bytes = N*(4m + 8*ceil(N_B/64)); peak = %s HBM copy; traffic = ncu dram bytes of "
             "the build launch + the 1000-query hash launch (0.1%%) (profiles/r01/traffic_cfg1.json)"
             % peaks["source"]))
    ms_sig = _time(lambda: nat.check(lib.ssh_signatures(ctx.handle, nat.ptr(X), N, m, nat.ptr(sig), None, st)))
    cws_ms = max(ms_sig - ms, 1e-6)
    b2 = N * (4 * m + 8 * params.d)
    res["shingle_cws"] = dict(name="shingle+CWS (K2+K3)", ms=cws_ms, evaluations=None, roofline=dict(
        bound="hbm", achieved=N * (8 * words + 8 * params.d) / cws_ms / 1e6, peak=hbm, unit="GB/s",
        frac=N * (8 * words + 8 * params.d) / cws_ms / 1e6 / hbm, traffic=_ncu_traffic("cws_fast_kernel<3, 5, 4>"),
        kernel="cws_fast_kernel<FUSED,5,4>",
        note="HBM bytes in/out only; the kernel is bound by L2 gathers of the CWS tables + FP64"))
    res["signatures_fused"] = dict(name="K1-K3", ms_total=ms_sig)

    def mk():
        h = ctypes.c_void_p()
        nat.check(lib.ssh_index_build(ctx.handle, nat.ptr(sig), N, 0, ctypes.byref(h), st))
        lib.ssh_index_destroy(h)

    ms_t = _time(mk, reps=3)
    bt = N * params.d * 20
    res["tables"] = dict(name="bucket tables (K4)", ms=ms_t, roofline=dict(
        bound="hbm", achieved=bt / ms_t / 1e6, peak=hbm, unit="GB/s", frac=bt / ms_t / 1e6 / hbm,
        traffic=None, kernel="rs_scatter/rs_hist/rle_*",
        note="algorithmic bytes = 20 B per (series, table): 8 B key in, 8 B key + 4 B id out"))
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
             "wave fp32 DTW (K8b dtwp_first/dtwp_level pooled passes)", "rescore+top-k (K9/K10)"]
    r = params.warping().radius(m)
    for i, n in enumerate(names):
        res[f"q{i}"] = dict(name=n, ms=prof[i])
    cells = prof[6]
    dtw_ms = prof[4]
    res["dtw_cells"] = cells
    res["dtw_cells_per_s"] = cells / (dtw_ms / 1e3) if dtw_ms > 0 else None
    # per cell: FADD + FFMA on the fma pipe, FMNMX3 + FMNMX (row min) on the alu
    # pipe; both pipes issue 16 lanes/clk/SMSP for these forms (B300_MICROARCH
    # "rt_SMSP=2"), so the cell peak is 148 x 64 lanes x f / 2 instr
    peak_cells = 148 * 64 * peaks["sm_max_mhz"] * 1e6 / 2.0
    res["q4"]["roofline"] = dict(bound="fp32", achieved=(cells / (dtw_ms / 1e3)) / 1e12 if dtw_ms else 0,
                                 peak=peak_cells / 1e12, unit="Tcells/s",
                                 frac=(cells / (dtw_ms / 1e3)) / peak_cells if dtw_ms else 0,
                                 traffic=_ncu_traffic("dtwp_level_kernel<26>"),
                                 kernel="dtwp_first_kernel + dtwp_level_kernel<26>",
                                 note="cells = alive lane-rows x (2r+1); 2 fma-pipe + 2 alu-pipe instr per cell; "
                                      "peak 148 x 64 x f_max / 2")
    res["dtw_evaluated"] = prof[8]
    res["rescored"] = prof[9]
    lb_bytes = prof[7]
    lb_ms = prof[3]
    if lb_ms > 0:
        res["q3"]["roofline"] = dict(
            bound="hbm", achieved=lb_bytes / lb_ms / 1e6, peak=hbm, unit="GB/s",
            frac=lb_bytes / lb_ms / 1e6 / hbm, traffic=_ncu_traffic("wave_lb_kernel"), kernel="wave_lb_kernel",
            note="algorithmic bytes = u8 envelope-code and sample-code blocks the LB_Keogh2/LB_Keogh "
                 "cascade reads before abandoning (device counter, per 1000-query batch); traffic = "
                 "ncu dram bytes of the same launches (profiles/r01/traffic_cfg1.json)")
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
    return res


def e2e_run(args, ds, X, Q, params, lo, nq):
    """Public API with HOST buffers: build_index from pinned host memory and
    query_index_batch from host numpy; H2D/D2H inside the timed region."""
    import numpy as np
    import torch

    import paper_1610_07328_b200 as ssh

    Xh = X.cpu().pin_memory()
    dsh = ssh.Dataset.__new__(ssh.Dataset)
    dsh.values, dsh.source = Xh, "pinned host"
    N, m = Xh.shape
    reps = 2
    tb, tq = [], []
    for i in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        index = ssh.build_index(dsh, params, id_base=lo)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        res = ssh.query_index_batch(index, Q, K_TOP)
        t2 = time.perf_counter()
        if i:
            tb.append(t1 - t0)
            tq.append(t2 - t1)
        del index, res
    h2d = N * m * 4 + Q.shape[0] * m * 4
    d2h = nq * K_TOP * 16 + nq * (4 + 8 + 40 + 4) + params.d * 8
    return {"value": N / statistics.median(tb), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "queries_per_s": nq / statistics.median(tq),
            "note": "build_index(Dataset(pinned host f32)) + query_index_batch(host numpy) "
                    "through the public API; wall clock with device sync"}


# ----------------------------------------------------------- reference arm

def cpu_baseline(X, Q, p, args, with_queries=False):
    """The oracle port (oracle/ssh_oracle.c, OpenMP over all host threads) on a
    bounded sample of the same workload."""
    import numpy as np

    from oracle import oracle as orc

    th = ncores()
    Xh = X.cpu().numpy() if hasattr(X, "cpu") else np.asarray(X)
    n_build = min(Xh.shape[0], args.cpu_build_sample)
    orc.get_tables(p["n"], p["d"] * p["K"], p["seed"], Xh.shape[1])
    t0 = time.perf_counter()
    sig = orc.signatures(Xh[:n_build], p["W"], p["delta"], p["n"], p["d"], p["K"], p["seed"], threads=th)
    csr = orc.tables_from_signatures(sig)
    tb = time.perf_counter() - t0
    out = {"value": n_build / tb, "unit": UNIT, "cores": th, "kind": "port",
           "sample": f"build_index (K=4 signatures + stable-argsort tables) over the first {n_build} "
                     f"series of the workload"}
    if not with_queries:
        return out
    n_idx = min(Xh.shape[0], args.cpu_query_index)
    idx = orc.build_index(Xh[:n_idx], p["W"], p["delta"], p["n"], p["d"], p["K"], p["seed"], p["band"],
                          threads=th)
    nq = min(Q.shape[0], args.cpu_queries)
    t0 = time.perf_counter()
    res = orc.query_batch(idx, Q[:nq], K_TOP, threads=th)
    tq = time.perf_counter() - t0
    out["queries_per_s"] = nq / tq
    out["query_sample"] = (f"{nq} queries against an oracle index over {n_idx} series "
                           f"(mean |R|={float(res['n_cand'].mean()):.0f}); full-N CPU query time not measured")
    return out


def run_reference(args):
    """--impl reference: the CPU oracle port of the reference path on host cores."""
    import numpy as np

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1610_07328_b200 import datagen

    dev = "cuda" if _cuda_ok() else "cpu"
    c = datagen.CONFIGS[args.cfg]
    N = min(args.n or c["N"], max(args.cpu_build_sample, args.cpu_query_index))
    X, Q, src, p = datagen.workload(args.cfg, lo=0, hi=N, device=dev, nq=args.cpu_queries,
                                    n_override=(args.n or c["N"]))
    Xh = X.cpu().numpy()
    vals = []
    qps = []
    base = None
    for i in range(args.warmup + args.steps):
        base = cpu_baseline(Xh, Q, p, args, with_queries=(i >= args.warmup))
        if i >= args.warmup:
            vals.append(base["value"])
            qps.append(base.get("queries_per_s"))
    v = statistics.median(vals)
    out = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic (BASELINE.json configs[%d] recipe, seeded)" % args.cfg,
        "config": {"workload": f"configs[{args.cfg}] (bounded CPU sample, see cpu_baseline.sample)",
                   "N": args.n or c["N"], "m": c["m"], "K": 4, "L": 20, "k": K_TOP},
        "queries_per_s": statistics.median([q for q in qps if q is not None]) if any(qps) else None,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": base["cores"], "kind": "port",
                         "sample": base["sample"], "query_sample": base.get("query_sample")},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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
    ap.add_argument("--n", type=int, default=None, help="override N per GPU (dev only)")
    ap.add_argument("--nq", type=int, default=None, help="override query count (dev only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-build-sample", type=int, default=20000)
    ap.add_argument("--cpu-query-index", type=int, default=100000)
    ap.add_argument("--cpu-queries", type=int, default=16)
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

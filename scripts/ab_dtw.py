"""Dev A/B: per-phase query times (ssh_ctx_profile) and a digest of the
results for one index + query batch, so variant libraries (SSH_LIB_PATH) and
env switches can be compared on identical inputs.

python scripts/ab_dtw.py --cfg 3 --n 1000000 --nq 200 [--reps 2]
"""
import argparse
import ctypes
import hashlib
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1610_07328_b200 as ssh  # noqa: E402
from paper_1610_07328_b200 import _native as nat  # noqa: E402
from paper_1610_07328_b200 import datagen  # noqa: E402
from paper_1610_07328_b200.index import query_batch_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--nq", type=int, default=200)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--tag", default=os.environ.get("SSH_LIB_PATH", "default"))
a = ap.parse_args()
X, Q, src, p = datagen.workload(a.cfg, device="cuda", nq=a.nq, n_override=a.n)
params = ssh.SshParams(**p)
idx = ssh.build_index(ssh.Dataset(X), params)
Qd = torch.from_numpy(Q).cuda()
ctx = idx.context()
lib = nat.lib()
out = query_batch_device(idx, Qd, 10)  # warm-up
torch.cuda.synchronize()
best = None
for _ in range(a.reps):
    nat.check(lib.ssh_ctx_set_profiling(ctx.handle, 1))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = query_batch_device(idx, Qd, 10)
    e1.record()
    torch.cuda.synchronize()
    prof = (ctypes.c_double * 24)()
    nat.check(lib.ssh_ctx_profile(ctx.handle, prof, 24))
    nat.check(lib.ssh_ctx_set_profiling(ctx.handle, 0))
    r = dict(total_ms=e0.elapsed_time(e1), phases_ms=[round(v, 3) for v in prof[:6]], cells=prof[6],
             cells_exec=prof[20], dtw_T_cells_s=prof[6] / prof[4] / 1e9 if prof[4] else None)
    if best is None or r["phases_ms"][4] < best["phases_ms"][4]:
        best = r
    # un-profiled timing
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
out = query_batch_device(idx, Qd, 10)
e1.record()
torch.cuda.synchronize()
best["plain_ms"] = e0.elapsed_time(e1)
h = hashlib.sha256()
for t in out[:4]:  # ids, d2, n_out, |R| (counters depend on the schedule)
    h.update(t.cpu().numpy().tobytes())
best["digest"] = h.hexdigest()[:16]
best["tag"] = a.tag
best["cfg"] = a.cfg
print(json.dumps(best), flush=True)

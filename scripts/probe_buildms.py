"""Dev probe: device time of build_index at a config (CUDA events, min/median of reps)."""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1610_07328_b200 as ssh  # noqa: E402
from paper_1610_07328_b200 import datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=1)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=8)
ap.add_argument("--tag", default="")
a = ap.parse_args()
X, Q, src, p = datagen.workload(a.cfg, device="cuda", nq=8, n_override=a.n)
params = ssh.SshParams(**p)
ds = ssh.Dataset(X)
ts = []
for i in range(a.reps + 2):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    idx = ssh.build_index(ds, params)
    e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
    del idx
print(f"{a.tag} cfg{a.cfg} N={X.shape[0]} build ms: min {min(ts):.3f} median {statistics.median(ts):.3f}", flush=True)

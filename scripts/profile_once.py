"""One index build + one query batch at a config's shape (for ncu captures).
The build + query are bracketed by cudaProfilerStart/Stop, so
`ncu --profile-from-start off` skips the data generation.

python scripts/profile_once.py [--cfg 1] [--nq 200] [--n N]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1610_07328_b200 as ssh  # noqa: E402
from paper_1610_07328_b200 import datagen  # noqa: E402
from paper_1610_07328_b200.index import query_batch_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=1)
ap.add_argument("--nq", type=int, default=200)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
X, Q, src, p = datagen.workload(a.cfg, device="cuda", nq=a.nq, n_override=a.n)
params = ssh.SshParams(**p)
ds = ssh.Dataset(X)
Qd = torch.from_numpy(Q).cuda()
ssh.index.get_context(0, params, X.shape[1])  # context setup (CWS tables) outside the range
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.reps):
    idx = ssh.build_index(ds, params)
    out = query_batch_device(idx, Qd, 10)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", float(out[3].double().mean()), out[4].double().mean(0).tolist())

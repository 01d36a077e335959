"""Dev probe: host/device timing of build_index in isolation and after a query batch."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1610_07328_b200 as ssh  # noqa: E402
from paper_1610_07328_b200 import datagen  # noqa: E402
from paper_1610_07328_b200.index import query_batch_device  # noqa: E402

X, Q, src, p = datagen.workload(1, device="cuda", nq=200)
params = ssh.SshParams(**p)
ds = ssh.Dataset(X)
Qd = torch.from_numpy(Q).cuda()


def tb(tag):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    idx = ssh.build_index(ds, params)
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{tag}: host {1e3 * (t1 - t0):.1f} ms, host+sync {1e3 * (t2 - t0):.1f} ms, "
          f"events {a.elapsed_time(b):.1f} ms", flush=True)
    return idx


for i in range(3):
    idx = tb(f"build {i}")
for i in range(2):
    t0 = time.perf_counter()
    out = query_batch_device(idx, Qd, 10)
    torch.cuda.synchronize()
    print(f"query: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    idx2 = tb(f"build after query {i}")
    del out
    idx = idx2

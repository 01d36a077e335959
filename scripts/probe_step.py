"""Dev probe: phase events inside the bench step loop (build sub-phases + query)."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1610_07328_b200 as ssh  # noqa: E402
from paper_1610_07328_b200 import _native as nat  # noqa: E402
from paper_1610_07328_b200 import datagen  # noqa: E402
from paper_1610_07328_b200.index import _stream_ptr, compute_signatures_device, get_context, query_batch_device  # noqa: E402

X, Q, src, p = datagen.workload(1, device="cuda", nq=1000)
params = ssh.SshParams(**p)
ds = ssh.Dataset(X)
Qd = torch.from_numpy(Q).cuda()
ctx = get_context(0, params, 512)
L = nat.lib()
N = X.shape[0]
for step in range(6):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    t0 = time.perf_counter()
    ev[0].record()
    sig = compute_signatures_device(ctx, X)
    ev[1].record()
    h = ctypes.c_void_p()
    nat.check(L.ssh_index_build(ctx.handle, nat.ptr(sig), N, 0, ctypes.byref(h), _stream_ptr(0)))
    ev[2].record()
    nat.check(L.ssh_index_summarize(ctx.handle, h, nat.ptr(X), 512, _stream_ptr(0)))
    ev[3].record()
    t1 = time.perf_counter()
    idx = ssh.build_index(ds, params)
    ev[4].record()
    out = query_batch_device(idx, Qd, 10)
    ev[5].record()
    torch.cuda.synchronize()
    L.ssh_index_destroy(h)
    print(f"step {step}: sig {ev[0].elapsed_time(ev[1]):.2f} tables {ev[1].elapsed_time(ev[2]):.2f} "
          f"paa {ev[2].elapsed_time(ev[3]):.2f} | build_index {ev[3].elapsed_time(ev[4]):.2f} "
          f"query {ev[4].elapsed_time(ev[5]):.2f} ms; host(build parts) {1e3 * (t1 - t0):.2f} ms", flush=True)

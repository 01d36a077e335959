"""Dev: time ssh_signatures at N=1M for alternative builds of libsshgpu (A/B)."""
import ctypes, shutil, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1610_07328_b200 import _native as nat, datagen
import paper_1610_07328_b200 as ssh
from paper_1610_07328_b200.index import get_context, _stream_ptr
if len(sys.argv) > 1:
    nat.LIB_PATH = Path(sys.argv[1]).resolve()
X, Q, src, p = datagen.workload(1, device="cuda", nq=1)
params = ssh.SshParams(**p)
ctx = get_context(0, params, 512)
L = nat.lib()
N = X.shape[0]
sig = torch.empty((N, 20), dtype=torch.int64, device="cuda")
ts = []
for _ in range(6):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); nat.check(L.ssh_signatures(ctx.handle, nat.ptr(X), N, 512, nat.ptr(sig), None, _stream_ptr(0))); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(sys.argv[1:] or "default", "signatures ms", sorted(ts)[:3])

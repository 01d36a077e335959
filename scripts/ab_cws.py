"""Dev: time ssh_signatures at configs[1] size and print a SHA-256 of the
signatures (run once with SSH_CWS_FAST=0 and once without to A/B the
order-free CWS path against the sorted-set kernel)."""
import hashlib, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1610_07328_b200 import _native as nat, datagen
import paper_1610_07328_b200 as ssh
from paper_1610_07328_b200.index import get_context, _stream_ptr
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nmax = int(sys.argv[2]) if len(sys.argv) > 2 else None
X, Q, src, p = datagen.workload(cfg, device="cuda", nq=1, n_override=nmax)
params = ssh.SshParams(**p)
m = X.shape[1]
ctx = get_context(0, params, m)
L = nat.lib()
N = X.shape[0]
sig = torch.empty((N, params.d), dtype=torch.int64, device="cuda")
ts = []
for _ in range(6):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); nat.check(L.ssh_signatures(ctx.handle, nat.ptr(X), N, m, nat.ptr(sig), None, _stream_ptr(0))); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
h = hashlib.sha256(sig.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"cfg{cfg} N={N} SSH_CWS_FAST={os.environ.get('SSH_CWS_FAST', '1')} signatures ms {sorted(ts)[:3]} sha {h}")

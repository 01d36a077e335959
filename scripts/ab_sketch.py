"""Dev: time ssh_sketch at a config size; prints ms, GB/s and a SHA-256 of the bits
(A/B the TMA-staged stream kernel against the polyphase pair kernel with
SSH_SKETCH_STREAM=0)."""
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
words = L.ssh_sketch_words(ctx.handle)
bits = torch.empty((N, words), dtype=torch.int64, device="cuda")
stats = torch.zeros(2, dtype=torch.int64, device="cuda")
ts = []
for _ in range(8):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); nat.check(L.ssh_sketch(ctx.handle, nat.ptr(X), N, m, nat.ptr(bits), nat.ptr(stats), _stream_ptr(0))); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
h = hashlib.sha256(bits.cpu().numpy().tobytes()).hexdigest()[:16]
gbs = N * (4 * m + 8 * words) / (sorted(ts)[0] * 1e-3) / 1e9
print(f"cfg{cfg} N={N} STREAM={os.environ.get('SSH_SKETCH_STREAM', '1')} sketch ms {sorted(ts)[:3]} {gbs:.0f} GB/s sha {h} rechecks {stats.tolist()}")

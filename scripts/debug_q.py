"""Dev: compare device vs oracle top-k for selected queries of a full-size config."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1610_07328_b200 as ssh
from paper_1610_07328_b200 import datagen
from oracle import oracle as O

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=1)
ap.add_argument("--nq", type=int, default=24)
ap.add_argument("--qs", default="16")
a = ap.parse_args()
X, Q, src, p = datagen.workload(a.cfg, device="cuda", nq=a.nq)
idx = ssh.build_index(ssh.Dataset(X), ssh.SshParams(**p))
qs = [int(v) for v in a.qs.split(",")]
res = ssh.query_index_batch(idx, Q[qs], 10)
Xh = X.cpu().numpy()
sig = idx.signatures
ocsr = O.tables_from_signatures(sig)
oidx = O.OracleIndex(Xh, 80, 3, 15, 20, 4, 0, p["band"], O.make_filter(80, 0), sig, ocsr)
ores = O.query_batch(oidx, Q[qs], 10, threads=16)
r_ = O.radius(p["band"], Xh.shape[1])
for t, qi in enumerate(qs):
    dev = res[t].ids
    orc = ores["ids"][t][: int(ores["n"][t])].tolist()
    print("query", qi, "match" if dev == orc else "DIFF", "cand", res[t].stats.candidates, int(ores["n_cand"][t]))
    if dev != orc:
        for i in sorted(set(dev) ^ set(orc)):
            print("  id", i, "in dev" if i in dev else "in oracle", "d2", O.dtw_sq(Xh[i], Q[qi], r_))
        print("  dev d", res[t].distances)
        print("  orc d", np.sqrt(ores["d2"][t][: int(ores["n"][t])]).tolist())

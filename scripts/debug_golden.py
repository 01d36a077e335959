"""Dev: run the rw512 golden query case once (for sanitizer / bisect runs)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests" / "golden")]
import json  # noqa: E402

import paper_1610_07328_b200 as ssh  # noqa: E402
from fixture_data import case_data  # noqa: E402

g = json.loads((ROOT / "tests/golden/golden.json").read_text())
X, Q, _, band = case_data("rw512")
idx = ssh.build_index(ssh.Dataset(X), ssh.SshParams(W=80, delta=3, n=15, d=20, seed=0, band=band, K=1))
res = ssh.query_index_batch(idx, Q, 10)
bad = [i for i, (r, c) in enumerate(zip(res, g["cases"]["rw512"]["queries_k1"])) if r.ids != c["ids"]]
print("mismatched queries:", bad)

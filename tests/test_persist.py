"""Index / dataset persistence on the CPU: file bytes
pinned to the reference's save_index / save_dataset (golden SHA-256 from
tests/golden/make_golden.py), parsing by the library's host routine, and the
reference's load-time error behaviour.  The GPU round trip is in
test_gpu_parity.py."""

import hashlib
import struct

import numpy as np
import pytest

from fixture_data import case_data
from oracle import oracle as O


def _sha(b):
    return hashlib.sha256(b).hexdigest()


def _golden_index_files(tmp_path):
    """Write the golden K=1 index (rw512[:200]) with this package's writer from
    oracle tables; returns the index path."""
    import paper_1610_07328_b200 as ssh
    from paper_1610_07328_b200.persist import index_file_bytes

    X, _, _, band = case_data("rw512")
    X = X[:200].astype(np.float64)
    ds = ssh.Dataset(X)
    params = ssh.SshParams(W=80, delta=3, n=15, d=20, seed=0, band=band, K=1)
    p = tmp_path / "idx.sshi"
    ssh.save_dataset(ds, tmp_path / "idx.sshi.sshd")
    sig = O.signatures(X, 80, 3, 15, 20, 1, 0)
    csr = O.tables_from_signatures(sig)
    w = O.make_filter(80, 0)
    p.write_bytes(index_file_bytes(params, True, 0, w, "idx.sshi.sshd",
                                   ssh.file_checksum(tmp_path / "idx.sshi.sshd"), csr))
    return p, sig, X


def test_dataset_formats_match_reference(golden, tmp_path):
    import paper_1610_07328_b200 as ssh

    X, _, _, _ = case_data("rw512")
    g = golden["persist"]
    ssh.save_dataset(ssh.Dataset(X[:200].astype(np.float64)), tmp_path / "a.sshd")
    assert _sha((tmp_path / "a.sshd").read_bytes()) == g["sidecar_sha256"]
    ssh.save_dataset(ssh.Dataset(X[:5].astype(np.float64)), tmp_path / "b.csv", fmt="csv")
    assert _sha((tmp_path / "b.csv").read_bytes()) == g["csv5_sha256"]
    back = ssh.load_dataset(tmp_path / "a.sshd")
    assert np.array_equal(back.values, X[:200].astype(np.float64))
    # like the reference's, the CSV round trip holds for plain float reprs
    (tmp_path / "c.csv").write_text("\n".join(",".join(repr(float(v)) for v in r) for r in X[:5]) + "\n")
    back = ssh.load_dataset(tmp_path / "c.csv", fmt="csv")
    assert np.array_equal(back.values, X[:5].astype(np.float64))


def test_dataset_load_errors(tmp_path):
    import paper_1610_07328_b200 as ssh

    (tmp_path / "s").write_bytes(b"SSHD")
    with pytest.raises(ssh.DataFormatError, match="file too short"):
        ssh.load_dataset(tmp_path / "s")
    (tmp_path / "m").write_bytes(b"XXXX" + struct.pack("<IQQ", 1, 1, 1) + b"\0" * 8)
    with pytest.raises(ssh.DataFormatError, match="bad magic"):
        ssh.load_dataset(tmp_path / "m")
    (tmp_path / "p").write_bytes(b"SSHD" + struct.pack("<IQQ", 1, 2, 3) + b"\0" * 8)
    with pytest.raises(ssh.DataFormatError, match="payload size mismatch"):
        ssh.load_dataset(tmp_path / "p")
    (tmp_path / "c.csv").write_text("1,2\n3\n")
    with pytest.raises(ssh.DataFormatError, match="ragged row"):
        ssh.load_dataset(tmp_path / "c.csv", fmt="csv")
    with pytest.raises(ssh.DataFormatError, match="no such file"):
        ssh.load_dataset(tmp_path / "none")


def test_index_bytes_match_reference(golden, tmp_path):
    p, _, _ = _golden_index_files(tmp_path)
    g = golden["persist"]
    data = p.read_bytes()
    assert len(data) == g["index_bytes"]
    assert _sha(data) == g["index_sha256"]


def test_read_index_file_recovers_signatures(tmp_path):
    import paper_1610_07328_b200 as ssh

    p, sig, X = _golden_index_files(tmp_path)
    params, w, fseed, normalized, ds, sig2 = ssh.read_index_file(p)
    assert params.K == 1 and params.W == 80 and params.d == 20 and normalized and fseed == 0
    assert np.array_equal(w, O.make_filter(80, 0))
    assert np.array_equal(ds.values, X)
    assert np.array_equal(sig2, sig)


def test_read_index_file_version2_k(tmp_path):
    import paper_1610_07328_b200 as ssh
    from paper_1610_07328_b200.persist import index_file_bytes

    X, _, _, band = case_data("rw512")
    X = X[:120].astype(np.float64)
    ssh.save_dataset(ssh.Dataset(X), tmp_path / "k.sshi.sshd")
    sig = O.signatures(X, 80, 3, 15, 20, 4, 0)
    params = ssh.SshParams(W=80, delta=3, n=15, d=20, seed=0, band=band, K=4)
    (tmp_path / "k.sshi").write_bytes(index_file_bytes(params, True, 0, O.make_filter(80, 0), "k.sshi.sshd",
                                                       ssh.file_checksum(tmp_path / "k.sshi.sshd"),
                                                       O.tables_from_signatures(sig)))
    got = ssh.read_index_file(tmp_path / "k.sshi")
    assert got[0] == params and np.array_equal(got[5], sig)


def test_read_index_file_errors(tmp_path):
    import paper_1610_07328_b200 as ssh

    p, _, _ = _golden_index_files(tmp_path)
    good = p.read_bytes()
    bad = tmp_path / "bad.sshi"

    def expect(data, pattern):
        bad.write_bytes(data)
        with pytest.raises(ssh.IndexLoadError, match=pattern):
            ssh.read_index_file(bad)

    # the sidecar name inside the file is idx.sshi.sshd, resolved next to the file
    expect(b"NOPE" + good[4:], "bad magic")
    expect(good[:4] + struct.pack("<I", 9) + good[8:], "unsupported index version 9")
    expect(good[:60], "truncated index file")
    expect(good[:-5], "truncated index file")
    expect(good + b"\0" * 8, "8 trailing bytes after tables")
    # first table, first bucket: its first id -> out of range / duplicate of the second
    hdr = good.index(b"idx.sshi.sshd") + len("idx.sshi.sshd") + 32
    first_id = hdr + 8 + 16
    cnt = struct.unpack_from("<Q", good, hdr + 16)[0]
    expect(good[:first_id] + struct.pack("<Q", 10 ** 6) + good[first_id + 8:], "outside \\[0, 200\\)")
    if cnt >= 2:
        second = struct.unpack_from("<Q", good, first_id + 8)[0]
        expect(good[:first_id] + struct.pack("<Q", second) + good[first_id + 8:], "more than once")
    (tmp_path / "idx.sshi.sshd").write_bytes((tmp_path / "idx.sshi.sshd").read_bytes()[:-8] + b"\1" * 8)
    with pytest.raises(ssh.IndexLoadError, match="checksum mismatch"):
        ssh.read_index_file(p)
    (tmp_path / "idx.sshi.sshd").unlink()
    with pytest.raises(ssh.IndexLoadError, match="is missing"):
        ssh.read_index_file(p)
    with pytest.raises(ssh.IndexLoadError, match="no such file"):
        ssh.read_index_file(tmp_path / "absent.sshi")


def test_ranking_metrics_match_reference(golden):
    """precision_at_k / ndcg_at_k (bench.py:63-90) on the golden rankings."""
    import paper_1610_07328_b200 as ssh

    retrieved = [5, 3, 9, 1, 7, 2, 8]
    gold = [3, 5, 1, 4, 9, 6, 0]
    for k, (p, n) in golden["srp"]["metrics"].items():
        assert ssh.precision_at_k(retrieved, gold, int(k)) == p
        assert ssh.ndcg_at_k(retrieved, gold, int(k)) == n
    with pytest.raises(ValueError, match="k must be >= 1"):
        ssh.ndcg_at_k(retrieved, gold, 0)

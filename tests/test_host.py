"""Host-side logic, tables and the C-ABI surface (CPU only, no kernel calls)."""

import ctypes
import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1610_07328_b200 as ssh
from oracle import oracle as O
from paper_1610_07328_b200 import _native, cws, datagen

ROOT = Path(__file__).resolve().parents[1]


def test_cws_tables_equal_oracle_restatement():
    """Product tables (cws.py) == oracle tables (independent restatement of wmh.py:60-72)."""
    r, lnc, beta = cws.cws_variates(15, 80, 0)
    o = O.get_tables(15, 80, 0, 131)
    assert np.array_equal(r, o.r) and np.array_equal(lnc, o.ln_c) and np.array_equal(beta, o.beta)
    assert np.array_equal(cws.ln_counts(643), O.ln_counts(643))


def test_cws_tables_match_reference_keys(golden):
    """Keys computed from the product tables with the oracle evaluator == golden keys."""
    r, lnc, beta = cws.tables(15, 80, 0)
    tabs = O.OracleTables(15, 80, 0, r, lnc, beta, cws.ln_counts(700))
    for cw in golden["cws"]:
        if cw["seed"]:
            continue
        keys = O.cws_keys_tab(np.array(cw["tokens"], dtype=np.uint64), np.array(cw["counts"]), 80, tabs)
        assert keys.tolist() == cw["keys"]


def test_make_filter_matches_reference(golden):
    assert cws.filter_weights(80, 0).tolist() == golden["spec"]["filter80"]
    with pytest.raises(ValueError):
        cws.filter_weights(0, 0)


def test_params_validation_messages():
    with pytest.raises(ssh.ConfigError, match="filter length W must be >= 1"):
        ssh.SshParams(W=0)
    with pytest.raises(ssh.ConfigError, match="step size delta must be >= 1"):
        ssh.SshParams(delta=0)
    with pytest.raises(ssh.ConfigError, match="shingle length n must be in"):
        ssh.SshParams(n=65)
    with pytest.raises(ssh.ConfigError, match="table count d must be >= 1"):
        ssh.SshParams(d=0)
    with pytest.raises(ssh.ConfigError, match="warping band must be in"):
        ssh.SshParams(band=1.5)
    with pytest.raises(ssh.ConfigError, match="concat order K"):
        ssh.SshParams(K=0)
    p = ssh.SshParams(W=80, delta=3, n=15)
    with pytest.raises(ssh.ConfigError, match=r"series length t=50 violates t >= W"):
        p.validate_for_length(50)
    with pytest.raises(ssh.ConfigError, match=r"violates >= n"):
        p.validate_for_length(100)
    p.validate_for_length(512)
    with pytest.raises(ssh.ConfigError, match="device limit"):
        ssh.SshParams(W=8, delta=1, n=24).validate_for_length(512)


def test_radius_bankers_rounding():
    # dtw.py:38-39 uses Python round (half to even)
    assert ssh.WarpingParams(0.05).radius(512) == 26
    assert ssh.WarpingParams(0.05).radius(1024) == 51
    assert ssh.WarpingParams(0.10).radius(2048) == 205
    assert ssh.WarpingParams(0.5).radius(5) == 2  # 2.5 -> 2
    assert ssh.WarpingParams(0.5).radius(7) == 4  # 3.5 -> 4


def test_num_sketch_bits():
    for m, W, d in [(512, 80, 3), (1024, 80, 3), (2048, 80, 3), (4, 2, 2), (80, 80, 3)]:
        assert ssh.num_sketch_bits(m, W, d) == O.num_sketch_bits(m, W, d)
    assert ssh.num_sketch_bits(512, 80, 3) == 145


def test_dataset_validation():
    with pytest.raises(ValueError, match="2-D"):
        ssh.Dataset(np.zeros(5))
    with pytest.raises(ValueError, match="non-finite"):
        ssh.Dataset(np.array([[1.0, np.nan]]))
    d = ssh.Dataset(np.ones((3, 4), dtype=np.float32))
    assert d.n_series == 3 and d.length == 4
    with pytest.raises(IndexError):
        d.series(3)


def test_znorm_matches_reference_semantics():
    v = np.array([[1.0, 2, 3, 4], [5, 5, 5, 5]])
    out = ssh.z_normalize_rows(v.copy())
    assert np.allclose(out[0].mean(), 0) and np.allclose(out[0].std(), 1)
    assert np.all(out[1] == 0)


def test_datagen_deterministic_and_sharded():
    a = datagen.random_walks(0, 300, 128, 11, device="cpu")
    b = datagen.random_walks(100, 250, 128, 11, device="cpu")
    assert np.array_equal(a[100:250].numpy(), b.numpy())
    q1 = datagen.warped_queries(a[:5].numpy(), 3)
    q2 = datagen.warped_queries(a[:5].numpy(), 3)
    assert np.array_equal(q1, q2) and q1.dtype == np.float32
    assert np.allclose(q1.mean(axis=1), 0, atol=1e-5)


def test_ecg_generator_shape():
    sig = datagen.ecg_signal(20_000, seed=4000)
    W = datagen.ecg_windows(sig, 1024, 64, 50)
    assert W.shape == (50, 1024) and np.isfinite(W).all()


def _header_functions():
    text = (ROOT / "include" / "sshgpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ssh_[a-z0-9_]+)\s*\(", text)))


def test_abi_exports_every_header_symbol():
    """libsshgpu.so loads (no GPU needed) and exports every function in include/sshgpu.h."""
    _native.build_native()
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    names = _header_functions()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_native.EXPORTED)
    assert lib.ssh_abi_version() == 1


def test_abi_built_for_sm100a():
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_abi_errors_without_gpu_are_loud():
    """No CUDA device here: context creation must fail with an error, never fall back."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _native.lib()
    h = ctypes.c_void_p()
    rc = lib.ssh_ctx_create(0, ctypes.byref(h))
    assert rc != 0
    assert lib.ssh_last_error()
    with pytest.raises(ssh.SshError):
        ssh.build_index(np.zeros((4, 128), dtype=np.float32), ssh.SshParams(W=8, delta=2, n=4))


def test_product_never_imports_oracle():
    for p in (ROOT / "paper_1610_07328_b200").rglob("*.py"):
        src = p.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", src, flags=re.M), p
        assert "import oracle" not in src and "from oracle" not in src, p


def test_results_from_arrays_match_dataclass_construction():
    """query_index_batch's fast result construction (field dicts, whole-batch
    tolist) yields objects equal to the normally constructed dataclasses, with
    the reference's statuses and sqrt distances (index.py:233-273)."""
    import dataclasses

    from paper_1610_07328_b200.index import QueryResult, QueryStats, SearchStats, _results_from_arrays

    rng = np.random.default_rng(3)
    nq, k, N = 5, 4, 1000
    ids = rng.integers(0, N, size=(nq, k)).astype(np.int64)
    d2 = rng.random((nq, k)) * 10.0
    d2[2, 1:] = -1.0  # entries past n_out are garbage and must not be used
    n_out = np.array([4, 4, 1, 0, 3], dtype=np.int32)
    n_cand = np.array([9, 7, 1, 0, 1000], dtype=np.int64)
    counters = rng.integers(0, 50, size=(nq, 5)).astype(np.int64)
    status = np.array([0, 0, 0, 1, 2], dtype=np.int32)
    got = _results_from_arrays(ids, d2, n_out, n_cand, counters, status, N, 0.5, "w", phase_ms=[10.0, 20.0, 30.0])
    for i, r in enumerate(got):
        # the reference's timing keys (index.py:235,265; cli.py:184-185) in seconds per query
        t = {"hash": 10.0 / 1e3 / nq, "probe": 20.0 / 1e3 / nq, "rerank": 30.0 / 1e3 / nq,
             "batch": 0.5, "per_query": 0.5 / nq}
        if status[i] == 1:
            want = QueryResult([], [], QueryStats(N, 0, SearchStats(0, 0, 0, 0, 0, 0)), t,
                               status="no-candidates", warning="w")
        else:
            c = [int(v) for v in counters[i]]
            st = QueryStats(N, int(n_cand[i]), SearchStats(int(n_cand[i]), *c))
            n = int(n_out[i])
            want = QueryResult([int(v) for v in ids[i, :n]], [float(v) for v in np.sqrt(d2[i, :n])], st, t,
                               status="fallback" if status[i] == 2 else "ok", warning="w")
        assert r == want
        assert type(r.ids[0] if r.ids else 0) is int and all(type(v) is float for v in r.distances)
        with pytest.raises(dataclasses.FrozenInstanceError):
            r.status = "x"
        assert r.stats.cascade.pruned == want.stats.cascade.pruned


def test_make_filter_returns_random_filter(golden):
    """make_filter returns the reference's RandomFilter (sketch.py:36-43)."""
    f = ssh.make_filter(80, 0)
    assert isinstance(f, ssh.RandomFilter) and f.seed == 0 and f.W == 80
    assert f.weights.tolist() == golden["spec"]["filter80"]
    with pytest.raises(ValueError, match="filter length W must be >= 1"):
        ssh.make_filter(0, 0)
    with pytest.raises(ValueError, match="seed must be non-negative"):
        ssh.make_filter(3, -1)


def test_reference_public_names_exported():
    """Every hot-path name of the reference's sshts/__init__.py that this
    drop-in covers is importable from the package."""
    for name in ["Dataset", "TimeSeries", "SshParams", "SshIndex", "QueryResult", "WarpingParams", "SearchStats",
                 "SearchResult", "Envelope", "RandomFilter", "build_index", "query_index", "save_index", "load_index",
                 "make_filter", "num_sketch_bits", "build_envelope", "dtw_distance", "lb_kim", "lb_keogh",
                 "lb_keogh2", "exact_search", "make_dataset", "extract_subsequences", "z_normalize",
                 "z_normalize_dataset", "save_dataset", "load_dataset", "srp_signature", "precision_at_k",
                 "ndcg_at_k", "ConfigError", "SshError", "IndexLoadError", "DataFormatError"]:
        assert hasattr(ssh, name), name


def test_float64_rounding_warning_policy():
    """float64 inputs that float32 cannot hold exactly warn (never silently
    rounded); exactly representable ones do not."""
    import warnings

    from paper_1610_07328_b200.index import Float32RoundingWarning, _warn_f32_rounding

    exact = np.arange(12, dtype=np.float64).reshape(3, 4) / 4.0
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        _warn_f32_rounding(exact, "dataset")
        _warn_f32_rounding(exact.astype(np.float32), "dataset")
    with pytest.warns(Float32RoundingWarning):
        _warn_f32_rounding(exact + 0.1, "dataset")

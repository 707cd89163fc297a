"""Host-side logic that needs no GPU: the C-ABI library loads and exports every
declared symbol, status codes map onto the reference's exception types, the
ER plan / schedules / configs match the reference, and the data-parallel
sharding covers every sample exactly once."""

import json
import re

import numpy as np
import pytest

from conftest import GOLDEN, REPO

import paper_2407_17437_b200 as smb  # noqa: E402
from paper_2407_17437_b200 import _lib  # noqa: E402
from paper_2407_17437_b200.engine import flat_layout, shard_epoch  # noqa: E402


def header_symbols():
    text = (REPO / "include" / "sparsemlp_b200.h").read_text()
    return sorted(set(re.findall(r"SMB_API\s+[\w\s\*]+?\b(smb_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert lib.smb_abi_version() == 1


def test_integration_doc_covers_every_entry_point():
    """INTEGRATION.md maps every C-ABI entry point to the reference interface
    it replaces (or says what it is for)."""
    doc = (REPO / "INTEGRATION.md").read_text()
    missing = [s for s in header_symbols() if s not in doc]
    assert not missing, missing


def test_status_codes_map_to_reference_exceptions():
    lib = _lib.load()
    # argument checks run on the host before any device work
    rc = lib.smb_axpby(7, 1.0, None, 1.0, None, 4, None)
    with pytest.raises(smb.InvalidArgumentError):
        _lib.check(rc)
    rc = lib.smb_spmm(0, None, None, None, -1, 2, None, 2, 2, None, 0, None, 2, None)
    assert rc == _lib.SMB_ERR_INVALID
    assert b"negative" in lib.smb_last_error()
    with pytest.raises(smb.StateError):
        _lib.check(_lib.SMB_ERR_STATE)
    with pytest.raises(smb.DeviceError):
        _lib.check(_lib.SMB_ERR_CUDA)
    assert issubclass(smb.InvalidArgumentError, ValueError)
    assert issubclass(smb.StateError, RuntimeError)


def test_er_plans_match_reference():
    plans = json.loads((GOLDEN / "plans_init.json").read_text())["plans"]
    for p in plans:
        got = smb.er_densities(p["chain"], p["density"])
        assert got.layer_nnz == p["layer_nnz"]
        assert got.layer_densities == p["layer_densities"]


def test_er_published_values():
    # pkg/tests/test_sparsity.py:25-43 / test_acceptance.py:60-85
    plan = smb.er_densities([3072, 1024, 512, 10], 0.01)
    d1, d2, d3 = plan.layer_densities
    assert round(d1, 3) == pytest.approx(0.008, abs=1.001e-3)
    assert round(d2, 3) == pytest.approx(0.018, abs=1.001e-3)
    assert round(d3, 1) == pytest.approx(0.6, abs=1.001e-3)
    assert smb.er_densities([3072, 1024, 512, 10], 0.001).total_nnz + 1546 == 5221
    sat = smb.er_densities([3072, 1024, 512, 10], 0.1)
    assert sat.layer_densities[2] == 1.0 and sat.layer_nnz[2] == 5120
    rng = np.random.default_rng(42)
    for _ in range(100):
        chain = rng.integers(1, 700, size=rng.integers(2, 7)).tolist()
        d = float(rng.uniform(0.001, 1.0))
        pl = smb.er_densities(chain, d)
        assert abs(pl.total_nnz - d * pl.total_size) <= 1.0


def test_er_rejects_bad_arguments():
    with pytest.raises(smb.InvalidArgumentError):
        smb.er_densities([10, 5], 0.0)
    with pytest.raises(smb.InvalidArgumentError):
        smb.er_densities([10], 0.5)
    with pytest.raises(smb.InvalidArgumentError):
        smb.er_densities([10, 0, 3], 0.5)


def test_schedules():
    s = smb.MultiStepSchedule(0.1, (0.5, 0.75), 0.1)
    assert [s(e, 8) for e in range(8)] == [0.1] * 4 + [0.1 * 0.1] * 2 + [0.1 * 0.1 ** 2] * 2
    assert smb.ConstantSchedule(0.3)(5) == 0.3
    with pytest.raises(smb.InvalidArgumentError):
        smb.MultiStepSchedule(0.1, (0.75, 0.5))
    with pytest.raises(smb.InvalidArgumentError):
        smb.lr_at(s, 8, 8)
    with pytest.raises(smb.InvalidArgumentError):
        smb.TrainConfig(epochs=1, batch_size=0, schedule=s)


def test_experiment_config_and_lr_table():
    assert smb.default_learning_rate(0.01) == 0.1
    assert smb.default_learning_rate(0.02) == 0.1
    assert smb.default_learning_rate(0.3) == 0.01
    cfg = smb.ExperimentConfig(density=0.05)
    assert cfg.resolved_lr() == 0.03 and cfg.nesterov and cfg.momentum == 0.9
    with pytest.raises(smb.ConfigurationError):
        smb.ExperimentConfig(density=1.5)
    with pytest.raises(smb.ConfigurationError):
        smb.Sparse(0, 0.5)
    with pytest.raises(smb.InvalidArgumentError):
        smb.Momentum(1.0)
    assert smb.ExperimentConfig(backend="masked").backend == "masked"  # bench.py:95-96
    with pytest.raises(smb.ConfigurationError):
        smb.ExperimentConfig(backend="dense")
    with pytest.raises(smb.ConfigurationError):
        smb.MaskedDense(10, 0.0)


def test_shard_epoch_covers_every_sample_once():
    perm = np.random.default_rng(0).permutation(10_007)
    G, B = 4, 250
    parts = [shard_epoch(perm, G * B, B, r * B) for r in range(G)]
    kb = parts[0][1]
    assert kb == 10_007 // (G * B)
    for k in range(kb):
        cols = np.concatenate([idx[k * B:(k + 1) * B] for idx, _ in parts])
        assert np.array_equal(cols, perm[k * G * B:(k + 1) * G * B])
    with pytest.raises(smb.InvalidArgumentError):
        shard_epoch(perm, 100, 60, 50)


def test_flat_layout():
    layout, total = flat_layout([(4, 10), (3, 12)])
    assert layout == [(0, 10), (14, 26)] and total == 29


def test_large_grid_pattern_sampler_matches_oracle(oracle):
    """Config-5 injection sampler (grids >= 2**31, which the reference
    refuses): exact nnz, sorted distinct columns, deterministic, and the
    oracle's restatement draws the identical pattern from the same stream."""
    from paper_2407_17437_b200.sparsity import sample_pattern_host, sample_pattern_large_host

    n_out, n_in, nnz = 65536, 65536, 40_000
    with pytest.raises(smb.InvalidArgumentError):
        sample_pattern_host(n_out, n_in, nnz, np.random.default_rng(0))
    rp, ci = sample_pattern_large_host(n_out, n_in, nnz, smb.Rng(5).stream("pattern"))
    assert rp[0] == 0 and rp[-1] == nnz and np.all(np.diff(rp) >= 0)
    for i in np.flatnonzero(np.diff(rp))[:2000]:
        row = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(row) > 0) and row[0] >= 0 and row[-1] < n_in
    rp2, ci2 = oracle.sample_pattern_large(n_out, n_in, nnz, oracle.Streams(5)("pattern"))
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2)

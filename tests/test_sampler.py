"""Device pattern sampler (scale mode; north_star "ER sparsity init generated
from a seed on the device"; reference sampler sparsity.py:183-216).

CPU: the Philox4x32-10 generator against the Random123 known-answer vector
(oracle restatement and the library's host-callable draw); the oracle's
restatement of the sampler's specification draws from the reference's
distribution (a uniform size-nnz subset of the grid) -- row occupancies
against the hypergeometric moments, column usage against uniformity, with
the reference's own host sampler (numpy stream) as the yardstick.
GPU: the device sampler equals the oracle restatement bit for bit (sparse
and complement modes, config-4 and config-5 layer sizes), and a model built
with pattern_sampler="device" trains through the fused step.
"""

import ctypes

import numpy as np
import pytest

import paper_2407_17437_b200 as smb
from paper_2407_17437_b200.sparsity import sample_pattern_host

# Random123 philox4x32-10 KAT: counter {0,0,0,0}, key {0,0}
KAT_ZERO = 0xE169C58D6627E8D5  # words 1:0 = 0xe169c58d : 0x6627e8d5


def test_philox_known_answer(oracle):
    assert oracle.lib().orc_philox_u64(0, 0, 0) == KAT_ZERO
    from paper_2407_17437_b200 import _lib

    assert _lib.load().smb_philox_u64(0, 0, 0) == KAT_ZERO
    for i in (1, 2, 12345, 2**40 + 3):
        assert _lib.load().smb_philox_u64(9, 5, i) == oracle.lib().orc_philox_u64(9, 5, i)


def _stats(rp, ci, m, k):
    counts = np.diff(rp)
    cols = np.bincount(ci, minlength=k)
    return counts, cols


@pytest.mark.parametrize("m,k,nnz", [(64, 80, 500), (40, 50, 1500)])  # sparse / complement
def test_spec_draws_the_reference_distribution(oracle, m, k, nnz):
    G = m * k
    rows_dev, cols_dev, rows_ref = [], [], []
    for seed in range(60):
        rp, ci = oracle.sample_pattern_device_spec(m, k, nnz, seed)
        assert rp[-1] == nnz and len(ci) == nnz
        pos = np.repeat(np.arange(m), np.diff(rp)) * k + ci
        assert np.all(np.diff(pos) > 0)  # distinct, CSR-sorted
        c, col = _stats(rp, ci, m, k)
        rows_dev.append(c)
        cols_dev.append(col)
        rrp, _ = sample_pattern_host(m, k, nnz, np.random.default_rng(seed))
        rows_ref.append(np.diff(rrp))
    rows_dev, rows_ref = np.concatenate(rows_dev), np.concatenate(rows_ref)
    # hypergeometric row occupancy (nnz draws from G cells, k of them in the
    # row): mean nnz/m, variance nnz (1/m) (1 - 1/m) (G - nnz) / (G - 1)
    var = nnz * (1 / m) * (1 - 1 / m) * (G - nnz) / (G - 1)
    for r in (rows_dev, rows_ref):
        assert abs(r.mean() - nnz / m) < 1e-9
        assert abs(r.var() - var) < 0.15 * var
    # every column equally likely: chi-square over the pooled column counts
    col = np.sum(cols_dev, axis=0)
    exp = col.sum() / k
    chi2 = float(np.sum((col - exp) ** 2 / exp))
    assert chi2 < k + 6 * np.sqrt(2 * k)


@pytest.mark.gpu
@pytest.mark.parametrize("m,k,nnz,seed,sid", [
    (1024, 3072, 24461, 0, 0),        # config-2 layer 0
    (512, 1024, 499759, 3, 1),        # config-2 d=0.5 layer 1 (complement mode)
    (8192, 8192, 562878, 1, 2),       # config-4 hidden layer
    (65536, 65536, 2521658, 0, 1),    # config-5 hidden layer (2^32 grid)
    (10, 7, 70, 5, 0),                # full grid
    (100, 100, 0, 5, 0),              # empty
])
def test_device_sampler_matches_spec(oracle, m, k, nnz, seed, sid):
    pat = smb.sample_pattern_device(m, k, nnz, seed, stream_id=sid)
    rp, ci = pat.host_arrays()
    erp, eci = oracle.sample_pattern_device_spec(m, k, nnz, seed, sid)
    assert np.array_equal(rp, erp) and np.array_equal(ci, eci)


@pytest.mark.gpu
def test_device_sampled_model_trains():
    import torch

    cfg = smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=0.01, seed=4,
                               batch_size=128)
    model, plan = smb.build_model(cfg, pattern_sampler="device")
    again, _ = smb.build_model(cfg, pattern_sampler="device")
    sparse = [l for l in model.layers if isinstance(l, smb.SparseLinearLayer)]
    assert [l.weights.nnz for l in sparse] == plan.layer_nnz
    for a, b in zip(sparse, [l for l in again.layers if isinstance(l, smb.SparseLinearLayer)]):
        assert np.array_equal(a.weights.pattern.host_arrays()[1], b.weights.pattern.host_arrays()[1])
    data = smb.synthetic_dataset(seed=1, n_samples=512, features=3072)
    st = smb.FusedTrainStep(model, 128)
    st.attach_dataset(smb.DeviceDataset(data))
    st.set_epoch(np.arange(512))
    losses = []
    for _ in range(4):
        st.step(0.05)
        losses.append(st.loss_value())
    torch.cuda.synchronize()
    assert all(np.isfinite(losses))

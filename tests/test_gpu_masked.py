"""Masked-dense baseline on the GPU: MaskedDense
layers (train.py:78-91, 159-170) whose DenseLinearLayer runs cuBLAS FP32
(TF32 off) and the masked update kernel (nn.py:201-264).

* initial dense weights and masks bit-exact with the oracle's restatement
  (same pattern / init draws as the sparse backend);
* smb_masked_optimizer_step bit-exact with the numpy sequence
  (grad*mask; velocity *= mask; _step_vector; weights *= mask);
* the fused step equals the layer-by-layer API; off-pattern weights stay
  exact zeros;
* the run behind the reference's recorded masked fingerprint
  (pkg/test_output.txt:26, cb8714b95a57...) within 1e-4 of the oracle, which
  reproduces that fingerprint bit for bit on the CPU.
"""

import numpy as np
import pytest
import torch

from conftest import bits_equal, rel_err

pytestmark = pytest.mark.gpu

import paper_2407_17437_b200 as smb  # noqa: E402
from paper_2407_17437_b200 import _lib  # noqa: E402
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr  # noqa: E402


def host(t):
    return t.detach().cpu().numpy()


def params_host(model):
    return [(n, host(t).reshape(-1)) for n, t in model.parameters()]


def max_rel(model, ref):
    return max(rel_err(a, b.reshape(-1))
               for (_, a), (_, b) in zip(params_host(model), ref.parameters()))


def masked_cfg(**kw):
    base = dict(layer_dims=[3072, 1024, 512, 10], density=0.01, seed=3, backend="masked")
    base.update(kw)
    return smb.ExperimentConfig(**base)


def test_masked_initial_weights_bit_exact(oracle):
    model, _ = smb.build_model(masked_cfg())
    ref = oracle.OracleMLP.build([3072, 1024, 512, 10], 0.01, seed=3, backend="masked")
    for (n1, a), (n2, b) in zip(params_host(model), ref.parameters()):
        assert n1 == n2
        assert bits_equal(a, b.reshape(-1)), n1
    dense = [l for l in model.layers if isinstance(l, smb.DenseLinearLayer)]
    masks = [l.mask for l in ref.layers if l.mask is not None]
    assert len(masks) == 3  # the 10x512 layer (ER density 0.609) is masked too
    for lay, mk in zip(dense, masks):
        assert bits_equal(host(lay.mask).reshape(-1), mk)
    # the sparse backend draws the same values: scattering them gives the same weights
    sp, _ = smb.build_model(masked_cfg(backend="sparse"))
    lay_s = [l for l in sp.layers if isinstance(l, smb.SparseLinearLayer)][0]
    assert bits_equal(host(smb.csr_to_dense(lay_s.weights)).reshape(-1),
                      host(dense[0].weights).reshape(-1))


@pytest.mark.parametrize("kind", [_lib.SMB_OPT_GD, _lib.SMB_OPT_MOMENTUM, _lib.SMB_OPT_NESTEROV])
@pytest.mark.parametrize("count", [4096, 1001])  # vector and scalar kernels
def test_masked_optimizer_step_bitwise(kind, count):
    rng = np.random.default_rng(count + kind)
    w = rng.standard_normal(count).astype(np.float32)
    v = rng.standard_normal(count).astype(np.float32)
    g = rng.standard_normal(count).astype(np.float32)
    mk = (rng.random(count) < 0.3).astype(np.float32)
    mu, eta = 0.9, 0.05
    tw, tv, tg, tm = (torch.from_numpy(a.copy()).cuda() for a in (w, v, g, mk))
    _lib.call("smb_masked_optimizer_step", _lib.SMB_F32, ptr(tw), ptr(tv), ptr(tg), ptr(tm),
              count, kind, mu, eta, stream_ptr())
    # numpy reference sequence (nn.py:255-263 with _step_vector nn.py:118-131)
    T = np.float32
    g = g * mk
    if kind != _lib.SMB_OPT_GD:
        v *= mk
        v *= T(mu)
        v += g
        if kind == _lib.SMB_OPT_NESTEROV:
            w += T(-eta * mu) * v
            w += T(-eta) * g
        else:
            w += T(-eta) * v
    else:
        w += T(-eta) * g
    w *= mk
    assert bits_equal(host(tw), w)
    if kind != _lib.SMB_OPT_GD:
        assert bits_equal(host(tv), v)


@pytest.mark.parametrize("B", [100, 128])
def test_masked_fused_step_equals_layer_api(B):
    chain, steps, eta = [3072, 1024, 512, 10], 3, 0.05
    data = smb.synthetic_dataset(seed=7, n_samples=B * steps, features=chain[0])
    cfg = masked_cfg(seed=5, batch_size=B, lr=eta)
    m_fused, _ = smb.build_model(cfg)
    m_layer, _ = smb.build_model(cfg)
    step = smb.FusedTrainStep(m_fused, B)
    step.attach_dataset(smb.DeviceDataset(data))
    perm = np.random.default_rng(1).permutation(B * steps)
    step.set_epoch(perm)
    loss = smb.SoftmaxCrossEntropyLoss()
    for k in range(steps):
        step.step(eta)
        b = perm[k * B:(k + 1) * B]
        xb = torch.from_numpy(np.ascontiguousarray(data.Xtrain[:, b])).cuda()
        tb = torch.from_numpy(np.ascontiguousarray(data.Ttrain[:, b])).cuda()
        y = m_layer.feedforward(xb)
        m_layer.backpropagate(y, loss.gradient_scaled(y, tb, B))
        m_layer.optimize(eta)
    torch.cuda.synchronize()
    for (n1, a), (n2, b) in zip(params_host(m_fused), params_host(m_layer)):
        assert n1 == n2
        assert rel_err(a, b) <= 1e-6, n1
    for lay in m_fused.layers:
        if isinstance(lay, smb.DenseLinearLayer) and lay.mask is not None:
            off = host(lay.weights)[host(lay.mask) == 0]
            assert np.all(off == 0)


def test_masked_reference_fingerprint_run(oracle):
    """The recorded masked run (seed 3, 2 epochs of B=100, lr 0.1 multistep,
    synthetic blobs) through sgd_train on the masked backend."""
    xtr, ttr, _, _ = oracle.synthetic_blobs(10, 3072, 50, 1.0, 3, 5)
    ref = oracle.OracleMLP.build([3072, 1024, 512, 10], 0.01, seed=3, backend="masked")
    ref.train(xtr, ttr, 2, 100, oracle.multistep(0.1))
    assert ref.fingerprint().startswith("cb8714b95a57")
    cfg = masked_cfg(epochs=2, batch_size=100, eval_metrics=False)
    model, _ = smb.build_model(cfg)
    smb.sgd_train(model, smb.Dataset(xtr, ttr),
                  smb.TrainConfig(epochs=2, batch_size=100, schedule=cfg.schedule(),
                                  eval_metrics=False))
    assert max_rel(model, ref) <= 1e-4

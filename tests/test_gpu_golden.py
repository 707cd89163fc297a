"""The CUDA path against the reference's own outputs (tests/golden/): kernels
bit-exact, optimizer trajectories bit-exact, initial models bit-exact (hashes
of patterns and Xavier values), and the 12-step reference training trace
within the north_star tolerance (softmax exp differs in the last ulp from
numpy's float32 exp, so training is tolerance-exact, not bit-exact)."""

import hashlib
import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN, bits_equal, rel_err

pytestmark = pytest.mark.gpu

import paper_2407_17437_b200 as smb  # noqa: E402

K = np.load(GOLDEN / "kernels.npz")


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("c", range(int(K["ncases"][0])))
def test_kernels_bit_exact_vs_reference(c):
    p = f"c{c:03d}_"
    m, k, n = (int(v) for v in K[p + "shape"])
    s = smb.CsrMatrix(m, k, K[p + "row_ptr"], K[p + "col_idx"], K[p + "values"])
    assert bits_equal(smb.spmm(s, K[p + "x"]), K[p + "spmm"])
    assert bits_equal(smb.spmm_transposed(s, K[p + "d"]), K[p + "spmm_t"])
    assert bits_equal(host(smb.sddmm(s.pattern, K[p + "a"], K[p + "b"]).values), K[p + "sddmm"])
    alpha, beta = K[p + "ab"]
    smb.sparse_combine(alpha, s, beta, s.pattern.with_values(K[p + "t"]))
    assert bits_equal(host(s.values), K[p + "combine"])


def test_empty_pattern():
    s = smb.SparsityPattern(4, 3, np.zeros(5, np.int32), np.zeros(0, np.int32)).zeros()
    x = np.ones((3, 6), np.float32)
    assert bits_equal(smb.spmm(s, x), np.zeros((4, 6), np.float32))


def test_optimizer_trajectories_bit_exact():
    O = np.load(GOLDEN / "optimizer.npz")
    pat = smb.SparsityPattern(6, 7, O["row_ptr"], O["col_idx"])
    for name, opt in (("gd", smb.GradientDescent()), ("mom", smb.Momentum(0.9)),
                      ("nesterov", smb.Momentum(0.9, nesterov=True))):
        layer = smb.SparseLinearLayer(pat, O["values0"], np.zeros(6, np.float32), opt)
        for s in range(10):
            layer.grad.values.copy_(torch.from_numpy(O["grads"][s]).cuda())
            layer.grad_bias = torch.from_numpy(O["gbias"][s].copy()).cuda()
            layer.optimize(0.05)
            assert bits_equal(host(layer.weights.values), O[name + "_values"][s]), (name, s)
            assert bits_equal(host(layer.bias), O[name + "_bias"][s]), (name, s)


def test_initial_models_bit_exact_vs_reference():
    init = json.loads((GOLDEN / "plans_init.json").read_text())["init"]
    for rec in init:
        model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=rec["chain"],
                                                        density=rec["density"], seed=rec["seed"]))
        got = [(n, hashlib.sha256(np.ascontiguousarray(host(t)).tobytes()).hexdigest())
               for n, t in model.parameters()]
        assert got == [(q["name"], q["sha256"]) for q in rec["params"]]
        assert smb.weights_fingerprint(model) == rec["fingerprint"]


def test_reference_training_trace_within_tolerance():
    """12 reference steps (config-1 shape, B=100, lr 0.01, Nesterov): per-step
    loss within 1e-4 relative, every parameter within rel_err 1e-4."""
    T = np.load(GOLDEN / "train_trace.npz")
    data = smb.synthetic_dataset(seed=5, n_samples=1200, features=3072)
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10],
                                                    density=0.01, seed=0, lr=0.01))
    step = smb.FusedTrainStep(model, 100)
    step.attach_dataset(smb.DeviceDataset(data))
    step.set_epoch(T["order"])
    for k in range(12):
        step.step(0.01)
        want = float(T["losses"][k])
        assert abs(step.loss_value() - want) <= 1e-4 * abs(want), k
    for name, t in model.parameters():
        assert rel_err(host(t), T["p_" + name]) <= 1e-4, name

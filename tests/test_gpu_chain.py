"""The column-chain kernel (csrc/chain.cu, smb_chain_run) against the separate
kernels it replaces inside the fused step: forward layers 1..L-1, the softmax
step and the input-gradient chain must give the same bits, so a fused step
with the chain equals one without it (weights, optimizer state, loss), and
both equal the oracle (test_gpu_bench_configs / test_gpu_training run the
default, chain-enabled step)."""

import numpy as np
import pytest
import torch

from conftest import bits_equal

pytestmark = pytest.mark.gpu

import paper_2407_17437_b200 as smb  # noqa: E402


def host(t):
    return t.detach().cpu().numpy()


def _run(chain_dims, density, B, steps, use_chain, seed=5, eta=0.05, graph=True):
    data = smb.synthetic_dataset(seed=seed, n_samples=B * steps, features=chain_dims[0],
                                 classes=chain_dims[-1])
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=chain_dims, density=density,
                                                    seed=seed, batch_size=B, lr=eta))
    st = smb.FusedTrainStep(model, B, chain=use_chain, use_graph=graph)
    st.attach_dataset(smb.DeviceDataset(data))
    st.set_epoch(np.random.default_rng(seed).permutation(B * steps))
    losses = []
    for _ in range(steps):
        st.step(eta)
        losses.append(st.loss_value())
    torch.cuda.synchronize()
    state = [host(t).reshape(-1).copy() for t in st.state_tensors()]
    params = [host(t).reshape(-1) for _, t in model.parameters()]
    return st, params, losses, state


@pytest.mark.parametrize("dims,density,B", [
    ([3072, 1024, 512, 10], 0.01, 1024),   # BASELINE config 2 point
    ([3072, 1024, 512, 10], 0.01, 100),    # partial column group (100 = 3*32 + 4)
    ([3072, 1024, 512, 10], 0.015, 512),   # cluster of 8
    ([200, 300, 16], 0.05, 37),            # two layers, 16 classes, padded leading dimension
    ([784, 512, 256, 128, 10], 0.02, 256),  # four layers: reloaded gradients
    ([3072, 1024, 512, 10], 0.01, 2048),   # two waves of clusters
])
def test_chain_step_equals_separate_kernels_bitwise(dims, density, B):
    st, p_chain, l_chain, _ = _run(dims, density, B, 3, True)
    assert st.chain_info() is not None, "the chain kernel should apply to this model"
    _, p_sep, l_sep, _ = _run(dims, density, B, 3, False)
    for a, b in zip(p_chain, p_sep):
        assert bits_equal(a, b)
    assert l_chain == l_sep


def test_chain_eager_equals_graph():
    dims = [3072, 1024, 512, 10]
    _, p_e, l_e, _ = _run(dims, 0.01, 256, 3, True, graph=False)
    _, p_g, l_g, _ = _run(dims, 0.01, 256, 3, True, graph=True)
    for a, b in zip(p_e, p_g):
        assert bits_equal(a, b)
    assert l_e == l_g


def test_chain_plan_shapes():
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10],
                                                    density=0.01, seed=1, batch_size=1024))
    info = smb.FusedTrainStep(model, 1024).chain_info()
    assert info["groups"] == 32 and info["cluster"] == 4 and info["layers"] == 3
    assert info["smem"] <= 227 * 1024


def test_chain_not_used_where_it_does_not_apply():
    # a saturated (dense) output layer and more than 16 classes run the
    # separate kernels
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10],
                                                    density=0.1, seed=1, batch_size=64))
    assert smb.FusedTrainStep(model, 64).chain_info() is None
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[100, 64, 20], density=0.3,
                                                    seed=1, batch_size=64))
    assert smb.FusedTrainStep(model, 64).chain_info() is None

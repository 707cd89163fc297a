"""Training-level parity on the GPU.

* initial weights (pattern + Xavier) bit-exact with the oracle's restatement of
  build_model / compile (bench.py:127-151, train.py:136-188);
* the fused, graph-captured step == the layer-by-layer drop-in API
  (feedforward / loss.gradient / backpropagate / optimize, train.py:398-401),
  bit for bit;
* 100 steps at the config-1 shape against the CPU oracle: per-step loss and
  weights within 1e-4 (rel_err of pkg/tests/conftest.py:46-53), final within
  1e-3 (BASELINE.json north_star tolerances).
"""

import numpy as np
import pytest
import torch

from conftest import bits_equal, rel_err

pytestmark = pytest.mark.gpu

import paper_2407_17437_b200 as smb  # noqa: E402


def host(t):
    return t.detach().cpu().numpy()


def params_host(model):
    return [(n, host(t).reshape(-1)) for n, t in model.parameters()]


def oracle_params(ref):
    return [(n, a.reshape(-1)) for n, a in ref.parameters()]


def max_rel(model, ref):
    return max(rel_err(a, b) for (_, a), (_, b) in zip(params_host(model), oracle_params(ref)))


@pytest.mark.parametrize("use_chain", [True, False])
def test_kernel_durations_time_every_sparse_launch(use_chain):
    """bench.py's per-kernel durations (KernelTimer.kernel_durations): one
    entry per C-ABI launch of the step, each a positive graph-timed duration."""
    chain, B = [3072, 1024, 512, 10], 256
    data = smb.synthetic_dataset(seed=2, n_samples=B * 4, features=chain[0])
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=0.01, seed=4,
                                                    batch_size=B))
    st = smb.FusedTrainStep(model, B, chain=use_chain)
    st.attach_dataset(smb.DeviceDataset(data))
    st.set_epoch(np.arange(B * 4))
    for _ in range(2):
        st.step(0.02)
    torch.cuda.synchronize()
    before = params_host(model)
    from paper_2407_17437_b200.engine import KernelTimer
    out = KernelTimer().kernel_durations(st, 0.02, reps=4, replays=2)
    # the timing pass replays in-place updates; it must leave the model as it was
    for (n1, a), (n2, b) in zip(before, params_host(model)):
        assert n1 == n2 and bits_equal(a, b), n1
    middle = (("chain",) if use_chain else
              ("spmm[1]", "spmm[2]", "softmax_ce", "spmm_t[2]", "spmm_t[1]"))
    for tag in ("spmm[0]",) + middle + ("sddmm_update[0]", "sddmm_update[1]", "sddmm_update[2]"):
        cnt, ms = out[tag]
        assert cnt == 8 and 0.0 < ms / cnt < 5.0, (tag, cnt, ms)
    assert st.timer is None and st.use_graph and st.overlap  # restored


@pytest.mark.parametrize("chain,density,seed", [
    ([3072, 1024, 512, 10], 0.01, 3),
    ([3072, 1024, 512, 10], 0.1, 1),      # last layer saturates -> Dense
    ([100, 64, 64, 10], 0.3, 9),
])
def test_initial_weights_bit_exact(oracle, chain, density, seed):
    model, plan = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=density, seed=seed))
    ref = oracle.OracleMLP.build(chain, density, seed=seed)
    for (n1, a), (n2, b) in zip(params_host(model), oracle_params(ref)):
        assert n1 == n2
        assert bits_equal(a, b), n1
    for lay, rl in zip([l for l in model.layers if isinstance(l, smb.SparseLinearLayer)],
                       [l for l in ref.layers if l.sparse]):
        rp, ci = lay.weights.pattern.host_arrays()
        assert np.array_equal(rp, rl.row_ptr) and np.array_equal(ci, rl.col_idx)


def _fused_and_layerwise(chain, density, seed, B, steps, eta=0.05):
    data = smb.synthetic_dataset(seed=seed, n_samples=B * steps, features=chain[0])
    cfg = smb.ExperimentConfig(layer_dims=chain, density=density, seed=seed, batch_size=B, lr=eta)
    m_fused, _ = smb.build_model(cfg)
    m_layer, _ = smb.build_model(cfg)
    step = smb.FusedTrainStep(m_fused, B)
    step.attach_dataset(smb.DeviceDataset(data))
    perm = np.random.default_rng(seed).permutation(B * steps)
    step.set_epoch(perm)
    loss = smb.SoftmaxCrossEntropyLoss()
    for k in range(steps):
        step.step(eta)
        b = perm[k * B:(k + 1) * B]
        xb = torch.from_numpy(np.ascontiguousarray(data.Xtrain[:, b])).cuda()
        tb = torch.from_numpy(np.ascontiguousarray(data.Ttrain[:, b])).cuda()
        y = m_layer.feedforward(xb)
        # (softmax(y) - t) / B with IEEE division like numpy (train.py:399);
        # torch's `cuda_tensor / python_scalar` multiplies by the reciprocal
        d = loss.gradient_scaled(y, tb, B)
        m_layer.backpropagate(y, d)
        m_layer.optimize(eta)
    torch.cuda.synchronize()
    return m_fused, m_layer


@pytest.mark.parametrize("chain,density,B", [
    ([3072, 1024, 512, 10], 0.01, 100),
    ([3072, 1024, 512, 10], 0.01, 1024),
    ([3072, 1024, 512, 10], 0.1, 256),    # dense last layer (cuBLAS on both paths)
    ([3072, 1024, 32, 10], 0.1, 128),     # small dense HIDDEN layer + ReLU (split-K forward)
    ([200, 300, 10], 0.2, 37),            # odd batch, padded leading dimension
])
def test_fused_step_equals_layer_api_bitwise(chain, density, B):
    m_fused, m_layer = _fused_and_layerwise(chain, density, 5, B, steps=4)
    for (n1, a), (n2, b) in zip(params_host(m_fused), params_host(m_layer)):
        assert n1 == n2
        assert bits_equal(a, b), n1




def test_graph_replay_equals_eager():
    chain, B = [3072, 1024, 512, 10], 128
    data = smb.synthetic_dataset(seed=2, n_samples=B * 6, features=chain[0])
    models = []
    for graph in (True, False):
        model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=0.01, seed=4,
                                                        batch_size=B))
        st = smb.FusedTrainStep(model, B, use_graph=graph)
        st.attach_dataset(smb.DeviceDataset(data))
        st.set_epoch(np.arange(B * 6))
        for _ in range(6):
            st.step(0.02)
        models.append(model)
    torch.cuda.synchronize()
    for (_, a), (_, b) in zip(params_host(models[0]), params_host(models[1])):
        assert bits_equal(a, b)


def test_hundred_steps_track_oracle(oracle):
    """Config-1 shape, B=100, lr 0.01, Nesterov 0.9, SURVEY 8(d) data: per-step
    loss/weights within 1e-4 and final weights within 1e-3 of the oracle."""
    chain, d, seed, B, steps, eta = [3072, 1024, 512, 10], 0.01, 0, 100, 100, 0.01
    data = smb.synthetic_dataset(seed=11, n_samples=B * steps, features=chain[0])
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=d, seed=seed,
                                                    batch_size=B, lr=eta))
    ref = oracle.OracleMLP.build(chain, d, seed=seed)
    step = smb.FusedTrainStep(model, B)
    step.attach_dataset(smb.DeviceDataset(data))
    perm = np.random.default_rng(0).permutation(B * steps)
    step.set_epoch(perm)
    worst_step = 0.0
    for k in range(steps):
        step.step(eta)
        b = perm[k * B:(k + 1) * B]
        ref_loss = ref.step(data.Xtrain[:, b], data.Ttrain[:, b], eta)
        gpu_loss = step.loss_value()
        assert abs(gpu_loss - ref_loss) <= 1e-4 * abs(ref_loss), (k, gpu_loss, ref_loss)
        if k < 10 or k % 10 == 9:
            worst_step = max(worst_step, max_rel(model, ref))
            assert worst_step <= 1e-4, (k, worst_step)
    assert max_rel(model, ref) <= 1e-3


def test_sgd_train_reference_fingerprint_run(oracle):
    """The run behind the reference's recorded fingerprint (pkg/test_output.txt:26:
    synthetic blobs seed 3, 2 epochs of B=100, lr 0.1 multistep) through the
    drop-in sgd_train: weights within 1e-4 of the oracle (which reproduces the
    fingerprint bit for bit on the CPU)."""
    xtr, ttr, _, _ = oracle.synthetic_blobs(10, 3072, 50, 1.0, 3, 5)
    ref = oracle.OracleMLP.build([3072, 1024, 512, 10], 0.01, seed=3)
    ref.train(xtr, ttr, 2, 100, oracle.multistep(0.1))
    assert ref.fingerprint().startswith("69a2e92774f1")
    cfg = smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=0.01, seed=3, epochs=2,
                               batch_size=100, eval_metrics=False)
    model, _ = smb.build_model(cfg)
    recs = smb.sgd_train(model, smb.Dataset(xtr, ttr),
                         smb.TrainConfig(epochs=2, batch_size=100, schedule=cfg.schedule(),
                                         eval_metrics=False))
    assert [r.lr for r in recs] == [0.1, 0.1 * 0.1 ** 2]
    assert max_rel(model, ref) <= 1e-4


@pytest.mark.parametrize("backend", ["sparse", "masked"])
def test_train_batch_host_buffers_equal_device_gather(backend):
    """FusedTrainStep.train_batch (pinned host batches, double-buffered copies:
    the e2e API bench.py times) == step() over the HBM dataset, bit for bit,
    including the loss copied back to the host."""
    chain, B, steps, eta = [3072, 1024, 512, 10], 128, 5, 0.03
    data = smb.synthetic_dataset(seed=4, n_samples=B * steps, features=chain[0])
    perm = np.random.default_rng(2).permutation(B * steps)
    cfg = smb.ExperimentConfig(layer_dims=chain, density=0.01, seed=6, batch_size=B, lr=eta,
                               backend=backend)
    m_dev, _ = smb.build_model(cfg)
    m_host, _ = smb.build_model(cfg)
    st_dev = smb.FusedTrainStep(m_dev, B)
    st_dev.attach_dataset(smb.DeviceDataset(data))
    st_dev.set_epoch(perm)
    st_host = smb.FusedTrainStep(m_host, B)
    loss_host = torch.empty(1, dtype=torch.float64).pin_memory()
    for k in range(steps):
        st_dev.step(eta)
        b = perm[k * B:(k + 1) * B]
        xb = torch.from_numpy(np.ascontiguousarray(data.Xtrain[:, b])).pin_memory()
        tb = torch.from_numpy(np.ascontiguousarray(data.Ttrain[:, b])).pin_memory()
        st_host.train_batch(xb, tb, eta, loss_host)
        torch.cuda.synchronize()
        assert float(loss_host[0]) == st_dev.loss_value(), k
    for (n1, a), (n2, b) in zip(params_host(m_dev), params_host(m_host)):
        assert n1 == n2
        assert bits_equal(a, b), n1


def test_config5_injected_patterns_track_oracle(oracle):
    """BASELINE config 5 shape (3072-65536-65536-10, d=0.001; the hidden-hidden
    grid exceeds the reference sampler's 2**31 limit, so its pattern is
    injected): initial weights bit-exact with the oracle's restatement, then
    two fused steps within the per-step tolerance."""
    chain, d, B, eta = [3072, 65536, 65536, 10], 0.001, 16, 0.01
    cfg = smb.ExperimentConfig(layer_dims=chain, density=d, seed=1, batch_size=B, lr=eta)
    with pytest.raises(smb.InvalidArgumentError):
        smb.build_model(cfg)  # the reference behaviour without injection
    model, plan = smb.build_model(cfg, large_patterns=True)
    assert plan.layer_nnz == [1319931, 2521658, 655360]
    ref = oracle.OracleMLP.build(chain, d, seed=1, large_patterns=True)
    for (n1, a), (n2, b) in zip(params_host(model), oracle_params(ref)):
        assert n1 == n2 and bits_equal(a, b), n1
    data = smb.synthetic_dataset(seed=3, n_samples=2 * B, features=chain[0])
    step = smb.FusedTrainStep(model, B)
    step.attach_dataset(smb.DeviceDataset(data))
    step.set_epoch(np.arange(2 * B))
    for k in range(2):
        step.step(eta)
        ref_loss = ref.step(data.Xtrain[:, k * B:(k + 1) * B], data.Ttrain[:, k * B:(k + 1) * B], eta)
        assert abs(step.loss_value() - ref_loss) <= 1e-4 * abs(ref_loss)
    assert max_rel(model, ref) <= 1e-4


@pytest.mark.parametrize("density,B", [(0.01, 128), (0.1, 100)])
def test_data_parallel_structure_on_one_gpu_equals_fused(density, B):
    """The data-parallel step structure (gradients into the flat buffer with
    side-stream overlap, [all-reduce], update pass from the flat buffer) run
    on one GPU (force_dp: the all-reduce is the identity) is bit-identical to
    the fused single-GPU step -- the update arithmetic is the same
    sparse_combine / _step_vector sequence either way."""
    chain, steps, eta = [3072, 1024, 512, 10], 4, 0.03
    data = smb.synthetic_dataset(seed=9, n_samples=B * steps, features=chain[0])
    cfg = smb.ExperimentConfig(layer_dims=chain, density=density, seed=2, batch_size=B, lr=eta)
    models = []
    for force_dp in (False, True):
        model, _ = smb.build_model(cfg)
        st = smb.FusedTrainStep(model, B, force_dp=force_dp)
        assert st.dp == force_dp
        st.attach_dataset(smb.DeviceDataset(data))
        st.set_epoch(np.arange(B * steps))
        for _ in range(steps):
            st.step(eta)
        models.append(model)
    torch.cuda.synchronize()
    for (n1, a), (n2, b) in zip(params_host(models[0]), params_host(models[1])):
        assert n1 == n2
        assert bits_equal(a, b), n1


@pytest.mark.parametrize("how", ["in_place", "assign", "layer_optimize"])
def test_step_follows_external_weight_change(how):
    """The step's value buffers and CSC-ordered copies (smb_spmm_t_csc) follow
    a change of the layer values made between steps -- an in-place torch op,
    a newly assigned tensor, or the layer API's optimize() -- without any
    explicit sync call: the next steps equal those of a fresh step object
    built on the changed model."""
    chain, B = [3072, 1024, 512, 10], 128
    data = smb.synthetic_dataset(seed=5, n_samples=B * 8, features=chain[0])
    models, steps = [], []
    for _ in range(2):
        model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=0.01, seed=6,
                                                        batch_size=B))
        st = smb.FusedTrainStep(model, B)
        st.attach_dataset(smb.DeviceDataset(data))
        st.set_epoch(np.arange(B * 8))
        models.append(model)
        steps.append(st)
    for _ in range(2):
        steps[0].step(0.02)
        steps[1].step(0.02)
    for m_ in models:  # same change on both replicas
        for lay in m_.layers:
            if isinstance(lay, smb.SparseLinearLayer):
                if how == "in_place":
                    lay.weights.values.mul_(0.5)
                elif how == "assign":
                    lay.weights.values = lay.weights.values * 0.5
                else:
                    lay.grad.values.fill_(0.25)
                    lay.grad_bias = torch.full_like(lay.bias, 0.5)
                    lay.optimize(0.1)
    # replica 1: a fresh step object on the changed model, same batch order
    fresh = smb.FusedTrainStep(models[1], B)
    fresh.attach_dataset(smb.DeviceDataset(data))
    fresh.set_epoch(np.arange(B * 8))
    fresh.counter.copy_(steps[1].counter)
    for _ in range(2):
        steps[0].step(0.02)
        fresh.step(0.02)
    torch.cuda.synchronize()
    for (_, a), (_, b) in zip(params_host(models[0]), params_host(models[1])):
        assert bits_equal(a, b)


def test_values_identity_stable_across_steps():
    """A caller holding `layer.weights.values` sees every update in place, as
    with the reference's in-place sparse_combine (nn.py:187-198): the
    overlapped step ping-pongs two buffers underneath, but the layer's tensor
    object is re-pointed at the current one."""
    chain, B = [3072, 1024, 512, 10], 128
    data = smb.synthetic_dataset(seed=5, n_samples=B * 8, features=chain[0])
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=0.01, seed=6,
                                                    batch_size=B))
    held = [lay.weights.values for lay in model.layers if isinstance(lay, smb.SparseLinearLayer)]
    before = [h.cpu().clone() for h in held]
    st = smb.FusedTrainStep(model, B)
    st.attach_dataset(smb.DeviceDataset(data))
    st.set_epoch(np.arange(B * 8))
    for n_steps in (1, 2, 3):
        st.step(0.02)
        torch.cuda.synchronize()
        now = [lay.weights.values for lay in model.layers
               if isinstance(lay, smb.SparseLinearLayer)]
        for h, cur in zip(held, now):
            assert h is cur
            assert h.data_ptr() == cur.data_ptr()
    for h, b in zip(held, before):
        assert not torch.equal(h.cpu(), b)  # the held tensors moved with training

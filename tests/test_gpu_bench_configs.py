"""Oracle parity at every configuration bench.py and scripts/kernel_bench.py time.

The kernels pick their variant (lane width, ring depth, tile size, blocked or
row-split form) from the batch width, the row/column lengths and the wave
count, so parity proven on small shapes does not cover the variants that run
at the benchmarked shapes.  These tests step the fused path (or launch the
single kernels) at exactly those shapes beside the CPU oracle:

* BASELINE config 2 point (3072-1024-512-10, d=0.01, B=1024): 20 fused steps,
  per-step loss and weights within 1e-4 (north_star tolerance);
* config 2 at d=0.05 / 0.5 (dense output layer) with B=100 and 1024;
* config 4 (3072-8192x3-10, d=0.01, B=1024): 3 steps;
* config 5 (3072-65536-65536-10, d=0.001, injected pattern) at B=512: 2 steps;
* config 3 (8192x8192 CSR, d in {0.001, 0.01, 0.1}, B in {128, 512, 2048}):
  forward SpMM, transposed SpMM (CSR-value and CSC-value forms) and
  SDDMM + Nesterov update, each BIT-EXACT against the oracle's restatement of
  _kernels.py:25-83 and nn.py:189-193.

Reference: train.py:398-401 (the step), _kernels.py:25-83 (the kernels).
"""

import os

import numpy as np
import pytest
import torch

from conftest import bits_equal, rel_err

pytestmark = pytest.mark.gpu

import paper_2407_17437_b200 as smb  # noqa: E402
from paper_2407_17437_b200 import _lib  # noqa: E402
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr  # noqa: E402


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle as O

    O.build()
    O.set_threads(os.cpu_count() or 1)
    return O


def _params(model):
    return [(n, t.detach().cpu().numpy().reshape(-1)) for n, t in model.parameters()]


def _max_rel(model, ref):
    return max(rel_err(a, b.reshape(-1))
               for (_, a), (_, b) in zip(_params(model), ref.parameters()))


def _track(orc, chain, density, B, steps, eta=0.01, seed=0, large=False, n_samples=None,
           check_every=1):
    """Fused steps beside the oracle on the same batches; asserts the north_star
    per-step tolerance and returns the worst parameter rel_err."""
    n_samples = n_samples or B * steps
    data = smb.synthetic_dataset(seed=seed + 7, n_samples=n_samples, features=chain[0],
                                 classes=chain[-1])
    cfg = smb.ExperimentConfig(layer_dims=chain, density=density, seed=seed, batch_size=B, lr=eta)
    model, _ = smb.build_model(cfg, large_patterns=large)
    ref = orc.OracleMLP.build(chain, density, seed=seed, large_patterns=large)
    for (n1, a), (n2, b) in zip(_params(model), ref.parameters()):
        assert n1 == n2 and bits_equal(a, b.reshape(-1)), n1  # same initial model
    step = smb.FusedTrainStep(model, B)
    step.attach_dataset(smb.DeviceDataset(data))
    perm = np.random.default_rng(seed).permutation(n_samples)
    step.set_epoch(perm)
    worst = 0.0
    for k in range(steps):
        step.step(eta)
        cols = perm[k * B:(k + 1) * B]
        ref_loss = ref.step(np.ascontiguousarray(data.Xtrain[:, cols]),
                            np.ascontiguousarray(data.Ttrain[:, cols]), eta)
        gpu_loss = step.loss_value()
        assert abs(gpu_loss - ref_loss) <= 1e-4 * abs(ref_loss), (k, gpu_loss, ref_loss)
        if k % check_every == check_every - 1 or k == steps - 1:
            worst = max(worst, _max_rel(model, ref))
            assert worst <= 1e-4, (k, worst)
    return worst


def test_config2_point_b1024_twenty_steps(orc):
    """The BENCH line's workload: 3072-1024-512-10, d=0.01, B=1024, 20 steps."""
    _track(orc, [3072, 1024, 512, 10], 0.01, 1024, 20, check_every=5)


@pytest.mark.parametrize("density", [0.05, 0.5])
@pytest.mark.parametrize("B", [100, 1024])
def test_config2_sweep_points(orc, density, B):
    """Sweep points with an ER-saturated (dense) output layer."""
    _track(orc, [3072, 1024, 512, 10], density, B, 4)


def test_config4_b1024_three_steps(orc):
    """BASELINE config 4: 3072-8192-8192-8192-10, d=0.01, B=1024."""
    _track(orc, [3072, 8192, 8192, 8192, 10], 0.01, 1024, 3)


def test_config5_b512_two_steps(orc):
    """BASELINE config 5 at the bench batch (B=512 per GPU), injected pattern."""
    _track(orc, [3072, 65536, 65536, 10], 0.001, 512, 2, large=True)


# ---------------------------------------------------------------------------
# config 3: the single-layer kernels at the kernel_bench.py shapes, bit-exact
# ---------------------------------------------------------------------------
_PATTERNS = {}


def _pattern(d):
    if d not in _PATTERNS:
        n = 8192
        nnz = int(round(d * n * n))
        _PATTERNS[d] = smb.sample_pattern(n, n, nnz, smb.Rng(0).stream("pattern"))
    return _PATTERNS[d]


@pytest.mark.parametrize("density", [0.001, 0.01, 0.1])
@pytest.mark.parametrize("B", [128, 512, 2048])
def test_config3_kernels_bit_exact(orc, density, B):
    n = 8192
    pat = _pattern(density)
    rp, ci = pat.host_arrays()
    nnz = ci.shape[0]
    rng = np.random.default_rng(int(density * 1e4) + B)
    vals_h = rng.standard_normal(nnz).astype(np.float32)
    x_h = rng.standard_normal((n, B)).astype(np.float32)
    dy_h = rng.standard_normal((n, B)).astype(np.float32)
    vel_h = (0.1 * rng.standard_normal(nnz)).astype(np.float32)
    dev = torch.device("cuda")
    vals = torch.from_numpy(vals_h).to(dev)
    X = torch.from_numpy(x_h).to(dev)
    dY = torch.from_numpy(dy_h).to(dev)
    out = torch.empty(n, B, device=dev)
    st = stream_ptr()

    # forward SpMM (_kernels.py:25-37)
    _lib.call("smb_spmm_p", 0, pat.handle, ptr(vals), ptr(X), B, B, None, 0, ptr(out), B, st)
    assert bits_equal(out.cpu().numpy(), orc.spmm(rp, ci, vals_h, x_h)), "spmm"

    # transposed SpMM (_kernels.py:40-59), CSR values and CSC-ordered values
    ref_t = orc.spmm_t(rp, ci, vals_h, n, dy_h)
    _lib.call("smb_spmm_t", 0, pat.handle, ptr(vals), ptr(dY), B, B, None, 0, ptr(out), B, st)
    assert bits_equal(out.cpu().numpy(), ref_t), "spmm_t"
    vcsc = torch.empty_like(vals)
    _lib.call("smb_values_to_csc", 0, pat.handle, ptr(vals), ptr(vcsc), st)
    out.zero_()
    _lib.call("smb_spmm_t_csc", 0, pat.handle, ptr(vcsc), ptr(dY), B, B, None, 0, ptr(out), B,
              st)
    assert bits_equal(out.cpu().numpy(), ref_t), "spmm_t_csc"

    # SDDMM + Nesterov update of values / velocity (_kernels.py:62-83, nn.py:189-193)
    mu, eta = 0.9, 1e-3
    vel = torch.from_numpy(vel_h).to(dev)
    vout = torch.empty_like(vals)
    _lib.call("smb_sddmm_update_into", 0, pat.handle, ptr(dY), B, ptr(X), B, B, ptr(vals),
              ptr(vout), ptr(vel), None, None, None, None, _lib.SMB_OPT_NESTEROV, mu, eta, st)
    g = orc.sddmm(rp, ci, dy_h, x_h)
    v_ref, w_ref = vel_h.copy(), vals_h.copy()
    orc.axpby(mu, v_ref, 1.0, g)
    orc.axpby(1.0, w_ref, -eta * mu, v_ref)
    orc.axpby(1.0, w_ref, -eta, g)
    assert bits_equal(vel.cpu().numpy(), v_ref), "sddmm velocity"
    assert bits_equal(vout.cpu().numpy(), w_ref), "sddmm values"
    # the gradient itself (SMB_OPT_NONE writes grad_out)
    gout = torch.empty_like(vals)
    _lib.call("smb_sddmm_update", 0, pat.handle, ptr(dY), B, ptr(X), B, B, ptr(vals), None,
              ptr(gout), None, None, None, _lib.SMB_OPT_NONE, 0.0, 0.0, st)
    assert bits_equal(gout.cpu().numpy(), g), "sddmm grad"


@pytest.mark.parametrize("B", [600, 1024])
def test_l2_sliced_spmm_bit_exact(orc, B):
    """Layers whose gathered operand is wider than the L2 budget run the SpMM
    in column slices (all output rows of one slice before the next, several
    rows per CTA).  Forward and transposed products must stay bit-identical
    to the oracle (_kernels.py:25-59), also with a ragged last slice."""
    m = k = 30000
    nnz = int(0.0005 * m * k)
    pat = smb.sample_pattern(m, k, nnz, smb.Rng(1).stream("pattern"))
    rp, ci = pat.host_arrays()
    rng = np.random.default_rng(B)
    vals_h = rng.standard_normal(nnz).astype(np.float32)
    x_h = rng.standard_normal((k, B)).astype(np.float32)
    dy_h = rng.standard_normal((m, B)).astype(np.float32)
    dev = torch.device("cuda")
    vals, X, dY = (torch.from_numpy(a).to(dev) for a in (vals_h, x_h, dy_h))
    out = torch.empty(m, B, device=dev)
    st = stream_ptr()
    _lib.call("smb_spmm_p", 0, pat.handle, ptr(vals), ptr(X), B, B, None, 0, ptr(out), B, st)
    assert bits_equal(out.cpu().numpy(), orc.spmm(rp, ci, vals_h, x_h)), "spmm"
    _lib.call("smb_spmm_t", 0, pat.handle, ptr(vals), ptr(dY), B, B, ptr(X), B, ptr(out), B, st)
    ref_t = orc.spmm_t(rp, ci, vals_h, k, dy_h) * (x_h > 0)
    assert bits_equal(out.cpu().numpy(), ref_t.astype(np.float32)), "spmm_t + mask"


def _pattern_from_row_lengths(lengths, k, rng):
    rows = [np.sort(rng.choice(k, size=int(L), replace=False)) for L in lengths]
    row_ptr = np.zeros(len(lengths) + 1, np.int32)
    np.cumsum(lengths, out=row_ptr[1:])
    col_idx = np.concatenate(rows).astype(np.int32)
    return row_ptr, col_idx


@pytest.mark.parametrize("n", [1, 37, 100, 1000, 1024])
@pytest.mark.parametrize("shape", ["uniform", "mixed_rows"])
def test_tma_sddmm_edge_cases_bit_exact(orc, n, shape):
    """The TMA gather4 SDDMM (many-wave layers, >= 16 nonzeros per row on
    average): ragged batch widths (the last 32-column chunk partly out of the
    tensor map, zero-filled by TMA and never summed), one column, and warps
    whose 32 nonzeros span more than the 4 staged d_out rows (short rows
    between long ones: d_out read from global memory) -- bit-exact with the
    oracle's sddmm + Nesterov sequence (_kernels.py:62-83, nn.py:189-193)."""
    rng = np.random.default_rng(n)
    m, k = 6144, 4096
    if shape == "uniform":
        lengths = np.full(m, 24)
    else:  # three 2-nonzero rows, then a 90-nonzero row: average 24
        lengths = np.tile([2, 2, 2, 90], m // 4)
    rp, ci = _pattern_from_row_lengths(lengths, k, rng)
    pat = smb.SparsityPattern(m, k, rp, ci)
    nnz = ci.shape[0]
    vals_h = rng.standard_normal(nnz).astype(np.float32)
    vel_h = (0.1 * rng.standard_normal(nnz)).astype(np.float32)
    x_h = rng.standard_normal((k, n)).astype(np.float32)
    dy_h = rng.standard_normal((m, n)).astype(np.float32)
    dev = torch.device("cuda")
    ld = (n + 3) // 4 * 4  # 16-byte rows (the TMA path's requirement)
    X = torch.zeros(k, ld, device=dev)
    dY = torch.zeros(m, ld, device=dev)
    X[:, :n] = torch.from_numpy(x_h)
    dY[:, :n] = torch.from_numpy(dy_h)
    vals = torch.from_numpy(vals_h).to(dev)
    vel = torch.from_numpy(vel_h).to(dev)
    vout = torch.empty_like(vals)
    mu, eta = 0.9, 1e-3
    _lib.call("smb_sddmm_update_into", 0, pat.handle, ptr(dY), ld, ptr(X), ld, n, ptr(vals),
              ptr(vout), ptr(vel), None, None, None, None, _lib.SMB_OPT_NESTEROV, mu, eta,
              stream_ptr())
    g = orc.sddmm(rp, ci, dy_h, x_h)
    v_ref, w_ref = vel_h.copy(), vals_h.copy()
    orc.axpby(mu, v_ref, 1.0, g)
    orc.axpby(1.0, w_ref, -eta * mu, v_ref)
    orc.axpby(1.0, w_ref, -eta, g)
    assert bits_equal(vel.cpu().numpy(), v_ref)
    assert bits_equal(vout.cpu().numpy(), w_ref)


def test_blocked_order_sddmm_bit_exact(orc):
    """Very wide layers (m, k >= 16384) whose x and d_out overflow L2 many
    times at the batch width walk their nonzeros in the pattern's L2-blocked
    order (row band x column band blocks, CSR order inside); each chain and
    the update are unchanged and land at the CSR index: bit-exact with the
    oracle, ragged batch width included.  The batch is walked in phases of
    256 columns (9 launches here, the last one ragged), the chain sums carried
    between them in the pattern's workspace."""
    m = k = 30000
    n = 2300  # (m + k) * n * 4 bytes > 512 MB -> blocked order
    nnz = int(0.0005 * m * k)
    pat = smb.sample_pattern(m, k, nnz, smb.Rng(2).stream("pattern"))
    rp, ci = pat.host_arrays()
    rng = np.random.default_rng(5)
    vals_h = rng.standard_normal(nnz).astype(np.float32)
    vel_h = (0.1 * rng.standard_normal(nnz)).astype(np.float32)
    x_h = rng.standard_normal((k, n)).astype(np.float32)
    dy_h = rng.standard_normal((m, n)).astype(np.float32)
    dev = torch.device("cuda")
    ld = (n + 3) // 4 * 4
    X = torch.zeros(k, ld, device=dev)
    dY = torch.zeros(m, ld, device=dev)
    X[:, :n] = torch.from_numpy(x_h)
    dY[:, :n] = torch.from_numpy(dy_h)
    vals = torch.from_numpy(vals_h).to(dev)
    vel = torch.from_numpy(vel_h).to(dev)
    vout = torch.empty_like(vals)
    gout = torch.empty_like(vals)
    mu, eta = 0.9, 1e-3
    _lib.call("smb_sddmm", 0, pat.handle, ptr(dY), ld, ptr(X), ld, n, ptr(gout), stream_ptr())
    _lib.call("smb_sddmm_update_into", 0, pat.handle, ptr(dY), ld, ptr(X), ld, n, ptr(vals),
              ptr(vout), ptr(vel), None, None, None, None, _lib.SMB_OPT_NESTEROV, mu, eta,
              stream_ptr())
    g = orc.sddmm(rp, ci, dy_h, x_h)
    assert bits_equal(gout.cpu().numpy(), g)
    v_ref, w_ref = vel_h.copy(), vals_h.copy()
    orc.axpby(mu, v_ref, 1.0, g)
    orc.axpby(1.0, w_ref, -eta * mu, v_ref)
    orc.axpby(1.0, w_ref, -eta, g)
    assert bits_equal(vel.cpu().numpy(), v_ref)
    assert bits_equal(vout.cpu().numpy(), w_ref)

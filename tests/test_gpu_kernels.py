"""Kernel parity on the GPU: every exact kernel must be BIT-IDENTICAL to the
CPU oracle (itself pinned to the reference in test_oracle_golden.py) on the
same seeded inputs -- random instances in the reference tests' shapes
(pkg/tests/test_tensor_core.py:96-182) plus the edge cases it covers (empty
pattern, empty rows, single nonzero, n = 0/1, odd n, fp64)."""

import numpy as np
import pytest
import torch

from conftest import bits_equal, random_csr, rel_err

pytestmark = pytest.mark.gpu

import paper_2407_17437_b200 as smb  # noqa: E402
from paper_2407_17437_b200 import _lib  # noqa: E402
from paper_2407_17437_b200 import tensor_core as tc  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy()


SHAPES = [(1, 1, 1), (2, 3, 4), (17, 13, 5), (40, 33, 37), (64, 96, 100), (129, 257, 128),
          (300, 200, 1), (512, 1024, 130), (1000, 700, 257)]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("density", [0.05, 0.3, 1.0])
def test_spmm_bit_exact(oracle, dtype, shape, density):
    m, k, n = shape
    rng = np.random.default_rng(hash((m, k, n, density)) % 2**32)
    rp, ci, v, dense = random_csr(rng, m, k, density, dtype, empty_rows=True)
    x = rng.standard_normal((k, n)).astype(dtype)
    s = smb.CsrMatrix(m, k, rp, ci, v)
    got = smb.spmm(s, x)
    want = oracle.spmm(rp, ci, v, x)
    assert bits_equal(got, want)
    # the reference's fp64-oracle tolerance holds for its own shape range (<= 40)
    tol = (1e-5 if dtype == np.float32 else 1e-12) * (1 if max(m, k) <= 40 else 10)
    assert rel_err(got, dense.astype(np.float64) @ x) <= tol


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("density", [0.05, 0.3, 1.0])
def test_spmm_transposed_bit_exact(oracle, dtype, shape, density):
    m, k, n = shape
    rng = np.random.default_rng(1 + hash((m, k, n, density)) % 2**32)
    rp, ci, v, dense = random_csr(rng, m, k, density, dtype, empty_rows=True)
    d = rng.standard_normal((m, n)).astype(dtype)
    s = smb.CsrMatrix(m, k, rp, ci, v)
    got = smb.spmm_transposed(s, d)
    want = oracle.spmm_t(rp, ci, v, k, d)
    assert bits_equal(got, want)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("density", [0.05, 0.3, 1.0])
def test_sddmm_bit_exact(oracle, dtype, shape, density):
    m, k, n = shape
    rng = np.random.default_rng(2 + hash((m, k, n, density)) % 2**32)
    rp, ci, v, _ = random_csr(rng, m, k, density, dtype, empty_rows=True)
    a = rng.standard_normal((m, n)).astype(dtype)
    b = rng.standard_normal((k, n)).astype(dtype)
    pat = smb.SparsityPattern(m, k, rp, ci)
    got = host(smb.sddmm(pat, dev(a), dev(b)).values)
    want = oracle.sddmm(rp, ci, a, b)
    assert bits_equal(got, want)


def test_sddmm_zero_batch_gives_zeros():
    pat = smb.csr_from_dense(np.ones((3, 4), dtype=np.float32)).pattern
    out = smb.sddmm(pat, torch.zeros((3, 0), device="cuda"), torch.zeros((4, 0), device="cuda"))
    assert torch.count_nonzero(out.values) == 0


def test_sddmm_many_empty_rows_window_fallback(oracle):
    # > 128 rows inside one 128-nonzero tile exercises the global row search
    m, k, n = 5000, 64, 9
    rng = np.random.default_rng(7)
    counts = np.zeros(m, dtype=np.int64)
    counts[rng.choice(m, size=40, replace=False)] = rng.integers(1, 8, size=40)
    rp = np.zeros(m + 1, dtype=np.int32)
    np.cumsum(counts, out=rp[1:])
    ci = np.concatenate([np.sort(rng.choice(k, size=c, replace=False)) for c in counts if c]).astype(np.int32)
    a = rng.standard_normal((m, n)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    got = host(smb.sddmm(smb.SparsityPattern(m, k, rp, ci), dev(a), dev(b)).values)
    assert bits_equal(got, oracle.sddmm(rp, ci, a, b))


@pytest.mark.parametrize("n", [1024, 70, 5])
def test_sddmm_very_sparse_rows_one_slot_per_nonzero(oracle, n):
    # 1-2 nonzeros per row: a 128-nonzero tile spans > 32 rows, so every
    # nonzero gets its own staged d_out row (SD = 1 tiles)
    m, k = 3000, 700
    rng = np.random.default_rng(n)
    counts = rng.integers(1, 3, size=m)
    rp = np.zeros(m + 1, dtype=np.int32)
    np.cumsum(counts, out=rp[1:])
    ci = np.concatenate([np.sort(rng.choice(k, size=c, replace=False)) for c in counts]).astype(np.int32)
    a = rng.standard_normal((m, n)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    got = host(smb.sddmm(smb.SparsityPattern(m, k, rp, ci), dev(a), dev(b)).values)
    assert bits_equal(got, oracle.sddmm(rp, ci, a, b))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_sparse_combine_bit_exact(oracle, dtype):
    rng = np.random.default_rng(55)
    rp, ci, v, _ = random_csr(rng, 90, 70, 0.4, dtype)
    t = rng.standard_normal(v.shape[0]).astype(dtype)
    for alpha, beta in [(0.9, 1.0), (1.0, -0.05 * 0.9), (1.0, -0.05), (0.3, 0.7)]:
        s = smb.CsrMatrix(90, 70, rp, ci, v.copy())
        smb.sparse_combine(alpha, s, beta, s.pattern.with_values(t))
        want = v.copy()
        oracle.axpby(alpha, want, beta, t)
        assert bits_equal(host(s.values), want)


def test_hand_values():
    # pkg/tests/test_tensor_core.py:81-84, 113-120, 144-150
    s = smb.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 2.0], np.float32))
    b = np.array([[1, 2], [3, 4]], dtype=np.float32)
    assert np.array_equal(smb.spmm(s, b), [[1, 2], [6, 8]])
    assert np.array_equal(smb.spmm_transposed(s, b), [[1, 2], [6, 8]])
    s1 = smb.CsrMatrix(1, 2, np.array([0, 1]), np.array([1]), np.array([3.0], np.float32))
    assert np.array_equal(smb.spmm_transposed(s1, np.array([[5.0, 7.0]], np.float32)),
                          [[0, 0], [15, 21]])
    pat = smb.SparsityPattern(1, 2, np.array([0, 1]), np.array([1]))
    out = smb.sddmm(pat, np.array([[1.0, 2.0]], np.float32),
                    np.array([[0.0, 0.0], [3.0, 4.0]], np.float32))
    assert host(out.values).tolist() == [11.0]


def test_empty_pattern_gives_zeros():
    s = smb.SparsityPattern(2, 2, np.zeros(3, np.int32), np.zeros(0, np.int32)).zeros()
    b = np.arange(4, dtype=np.float32).reshape(2, 2)
    assert np.array_equal(smb.spmm(s, b), np.zeros((2, 2)))
    assert np.array_equal(smb.spmm_transposed(s, b), np.zeros((2, 2)))


def test_invalid_structures_rejected():
    bad = [
        (2, 2, [0, 1, 3], [0]),        # row_ptr end != nnz
        (2, 2, [0, 2, 1], [0, 1]),     # decreasing row_ptr
        (1, 2, [0, 1], [2]),           # col out of range
        (1, 3, [0, 2], [1, 1]),        # duplicate col within a row
    ]
    for m, k, rp, ci in bad:
        with pytest.raises(smb.InvalidArgumentError):
            smb.CsrMatrix(m, k, np.array(rp), np.array(ci), np.ones(len(ci), np.float32))
    with pytest.raises(smb.InvalidArgumentError):
        smb.CsrMatrix(2, 2, np.array([0, 1]), np.array([0]), np.array([1.0], np.float32))
    with pytest.raises(smb.InvalidArgumentError):
        smb.CsrMatrix(1, 1, np.array([0, 1]), np.array([0]), np.array([1]))


def test_csc_index_is_row_sorted(oracle):
    rng = np.random.default_rng(3)
    rp, ci, v, dense = random_csr(rng, 300, 200, 0.2)
    pat = smb.SparsityPattern(300, 200, rp, ci)
    col_ptr, row_idx, perm = (host(t) for t in pat.csc())
    want_order = np.argsort(ci, kind="stable")
    rows = np.repeat(np.arange(300), np.diff(rp))
    assert np.array_equal(perm, want_order)
    assert np.array_equal(row_idx, rows[want_order])
    assert np.array_equal(col_ptr[1:], np.cumsum(np.bincount(ci, minlength=200)))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_row_sums_numpy_pairwise_order(dtype):
    rng = np.random.default_rng(12)
    # (256 ... 16384 = 128 * 2^p: the balanced-tree fast path)
    for n in [1, 7, 8, 9, 100, 128, 129, 256, 257, 384, 512, 1000, 1024, 2048, 4096, 8192, 16384,
              16512]:
        a = (rng.standard_normal((33, n)) * np.exp(3 * rng.standard_normal((33, n)))).astype(dtype)
        assert bits_equal(smb.row_sums(a), a.sum(axis=1))


@pytest.mark.parametrize("nesterov", [False, True])
def test_optimizer_ten_steps_bitwise(nesterov):
    # pkg/tests/test_nn.py:437-467: fp32 scalar recurrence with explicit rounding
    mu, eta = 0.9, 0.05
    rng = np.random.default_rng(33)
    rp, ci, v, _ = random_csr(rng, 3, 3, 1.0)
    layer = smb.SparseLinearLayer(smb.SparsityPattern(3, 3, rp, ci), v, np.zeros(3, np.float32),
                                  smb.Momentum(mu, nesterov=nesterov))
    nnz = layer.weights.nnz
    grads = rng.standard_normal((10, nnz)).astype(np.float32)
    w, vv = v.copy(), np.zeros(nnz, np.float32)
    mu32, one, c_v, c_g = np.float32(mu), np.float32(1), np.float32(-eta * mu), np.float32(-eta)
    for g in grads:
        for i in range(nnz):
            vv[i] = np.float32(np.float32(mu32 * vv[i]) + np.float32(one * g[i]))
            if nesterov:
                w[i] = np.float32(np.float32(one * w[i]) + np.float32(c_v * vv[i]))
                w[i] = np.float32(np.float32(one * w[i]) + np.float32(c_g * g[i]))
            else:
                w[i] = np.float32(np.float32(one * w[i]) + np.float32(c_g * vv[i]))
    for g in grads:
        layer.grad.values.copy_(dev(g))
        layer.grad_bias.zero_()
        layer.optimize(eta)
    assert bits_equal(host(layer.weights.values), w)
    assert bits_equal(host(layer.velocity.values), vv)


def test_fused_sddmm_update_matches_separate_ops(oracle):
    """smb_sddmm_update == sddmm + row_sums + the Nesterov sparse_combine
    sequence, bit for bit (nn.py:183-198)."""
    rng = np.random.default_rng(8)
    m, k, n = 257, 300, 100
    rp, ci, v, _ = random_csr(rng, m, k, 0.1)
    d = rng.standard_normal((m, n)).astype(np.float32)
    x = rng.standard_normal((k, n)).astype(np.float32)
    vel = rng.standard_normal(v.shape[0]).astype(np.float32)
    bias = rng.standard_normal(m).astype(np.float32)
    vb = rng.standard_normal(m).astype(np.float32)
    eta, mu = 0.01, 0.9
    # oracle sequence
    g = oracle.sddmm(rp, ci, d, x)
    gb = d.sum(axis=1)
    w_o, v_o, b_o, vb_o = v.copy(), vel.copy(), bias.copy(), vb.copy()
    oracle.axpby(mu, v_o, 1.0, g)
    oracle.axpby(1.0, w_o, -eta * mu, v_o)
    oracle.axpby(1.0, w_o, -eta, g)
    vb_o *= np.float32(mu)
    vb_o += gb
    b_o += np.float32(-eta * mu) * vb_o
    b_o += np.float32(-eta) * gb
    # fused kernel
    pat = smb.SparsityPattern(m, k, rp, ci)
    tv, tvel, tb, tvb = dev(v), dev(vel), dev(bias), dev(vb)
    td, tx = dev(d), dev(x)  # keep the operands alive across the async launch
    from paper_2407_17437_b200 import _lib
    _lib.call("smb_sddmm_update", _lib.SMB_F32, pat.handle, tc.ptr(td), n, tc.ptr(tx), n, n,
              tc.ptr(tv), tc.ptr(tvel), None, tc.ptr(tb), tc.ptr(tvb), None,
              _lib.SMB_OPT_NESTEROV, mu, eta, tc.stream_ptr())
    torch.cuda.synchronize()
    for got, want in [(tv, w_o), (tvel, v_o), (tb, b_o), (tvb, vb_o)]:
        assert bits_equal(host(got), want)


def test_relu_and_mask_match_numpy():
    # bit-exact including signed zeros; NaN payloads are unspecified by IEEE
    # (the GPU returns the canonical NaN), so NaNs only need to stay NaN
    def same(a, b):
        nan = np.isnan(a)
        return np.array_equal(nan, np.isnan(b)) and bits_equal(a[~nan], b[~nan])

    x = np.array([[-1.0, -0.0, 0.0, 2.0, np.nan]], np.float32)
    y = host(smb.ReLU().forward(dev(x)))
    assert same(y, np.maximum(x, 0))
    d = np.array([[-3.0, 1.0, -2.0, 4.0, 5.0]], np.float32)
    got = host(smb.ReLU().backward(dev(d), dev(x)))
    assert same(got, d * (x > 0))


def test_xavier_device_matches_numpy_stream():
    from paper_2407_17437_b200.sparsity import Rng
    for seed, n_in, n_out, nnz in [(3, 3072, 1024, 24461), (0, 10, 7, None), (11, 512, 10, 3117)]:
        r1, r2 = Rng(seed).stream("init"), Rng(seed).stream("init")
        a = np.sqrt(6.0 / (n_in + n_out))
        size = n_out * n_in if nnz is None else nnz
        want = r1.uniform(-a, a, size=size).astype(np.float32)
        got = host(smb.xavier_init(n_in, n_out, r2, nnz=nnz))
        assert bits_equal(got, want)
        # the host stream advanced identically
        assert r1.random() == r2.random()


def test_softmax_ce_gradient_tolerance():
    rng = np.random.default_rng(4)
    y = (3 * rng.standard_normal((10, 333))).astype(np.float32)
    lab = rng.integers(0, 10, 333)
    t = np.zeros((10, 333), np.float32)
    t[lab, np.arange(333)] = 1
    z = y - y.max(axis=0, keepdims=True)
    e = np.exp(z)
    want = (e / e.sum(axis=0, keepdims=True) - t) / 333
    got = host(smb.SoftmaxCrossEntropyLoss().gradient_scaled(dev(y), dev(t), 333))
    assert rel_err(got, want) <= 1e-6
    loss_want = float(np.sum(np.log(e.sum(axis=0)) - (z * t).sum(axis=0)))
    assert abs(smb.softmax_ce_loss(dev(y), dev(t)) - loss_want) <= 1e-4 * abs(loss_want)




@pytest.mark.parametrize("relu", [True, False])
def test_spmv_single_column_strided_with_epilogue(oracle, relu):
    """n == 1 (batch-1 inference) through the warp-per-row SpMV, with padded
    leading dimensions (ld 4, like the fused step at B = 1) and bias + ReLU."""
    from paper_2407_17437_b200 import _lib

    rng = np.random.default_rng(3 if relu else 4)
    m, k, ld = 700, 500, 4
    rp, ci, v, _ = random_csr(rng, m, k, 0.15, np.float32, empty_rows=True)
    s = smb.CsrMatrix(m, k, rp, ci, v)
    x = rng.standard_normal((k, 1)).astype(np.float32)
    b = rng.standard_normal(m).astype(np.float32)
    xp = np.zeros((k, ld), np.float32)
    xp[:, :1] = x
    out = torch.full((m, ld), 7.0, device="cuda")
    tx, tb = dev(xp), dev(b)
    _lib.call("smb_spmm", _lib.SMB_F32, tc.ptr(s.row_ptr), tc.ptr(s.col_idx), tc.ptr(s.values),
              m, k, tc.ptr(tx), ld, 1, tc.ptr(tb), _lib.SMB_EPI_RELU if relu else _lib.SMB_EPI_NONE,
              tc.ptr(out), ld, tc.stream_ptr())
    want = oracle.spmm(rp, ci, v, x) + b[:, None]
    if relu:
        want = np.maximum(want, 0)
    got = host(out)
    assert bits_equal(got[:, :1], want)
    assert np.all(got[:, 1:] == 7.0)  # padding columns untouched


@pytest.mark.parametrize("shape,density", [((10, 512, 1024), 0.6), ((7, 300, 777), 0.9),
                                           ((20, 2000, 600), 0.3), ((3, 50, 515), 0.05),
                                           ((10, 512, 100), 0.6), ((5, 1000, 37), 0.4),
                                           ((12, 64, 300), 0.9), ((16, 700, 512), 0.5),
                                           ((4, 300, 64), 0.9), ((6, 1200, 256), 0.5)])
def test_few_long_rows_wide_batch_bit_exact(oracle, shape, density):
    """Few output rows (the output layer): the three-group register-pipelined
    kernel (batch >= 512) and the parallel-products kernel (narrower
    batches, rows of several 128-nonzero segments), forward with bias + ReLU
    and transposed with mask, bit-exact."""
    m, k, n = shape
    rng = np.random.default_rng(m * 7 + n)
    rp, ci, v, _ = random_csr(rng, m, k, density, np.float32, empty_rows=True)
    s = smb.CsrMatrix(m, k, rp, ci, v)
    x = rng.standard_normal((k, n)).astype(np.float32)
    b = rng.standard_normal(m).astype(np.float32)
    got = smb.spmm(s, x, bias=dev(b), relu=True)
    assert bits_equal(got, np.maximum(oracle.spmm(rp, ci, v, x) + b[:, None], 0))
    # transposed over the CSC of a few-column matrix: few output rows again
    st = smb.CsrMatrix(k, m, *random_csr(rng, k, m, density, np.float32)[:3])
    d = rng.standard_normal((k, n)).astype(np.float32)
    mk = rng.standard_normal((m, n)).astype(np.float32)
    rp2, ci2 = tc.to_numpy(st.row_ptr), tc.to_numpy(st.col_idx)
    want = oracle.spmm_t(rp2, ci2, tc.to_numpy(st.values), m, d)
    want = want * (mk > 0)
    assert bits_equal(smb.spmm_transposed(st, d, mask=dev(mk)), want)




@pytest.mark.parametrize("n", [1024, 100, 37])
def test_sddmm_many_waves_long_rows_bit_exact(oracle, n):
    """> 296 tiles of 128 nonzeros whose rows hold >= ~60 nonzeros: the
    warp-independent SDDMM (per-warp staging, no CTA barrier); partial last
    chunks for n = 100 / 37."""
    m, k = 1000, 4000
    rng = np.random.default_rng(n + 11)
    counts = rng.integers(60, 100, size=m)
    rp = np.zeros(m + 1, dtype=np.int32)
    np.cumsum(counts, out=rp[1:])
    ci = np.concatenate([np.sort(rng.choice(k, size=c, replace=False)) for c in counts]).astype(np.int32)
    assert rp[-1] > 296 * 128
    a = rng.standard_normal((m, n)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    got = host(smb.sddmm(smb.SparsityPattern(m, k, rp, ci), dev(a), dev(b)).values)
    assert bits_equal(got, oracle.sddmm(rp, ci, a, b))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("m,k,n", [(10, 512, 1024), (10, 8192, 100), (1, 7, 3), (32, 300, 257),
                                   (17, 1000, 1), (10, 4099, 512), (32, 1000, 64), (5, 77, 12),
                                   (10, 20000, 4)])
@pytest.mark.parametrize("with_mask", [True, False])
def test_dense_backward_input_sequential_sum(dtype, m, k, n, with_mask):
    """smb_dense_backward_input: W^T d summed over ascending rows with
    separate roundings (bit-exact against that sequence on the host), times
    (mask > 0); within BLAS tolerance of numpy's W.T @ d (nn.py:241-255)."""
    from paper_2407_17437_b200 import _lib

    rng = np.random.default_rng(m * 1000 + n)
    w = rng.standard_normal((m, k)).astype(dtype)
    d = rng.standard_normal((m, n)).astype(dtype)
    mk = rng.standard_normal((k, n)).astype(dtype)
    want = np.zeros((k, n), dtype)
    for i in range(m):  # acc = fl(acc + fl(w * d)), ascending i
        want = (want + (w[i][:, None] * d[i][None, :]).astype(dtype)).astype(dtype)
    if with_mask:
        want = want * (mk > 0).astype(dtype)
    tw, td, tm = dev(w), dev(d), dev(mk)
    out = torch.full((k, n), float("nan"), dtype=td.dtype, device="cuda")
    code = _lib.SMB_F32 if dtype == np.float32 else _lib.SMB_F64
    _lib.call("smb_dense_backward_input", code, tc.ptr(tw), k, m, k, tc.ptr(td), n, n,
              tc.ptr(tm) if with_mask else None, n if with_mask else 0, tc.ptr(out), n,
              tc.stream_ptr())
    torch.cuda.synchronize()
    got = host(out)
    assert bits_equal(got, want)
    ref = (w.astype(np.float64).T @ d.astype(np.float64)) * ((mk > 0) if with_mask else 1)
    assert rel_err(got, ref) < (1e-5 if dtype == np.float32 else 1e-12)


@pytest.mark.parametrize("m,k,n", [(10, 512, 1024), (512, 1024, 1024), (64, 300, 100), (40, 90, 37)])
@pytest.mark.parametrize("kind", [0, 3])
def test_sddmm_concurrent_hint_bit_exact(oracle, m, k, n, kind):
    """SMB_HINT_CONCURRENT (the overlapped step's small-footprint staging ring
    for small layers): gradient and Nesterov update bit-identical to the
    oracle / to the launch without the hint."""
    from paper_2407_17437_b200 import _lib
    rng = np.random.default_rng(m * 7 + n)
    rp, ci, v, _ = random_csr(rng, m, k, 0.3 if m < 100 else 0.02, np.float32, empty_rows=True)
    a = rng.standard_normal((m, n)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    pat = smb.SparsityPattern(m, k, rp, ci)
    da, db = dev(a), dev(b)  # kept alive until the launches complete
    outs = []
    for hint in (0, _lib.SMB_HINT_CONCURRENT):
        vals, vel = dev(v.copy()), dev(np.full(v.shape, 0.25, np.float32))
        grad = torch.empty_like(vals)
        _lib.call("smb_sddmm_update_into", _lib.SMB_F32, pat.handle, tc.ptr(da), n,
                  tc.ptr(db), n, n, tc.ptr(vals), tc.ptr(vals), tc.ptr(vel), tc.ptr(grad),
                  None, None, None, kind | hint, 0.9, 0.01, tc.stream_ptr())
        torch.cuda.synchronize()
        outs.append((host(grad), host(vals), host(vel)))
    assert bits_equal(outs[0][0], oracle.sddmm(rp, ci, a, b))
    for x, y in zip(*outs):
        assert bits_equal(x, y)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("features,batch", [(3072, 1024), (130, 37), (100, 64), (7, 5), (256, 1)])
def test_gather_columns_equals_host_gather(dtype, features, batch):
    """smb_gather_columns: dst[f, j] = src[perm[base + j], f] (the host gather
    Xtrain[:, batch] of train.py:390-396), ragged feature / batch tails."""
    from paper_2407_17437_b200 import _lib
    rng = np.random.default_rng(features + batch)
    n = 3 * batch + 5
    src = rng.standard_normal((n, features)).astype(dtype)
    perm = rng.permutation(n).astype(np.int32)
    base = batch + 2
    d_src, d_perm = dev(src), dev(perm)
    ld = batch + 3
    out = torch.full((features, ld), -7.0, dtype=d_src.dtype, device="cuda")
    code = _lib.SMB_F32 if dtype == np.float32 else _lib.SMB_F64
    _lib.call("smb_gather_columns", code, tc.ptr(d_src), n, features, tc.ptr(d_perm), None, base,
              batch, tc.ptr(out), ld, tc.stream_ptr())
    got = host(out)
    assert bits_equal(got[:, :batch], src[perm[base:base + batch]].T)
    assert np.all(got[:, batch:] == -7.0)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", [(1, 1, 1), (17, 13, 5), (512, 1024, 130), (300, 200, 1),
                                   (1000, 700, 257)])
@pytest.mark.parametrize("density", [0.0, 0.05, 1.0])
@pytest.mark.parametrize("with_mask", [False, True])
def test_spmm_t_csc_values_equal_perm_path(dtype, shape, density, with_mask):
    """smb_values_to_csc + smb_spmm_t_csc (the training step's transposed
    SpMM) == smb_spmm_t through perm, bit for bit."""
    from paper_2407_17437_b200 import _lib
    m, k, n = shape
    rng = np.random.default_rng(m + 3 * k + n)
    rp, ci, v, _ = random_csr(rng, m, k, density, dtype, empty_rows=True)
    pat = smb.SparsityPattern(m, k, rp, ci)
    code = _lib.SMB_F32 if dtype == np.float32 else _lib.SMB_F64
    d_v = dev(v) if v.size else torch.zeros(1, dtype=torch.float64 if dtype == np.float64 else torch.float32, device="cuda")
    d = dev(rng.standard_normal((m, n)).astype(dtype))
    mask = dev(rng.standard_normal((k, n)).astype(dtype)) if with_mask else None
    csc = torch.empty_like(d_v)
    _lib.call("smb_values_to_csc", code, pat.handle, tc.ptr(d_v), tc.ptr(csc), tc.stream_ptr())
    outs = []
    for name, vals in (("smb_spmm_t", d_v), ("smb_spmm_t_csc", csc)):
        out = torch.full((k, n), 5.0, dtype=d.dtype, device="cuda")
        _lib.call(name, code, pat.handle, tc.ptr(vals), tc.ptr(d), n, n,
                  tc.ptr(mask) if mask is not None else None, n if mask is not None else 0,
                  tc.ptr(out), n, tc.stream_ptr())
        outs.append(host(out))
    assert bits_equal(outs[0], outs[1])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("m,k,n", [(10, 8192, 1024), (10, 512, 100), (10, 65536, 64), (3, 7, 5),
                                   (32, 300, 257), (17, 1000, 1), (10, 0, 4), (10, 3000, 6)])
def test_dense_forward_small_matches_blas(dtype, m, k, n):
    """smb_dense_forward_small (split-K, fixed order): deterministic and within
    BLAS tolerance of W @ x + b (DenseLinearLayer.forward, nn.py:241-255)."""
    from paper_2407_17437_b200.nn import dense_forward_small
    rng = np.random.default_rng(m * k + n)
    w = rng.standard_normal((m, k)).astype(dtype)
    x = rng.standard_normal((k, n)).astype(dtype)
    b = rng.standard_normal(m).astype(dtype)
    y1 = host(dense_forward_small(dev(w), dev(x), dev(b)))
    y2 = host(dense_forward_small(dev(w), dev(x), dev(b)))
    assert bits_equal(y1, y2)
    want = w.astype(np.float64) @ x.astype(np.float64) + b[:, None]
    # rounding of a k-term fp32 sum grows ~sqrt(k) (cuBLAS / numpy BLAS alike)
    tol = (1e-5 if dtype == np.float32 else 1e-12) * max(1.0, np.sqrt(k) / 16)
    assert rel_err(y1, want) <= tol


@pytest.mark.parametrize("m,k,n", [(10, 8192, 1024), (10, 512, 100), (3, 1000, 37),
                                   (32, 700, 1), (17, 300, 64), (10, 65536, 8)])
@pytest.mark.parametrize("kind", ["none", "nesterov"])
def test_dense_grad_update_is_full_pattern_sddmm(oracle, m, k, n, kind):
    """smb_dense_grad_update (the ER-saturated output layer's weight side,
    DenseLinearLayer.backward + optimize, nn.py:241-264): every gradient
    element is the SDDMM chain of _kernels.py:62-75 over a full pattern --
    bit-identical to the oracle's sddmm of an all-ones CSR pattern -- and the
    fused update follows the exact _step_vector sequence."""
    rng = np.random.default_rng(m * 7 + k + n)
    d = rng.standard_normal((m, n)).astype(np.float32)
    x = rng.standard_normal((k, n)).astype(np.float32)
    w = rng.standard_normal((m, k)).astype(np.float32)
    v = (0.1 * rng.standard_normal((m, k))).astype(np.float32)
    row_ptr = (np.arange(m + 1) * k).astype(np.int32)
    col_idx = np.tile(np.arange(k, dtype=np.int32), m)
    g_ref = oracle.sddmm(row_ptr, col_idx, d, x).reshape(m, k)
    dt, xt = torch.from_numpy(d).cuda(), torch.from_numpy(x).cuda()
    wt, vt = torch.from_numpy(w).cuda(), torch.from_numpy(v).cuda()
    gt = torch.empty(m, k, device="cuda")
    mu, eta = 0.9, 0.05
    opt = _lib.SMB_OPT_NONE if kind == "none" else _lib.SMB_OPT_NESTEROV
    _lib.call("smb_dense_grad_update", _lib.SMB_F32, tc.ptr(dt), n, m, tc.ptr(xt), n, k, n,
              tc.ptr(wt), k, tc.ptr(vt), tc.ptr(gt), opt, mu, eta, tc.stream_ptr())
    torch.cuda.synchronize()
    assert bits_equal(gt.cpu().numpy(), g_ref)
    # within tolerance of the reference's numpy BLAS product d @ x.T
    assert rel_err(gt.cpu().numpy(), d @ x.T) <= 1e-4
    if kind == "nesterov":
        v_ref, w_ref = v.reshape(-1).copy(), w.reshape(-1).copy()
        g = g_ref.reshape(-1)
        oracle.axpby(mu, v_ref, 1.0, g)
        oracle.axpby(1.0, w_ref, -eta * mu, v_ref)
        oracle.axpby(1.0, w_ref, -eta, g)
        assert bits_equal(vt.cpu().numpy().reshape(-1), v_ref)
        assert bits_equal(wt.cpu().numpy().reshape(-1), w_ref)
    else:  # OPT_NONE leaves the parameters alone
        assert bits_equal(wt.cpu().numpy(), w) and bits_equal(vt.cpu().numpy(), v)

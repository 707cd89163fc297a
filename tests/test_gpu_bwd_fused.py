"""smb_backward_fused (csrc/bwd_fused.cu): the transposed SpMM + ReLU.backward
and the SDDMM + optimizer update of one layer in a single CSC-order launch.
Must be BIT-IDENTICAL to the oracle's spmm_t / sddmm / sparse_combine
sequence (_kernels.py:40-83, nn.py:89-91, 183-197) and to the separate
library kernels, on ragged batches, empty columns, fp64, in place and out of
place, with every optimizer kind."""

import numpy as np
import pytest
import torch

from conftest import bits_equal, random_csr

pytestmark = pytest.mark.gpu

import paper_2407_17437_b200 as smb  # noqa: E402
from paper_2407_17437_b200 import _lib  # noqa: E402
from paper_2407_17437_b200 import tensor_core as tc  # noqa: E402
from paper_2407_17437_b200.errors import InvalidArgumentError  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def oracle_backward(oracle, rp, ci, v, vel, d, x, mask, kind, mu, eta):
    """spmm_t (+ mask) with the pre-update weights, then sddmm and the
    sparse_combine sequence of SparseLinearLayer.optimize (nn.py:187-197)."""
    k = x.shape[0]
    dx = oracle.spmm_t(rp, ci, v, k, d)
    if mask:
        dx = dx * (x > 0).astype(dx.dtype)
    g = oracle.sddmm(rp, ci, d, x)
    w, vv = v.copy(), vel.copy()
    if kind == _lib.SMB_OPT_NESTEROV:
        oracle.axpby(mu, vv, 1.0, g)
        oracle.axpby(1.0, w, -eta * mu, vv)
        oracle.axpby(1.0, w, -eta, g)
    elif kind == _lib.SMB_OPT_MOMENTUM:
        oracle.axpby(mu, vv, 1.0, g)
        oracle.axpby(1.0, w, -eta, vv)
    elif kind == _lib.SMB_OPT_GD:
        oracle.axpby(1.0, w, -eta, g)
    return dx, g, w, vv


def run_fused(pat, dtype, d, x, v, vel, mask, kind, mu, eta, inplace, want_grad):
    code = _lib.SMB_F32 if dtype == np.float32 else _lib.SMB_F64
    m, n = d.shape
    k = x.shape[0]
    td, tx = dev(d), dev(x)
    tdx = torch.full((k, n), float("nan"), dtype=td.dtype, device="cuda")
    tv, tvel = dev(v), dev(vel)
    tout = tv if inplace else torch.full_like(tv, float("nan"))
    tg = torch.full_like(tv, float("nan")) if want_grad else None
    _lib.call("smb_backward_fused", code, pat.handle, tc.ptr(td), n, tc.ptr(tx), n, n,
              1 if mask else 0, tc.ptr(tdx), n, tc.ptr(tv), tc.ptr(tout), tc.ptr(tvel),
              tc.ptr(tg) if tg is not None else None, kind, mu, eta, tc.stream_ptr())
    torch.cuda.synchronize()
    return host(tdx), (host(tg) if tg is not None else None), host(tout), host(tvel)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("m,k,n,density", [(300, 400, 1024, 0.05), (129, 257, 100, 0.2),
                                           (64, 96, 37, 0.3), (40, 33, 5, 0.5),
                                           (1000, 700, 256, 0.01), (17, 13, 1, 0.4)])
def test_backward_fused_equals_oracle(oracle, dtype, m, k, n, density):
    rng = np.random.default_rng(m * 7 + n)
    rp, ci, v, _ = random_csr(rng, m, k, density, dtype=dtype, empty_rows=True)
    vel = rng.standard_normal(v.shape[0]).astype(dtype)
    d = rng.standard_normal((m, n)).astype(dtype)
    x = np.maximum(rng.standard_normal((k, n)), 0).astype(dtype)  # post-ReLU input
    mu, eta = 0.9, 0.01
    pat = smb.SparsityPattern(m, k, rp, ci)
    assert _lib.load().smb_backward_fused_supported(
                     _lib.SMB_F32 if dtype == np.float32 else _lib.SMB_F64, pat.handle) == 1
    dx_o, g_o, w_o, v_o = oracle_backward(oracle, rp, ci, v, vel, d, x, True,
                                          _lib.SMB_OPT_NESTEROV, mu, eta)
    dx, _, w, vv = run_fused(pat, dtype, d, x, v, vel, True, _lib.SMB_OPT_NESTEROV, mu, eta,
                             inplace=False, want_grad=False)
    assert bits_equal(dx, dx_o)
    assert bits_equal(w, w_o)
    assert bits_equal(vv, v_o)


@pytest.mark.parametrize("kind", [_lib.SMB_OPT_NONE, _lib.SMB_OPT_GD, _lib.SMB_OPT_MOMENTUM,
                                  _lib.SMB_OPT_NESTEROV])
@pytest.mark.parametrize("inplace", [True, False])
@pytest.mark.parametrize("mask", [True, False])
def test_backward_fused_modes(oracle, kind, inplace, mask):
    rng = np.random.default_rng(kind * 4 + inplace * 2 + mask)
    m, k, n = 700, 900, 200
    rp, ci, v, _ = random_csr(rng, m, k, 0.03)
    vel = rng.standard_normal(v.shape[0]).astype(np.float32)
    d = rng.standard_normal((m, n)).astype(np.float32)
    x = rng.standard_normal((k, n)).astype(np.float32)  # signed: the mask matters
    mu, eta = 0.9, 0.05
    pat = smb.SparsityPattern(m, k, rp, ci)
    dx_o, g_o, w_o, v_o = oracle_backward(oracle, rp, ci, v, vel, d, x, mask, kind, mu, eta)
    dx, g, w, vv = run_fused(pat, np.float32, d, x, v, vel, mask, kind, mu, eta,
                             inplace=inplace, want_grad=True)
    assert bits_equal(dx, dx_o)
    assert bits_equal(g, g_o)
    if kind != _lib.SMB_OPT_NONE:
        assert bits_equal(w, w_o)
        assert bits_equal(vv, v_o)
    elif inplace:
        assert bits_equal(w, v)  # nothing updated


def test_backward_fused_equals_separate_kernels():
    """Same bits as smb_spmm_t + smb_sddmm_update_into (the unfused step)."""
    rng = np.random.default_rng(5)
    m, k, n = 2048, 2048, 512
    rp, ci, v, _ = random_csr(rng, m, k, 0.02, empty_rows=True)
    vel = rng.standard_normal(v.shape[0]).astype(np.float32)
    d = rng.standard_normal((m, n)).astype(np.float32)
    x = np.maximum(rng.standard_normal((k, n)), 0).astype(np.float32)
    pat = smb.SparsityPattern(m, k, rp, ci)
    td, tx = dev(d), dev(x)
    tdx = torch.empty(k, n, device="cuda")
    tv, tvel = dev(v), dev(vel)
    tw = torch.empty_like(tv)
    st = tc.stream_ptr()
    _lib.call("smb_spmm_t", _lib.SMB_F32, pat.handle, tc.ptr(tv), tc.ptr(td), n, n, tc.ptr(tx), n,
              tc.ptr(tdx), n, st)
    _lib.call("smb_sddmm_update_into", _lib.SMB_F32, pat.handle, tc.ptr(td), n, tc.ptr(tx), n, n,
              tc.ptr(tv), tc.ptr(tw), tc.ptr(tvel), None, None, None, None,
              _lib.SMB_OPT_NESTEROV, 0.9, 0.01, st)
    torch.cuda.synchronize()
    dx, _, w, vv = run_fused(pat, np.float32, d, x, v, vel, True, _lib.SMB_OPT_NESTEROV, 0.9,
                             0.01, inplace=False, want_grad=False)
    assert bits_equal(dx, host(tdx))
    assert bits_equal(w, host(tw))
    assert bits_equal(vv, host(tvel))


def test_backward_fused_empty_columns_and_pattern(oracle):
    """Columns without nonzeros give zero rows of d_x; an empty pattern only
    zeroes d_x."""
    m, k, n = 50, 300, 64
    rng = np.random.default_rng(3)
    rp, ci, v, _ = random_csr(rng, m, k, 0.01)
    d = rng.standard_normal((m, n)).astype(np.float32)
    x = np.abs(rng.standard_normal((k, n))).astype(np.float32)
    vel = np.zeros_like(v)
    pat = smb.SparsityPattern(m, k, rp, ci)
    dx_o, _, w_o, _ = oracle_backward(oracle, rp, ci, v, vel, d, x, True, _lib.SMB_OPT_GD, 0.0,
                                      0.1)
    dx, _, w, _ = run_fused(pat, np.float32, d, x, v, vel, True, _lib.SMB_OPT_GD, 0.0, 0.1,
                            inplace=True, want_grad=False)
    assert bits_equal(dx, dx_o) and bits_equal(w, w_o)
    rp0 = np.zeros(m + 1, dtype=np.int32)
    pat0 = smb.SparsityPattern(m, k, rp0, np.zeros(0, dtype=np.int32))
    dx0, _, _, _ = run_fused(pat0, np.float32, d, x, np.zeros(0, np.float32),
                             np.zeros(0, np.float32), True, _lib.SMB_OPT_GD, 0.0, 0.1,
                             inplace=True, want_grad=False)
    assert bits_equal(dx0, np.zeros((k, n), np.float32))


def test_backward_fused_rejects_long_columns():
    """A column with > 256 nonzeros: unsupported, with the reference's error type."""
    m, k, n = 400, 8, 16
    rp = np.arange(0, m * k + 1, k, dtype=np.int32)  # dense 400 x 8: columns of 400
    ci = np.tile(np.arange(k, dtype=np.int32), m)
    pat = smb.SparsityPattern(m, k, rp, ci)
    assert _lib.load().smb_backward_fused_supported( _lib.SMB_F32, pat.handle) == 0
    d = torch.zeros(m, n, device="cuda")
    x = torch.zeros(k, n, device="cuda")
    v = torch.zeros(m * k, device="cuda")
    with pytest.raises(InvalidArgumentError):
        _lib.call("smb_backward_fused", _lib.SMB_F32, pat.handle, tc.ptr(d), n, tc.ptr(x), n, n,
                  1, tc.ptr(x), n, tc.ptr(v), tc.ptr(v), None, None, _lib.SMB_OPT_GD, 0.0, 0.1,
                  tc.stream_ptr())

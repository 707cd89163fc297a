"""Layers, loss and optimizers on device-resident state.

Drop-in for pkg/src/sparsemlp/nn.py (same classes, attributes, call order and
exception types).  Activations are feature-major ``[features, batch]`` CUDA
tensors (nn.py:3-8); numpy inputs are accepted and uploaded.  Every
arithmetic step runs in the sm_100a library:

    SparseLinearLayer.forward   spmm (+bias fused)                     nn.py:169-176
    SparseLinearLayer.backward  sddmm, row_sums, spmm_transposed       nn.py:178-185
    SparseLinearLayer.optimize  smb_optimizer_step (sparse_combine
                                order, bit-identical)                  nn.py:187-198
    ReLU forward/backward       smb_relu / smb_relu_backward           nn.py:83-95
    softmax CE gradient / loss  smb_softmax_ce_grad                    nn.py:385-432

Dense (saturated) layers use cuBLAS FP32 GEMMs with TF32 disabled -- the
reference runs them through numpy BLAS (nn.py:241-255), so they are
tolerance-exact, not bit-exact, on both sides.  BatchNorm and Dropout are not
part of this hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import InvalidArgumentError, StateError
from .tensor_core import (
    SparsityPattern,
    _TORCH_TO_NP,
    _no_tf32,
    _values_tensor,
    device,
    dtype_code,
    ptr,
    row_sums,
    sddmm,
    spmm,
    spmm_transposed,
    stream_ptr,
)

__all__ = [
    "GradientDescent",
    "Momentum",
    "ReLU",
    "NoActivation",
    "SparseLinearLayer",
    "DenseLinearLayer",
    "ActivationLayer",
    "SoftmaxCrossEntropyLoss",
    "softmax_columns",
    "softmax_ce_loss",
    "softmax_ce_gradient",
    "optimizer_kind",
]


class GradientDescent:
    """Plain SGD step: w <- w - eta * g."""

    mu = 0.0
    nesterov = False
    uses_velocity = False

    def __repr__(self):
        return "GradientDescent()"

    def to_dict(self):
        return {"kind": "gd"}


class Momentum:
    """v <- mu*v + g, then w <- w - eta*v, or Nesterov w <- w - eta*(g + mu*v)."""

    uses_velocity = True

    def __init__(self, mu: float, nesterov: bool = False):
        if not 0.0 <= mu < 1.0:
            raise InvalidArgumentError(f"momentum coefficient must be in [0, 1), got {mu}")
        self.mu = float(mu)
        self.nesterov = bool(nesterov)

    def __repr__(self):
        return f"Momentum({self.mu}, nesterov={self.nesterov})"

    def to_dict(self):
        return {"kind": "momentum", "mu": self.mu, "nesterov": self.nesterov}


def optimizer_from_dict(d: dict):
    if d["kind"] == "gd":
        return GradientDescent()
    if d["kind"] == "momentum":
        return Momentum(d["mu"], d.get("nesterov", False))
    raise InvalidArgumentError(f"unknown optimizer kind {d['kind']!r}")


def optimizer_kind(opt) -> int:
    if not opt.uses_velocity:
        return _lib.SMB_OPT_GD
    return _lib.SMB_OPT_NESTEROV if opt.nesterov else _lib.SMB_OPT_MOMENTUM


def _step(param: torch.Tensor, grad: torch.Tensor, velocity, opt, eta: float) -> None:
    """The sparse_combine / _step_vector arithmetic (nn.py:118-131, 187-197) on
    a flat parameter, bit-identical to the reference's rounding sequence."""
    n = param.numel()
    if n == 0:
        return
    _lib.call(
        "smb_optimizer_step", dtype_code(param.dtype), ptr(param), ptr(velocity), ptr(grad), n,
        optimizer_kind(opt), float(opt.mu), float(eta), stream_ptr(),
    )
    # the kernel wrote through a raw pointer: bump the tensor's version like
    # an in-place torch op would, so FusedTrainStep sees the changed weights
    torch.autograd.graph.increment_version(param)


def _act(x, rows: int, dtype: torch.dtype) -> torch.Tensor:
    """Validated device activation [rows, batch] of the layer dtype."""
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor) or x.dim() != 2:
        raise InvalidArgumentError("activations must be 2-D [features, batch]")
    if x.shape[0] != rows:
        raise InvalidArgumentError(f"expected {rows} input rows, got {x.shape[0]}")
    if x.dtype != dtype:
        x = x.to(dtype)
    return x.to(device())


class ReLU:
    name = "relu"

    def forward(self, x):
        x = _act(x, x.shape[0], x.dtype if isinstance(x, torch.Tensor) else torch.float32)
        y = torch.empty((x.shape[0], x.shape[1]), dtype=x.dtype, device=x.device)
        if x.numel():
            _lib.call("smb_relu", dtype_code(x.dtype), ptr(x), _ld(x), x.shape[0], x.shape[1],
                      ptr(y), _ld(y), stream_ptr())
        return y

    def backward(self, d_out, x_cached):
        d = _act(d_out, d_out.shape[0], x_cached.dtype)
        out = torch.empty((d.shape[0], d.shape[1]), dtype=d.dtype, device=d.device)
        if d.numel():
            _lib.call("smb_relu_backward", dtype_code(d.dtype), ptr(d), _ld(d), ptr(x_cached),
                      _ld(x_cached), d.shape[0], d.shape[1], ptr(out), _ld(out), stream_ptr())
        return out

    def __repr__(self):
        return "ReLU()"


class NoActivation:
    name = "none"

    def forward(self, x):
        return x

    def backward(self, d_out, x_cached):
        return d_out

    def __repr__(self):
        return "NoActivation()"


def activation_from_name(name: str):
    if name == "relu":
        return ReLU()
    if name == "none":
        return NoActivation()
    raise InvalidArgumentError(f"unknown activation {name!r}")


def _ld(t: torch.Tensor) -> int:
    return int(t.stride(0)) if t.shape[0] > 1 else max(int(t.shape[1]), 1)


class SparseLinearLayer:
    """Linear layer with truly sparse weights on a fixed pattern; weights, grad
    and velocity share one SparsityPattern (and its CSC index) for the whole
    run; the bias is dense (nn.py:134-198)."""

    kind = "sparse"

    def __init__(self, pattern: SparsityPattern, values, bias, optimizer=None):
        self.n_out = pattern.nrows
        self.n_in = pattern.ncols
        vals = _values_tensor(values)
        if vals.shape[0] != pattern.nnz:
            raise InvalidArgumentError("values length must equal pattern nnz")
        self.weights = pattern.with_values(vals)
        b = _values_tensor(bias).to(vals.dtype)
        if tuple(b.shape) != (self.n_out,):
            raise InvalidArgumentError(f"bias must have shape ({self.n_out},)")
        self.bias = b.clone()
        np_dt = _TORCH_TO_NP[vals.dtype]
        self.grad = pattern.zeros(dtype=np_dt)
        self.grad_bias = torch.zeros(self.n_out, dtype=vals.dtype, device=vals.device)
        self.optimizer = optimizer or GradientDescent()
        uv = self.optimizer.uses_velocity
        self.velocity = pattern.zeros(dtype=np_dt) if uv else None
        self.velocity_bias = torch.zeros_like(self.grad_bias) if uv else None
        self._cached_input = None

    @property
    def dtype(self):
        return self.weights.dtype

    @property
    def density(self):
        return self.weights.nnz / (self.n_in * self.n_out)

    def forward(self, x, training=True):
        x = _act(x, self.n_in, self.weights.values.dtype)
        y = spmm(self.weights, x, bias=self.bias)
        if training:
            self._cached_input = x
        return y

    def backward(self, d_out):
        x = self._cached_input
        if x is None:
            raise StateError("backward called before forward")
        d = _act(d_out, self.n_out, self.weights.values.dtype)
        sddmm(self.weights.pattern, d, x, out=self.grad)
        self.grad_bias = row_sums(d)
        return spmm_transposed(self.weights, d)

    def optimize(self, eta):
        v = self.velocity.values if self.velocity is not None else None
        _step(self.weights.values, self.grad.values, v, self.optimizer, eta)
        _step(self.bias, self.grad_bias, self.velocity_bias, self.optimizer, eta)


# output layers up to this many rows take smb_dense_backward_input for W^T d
# and (unmasked) smb_dense_forward_small for W x + b
DENSE_T_MAX_ROWS = 32


def dense_forward_small(w, x, bias, out=None, workspace=None, stream=None):
    """y = w @ x + bias for m <= DENSE_T_MAX_ROWS rows (smb_dense_forward_small:
    deterministic split-K; the reference's numpy BLAS order is unspecified,
    nn.py:241-255).  x is [k, n] with a unit column stride."""
    m, k = w.shape
    n = x.shape[1]
    if n > 1 and (x.stride(1) != 1 or (k > 1 and x.stride(0) < n)):
        x = x.contiguous()  # the kernel reads rows of unit column stride
    if out is None:
        out = torch.empty((m, n), dtype=w.dtype, device=w.device)
    if workspace is None:
        nb = int(_lib.load().smb_dense_forward_workspace_bytes(m, k, n))
        workspace = torch.empty(nb, dtype=torch.uint8, device=w.device)
    _lib.call("smb_dense_forward_small", dtype_code(w.dtype), ptr(w), w.stride(0), m, k, ptr(x),
              x.stride(0), n, ptr(bias), ptr(out), out.stride(0), ptr(workspace),
              stream if stream is not None else stream_ptr())
    return out


class DenseLinearLayer:
    """Dense linear layer; with a mask it is the masked-sparse baseline
    (nn.py:201-264).  Weights are an [n_out, n_in] CUDA tensor."""

    kind = "dense"

    def __init__(self, weights, bias, optimizer=None, mask=None):
        w = _values_tensor(weights)
        if w.dim() != 2:
            raise InvalidArgumentError("weights must be 2-D")
        self.weights = w.clone()
        self.n_out, self.n_in = self.weights.shape
        b = _values_tensor(bias).to(w.dtype)
        if tuple(b.shape) != (self.n_out,):
            raise InvalidArgumentError(f"bias must have shape ({self.n_out},)")
        self.bias = b.clone()
        self.mask = None if mask is None else _values_tensor(mask).to(w.dtype)
        if self.mask is not None and self.mask.shape != self.weights.shape:
            raise InvalidArgumentError("mask shape must match weights")
        self.grad = torch.zeros_like(self.weights)
        self.grad_bias = torch.zeros(self.n_out, dtype=w.dtype, device=w.device)
        self.optimizer = optimizer or GradientDescent()
        uv = self.optimizer.uses_velocity
        self.velocity = torch.zeros_like(self.weights) if uv else None
        self.velocity_bias = torch.zeros_like(self.grad_bias) if uv else None
        self._cached_input = None

    @property
    def dtype(self):
        return _TORCH_TO_NP[self.weights.dtype]

    @property
    def density(self):
        if self.mask is None:
            return 1.0
        return float(torch.count_nonzero(self.mask)) / (self.n_in * self.n_out)

    def forward(self, x, training=True):
        x = _act(x, self.n_in, self.weights.dtype)
        if self.n_out <= DENSE_T_MAX_ROWS and self.mask is None:
            # small (ER-saturated output) layer: the fused step's split-K kernel
            y = dense_forward_small(self.weights, x, self.bias)
        else:
            with _no_tf32():
                y = torch.addmm(self.bias[:, None], self.weights, x)
        if training:
            self._cached_input = x
        return y

    def backward(self, d_out):
        x = self._cached_input
        if x is None:
            raise StateError("backward called before forward")
        d = _act(d_out, self.n_out, self.weights.dtype)
        small = self.n_out <= DENSE_T_MAX_ROWS and self.mask is None
        if small:
            # ER-saturated output layer: one sequential chain per gradient
            # element (smb_dense_grad_update, the fused step's kernel; numpy
            # BLAS order is unspecified, nn.py:241-255)
            d = d.contiguous()
            if x.shape[1] > 1 and (x.stride(1) != 1 or x.stride(0) < x.shape[1]):
                x = x.contiguous()
            self.grad = torch.empty_like(self.weights)
            _lib.call("smb_dense_grad_update", dtype_code(d.dtype), ptr(d), _ld(d), self.n_out,
                      ptr(x), _ld(x), self.n_in, d.shape[1], None, self.n_in, None,
                      ptr(self.grad), _lib.SMB_OPT_NONE, 0.0, 0.0, stream_ptr())
        with _no_tf32():
            if not small:
                self.grad = d @ x.T
            if self.mask is not None:
                self.grad *= self.mask
            if self.n_out > DENSE_T_MAX_ROWS:
                dx = self.weights.T @ d
        if self.n_out <= DENSE_T_MAX_ROWS:
            # small output layer: the same kernel as the fused step (ascending
            # rows, separately rounded; numpy BLAS order is unspecified)
            d = d.contiguous()
            dx = torch.empty((self.n_in, d.shape[1]), dtype=d.dtype, device=d.device)
            _lib.call("smb_dense_backward_input", dtype_code(d.dtype), ptr(self.weights),
                      self.n_in, self.n_out, self.n_in, ptr(d), d.shape[1], d.shape[1], None, 0,
                      ptr(dx), d.shape[1], stream_ptr())
        self.grad_bias = row_sums(d)
        return dx

    def optimize(self, eta):
        vel = None if self.velocity is None else self.velocity.view(-1)
        if self.mask is None:
            _step(self.weights.view(-1), self.grad.contiguous().view(-1), vel, self.optimizer, eta)
        else:
            # velocity *= mask; _step_vector; weights *= mask (nn.py:258-263), one pass
            opt = self.optimizer
            _lib.call("smb_masked_optimizer_step", dtype_code(self.weights.dtype),
                      ptr(self.weights), ptr(vel), ptr(self.grad.contiguous()), ptr(self.mask),
                      self.weights.numel(), optimizer_kind(opt), float(opt.mu), float(eta),
                      stream_ptr())
        _step(self.bias, self.grad_bias, self.velocity_bias, self.optimizer, eta)


class ActivationLayer:
    kind = "activation"

    def __init__(self, fn):
        self.fn = fn
        self._cached_input = None

    def forward(self, x, training=True):
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x)).to(device())
        if training:
            self._cached_input = x
        return self.fn.forward(x)

    def backward(self, d_out):
        if self._cached_input is None:
            raise StateError("backward called before forward")
        return self.fn.backward(d_out, self._cached_input)

    def optimize(self, eta):
        pass


# ---------------------------------------------------------------------------
# softmax cross-entropy (nn.py:385-432)
# ---------------------------------------------------------------------------
def _ce_call(y, t, divisor):
    if tuple(y.shape) != tuple(t.shape):
        raise InvalidArgumentError(f"shape mismatch: {tuple(y.shape)} vs {tuple(t.shape)}")
    yd = _act(y, y.shape[0], y.dtype if isinstance(y, torch.Tensor) else torch.float32)
    td = _act(t, t.shape[0], yd.dtype)
    d = torch.empty((yd.shape[0], yd.shape[1]), dtype=yd.dtype, device=yd.device)
    loss = torch.zeros(1, dtype=torch.float64, device=yd.device)
    _lib.call("smb_softmax_ce_grad", dtype_code(yd.dtype), ptr(yd), _ld(yd), ptr(td), _ld(td),
              yd.shape[0], yd.shape[1], float(divisor), ptr(d), _ld(d), ptr(loss), stream_ptr())
    return d, loss


def _check_one_hot(t):
    t = torch.as_tensor(t)
    if not (bool(((t == 0) | (t == 1)).all()) and bool((t.sum(dim=0) == 1).all())):
        raise InvalidArgumentError("target columns must be one-hot")


def softmax_columns(y):
    """Columnwise softmax with max subtraction."""
    yt = torch.as_tensor(y)
    z = yt - yt.max(dim=0, keepdim=True).values
    e = torch.exp(z)
    return e / e.sum(dim=0, keepdim=True)


def softmax_ce_loss(y, t, check_targets: bool = False) -> float:
    """Softmax cross-entropy summed over the batch (the loop divides by B)."""
    if check_targets:
        _check_one_hot(t)
    _, loss = _ce_call(y, t, 1.0)
    return float(loss.item())


def softmax_ce_gradient(y, t, check_targets: bool = False):
    """softmax(y) - t, columnwise."""
    if check_targets:
        _check_one_hot(t)
    d, _ = _ce_call(y, t, 1.0)
    return d


class SoftmaxCrossEntropyLoss:
    """Object form of the loss (nn.py:420-432)."""

    def __call__(self, y, t):
        return softmax_ce_loss(y, t)

    loss = __call__

    def gradient(self, y, t):
        return softmax_ce_gradient(y, t)

    def gradient_scaled(self, y, t, divisor):
        """(softmax(y) - t) / divisor in one kernel (train.py:399)."""
        d, _ = _ce_call(y, t, divisor)
        return d

    def __repr__(self):
        return "SoftmaxCrossEntropyLoss()"

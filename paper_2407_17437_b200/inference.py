"""Batch-1 (small-batch) inference on the GPU.

Replaces the reference's single-example latency path (bench.py:366-399:
``model.feedforward(x)`` on a [features, 1] column in eval mode).
``InferenceSession`` keeps every buffer resident and captures ONE CUDA graph
per session: the pinned-host -> HBM copy of the input, the forward chain
(smb_spmm with bias + ReLU fused per sparse layer; smb_dense_forward_small for
small dense output layers, cuBLAS FP32 for other dense /
masked-dense layers) and the HBM -> pinned-host copy of the logits.  A call
is one graph replay plus one stream synchronisation.  Results are bit-identical
to ``Sequential.feedforward`` (same kernels, same rounding order).
"""

from __future__ import annotations

import time

import numpy as np
import torch

from . import _lib
from .errors import InvalidArgumentError
from .nn import (DENSE_T_MAX_ROWS, ActivationLayer, DenseLinearLayer, ReLU,
                 SparseLinearLayer, dense_forward_small)
from .sparsity import Rng
from .tensor_core import _no_tf32, ptr, stream_ptr

__all__ = ["InferenceSession", "bench_inference"]


class InferenceSession:
    """Graph-captured forward pass of a compiled model for a fixed batch."""

    def __init__(self, model, batch: int = 1, use_graph: bool = True):
        model._require_compiled()
        if batch <= 0:
            raise InvalidArgumentError("batch must be positive")
        self.model = model
        self.B = int(batch)
        self.units = []  # (layer, relu)
        layers = list(model.layers)
        i = 0
        while i < len(layers):
            lay = layers[i]
            if not isinstance(lay, (SparseLinearLayer, DenseLinearLayer)):
                raise InvalidArgumentError(
                    f"inference supports Sparse/Dense layers (+ReLU), got {type(lay).__name__}")
            relu = False
            if i + 1 < len(layers) and isinstance(layers[i + 1], ActivationLayer):
                relu = isinstance(layers[i + 1].fn, ReLU)
                i += 1
            self.units.append((lay, relu))
            i += 1
        dev = self.units[0][0].bias.device
        dt = self.units[0][0].bias.dtype
        self.dtype = dt
        n_in = self.units[0][0].n_in
        self.x = torch.zeros((n_in, self.B), dtype=dt, device=dev)
        self.acts = [torch.zeros((lay.n_out, self.B), dtype=dt, device=dev)
                     for lay, _ in self.units]
        self.x_host = torch.zeros((n_in, self.B), dtype=dt).pin_memory()
        self.y_host = torch.zeros((self.units[-1][0].n_out, self.B), dtype=dt).pin_memory()
        self._xh, self._yh = self.x_host.numpy(), self.y_host.numpy()
        # split-K workspace of the small (ER-saturated output) dense layers
        nb = max([int(_lib.load().smb_dense_forward_workspace_bytes(l.n_out, l.n_in, self.B))
                  for l, _ in self.units if isinstance(l, DenseLinearLayer)
                  and l.n_out <= DENSE_T_MAX_ROWS and l.mask is None] or [0])
        self._dws = torch.empty(nb, dtype=torch.uint8, device=dev) if nb else None
        self.use_graph = use_graph
        self._graph = None
        self._stream = torch.cuda.Stream(device=dev)

    def _enqueue(self) -> None:
        B = self.B
        code = _lib.SMB_F32 if self.dtype == torch.float32 else _lib.SMB_F64
        self.x.copy_(self.x_host, non_blocking=True)
        x = self.x
        st = stream_ptr()
        for (lay, relu), a in zip(self.units, self.acts):
            if isinstance(lay, SparseLinearLayer):
                w = lay.weights
                _lib.call("smb_spmm", code, ptr(w.row_ptr), ptr(w.col_idx), ptr(w.values),
                          lay.n_out, lay.n_in, ptr(x), B, B, ptr(lay.bias),
                          _lib.SMB_EPI_RELU if relu else _lib.SMB_EPI_NONE, ptr(a), B, st)
            else:
                if lay.n_out <= DENSE_T_MAX_ROWS and lay.mask is None:
                    # the same kernel as DenseLinearLayer.forward / the step
                    dense_forward_small(lay.weights, x, lay.bias, out=a, workspace=self._dws,
                                        stream=st)
                else:
                    with _no_tf32():
                        torch.addmm(lay.bias[:, None], lay.weights, x, out=a)
                if relu:
                    _lib.call("smb_relu", code, ptr(a), B, lay.n_out, B, ptr(a), B, st)
            x = a
        self.y_host.copy_(self.acts[-1], non_blocking=True)

    def __call__(self, x) -> np.ndarray:
        """Logits [classes, batch] on the host for input x [features, batch]."""
        xh = self._xh
        if getattr(x, "shape", None) != xh.shape:
            raise InvalidArgumentError(
                f"expected input of shape {xh.shape}, got {getattr(x, 'shape', None)}")
        xh[...] = x
        cur = torch.cuda.current_stream()
        if self._graph is not None:
            self._graph.replay()  # replays on the current stream
        elif not self.use_graph:
            self._enqueue()
        else:
            self._stream.wait_stream(cur)
            with torch.cuda.stream(self._stream):
                self._enqueue()  # eager warm-up on the captured stream
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self._stream):
                    self._enqueue()
                self._graph = g
            cur.wait_stream(self._stream)
            g.replay()
        cur.synchronize()
        return self._yh.copy()


def bench_inference(config, n_repeats: int = 100, warmup: int = 10, model=None) -> dict:
    """Latency of a single-example forward pass (bench.py:366-399): host wall
    clock around each call, input copy and logits read-back included."""
    if n_repeats < 1:
        raise InvalidArgumentError("n_repeats must be >= 1")
    if model is None:
        from .experiment import build_model

        model, _ = build_model(config)
    model.eval_mode()
    x = Rng(config.seed).stream("data").standard_normal((model.input_size, 1)).astype(
        np.dtype(model.dtype))
    sess = InferenceSession(model, batch=1)
    for _ in range(warmup):
        sess(x)
    times = np.empty(n_repeats)
    for i in range(n_repeats):
        t0 = time.perf_counter()
        sess(x)
        times[i] = time.perf_counter() - t0
    times *= 1e3
    return {
        "backend": config.backend,
        "density": config.density,
        "layer_dims": list(config.layer_dims),
        "repeats": n_repeats,
        "mean_ms": float(times.mean()),
        "median_ms": float(np.median(times)),
        "min_ms": float(times.min()),
        "max_ms": float(times.max()),
    }

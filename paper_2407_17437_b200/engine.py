"""Fused, graph-captured training step (one pass of sgd_train's hot loop).

One call of ``FusedTrainStep.step()`` performs, entirely on the GPU, the body
of the reference's per-batch loop (train.py:389-402):

    gather      xb = Xtrain[:, batch], tb = Ttrain[:, batch]    smb_gather_columns
    forward     a_l = relu(W_l a_{l-1} + b_l)                   smb_spmm (bias+ReLU fused)
    loss grad   d_L = (softmax(y) - t) / B                      smb_softmax_ce_grad
    backward    d_{l-1} = (W_l^T d_l) * (a_{l-1} > 0)           smb_spmm_t (mask fused)
                grad_l = sddmm(d_l, a_{l-1}); update W_l, b_l   smb_sddmm_update (fused)
    next batch  step counter += 1                               smb_step_counter_advance

spmm_t of layer l runs before the update of layer l (pre-update weights,
train.py:400-401).  The layer-1 input gradient is never computed: the
reference computes and discards it (train.py:216-220).  Dense (ER-saturated)
layers use cuBLAS FP32 (TF32 off) plus the same exact bias/optimizer kernels.

The kernel sequence is captured once into a CUDA graph per learning rate and
replayed (a step is ~10 launches; replay removes the host launch cost).

Data parallel (``process_group`` with world size G > 1): every rank runs the
step on its B/G slice of the same global batch; the loss gradient is scaled
by 1/B_global; the value, dense-weight and bias gradients of all layers land
in ONE flat fp32 buffer that is summed with a single NCCL all-reduce, after
which every rank applies the identical update.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import ConfigurationError, InvalidArgumentError
from .nn import ActivationLayer, DenseLinearLayer, ReLU, SparseLinearLayer, optimizer_kind
from .tensor_core import _no_tf32, ptr, stream_ptr

__all__ = ["FusedTrainStep"]


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


class _Unit:
    __slots__ = ("layer", "relu", "sparse", "m", "k", "grad_off", "bias_off", "nvals")

    def __init__(self, layer, relu):
        self.layer = layer
        self.relu = relu
        self.sparse = isinstance(layer, SparseLinearLayer)
        self.m = layer.n_out
        self.k = layer.n_in
        self.nvals = layer.weights.nnz if self.sparse else self.m * self.k


class FusedTrainStep:
    def __init__(self, model, batch_size: int, global_batch: int | None = None,
                 process_group=None, use_graph: bool = True):
        self.units = self._parse(model)
        self.model = model
        self.B = int(batch_size)
        self.B_global = int(global_batch or batch_size)
        if self.B <= 0:
            raise InvalidArgumentError("batch_size must be positive")
        self.pg = process_group
        self.world = 1
        if process_group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(process_group)
        self.use_graph = use_graph
        dev = self.units[0].layer.bias.device
        self.dev = dev
        ld = _round_up(self.B, 4)
        self.ld = ld
        f32 = torch.float32
        self.n_in = self.units[0].k
        self.classes = self.units[-1].m
        self.x_in = torch.zeros((self.n_in, ld), dtype=f32, device=dev)
        self.t_in = torch.zeros((self.classes, ld), dtype=f32, device=dev)
        self.acts = [torch.zeros((u.m, ld), dtype=f32, device=dev) for u in self.units]
        self.dys = [torch.zeros((u.m, ld), dtype=f32, device=dev) for u in self.units]
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.counter = torch.zeros(1, dtype=torch.int32, device=dev)
        self.perm = None
        self.data = None
        self.steps_per_epoch = 0
        # scratch for dense layers' bias gradient
        self._dense_gb = {id(u): torch.zeros(u.m, dtype=f32, device=dev)
                          for u in self.units if not u.sparse}
        # data-parallel flat gradient buffer: [values | bias] per layer
        self.flat = None
        if self.world > 1:
            off = 0
            for u in self.units:
                u.grad_off = off
                off += u.nvals
                u.bias_off = off
                off += u.m
            self.flat = torch.zeros(off, dtype=f32, device=dev)
        self._graphs = {}

    # ------------------------------------------------------------------
    @staticmethod
    def _parse(model):
        layers = list(model.layers)
        units = []
        i = 0
        while i < len(layers):
            lay = layers[i]
            if not isinstance(lay, (SparseLinearLayer, DenseLinearLayer)):
                raise ConfigurationError(
                    f"fused step supports Sparse/Dense layers with ReLU only, got {type(lay).__name__}")
            if isinstance(lay, DenseLinearLayer) and lay.mask is not None:
                raise ConfigurationError("fused step does not run the masked-dense baseline")
            relu = False
            if i + 1 < len(layers) and isinstance(layers[i + 1], ActivationLayer):
                if not isinstance(layers[i + 1].fn, ReLU):
                    raise ConfigurationError("fused step supports ReLU activations only")
                relu = True
                i += 1
            if lay.weights.dtype not in (np.float32, torch.float32):
                raise ConfigurationError("fused step runs float32 models")
            units.append(_Unit(lay, relu))
            i += 1
        if not units:
            raise ConfigurationError("model has no linear layers")
        return units

    # ------------------------------------------------------------------
    def attach_dataset(self, ddata) -> None:
        """Gather batches on the device from a DeviceDataset."""
        if ddata.features != self.n_in or ddata.classes != self.classes:
            raise InvalidArgumentError("dataset shape does not match the model")
        self.data = ddata
        self._graphs.clear()

    def set_epoch(self, perm: np.ndarray, rank_offset: int = 0) -> None:
        """Upload the epoch's sample order; this rank's batch k is
        perm[k*B_global + rank_offset : ... + B]."""
        p = np.ascontiguousarray(perm, dtype=np.int64)
        kb = p.shape[0] // self.B_global
        # lay the rank's slices out contiguously so batch k starts at k*B
        idx = p[: kb * self.B_global].reshape(kb, self.B_global)[:, rank_offset:rank_offset + self.B]
        flat = torch.from_numpy(np.ascontiguousarray(idx.reshape(-1)).astype(np.int32))
        if self.perm is None or self.perm.numel() != flat.numel():
            self.perm = torch.empty(flat.numel(), dtype=torch.int32, device=self.dev)
            self._graphs.clear()
        self.perm.copy_(flat)
        self.counter.zero_()
        self.steps_per_epoch = kb

    # ------------------------------------------------------------------
    def _launch_forward_backward(self, eta: float, fuse_update: bool, gather: bool) -> None:
        st = stream_ptr()
        B, ld = self.B, self.ld
        F32 = _lib.SMB_F32
        if gather:
            d = self.data
            _lib.call("smb_gather_columns", F32, ptr(d.X), d.n_samples, d.features, ptr(self.perm),
                      ptr(self.counter), 0, B, ptr(self.x_in), ld, st)
            _lib.call("smb_gather_columns", F32, ptr(d.T), d.n_samples, d.classes, ptr(self.perm),
                      ptr(self.counter), 0, B, ptr(self.t_in), ld, st)
        # forward
        x = self.x_in
        for u, a in zip(self.units, self.acts):
            lay = u.layer
            if u.sparse:
                _lib.call("smb_spmm", F32, ptr(lay.weights.row_ptr), ptr(lay.weights.col_idx),
                          ptr(lay.weights.values), u.m, u.k, ptr(x), ld, B, ptr(lay.bias),
                          _lib.SMB_EPI_RELU if u.relu else _lib.SMB_EPI_NONE, ptr(a), ld, st)
            else:
                with _no_tf32():
                    torch.addmm(lay.bias[:, None], lay.weights, x[:, :B], out=a[:, :B])
                if u.relu:
                    _lib.call("smb_relu", F32, ptr(a), ld, u.m, B, ptr(a), ld, st)
            x = a
        # loss gradient (softmax CE), scaled by 1/B_global
        _lib.call("smb_softmax_ce_grad", F32, ptr(self.acts[-1]), ld, ptr(self.t_in), ld,
                  self.classes, B, float(self.B_global), ptr(self.dys[-1]), ld, ptr(self.loss), st)
        # backward, last layer first
        for li in range(len(self.units) - 1, -1, -1):
            u = self.units[li]
            lay = u.layer
            dy = self.dys[li]
            x_prev = self.acts[li - 1] if li > 0 else self.x_in
            if li > 0:
                below = self.units[li - 1]
                mask = self.acts[li - 1] if below.relu else None
                if u.sparse:
                    _lib.call("smb_spmm_t", F32, lay.weights.pattern.handle, ptr(lay.weights.values),
                              ptr(dy), ld, B, ptr(mask), ld if mask is not None else 0,
                              ptr(self.dys[li - 1]), ld, st)
                else:
                    dst = self.dys[li - 1]
                    with _no_tf32():
                        torch.mm(lay.weights.T, dy[:, :B], out=dst[:, :B])
                    if mask is not None:
                        _lib.call("smb_relu_backward", F32, ptr(dst), ld, ptr(mask), ld, u.k, B,
                                  ptr(dst), ld, st)
            self._weight_side(u, dy, x_prev, eta, fuse_update, st)

    def _weight_side(self, u, dy, x_prev, eta, fuse_update, st):
        lay = u.layer
        B, ld = self.B, self.ld
        F32 = _lib.SMB_F32
        opt = lay.optimizer
        kind = optimizer_kind(opt) if fuse_update else _lib.SMB_OPT_NONE
        if u.sparse:
            vel = lay.velocity.values if lay.velocity is not None else None
            g_out = None if fuse_update else self.flat[u.grad_off:u.grad_off + u.nvals]
            gb_out = None if fuse_update else self.flat[u.bias_off:u.bias_off + u.m]
            _lib.call("smb_sddmm_update", F32, lay.weights.pattern.handle, ptr(dy), ld, ptr(x_prev),
                      ld, B, ptr(lay.weights.values), ptr(vel), ptr(g_out), ptr(lay.bias),
                      ptr(lay.velocity_bias), ptr(gb_out), kind, float(opt.mu), float(eta), st)
            return
        # dense layer: cuBLAS gradient, exact pairwise bias sum, exact update
        if fuse_update:
            gw = lay.grad
            gb = self._dense_gb[id(u)]
        else:
            gw = self.flat[u.grad_off:u.grad_off + u.nvals].view(u.m, u.k)
            gb = self.flat[u.bias_off:u.bias_off + u.m]
        with _no_tf32():
            torch.mm(dy[:, :B], x_prev[:, :B].T, out=gw)
        _lib.call("smb_row_sums", F32, ptr(dy), u.m, B, ld, ptr(gb), st)
        if fuse_update:
            self._dense_update(u, gw, gb, eta, st)

    def _dense_update(self, u, gw, gb, eta, st):
        lay = u.layer
        opt = lay.optimizer
        kind = optimizer_kind(opt)
        vel = lay.velocity.view(-1) if lay.velocity is not None else None
        _lib.call("smb_optimizer_step", _lib.SMB_F32, ptr(lay.weights), ptr(vel), ptr(gw),
                  u.nvals, kind, float(opt.mu), float(eta), st)
        _lib.call("smb_optimizer_step", _lib.SMB_F32, ptr(lay.bias), ptr(lay.velocity_bias),
                  ptr(gb), u.m, kind, float(opt.mu), float(eta), st)

    def _launch_updates_from_flat(self, eta: float) -> None:
        st = stream_ptr()
        for u in self.units:
            lay = u.layer
            opt = lay.optimizer
            kind = optimizer_kind(opt)
            g = self.flat[u.grad_off:u.grad_off + u.nvals]
            gb = self.flat[u.bias_off:u.bias_off + u.m]
            if u.sparse:
                vel = lay.velocity.values if lay.velocity is not None else None
                _lib.call("smb_optimizer_step", _lib.SMB_F32, ptr(lay.weights.values), ptr(vel),
                          ptr(g), u.nvals, kind, float(opt.mu), float(eta), st)
                _lib.call("smb_optimizer_step", _lib.SMB_F32, ptr(lay.bias), ptr(lay.velocity_bias),
                          ptr(gb), u.m, kind, float(opt.mu), float(eta), st)
            else:
                self._dense_update(u, g.view(u.m, u.k), gb, eta, st)

    def _advance(self, gather: bool) -> None:
        if gather:
            _lib.call("smb_step_counter_advance", ptr(self.counter), int(self.steps_per_epoch),
                      stream_ptr())

    # ------------------------------------------------------------------
    def _run_eager(self, eta: float, gather: bool, part: str) -> None:
        if self.world == 1:
            self._launch_forward_backward(eta, True, gather)
            self._advance(gather)
        elif part == "fb":
            self._launch_forward_backward(eta, False, gather)
        else:
            self._launch_updates_from_flat(eta)
            self._advance(gather)

    def _graph(self, eta: float, gather: bool, part: str):
        key = (float(eta), gather, part)
        g = self._graphs.get(key)
        if g is None:
            # warm up eagerly on a side stream (cuBLAS handles, smem attributes),
            # then restore the state the warm-up touched by re-running nothing:
            # capture only records, it does not execute.
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._run_eager(eta, gather, part)
            self._graphs[key] = g
        return g

    def step(self, eta: float, gather: bool | None = None) -> None:
        """One training step.  With gather (default when a dataset is
        attached) the batch comes from the device dataset at the device step
        counter; otherwise the caller has filled ``x_in`` / ``t_in``."""
        if gather is None:
            gather = self.data is not None
        if gather and (self.data is None or self.perm is None):
            raise InvalidArgumentError("attach_dataset() and set_epoch() before gathering steps")
        if self.world == 1:
            self._replay_or_run(eta, gather, "all")
            return
        import torch.distributed as dist

        self._replay_or_run(eta, gather, "fb")
        dist.all_reduce(self.flat, group=self.pg)
        self._replay_or_run(eta, gather, "upd")

    def _replay_or_run(self, eta, gather, part):
        if not self.use_graph:
            self._run_eager(eta, gather, part)
            return
        key = (float(eta), gather, part)
        if key not in self._graphs:
            # the first execution is eager (initialises cuBLAS / kernel
            # attributes outside capture); later ones replay the graph
            self._run_eager(eta, gather, part)
            self._graph(eta, gather, part)
            return
        self._graphs[key].replay()

    def loss_value(self) -> float:
        """Summed softmax-CE loss of the last step's local batch (syncs)."""
        return float(self.loss.item())

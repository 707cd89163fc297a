"""Fused, graph-captured training step (one pass of sgd_train's hot loop).

One call of ``FusedTrainStep.step()`` performs, entirely on the GPU, the body
of the reference's per-batch loop (train.py:389-402):

    gather      xb = Xtrain[:, batch], tb = Ttrain[:, batch]    smb_gather_columns
    forward     a_l = relu(W_l a_{l-1} + b_l)                   smb_spmm (bias+ReLU fused)
    loss grad   d_L = (softmax(y) - t) / B                      smb_softmax_ce_grad
    backward    d_{l-1} = (W_l^T d_l) * (a_{l-1} > 0)           smb_spmm_t_bias (mask fused,
                + row_sums(d_{l-1}), update b_{l-1}              + bias side of layer l-1)
                grad_l = sddmm(d_l, a_{l-1}); update W_l        smb_sddmm_update (fused)
    next batch  gathered ahead into the other input slot, step  smb_gather_columns_ahead +
                counter += 1 (own stream, beside the last SDDMM) smb_step_counter_advance

spmm_t of layer l runs before the update of layer l (pre-update weights,
train.py:400-401).  The layer-1 input gradient is never computed: the
reference computes and discards it (train.py:216-220).  Dense (ER-saturated)
layers use cuBLAS FP32 (TF32 off) plus the same exact bias/optimizer kernels;
masked-dense baseline layers (MaskedDense) add the mask in one fused update
kernel (smb_masked_optimizer_step, nn.py:255-263).

The kernel sequence is captured once into a CUDA graph per learning rate and
replayed (a step is ~10 launches; replay removes the host launch cost).

Data parallel (``process_group`` with world size G > 1): every rank runs the
step on its B/G slice of the same global batch; the loss gradient is scaled
by 1/B_global; the value, dense-weight and bias gradients of all layers land
in ONE flat fp32 buffer that is summed with a single NCCL all-reduce, after
which every rank applies the identical update.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from .errors import ConfigurationError, InvalidArgumentError
from .nn import DENSE_T_MAX_ROWS, ActivationLayer, DenseLinearLayer, ReLU, SparseLinearLayer, optimizer_kind
from .tensor_core import _no_tf32, ptr, stream_ptr

__all__ = ["FusedTrainStep", "KernelTimer"]


class KernelTimer:
    """CUDA-event spans around individual launches on the launching stream."""

    def __init__(self):
        self.records = []  # (tag, start_event, end_event)
        self.calls = None  # (tag, name, args) while kernel_durations records

    @staticmethod
    def hold_gpu(cycles: int = 40_000_000) -> None:
        """Enqueue a spin kernel so the host can enqueue a whole step before the
        GPU reaches it: the spans then time kernels, not host launch gaps."""
        torch.cuda._sleep(cycles)

    def span(self, tag):
        timer = self

        class _Span:
            def __enter__(self):
                self.s = torch.cuda.Event(enable_timing=True)
                self.e = torch.cuda.Event(enable_timing=True)
                self.s.record()

            def __exit__(self, *exc):
                self.e.record()
                timer.records.append((tag, self.s, self.e))

        return _Span()

    def kernel_durations(self, step, eta: float, reps: int = 20, replays: int = 5):
        """{tag: (launches, total_ms)}: every C-ABI launch of one step (the
        kernels of the overlapped step itself; the input slot already filled)
        is recorded once from an eager run, then timed alone as `reps` back-to-back launches
        captured in a CUDA graph and replayed `replays` times between two
        events, so the average is the kernel's own launch duration with its
        operands resident in L2 as they are inside the step.  (Event pairs
        around single launches would not do: stream launches and event nodes
        round every kernel up to the ~2 us period of the stream's dependency
        polling -- scripts/launch_gap_lab.cu -- which swamps the 5-25 us
        kernels of the small configs.)  The stream is the last argument of
        every recorded call; sddmm_update writes the other value buffer, so
        repeats recompute the same update."""
        cur = torch.cuda.current_stream()
        # every replayed launch writes its outputs again (velocity, bias,
        # dense weights are updated in place): snapshot the step's whole
        # mutable state and restore it afterwards
        snapshot = [(t, t.clone()) for t in step.state_tensors()]
        saved = (step.timer, step.use_graph)
        self.calls = []
        step.timer, step.use_graph = self, False
        try:
            step._launch_forward_backward(eta, not step.dp, False)
        finally:
            step.timer, step.use_graph = saved
            self.calls, calls = None, self.calls
        torch.cuda.synchronize()
        cs = torch.cuda.Stream(device=step.dev)
        out = {}
        for tag, name, args in calls:
            g = torch.cuda.CUDAGraph()
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                _lib.call(name, *args[:-1], stream_ptr())
            with torch.cuda.graph(g, stream=cs):
                for _ in range(reps):
                    _lib.call(name, *args[:-1], stream_ptr())
            cur.wait_stream(cs)
            g.replay()
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record()
            for _ in range(replays):
                g.replay()
            e_.record()
            e_.synchronize()
            c, t = out.get(tag, (0, 0.0))
            out[tag] = (c + reps * replays, t + s_.elapsed_time(e_))
        torch.cuda.synchronize()
        for t, saved_t in snapshot:
            t.copy_(saved_t)
        step.sync_weights()  # derived copies (CSC / padded) of the restored values
        torch.cuda.synchronize()
        return out

    def summary(self):
        """{tag: (count, total_ms)} after synchronising."""
        torch.cuda.synchronize()
        out = {}
        for tag, s, e in self.records:
            c, t = out.get(tag, (0, 0.0))
            out[tag] = (c + 1, t + s.elapsed_time(e))
        return out


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def shard_epoch(perm, global_batch: int, local_batch: int, rank_offset: int):
    """This rank's sample order for one epoch, laid out so its batch k is
    entries [k*local_batch, (k+1)*local_batch): the columns
    [rank_offset, rank_offset + local_batch) of every global batch of the
    shuffled order (K = N // global_batch batches; the partial batch is
    dropped like train.py:389).  Returns (int32 indices, K)."""
    p = np.ascontiguousarray(perm, dtype=np.int64)
    if not 0 <= rank_offset <= global_batch - local_batch:
        raise InvalidArgumentError("rank slice outside the global batch")
    kb = p.shape[0] // global_batch
    idx = p[: kb * global_batch].reshape(kb, global_batch)[:, rank_offset:rank_offset + local_batch]
    return np.ascontiguousarray(idx.reshape(-1)).astype(np.int32), kb


def flat_layout(units):
    """Offsets of the data-parallel gradient buffer: per layer [values | bias]."""
    off, layout = 0, []
    for m, nvals in units:
        layout.append((off, off + nvals))
        off += nvals + m
    return layout, off


class _ChainPlan:
    """Owns an smb_chain_plan handle."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            _lib.load().smb_chain_plan_destroy(self.h)
        except Exception:
            pass


class _Unit:
    __slots__ = ("layer", "relu", "sparse", "m", "k", "grad_off", "bias_off", "nvals", "index",
                 "vals", "vals_csc", "seen")

    def __init__(self, layer, relu, index=0):
        self.index = index
        self.layer = layer
        self.relu = relu
        self.sparse = isinstance(layer, SparseLinearLayer)
        self.m = layer.n_out
        self.k = layer.n_in
        self.nvals = layer.weights.nnz if self.sparse else self.m * self.k


class FusedTrainStep:
    def __init__(self, model, batch_size: int, global_batch: int | None = None,
                 process_group=None, use_graph: bool = True, force_dp: bool = False,
                 bucketed: bool | None = None, chain: bool = True):
        self.units = self._parse(model)
        self.model = model
        self.B = int(batch_size)
        self.B_global = int(global_batch or batch_size)
        if self.B <= 0:
            raise InvalidArgumentError("batch_size must be positive")
        self.pg = process_group
        self.world = 1
        backend = None
        if process_group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(process_group)
            backend = str(dist.get_backend(process_group)).lower()
        # data parallel: one all-reduce per layer bucket, issued as soon as the
        # layer's gradients exist and followed by that layer's update, so the
        # collectives overlap the backward of the layers below (bucketed);
        # with NCCL the collectives are captured into the step's CUDA graph
        # (graph_comm), other backends (gloo) run the same sequence eagerly.
        # bucketed=False: one all-reduce of the whole flat buffer after the
        # backward, then one update launch (the round-1 structure).
        self.bucketed = (os.environ.get("SMB_DP_BUCKETED", "1") != "0"
                         if bucketed is None else bool(bucketed))
        self.graph_comm = process_group is None or backend == "nccl"
        # data-parallel structure: a forward/backward pass that only produces
        # gradients (flat buffer), the all-reduce, then the update pass.
        # force_dp runs that structure on one process (testing; the
        # all-reduce is then skipped)
        self.dp = self.world > 1 or bool(force_dp)
        self.use_graph = use_graph
        dev = self.units[0].layer.bias.device
        self.dev = dev
        ld = _round_up(self.B, 4)
        self.ld = ld
        f32 = torch.float32
        self.n_in = self.units[0].k
        self.classes = self.units[-1].m
        # two input slots: train_batch() copies batch k+1 into one slot on a
        # copy stream while the step of batch k reads the other
        self.x_slots = [torch.zeros((self.n_in, ld), dtype=f32, device=dev) for _ in range(2)]
        self.t_slots = [torch.zeros((self.classes, ld), dtype=f32, device=dev) for _ in range(2)]
        self.x_in, self.t_in = self.x_slots[0], self.t_slots[0]
        self._slot = 0
        self._next_slot = 0
        self._copy_stream = None
        self._slot_ready = self._slot_free = None
        self.acts = [torch.zeros((u.m, ld), dtype=f32, device=dev) for u in self.units]
        self.dys = [torch.zeros((u.m, ld), dtype=f32, device=dev) for u in self.units]
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.counter = torch.zeros(1, dtype=torch.int32, device=dev)
        ws = int(_lib.load().smb_softmax_ce_workspace_bytes(self.B))
        self._ce_ws = torch.zeros(ws, dtype=torch.uint8, device=dev)
        self.perm = None
        self.data = None
        self.steps_per_epoch = 0
        # device-gather steps prefetch the NEXT batch into the other input
        # slot right after the softmax step advanced the counter (side
        # stream, overlapping the backward); _gslot is the slot the next
        # gather step reads, _prefetched whether it already holds that batch
        self._gslot = 0
        self._prefetched = False
        # data-parallel flat gradient buffer: [values | bias] per layer
        self.flat = None
        if self.dp:
            layout, total = flat_layout([(u.m, u.nvals) for u in self.units])
            for u, (g_off, b_off) in zip(self.units, layout):
                u.grad_off, u.bias_off = g_off, b_off
            self.flat = torch.zeros(total, dtype=f32, device=dev)
        # single GPU: bias row sums of transposed-SpMM outputs on a side stream
        # instead of fused into the critical-path kernel's epilogue
        self.split_bias = True
        self._segs = None  # data-parallel update segment table (built on first use)
        self._graphs = {}
        self._cap_stream = None
        self.timer = None  # optional KernelTimer: per-launch CUDA events (eager only)
        # Each sparse layer's weight side (SDDMM + update, or SDDMM into the
        # flat buffer when data parallel) runs on its own side stream,
        # concurrently with the transposed-SpMM chain.  A single-GPU update
        # writes the second of two value buffers (ping-pong), so the
        # transposed SpMM of the same layer keeps reading the pre-update
        # weights (train.py:400-401); `parity` selects the current buffer.
        nb = max([int(_lib.load().smb_dense_forward_workspace_bytes(u.m, u.k, self.B))
                  for u in self.units if not u.sparse and u.m <= DENSE_T_MAX_ROWS] or [0])
        self._dense_ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=dev) if nb else None
        self.overlap = True
        # where the next batch is gathered in the chain-kernel step: beside the
        # chain kernel (True) or beside the weight sides at the end (False)
        # (config 2: 56.5 -> 53.6 us back to back once the lean SDDMMs left the
        # gather as the tail of the step; before them it was within 1 us)
        self.prefetch_beside_chain = True
        self._parity = 0
        self._sides = {}
        for u in self.units:
            u.vals = None
            u.vals_csc = None
            u.seen = None
            if u.sparse and self.overlap and not self.dp:
                # two value buffers; the layer's own `weights.values` tensor
                # object stays the same and is re-pointed (set_) at the current
                # buffer after every step, so a caller holding it always reads
                # the updated weights, like the reference's in-place update
                # (nn.py:187-198)
                cur = u.layer.weights.values
                u.vals = [cur.view_as(cur), cur.clone()]
                if u.index > 0:
                    # the transposed SpMM reads a CSC-ordered copy of the
                    # values (no per-nonzero perm indirection), refreshed
                    # after every update on the update's stream
                    u.vals_csc = [torch.empty_like(cur), torch.empty_like(cur)]
            elif u.sparse and self.overlap and self.dp and u.index > 0:
                # data parallel: no ping-pong (the update waits for the
                # layer's transposed SpMM), one CSC copy refreshed after the
                # update on the same stream
                c = torch.empty_like(u.layer.weights.values)
                u.vals_csc = [c, c]
        # column-chain kernel (csrc/chain.cu): layers 1..L-1 forward, the
        # softmax step and the input-gradient chain in one cluster launch,
        # when the model fits it (all layers sparse, ReLU between them, at
        # most 16 classes, operands within shared memory)
        self._chain = None
        self._chain_ws = None
        if chain and self.overlap:
            self._chain = self._make_chain_plan()
        self.sync_weights()

    def _make_chain_plan(self):
        import ctypes as C

        us = self.units
        if len(us) < 2 or not all(u.sparse for u in us):
            return None
        if not all(u.relu for u in us[:-1]) or us[-1].relu:
            return None
        lib = _lib.load()
        L = len(us)
        pats = (C.c_void_p * L)(*[u.layer.weights.pattern.handle for u in us])
        relu = (C.c_int * L)(*[int(u.relu) for u in us])
        out = C.c_void_p()
        rc = lib.smb_chain_plan_create(L, pats, relu, self.B, self.ld, C.byref(out))
        if rc != _lib.SMB_OK:
            msg = lib.smb_last_error().decode(errors="replace")
            if rc == _lib.SMB_ERR_INVALID and "unsupported" in msg:
                return None  # the separate kernels run this model
            _lib.check(rc, "smb_chain_plan_create")
        self._chain_ws = torch.zeros(int(lib.smb_chain_workspace_bytes(self.B)), dtype=torch.uint8,
                                     device=self.dev)
        # the chain reads the plan's padded value copies (refreshed after
        # every update), not the CSC-ordered copies of the separate kernels
        for u in us:
            u.vals_csc = None
        return _ChainPlan(out.value)

    def chain_info(self):
        """{cluster, groups, smem, layers} of the column-chain plan, or None."""
        if self._chain is None:
            return None
        import ctypes as C

        info = (C.c_int64 * 4)()
        _lib.call("smb_chain_plan_info", self._chain.h, info)
        return dict(zip(("cluster", "groups", "smem", "layers"), list(info)))

    def sync_weights(self) -> None:
        """Re-derive the CSC-ordered value copies from the layers' current
        values.  Not needed by callers: every step first checks each layer's
        `weights.values` (a replaced tensor or a bumped version counter, i.e. an
        in-place torch op or a layer-API optimize()) and re-syncs itself."""
        for u in self.units:
            self._sync_unit(u)

    def _sync_unit(self, u) -> None:
        if u.vals is not None:
            v = u.layer.weights.values
            cur = u.vals[self._parity]
            if v.data_ptr() != cur.data_ptr():
                # the caller assigned a new value tensor: adopt its contents
                # into the current buffer and point the tensor at that buffer
                if v.shape != cur.shape or v.dtype != cur.dtype:
                    raise InvalidArgumentError("weights.values changed shape or dtype")
                cur.copy_(v)
                v.set_(cur)
        if u.sparse:
            u.seen = u.layer.weights.values._version
        if u.vals_csc is not None:
            _lib.call("smb_values_to_csc", _lib.SMB_F32, u.layer.weights.pattern.handle,
                      ptr(self._vals(u)), ptr(u.vals_csc[self._parity]), stream_ptr())
        if self._chain is not None and u.index > 0:
            _lib.call("smb_chain_refresh", self._chain.h, u.index, ptr(self._vals(u)),
                      stream_ptr())

    def _adopt_external_changes(self) -> None:
        """Re-sync any layer whose values changed outside the step."""
        for u in self.units:
            if u.vals is None and u.vals_csc is None and self._chain is None:
                continue
            v = u.layer.weights.values
            if v._version != u.seen or (
                    u.vals is not None and v.data_ptr() != u.vals[self._parity].data_ptr()):
                self._sync_unit(u)

    def state_tensors(self):
        """Every tensor a step mutates (parameters, optimizer state, both value
        buffers and the CSC copies): KernelTimer snapshots and restores them."""
        out = []
        for u in self.units:
            lay = u.layer
            if u.sparse:
                out += list(u.vals) if u.vals is not None else [lay.weights.values]
                out += list(u.vals_csc) if u.vals_csc is not None else []
                out += [lay.velocity.values] if lay.velocity is not None else []
                out += [lay.grad.values]
            else:
                out += [lay.weights, lay.grad]
                out += [lay.velocity] if lay.velocity is not None else []
            out += [lay.bias] + ([lay.velocity_bias] if lay.velocity_bias is not None else [])
        out += [self.loss, self.counter] + self.acts + self.dys
        if self.flat is not None:
            out.append(self.flat)
        return out

    def _call(self, tag: str, name: str, *args) -> None:
        t = self.timer
        if t is None:
            _lib.call(name, *args)
            return
        if t.calls is not None:  # KernelTimer.kernel_durations records the launch
            t.calls.append((tag, name, args))
            _lib.call(name, *args)
            return
        with t.span(tag):
            _lib.call(name, *args)

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
            relu = False
            if i + 1 < len(layers) and isinstance(layers[i + 1], ActivationLayer):
                if not isinstance(layers[i + 1].fn, ReLU):
                    raise ConfigurationError("fused step supports ReLU activations only")
                relu = True
                i += 1
            if lay.weights.dtype not in (np.float32, torch.float32):
                raise ConfigurationError("fused step runs float32 models")
            units.append(_Unit(lay, relu, len(units)))
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
        self._prefetched = False
        self.sync_weights()

    def set_epoch(self, perm: np.ndarray, rank_offset: int = 0) -> None:
        """Upload the epoch's sample order; this rank's batch k is
        perm[k*B_global + rank_offset : ... + B]."""
        idx, kb = shard_epoch(perm, self.B_global, self.B, rank_offset)
        flat = torch.from_numpy(idx)
        if self.perm is None or self.perm.numel() != flat.numel():
            self.perm = torch.empty(flat.numel(), dtype=torch.int32, device=self.dev)
            self._graphs.clear()
        self.perm.copy_(flat)
        self.counter.zero_()
        self.sync_weights()
        self.steps_per_epoch = kb
        self._prefetched = False  # the next step gathers batch 0 of this order first

    def _gather_into(self, slot: int, st, ahead: bool = False) -> None:
        """xb / tb of the batch at the device step counter (ahead: the next
        batch, then advance the counter) into input `slot`.  The counter
        names the batch in the slot the current step reads; only this
        gather stream reads or writes it during a step."""
        d, B, ld, F32 = self.data, self.B, self.ld, _lib.SMB_F32
        if not ahead:
            self._call("gather", "smb_gather_columns", F32, ptr(d.X), d.n_samples, d.features,
                       ptr(self.perm), ptr(self.counter), 0, B, ptr(self.x_slots[slot]), ld, st)
            self._call("gather_t", "smb_gather_columns", F32, ptr(d.T), d.n_samples, d.classes,
                       ptr(self.perm), ptr(self.counter), 0, B, ptr(self.t_slots[slot]), ld, st)
            return
        kb = int(self.steps_per_epoch)
        self._call("gather", "smb_gather_columns_ahead", F32, ptr(d.X), d.n_samples, d.features,
                   ptr(self.perm), ptr(self.counter), 1, kb, B, ptr(self.x_slots[slot]), ld, st)
        self._call("gather_t", "smb_gather_columns_ahead", F32, ptr(d.T), d.n_samples,
                   d.classes, ptr(self.perm), ptr(self.counter), 1, kb, B,
                   ptr(self.t_slots[slot]), ld, st)
        self._call("counter", "smb_step_counter_advance", ptr(self.counter), kb, st)

    # ------------------------------------------------------------------
    def _bias_target(self, u, fuse_update: bool):
        """(bias, velocity_bias, grad_bias_out, opt_kind, mu) for unit u's bias side."""
        lay = u.layer
        opt = lay.optimizer
        if fuse_update:
            return (ptr(lay.bias), ptr(lay.velocity_bias), None, optimizer_kind(opt),
                    float(opt.mu))
        return (None, None, ptr(self.flat[u.bias_off:u.bias_off + u.m]), _lib.SMB_OPT_NONE,
                float(opt.mu))

    def _allreduce_bucket(self, u) -> None:
        """SUM-all-reduce of unit u's flat-buffer bucket [values | bias].
        Buckets are issued in the same order (last layer first) on every rank,
        so the communicator sees one consistent sequence of collectives."""
        if self.pg is None:  # force_dp on one process: the identity
            return
        import torch.distributed as dist

        work = dist.all_reduce(self.flat[u.grad_off:u.bias_off + u.m], group=self.pg,
                               async_op=True)
        work.wait()  # the current (weights) stream waits for the collective

    def _update_unit_from_flat(self, u, eta: float, st) -> None:
        """The exact optimizer update of unit u from its summed bucket."""
        lay = u.layer
        opt = lay.optimizer
        kind = optimizer_kind(opt)
        g = self.flat[u.grad_off:u.grad_off + u.nvals]
        gb = self.flat[u.bias_off:u.bias_off + u.m]
        if u.sparse:
            vals = lay.weights.values
            vel = lay.velocity.values if lay.velocity is not None else None
        else:
            vals = lay.weights
            vel = lay.velocity.view(-1) if lay.velocity is not None else None
        if not u.sparse and lay.mask is not None:
            self._call(f"update[{u.index}]", "smb_masked_optimizer_step", _lib.SMB_F32,
                       ptr(vals), ptr(vel), ptr(g), ptr(lay.mask), u.nvals, kind,
                       float(opt.mu), float(eta), st)
        else:
            self._call(f"update[{u.index}]", "smb_optimizer_step", _lib.SMB_F32, ptr(vals),
                       ptr(vel), ptr(g), u.nvals, kind, float(opt.mu), float(eta), st)
        self._call(f"update_bias[{u.index}]", "smb_optimizer_step", _lib.SMB_F32,
                   ptr(lay.bias), ptr(lay.velocity_bias), ptr(gb), u.m, kind, float(opt.mu),
                   float(eta), st)
        self._refresh_csc(u, st)

    def _refresh_csc(self, u, st) -> None:
        if u.vals_csc is not None and u.vals is None:  # data parallel: one CSC copy
            self._call(f"to_csc[{u.index}]", "smb_values_to_csc", _lib.SMB_F32,
                       u.layer.weights.pattern.handle, ptr(u.layer.weights.values),
                       ptr(u.vals_csc[0]), st)

    def _launch_forward_backward(self, eta: float, fuse_update: bool, gather: bool,
                                 comm: bool = False) -> None:
        st = stream_ptr()
        B, ld = self.B, self.ld
        F32 = _lib.SMB_F32
        x_in, t_in = self.x_slots[self._slot], self.t_slots[self._slot]
        overlap = self.overlap
        forked = []  # side streams this step forked onto (joined at the end)

        def fork(key):
            """A side stream (one per purpose, so the layers' updates and the
            batch prefetch overlap each other as well as the main chain) that
            starts after everything enqueued on main so far."""
            s_ = self._side_stream(key)
            s_.wait_stream(main)
            if s_ not in forked:
                forked.append(s_)
            return s_
        main = torch.cuda.current_stream()
        # gather steps: this batch is already in x_in / t_in (prefetched by
        # the previous step or by step()'s prologue); the next one is
        # gathered into the other slot on its own stream, beside the layer-0
        # SDDMM at the end of the backward (measured 78.2 -> 76.5 us/step at
        # config 2 against launching it at the step start, where it competed
        # with the L2-bound first-layer SpMM)

        def prefetch():
            # (serialised on the main stream when overlap is off: the
            # per-kernel timing pass then sees each kernel alone)
            with torch.cuda.stream(fork("prefetch")) if overlap else _nullctx():
                self._gather_into(1 - self._slot, stream_ptr(), ahead=True)

        if self._chain is not None and overlap and (fuse_update or comm):
            early = gather and self.prefetch_beside_chain
            self._launch_chain_step(eta, x_in, t_in, fork, main, prefetch if early else None,
                                    comm=comm)
            if gather and not early:
                prefetch()
            for s_ in forked:
                main.wait_stream(s_)
            return
        # forward: a_l = act(W_l a_{l-1} + b_l)
        x = x_in
        for li, (u, a) in enumerate(zip(self.units, self.acts)):
            lay = u.layer
            if u.sparse:
                self._call(f"spmm[{li}]", "smb_spmm_p", F32, lay.weights.pattern.handle,
                           ptr(self._vals(u)), ptr(x), ld, B, ptr(lay.bias),
                           _lib.SMB_EPI_RELU if u.relu else _lib.SMB_EPI_NONE, ptr(a), ld, st)
            elif u.m <= DENSE_T_MAX_ROWS and lay.mask is None:
                # small (ER-saturated output) layer: split-K kernel, not a
                # cuBLAS SIMT GEMM (config 4: ~7 vs ~36 us)
                self._call(f"dense_fwd[{li}]", "smb_dense_forward_small", F32, ptr(lay.weights),
                           u.k, u.m, u.k, ptr(x), ld, B, ptr(lay.bias), ptr(a), ld,
                           ptr(self._dense_ws), st)
            else:
                with _no_tf32():
                    torch.addmm(lay.bias[:, None], lay.weights, x[:, :B], out=a[:, :B])
            if not u.sparse and u.relu:
                self._call(f"relu[{li}]", "smb_relu", F32, ptr(a), ld, u.m, B, ptr(a), ld, st)
            x = a
        # loss gradient (softmax CE) scaled by 1/B_global; the same launch
        # applies the last layer's bias side and advances the step counter
        top = self.units[-1]
        b, vb, gb, kind, mu = self._bias_target(top, fuse_update)
        if overlap:
            # the column-parallel softmax step on the critical path; the last
            # layer's bias row sums + update (they cross columns) beside it
            self._call("softmax_ce", "smb_softmax_ce_step", F32, ptr(self.acts[-1]), ld,
                       ptr(t_in), ld, self.classes, B, float(self.B_global), ptr(self.dys[-1]),
                       ld, ptr(self.loss), None, None, None, _lib.SMB_OPT_NONE, 0.0, float(eta),
                       None, 0, ptr(self._ce_ws), st)
            with torch.cuda.stream(fork(("weights", len(self.units) - 1))):
                self._call(f"bias[{top.index}]", "smb_bias_grad_update", F32, ptr(self.dys[-1]),
                           ld, top.m, B, b, vb, gb, kind, mu, float(eta), stream_ptr())
        else:
            self._call("softmax_ce", "smb_softmax_ce_step", F32, ptr(self.acts[-1]), ld,
                       ptr(t_in), ld, self.classes, B, float(self.B_global), ptr(self.dys[-1]),
                       ld, ptr(self.loss), b, vb, gb, kind, mu, float(eta), None, 0,
                       ptr(self._ce_ws), st)
        # backward, last layer first: d_{l-1} (+ bias side of layer l-1) on the
        # main stream; the weight side of layer l (SDDMM + update) either
        # follows it in order, or -- single GPU -- runs on the side stream as
        # soon as d_l exists, writing the other value buffer (spmm_t keeps
        # reading the pre-update W_l, train.py:400-401)
        for li in range(len(self.units) - 1, -1, -1):
            u = self.units[li]
            lay = u.layer
            dy = self.dys[li]
            x_prev = self.acts[li - 1] if li > 0 else x_in
            if overlap and u.sparse:
                with torch.cuda.stream(fork(("weights", li))):  # d_l is ready
                    self._weight_side(u, dy, x_prev, eta, fuse_update, stream_ptr())
            if li > 0:
                below = self.units[li - 1]
                mask = self.acts[li - 1] if below.relu else None
                dst = self.dys[li - 1]
                b, vb, gb, kind, mu = self._bias_target(below, fuse_update)
                if u.sparse and overlap and self.split_bias:
                    # d_{l-1} alone on the critical path; the bias side of
                    # layer l-1 (row sums cross the batch) beside it
                    if u.vals_csc is not None:
                        self._call(f"spmm_t[{li}]", "smb_spmm_t_csc", F32,
                                   lay.weights.pattern.handle, ptr(u.vals_csc[self._parity]),
                                   ptr(dy), ld, B, ptr(mask), ld if mask is not None else 0,
                                   ptr(dst), ld, st)
                    else:
                        self._call(f"spmm_t[{li}]", "smb_spmm_t", F32, lay.weights.pattern.handle,
                                   ptr(self._vals(u)), ptr(dy), ld, B, ptr(mask),
                                   ld if mask is not None else 0, ptr(dst), ld, st)
                    with torch.cuda.stream(fork(("weights", li - 1))):
                        self._call(f"bias[{li - 1}]", "smb_bias_grad_update", F32, ptr(dst), ld,
                                   u.k, B, b, vb, gb, kind, mu, float(eta), stream_ptr())
                elif u.sparse:
                    self._call(f"spmm_t[{li}]", "smb_spmm_t_bias", F32, lay.weights.pattern.handle,
                               ptr(self._vals(u)), ptr(dy), ld, B, ptr(mask),
                               ld if mask is not None else 0, ptr(dst), ld, b, vb, gb, kind, mu,
                               float(eta), st)
                elif u.m <= DENSE_T_MAX_ROWS:
                    # small dense output layer: W^T d and the mask in one pass
                    self._call(f"dense_t[{li}]", "smb_dense_backward_input", F32,
                               ptr(lay.weights), u.k, u.m, u.k, ptr(dy), ld, B, ptr(mask),
                               ld if mask is not None else 0, ptr(dst), ld, st)
                    # (the bias side of the layer below stays on the main
                    # stream here: forked, it delays the SDDMM queued behind
                    # it on that layer's stream -- config 4: 1448 vs 1520 us)
                    self._call(f"bias[{li - 1}]", "smb_bias_grad_update", F32, ptr(dst), ld, u.k,
                               B, b, vb, gb, kind, mu, float(eta), st)
                else:
                    with _no_tf32():
                        torch.mm(lay.weights.T, dy[:, :B], out=dst[:, :B])
                    if mask is not None:
                        self._call(f"relu_bwd[{li}]", "smb_relu_backward", F32, ptr(dst), ld,
                                   ptr(mask), ld, u.k, B, ptr(dst), ld, st)
                    self._call(f"bias[{li - 1}]", "smb_bias_grad_update", F32, ptr(dst), ld, u.k,
                               B, b, vb, gb, kind, mu, float(eta), st)
            if overlap and not u.sparse:
                # dense layer: its weight gradient GEMM + update beside the
                # chain, forked after the kernel that reads the pre-update
                # weights (dense_t / the W^T d GEMM above) was enqueued
                with torch.cuda.stream(fork(("weights", li))):
                    self._weight_side(u, dy, x_prev, eta, fuse_update, stream_ptr())
            elif not (overlap and u.sparse):
                self._weight_side(u, dy, x_prev, eta, fuse_update, st)
            if comm:
                # data parallel, per-layer bucket: layer li's [values | bias]
                # gradients are complete on its weights stream (bias side
                # forked at layer li+1, SDDMM / dense GEMM above); the
                # stream also waits for main, which now holds the last reader
                # of the pre-update W_li (its transposed product).  Sum the
                # bucket over the ranks, then update layer li there, while
                # the backward of the layers below continues on main.
                with torch.cuda.stream(fork(("weights", li)) if overlap else main):
                    self._allreduce_bucket(u)
                    self._update_unit_from_flat(u, eta, stream_ptr())
        if gather:
            prefetch()
        for s_ in forked:
            main.wait_stream(s_)  # join: the step ends when every update has

    def _launch_chain_step(self, eta, x_in, t_in, fork, main, prefetch=None,
                           comm: bool = False) -> None:
        """Step through the column-chain kernel: layer 0's forward SpMM, then
        ONE cluster launch for layers 1..L-1 forward, the softmax step and
        every input gradient (csrc/chain.cu), then every layer's weight side
        concurrently on the layers' side streams, the first layer's (the
        longest SDDMM) first.  Single GPU: SDDMM + update and bias row sums +
        update fused.  Data parallel (comm): the gradients go to the layer's
        flat bucket, which is summed over the ranks and applied on that
        stream (same bucket order on every rank), then the chain's padded
        value copies are refreshed."""
        import ctypes as C

        st = stream_ptr()
        B, ld, F32 = self.B, self.ld, _lib.SMB_F32
        us = self.units
        L = len(us)
        u0 = us[0]
        self._call("spmm[0]", "smb_spmm_p", F32, u0.layer.weights.pattern.handle,
                   ptr(self._vals(u0)), ptr(x_in), ld, B, ptr(u0.layer.bias),
                   _lib.SMB_EPI_RELU if u0.relu else _lib.SMB_EPI_NONE, ptr(self.acts[0]), ld, st)
        if prefetch is not None:
            prefetch()  # the next batch's gather beside the chain kernel
        arr = C.c_void_p * L
        bias = arr(*[ptr(u.layer.bias) for u in us])
        acts = arr(*[ptr(a) for a in self.acts])
        dys = arr(*[ptr(d) for d in self.dys])
        self._call("chain", "smb_chain_run", self._chain.h, bias, acts, dys, ptr(t_in), ld,
                   float(self.B_global), ptr(self.loss), ptr(self._chain_ws), st)
        for li in [0] + list(range(L - 1, 0, -1)):
            u = us[li]
            x_prev = self.acts[li - 1] if li > 0 else x_in
            b, vb, gb, kind, mu = self._bias_target(u, not comm)
            with torch.cuda.stream(fork(("weights", li))):
                self._weight_side(u, self.dys[li], x_prev, eta, not comm, stream_ptr())
                self._call(f"bias[{li}]", "smb_bias_grad_update", F32, ptr(self.dys[li]), ld,
                           u.m, B, b, vb, gb, kind, mu, float(eta), stream_ptr())
                if comm:
                    self._allreduce_bucket(u)
                    self._update_unit_from_flat(u, eta, stream_ptr())
                    if li > 0:
                        self._call(f"chain_refresh[{li}]", "smb_chain_refresh", self._chain.h,
                                   li, ptr(self._vals(u)), stream_ptr())

    def _side_stream(self, key):
        s_ = self._sides.get(key)
        if s_ is None:
            # lowest priority: the main chain's CTAs are scheduled first
            lo, _hi = torch.cuda.Stream.priority_range()
            s_ = self._sides[key] = torch.cuda.Stream(device=self.dev, priority=lo)
        return s_

    def _vals(self, u):
        """The current (pre-update) value buffer of sparse unit u."""
        return u.vals[self._parity] if u.vals is not None else u.layer.weights.values

    def _flip_parity(self) -> None:
        """After an overlapped step the updated weights live in the other
        buffer: point the layer's CsrMatrix at it."""
        if not any(u.vals is not None for u in self.units):
            return
        self._parity ^= 1
        for u in self.units:
            if u.vals is not None:
                v = u.layer.weights.values
                v.set_(u.vals[self._parity])
                u.seen = v._version

    def _weight_side(self, u, dy, x_prev, eta, fuse_update, st):
        lay = u.layer
        B, ld = self.B, self.ld
        F32 = _lib.SMB_F32
        opt = lay.optimizer
        kind = optimizer_kind(opt) if fuse_update else _lib.SMB_OPT_NONE
        if u.sparse:
            vel = lay.velocity.values if lay.velocity is not None else None
            g_out = None if fuse_update else self.flat[u.grad_off:u.grad_off + u.nvals]
            w_in = self._vals(u)
            w_out = u.vals[self._parity ^ 1] if (u.vals is not None and fuse_update) else w_in
            # on a side stream beside the critical path: the small-footprint
            # staging ring (include/sparsemlp_b200.h SMB_HINT_CONCURRENT)
            hint = _lib.SMB_HINT_CONCURRENT if self.overlap else 0
            self._call(f"sddmm_update[{u.index}]", "smb_sddmm_update_into", F32,
                       lay.weights.pattern.handle, ptr(dy), ld, ptr(x_prev), ld, B,
                       ptr(w_in), ptr(w_out), ptr(vel), ptr(g_out), None, None, None,
                       kind | hint, float(opt.mu), float(eta), st)
            if u.vals_csc is not None and fuse_update:
                self._call(f"to_csc[{u.index}]", "smb_values_to_csc", F32,
                           lay.weights.pattern.handle, ptr(w_out),
                           ptr(u.vals_csc[self._parity ^ 1]), st)
            if self._chain is not None and fuse_update and u.index > 0:
                self._call(f"chain_refresh[{u.index}]", "smb_chain_refresh", self._chain.h,
                           u.index, ptr(w_out), st)
            return
        if u.m <= DENSE_T_MAX_ROWS and lay.mask is None:
            # ER-saturated output layer: gradient chains + update in one
            # launch (smb_dense_grad_update), no dense gradient round trip
            vel = lay.velocity.view(-1) if lay.velocity is not None else None
            g_out = None if fuse_update else self.flat[u.grad_off:u.grad_off + u.nvals]
            self._call(f"dense_grad[{u.index}]", "smb_dense_grad_update", F32, ptr(dy), ld, u.m,
                       ptr(x_prev), ld, u.k, B, ptr(lay.weights), u.k, ptr(vel), ptr(g_out),
                       kind, float(opt.mu), float(eta), st)
            return
        # wider dense / masked-dense baseline layer: cuBLAS FP32 weight
        # gradient + exact (masked) update
        gw = lay.grad if fuse_update else self.flat[u.grad_off:u.grad_off + u.nvals].view(u.m, u.k)
        with _no_tf32():
            torch.mm(dy[:, :B], x_prev[:, :B].T, out=gw)
        if fuse_update:
            vel = lay.velocity.view(-1) if lay.velocity is not None else None
            if lay.mask is not None:  # masked-dense baseline (nn.py:255-263)
                self._call(f"update[{u.index}]", "smb_masked_optimizer_step", F32,
                           ptr(lay.weights), ptr(vel), ptr(gw), ptr(lay.mask), u.nvals,
                           optimizer_kind(opt), float(opt.mu), float(eta), st)
            else:
                self._call(f"update[{u.index}]", "smb_optimizer_step", F32, ptr(lay.weights),
                           ptr(vel), ptr(gw), u.nvals, optimizer_kind(opt), float(opt.mu),
                           float(eta), st)

    def _segment_table(self):
        """Device table for smb_optimizer_step_multi: one record per
        parameter (values or dense weights, then bias) in flat-buffer order,
        or None when the layers' optimizers differ."""
        if self._segs is not None:
            return self._segs if self._segs is not False else None
        opts = {(optimizer_kind(u.layer.optimizer), float(u.layer.optimizer.mu)) for u in self.units}
        if len(opts) != 1 or 2 * len(self.units) > 32:
            self._segs = False
            return None
        rec = np.zeros((2 * len(self.units), 5), dtype=np.int64)
        fp = self.flat.data_ptr()
        for i, u in enumerate(self.units):
            lay = u.layer
            if u.sparse:
                w = lay.weights.values
                vel = lay.velocity.values if lay.velocity is not None else None
                mk = None
            else:
                w = lay.weights
                vel = lay.velocity
                mk = lay.mask
            rec[2 * i] = [w.data_ptr(), vel.data_ptr() if vel is not None else 0,
                          fp + 4 * u.grad_off, mk.data_ptr() if mk is not None else 0, u.grad_off]
            vb = lay.velocity_bias
            rec[2 * i + 1] = [lay.bias.data_ptr(), vb.data_ptr() if vb is not None else 0,
                              fp + 4 * u.bias_off, 0, u.bias_off]
        self._segs = torch.from_numpy(rec.view(np.uint8).reshape(-1)).to(self.dev)
        self._seg_kind = opts.pop()
        return self._segs

    def _launch_updates_from_flat(self, eta: float) -> None:
        st = stream_ptr()
        segs = self._segment_table()
        if segs is not None:
            kind, mu = self._seg_kind
            self._call("update", "smb_optimizer_step_multi", _lib.SMB_F32, ptr(segs),
                       2 * len(self.units), self.flat.numel(), kind, mu, float(eta), st)
            for u in self.units:
                self._refresh_csc(u, st)
            return
        for u in self.units:
            lay = u.layer
            opt = lay.optimizer
            kind = optimizer_kind(opt)
            g = self.flat[u.grad_off:u.grad_off + u.nvals]
            gb = self.flat[u.bias_off:u.bias_off + u.m]
            if u.sparse:
                vals = lay.weights.values
                vel = lay.velocity.values if lay.velocity is not None else None
            else:
                vals = lay.weights
                vel = lay.velocity.view(-1) if lay.velocity is not None else None
            if not u.sparse and lay.mask is not None:
                self._call(f"update[{u.index}]", "smb_masked_optimizer_step", _lib.SMB_F32,
                           ptr(vals), ptr(vel), ptr(g), ptr(lay.mask), u.nvals, kind,
                           float(opt.mu), float(eta), st)
            else:
                self._call(f"update[{u.index}]", "smb_optimizer_step", _lib.SMB_F32, ptr(vals),
                           ptr(vel), ptr(g), u.nvals, kind, float(opt.mu), float(eta), st)
            self._call(f"update_bias[{u.index}]", "smb_optimizer_step", _lib.SMB_F32,
                       ptr(lay.bias), ptr(lay.velocity_bias), ptr(gb), u.m, kind, float(opt.mu),
                       float(eta), st)
            self._refresh_csc(u, st)

    # ------------------------------------------------------------------
    def _run_eager(self, eta: float, gather: bool, part: str) -> None:
        if not self.dp:
            self._launch_forward_backward(eta, True, gather)
        elif part == "dp":  # gradients, per-layer all-reduce buckets and updates
            self._launch_forward_backward(eta, False, gather, comm=True)
        elif part == "fb":
            self._launch_forward_backward(eta, False, gather)
        else:
            self._launch_updates_from_flat(eta)

    def step(self, eta: float, gather: bool | None = None, slot: int = 0) -> None:
        """One training step.  With gather (default when a dataset is
        attached) the batch comes from the device dataset at the device step
        counter; otherwise the caller has filled input slot `slot`
        (``x_slots[slot]`` / ``t_slots[slot]``; slot 0 is ``x_in`` / ``t_in``)."""
        if gather is None:
            gather = self.data is not None
        self._adopt_external_changes()
        if gather and (self.data is None or self.perm is None):
            raise InvalidArgumentError("attach_dataset() and set_epoch() before gathering steps")
        if gather:
            if not self._prefetched:  # prologue: the first batch of this order
                self._gather_into(self._gslot, stream_ptr())
                self._prefetched = True
            self._slot = self._gslot
        else:
            self._slot = int(slot)
        if not self.dp:
            self._replay_or_run(eta, gather, "all")
            self._flip_parity()
        elif self.bucketed:
            self._replay_or_run(eta, gather, "dp")
        else:
            self._replay_or_run(eta, gather, "fb")
            if self.pg is not None:  # (a world of 1 is the identity)
                import torch.distributed as dist

                dist.all_reduce(self.flat, group=self.pg)
            self._replay_or_run(eta, gather, "upd")
        if gather:
            self._gslot ^= 1  # the next batch was prefetched into the other slot

    def _replay_or_run(self, eta, gather, part):
        if not self.use_graph or (part == "dp" and not self.graph_comm):
            self._run_eager(eta, gather, part)
            return
        key = (float(eta), gather, part, self._slot, self._parity)
        g = self._graphs.get(key)
        if g is None:
            # the first execution is eager, on the stream that is then
            # captured (initialises cuBLAS handles / per-stream workspaces and
            # kernel attributes outside capture); capture only records, it
            # does not execute, so the captured graph replays from step 2 on
            cur = torch.cuda.current_stream()
            if self._cap_stream is None:
                _lo, hi = torch.cuda.Stream.priority_range()
                self._cap_stream = torch.cuda.Stream(device=self.dev, priority=hi)
            cs = self._cap_stream
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                self._run_eager(eta, gather, part)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                self._run_eager(eta, gather, part)
            cur.wait_stream(cs)
            self._graphs[key] = g
            return
        g.replay()

    def train_batch(self, xb, tb, eta: float, loss_out=None) -> None:
        """One step on a host-supplied batch (the reference's per-batch call
        sequence, train.py:398-401): xb [features, B] and tb [classes, B]
        (pinned host tensors for asynchronous copies) are copied into one of
        two device input slots on a copy stream, so the copy of batch k+1
        overlaps the step of batch k; the captured step then runs on the
        current stream and the batch loss is copied into `loss_out` (a pinned
        float64 host tensor) when given.  Stream-ordered; nothing
        synchronises with the host."""
        B = self.B
        if tuple(xb.shape) != (self.n_in, B) or tuple(tb.shape) != (self.classes, B):
            raise InvalidArgumentError(
                f"expected batch shapes {(self.n_in, B)} / {(self.classes, B)}")
        if self._copy_stream is None:
            # two copy streams, each moving half of the feature rows: one
            # host->device copy reached 29 GB/s on the B200 box's PCIe link,
            # two in flight 53 GB/s (scripts/probe_h2d.py)
            self._copy_stream = [torch.cuda.Stream(device=self.dev) for _ in range(2)]
            self._slot_ready = [[torch.cuda.Event() for _ in range(2)] for _ in range(2)]
            self._slot_free = [torch.cuda.Event() for _ in range(2)]
            for e in self._slot_free:
                e.record()
        slot = self._next_slot
        self._next_slot ^= 1
        main = torch.cuda.current_stream()
        x_src = torch.as_tensor(xb)
        h = (self.n_in + 1) // 2
        parts = ((0, h), (h, self.n_in))
        for half, (cs, (r0, r1)) in enumerate(zip(self._copy_stream, parts)):
            cs.wait_event(self._slot_free[slot])  # the step that read this slot is done
            with torch.cuda.stream(cs):
                if r1 > r0:
                    self.x_slots[slot][r0:r1, :B].copy_(x_src[r0:r1], non_blocking=True)
                if half == 0:
                    self.t_slots[slot][:, :B].copy_(torch.as_tensor(tb), non_blocking=True)
                self._slot_ready[slot][half].record(cs)
        for e in self._slot_ready[slot]:
            main.wait_event(e)
        self.step(eta, gather=False, slot=slot)
        self._slot_free[slot].record(main)
        if loss_out is not None:
            loss_out.copy_(self.loss, non_blocking=True)

    def loss_value(self) -> float:
        """Summed softmax-CE loss of the last step's local batch (syncs)."""
        return float(self.loss.item())

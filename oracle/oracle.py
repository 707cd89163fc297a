"""CPU oracle for the static-sparse MLP training path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module, and only as the checker or the timed CPU
baseline; the product package (paper_2407_17437_b200) never does.

It restates the reference package's algorithm (arxiv 2407.17437 "sparsemlp",
pkg/src/sparsemlp) on the CPU:

* the four CSR kernels: oracle/csr_oracle.c (_kernels.py:25-83), via ctypes;
* the step glue with the same numpy operations the reference applies
  (bias nn.py:173, ReLU nn.py:86-91, softmax CE nn.py:385-417, the /B of
  train.py:399, row sums tensor_core.py:353-356, the optimizer sequence
  nn.py:118-131,187-198, BLAS for dense layers nn.py:241-255);
* the seeded construction: streams (sparsity.py:31-55), ER solve
  (sparsity.py:103-180), pattern sampler (sparsity.py:183-216), Xavier
  (sparsity.py:223-237), build_model (bench.py:127-151), sgd_train's epoch
  loop (train.py:357-423) and synthetic_blobs (data_io.py:215-248);
* a pure-Python PCG64 (XSL-RR 128/64) with LCG jump-ahead -- the algorithm the
  device Xavier kernel uses -- checked against numpy's own generator.

Parity pins: tests/golden/ (written by tests/golden/make_golden.py from the
reference itself in the build container) -- kernel outputs, bitwise optimizer
trajectories, ER plans, patterns/Xavier hashes, and the reference's recorded
weight fingerprints (pkg/test_output.txt:26), which this oracle reproduces.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liborcl.so"
_lib = None


def build() -> Path:
    srcs = [HERE / "csr_oracle.c", HERE / "pattern_oracle.c"]
    if not LIB.exists() or LIB.stat().st_mtime < max(p.stat().st_mtime for p in srcs):
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        p, i64 = C.c_void_p, C.c_int64
        for suf, T in (("f32", C.c_float), ("f64", C.c_double)):
            getattr(L, f"orc_spmm_{suf}").argtypes = [p, p, p, i64, p, i64, p]
            getattr(L, f"orc_spmm_t_{suf}").argtypes = [p, p, p, i64, i64, p, i64, p, i64]
            getattr(L, f"orc_sddmm_{suf}").argtypes = [p, p, i64, p, p, i64, p]
            getattr(L, f"orc_axpby_{suf}").argtypes = [T, p, T, p, i64]
            getattr(L, f"orc_row_sums_{suf}").argtypes = [p, i64, i64, p]
        L.orc_philox_u64.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_philox_u64.restype = C.c_uint64
        L.orc_sample_pattern.argtypes = [i64, i64, i64, C.c_uint64, C.c_uint64, p, p]
        L.orc_sample_pattern.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def sample_pattern_device_spec(n_out, n_in, nnz, seed, stream_id=0):
    """CPU restatement of the device sampler (csrc/sampler.cu): the first nnz
    distinct Philox candidates of the grid, as CSR (row_ptr, col_idx)."""
    rp = np.zeros(n_out + 1, np.int32)
    ci = np.zeros(max(nnz, 1), np.int32)
    rc = lib().orc_sample_pattern(n_out, n_in, nnz, seed, stream_id, _p(rp), _p(ci))
    if rc != 0:
        raise ValueError("orc_sample_pattern failed")
    return rp, ci[:nnz]


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _suf(dt) -> str:
    return "f32" if np.dtype(dt) == np.float32 else "f64"


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c(a, dt=None):
    return np.ascontiguousarray(a, dtype=dt)


# ---------------------------------------------------------------------------
# kernels (tensor_core.py:227-306 wrappers around _kernels.py)
# ---------------------------------------------------------------------------
def spmm(row_ptr, col_idx, values, dense):
    values = _c(values)
    dense = _c(dense, values.dtype)
    m, n = len(row_ptr) - 1, dense.shape[1]
    out = np.empty((m, n), dtype=values.dtype)
    getattr(lib(), f"orc_spmm_{_suf(values.dtype)}")(
        _p(_c(row_ptr, np.int32)), _p(_c(col_idx, np.int32)), _p(values), m, _p(dense), n, _p(out))
    return out


def spmm_t(row_ptr, col_idx, values, ncols, dense, nblocks=None):
    values = _c(values)
    dense = _c(dense, values.dtype)
    m, n = len(row_ptr) - 1, dense.shape[1]
    if nblocks is None:
        nblocks = max(1, min(max_threads(), ncols))
    out = np.empty((ncols, n), dtype=values.dtype)
    getattr(lib(), f"orc_spmm_t_{_suf(values.dtype)}")(
        _p(_c(row_ptr, np.int32)), _p(_c(col_idx, np.int32)), _p(values), m, ncols, _p(dense), n,
        _p(out), int(nblocks))
    return out


def sddmm(row_ptr, col_idx, a, b):
    a = _c(a)
    b = _c(b, a.dtype)
    m, kk = len(row_ptr) - 1, a.shape[1]
    out = np.empty(len(col_idx), dtype=a.dtype)
    getattr(lib(), f"orc_sddmm_{_suf(a.dtype)}")(
        _p(_c(row_ptr, np.int32)), _p(_c(col_idx, np.int32)), m, _p(a), _p(b), kk, _p(out))
    return out


def axpby(alpha, s: np.ndarray, beta, t: np.ndarray) -> None:
    """In place s = T(alpha) s + T(beta) t (tensor_core.py:304-305 casts)."""
    T = s.dtype.type
    getattr(lib(), f"orc_axpby_{_suf(s.dtype)}")(T(alpha), _p(s), T(beta), _p(_c(t, s.dtype)),
                                                 s.shape[0])


def row_sums(a):
    a = _c(a)
    out = np.empty(a.shape[0], dtype=a.dtype)
    getattr(lib(), f"orc_row_sums_{_suf(a.dtype)}")(_p(a), a.shape[0], a.shape[1], _p(out))
    return out


# ---------------------------------------------------------------------------
# seeded construction
# ---------------------------------------------------------------------------
STREAMS = ("pattern", "init", "shuffle", "dropout", "augment", "data")


class Streams:
    """Per-purpose PCG64 generators from SeedSequence spawn keys."""

    def __init__(self, seed):
        self.seed = int(seed)
        self._g = {}

    def __call__(self, purpose):
        if purpose not in self._g:
            seq = np.random.SeedSequence(entropy=self.seed, spawn_key=(STREAMS.index(purpose),))
            self._g[purpose] = np.random.Generator(np.random.PCG64(seq))
        return self._g[purpose]


def er_plan(chain, density):
    """(densities, nnz) of the ER solve with round-half-even + drift fix."""
    pairs = list(zip(chain[:-1], chain[1:]))
    sizes = [a * b for a, b in pairs]
    ratio = [(a + b) / (a * b) for a, b in pairs]  # sparsity.py:127
    target = density * sum(sizes)
    sat = [False] * len(pairs)
    dens = [0.0] * len(pairs)
    while True:
        denom = sum(a + b for (a, b), s in zip(pairs, sat) if not s)
        if denom == 0:
            break
        eps = (target - sum(sz for sz, s in zip(sizes, sat) if s)) / denom
        new = [i for i in range(len(pairs)) if not sat[i] and eps * ratio[i] >= 1.0]
        for i in new:
            sat[i], dens[i] = True, 1.0
        if new:
            continue
        for i in range(len(pairs)):
            if not sat[i]:
                dens[i] = eps * ratio[i]
        break
    nnz = [sz if s else int(round(d * sz)) for d, sz, s in zip(dens, sizes, sat)]
    drift = int(round(target)) - sum(nnz)
    order = sorted(range(len(pairs)), key=lambda i: -sizes[i])
    step = 1 if drift > 0 else -1
    while drift:
        moved = False
        for i in order:
            if 0 <= nnz[i] + step <= sizes[i]:
                nnz[i] += step
                drift -= step
                moved = True
                break
        if not moved:
            break
    return dens, nnz


def sample_pattern(n_out, n_in, nnz, rng):
    row_ptr = np.zeros(n_out + 1, dtype=np.int64)
    col_idx = np.empty(nnz, dtype=np.int32)
    if nnz:
        counts = rng.multivariate_hypergeometric([n_in] * n_out, nnz)
        np.cumsum(counts, out=row_ptr[1:])
        for i in range(n_out):
            if counts[i]:
                cols = rng.choice(n_in, size=counts[i], replace=False, shuffle=False)
                col_idx[row_ptr[i]:row_ptr[i + 1]] = np.sort(cols)
    return row_ptr.astype(np.int32), col_idx


def sample_pattern_large(n_out, n_in, nnz, rng):
    """Injected pattern for grids >= 2**31 (config 5; the reference refuses
    them, sparsity.py:193-195): multinomial row counts redrawn until every row
    fits, then sorted distinct columns per row -- the same numpy call
    sequence as the package's sample_pattern_large_host."""
    while True:
        counts = rng.multinomial(nnz, np.full(n_out, 1.0 / n_out))
        if counts.max(initial=0) <= n_in:
            break
    row_ptr = np.zeros(n_out + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col_idx = np.empty(nnz, dtype=np.int32)
    for i in range(n_out):
        if counts[i]:
            cols = rng.choice(n_in, size=counts[i], replace=False, shuffle=False)
            col_idx[row_ptr[i]:row_ptr[i + 1]] = np.sort(cols)
    return row_ptr.astype(np.int32), col_idx


def xavier(n_in, n_out, rng, nnz=None, dtype=np.float32):
    a = float(np.sqrt(6.0 / (n_in + n_out)))
    size = n_out * n_in if nnz is None else nnz
    return rng.uniform(-a, a, size=size).astype(dtype)


# pure-Python PCG64 (XSL-RR 128/64), the device kernel's algorithm
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
M128 = (1 << 128) - 1


def pcg_advance(state, inc, delta):
    cur_mult, cur_plus, acc_mult, acc_plus = PCG_MULT, inc, 1, 0
    while delta:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & M128
        cur_plus = ((cur_mult + 1) * cur_plus) & M128
        cur_mult = (cur_mult * cur_mult) & M128
        delta >>= 1
    return (acc_mult * state + acc_plus) & M128


def pcg_output(state):
    hi, lo = state >> 64, state & ((1 << 64) - 1)
    x = hi ^ lo
    rot = hi >> 58
    return ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)


def pcg_uniform(state, inc, offset, count, a):
    """Xavier values offset..offset+count-1 of a stream at (state, inc)."""
    st = pcg_advance(state, inc, offset)
    out = np.empty(count, dtype=np.float64)
    for i in range(count):
        st = (st * PCG_MULT + inc) & M128
        u = (pcg_output(st) >> 11) * (1.0 / 9007199254740992.0)
        out[i] = -a + (2.0 * a) * u
    return out


def synthetic_blobs(n_classes, n_features, n_per_class, spread, seed, n_test_per_class=None):
    """data_io.synthetic_blobs restated: Gaussian blobs from the "data" stream."""
    rng = Streams(seed)("data")
    if n_test_per_class is None:
        n_test_per_class = max(1, n_per_class // 5)
    centers = rng.standard_normal((n_classes, n_features))

    def draw(per_class):
        xs, labels = [], []
        for c in range(n_classes):
            noise = rng.standard_normal((per_class, n_features))
            xs.append(centers[c] + spread * noise)
            labels.append(np.full(per_class, c))
        x = np.concatenate(xs).astype(np.float32)
        y = np.concatenate(labels)
        order = rng.permutation(len(y))
        t = np.zeros((n_classes, len(y)), dtype=np.float32)
        t[y[order], np.arange(len(y))] = 1.0
        return np.ascontiguousarray(x[order].T), t

    xtr, ttr = draw(n_per_class)
    xte, tte = draw(n_test_per_class)
    return xtr, ttr, xte, tte


# ---------------------------------------------------------------------------
# model + step
# ---------------------------------------------------------------------------
class Layer:
    def __init__(self, n_in, n_out, relu, sparse, values, row_ptr=None, col_idx=None,
                 mu=0.9, nesterov=True, dtype=np.float32):
        self.n_in, self.n_out, self.relu, self.sparse = n_in, n_out, relu, sparse
        self.values = np.array(values, dtype=dtype)  # sparse: [nnz]; dense: [n_out*n_in]
        self.row_ptr = None if row_ptr is None else np.asarray(row_ptr, np.int32)
        self.col_idx = None if col_idx is None else np.asarray(col_idx, np.int32)
        self.bias = np.zeros(n_out, dtype=dtype)
        self.vel = np.zeros_like(self.values)
        self.vbias = np.zeros_like(self.bias)
        self.mu, self.nesterov = mu, nesterov
        self.mask = None  # masked-dense baseline: [n_out*n_in] 0/1 (nn.py:201-264)

    @property
    def W(self):
        return self.values.reshape(self.n_out, self.n_in)


class OracleMLP:
    """The reference's compiled Sequential of Sparse/Dense(+ReLU) layers with
    Momentum optimizers, restated on the CPU."""

    def __init__(self, layers, seed=0):
        self.layers = layers
        self.streams = Streams(seed)

    @classmethod
    def build(cls, chain, density, seed=0, momentum=0.9, nesterov=True, dtype=np.float32,
              backend="sparse", large_patterns=False):
        """bench.build_model + Sequential.compile (bench.py:127-151, train.py:136-188).
        backend "masked": the MaskedDense baseline -- the same pattern / init
        draws scattered into dense storage plus a 0/1 mask (train.py:159-170)."""
        dens, nnz = er_plan(list(chain), density)
        st = Streams(seed)
        prng, irng = st("pattern"), st("init")
        layers = []
        for i, (n_in, n_out) in enumerate(zip(chain[:-1], chain[1:])):
            relu = i < len(chain) - 2
            if dens[i] >= 1.0:
                w = xavier(n_in, n_out, irng, dtype=dtype)
                layers.append(Layer(n_in, n_out, relu, False, w, mu=momentum, nesterov=nesterov,
                                    dtype=dtype))
            else:
                if large_patterns and n_out * n_in >= 2**31:
                    rp, ci = sample_pattern_large(n_out, n_in, nnz[i], prng)
                else:
                    rp, ci = sample_pattern(n_out, n_in, nnz[i], prng)
                v = xavier(n_in, n_out, irng, nnz=nnz[i], dtype=dtype)
                if backend == "masked":
                    rows = np.repeat(np.arange(n_out), np.diff(rp))
                    w = np.zeros((n_out, n_in), dtype=dtype)
                    w[rows, ci] = v
                    mk = np.zeros((n_out, n_in), dtype=dtype)
                    mk[rows, ci] = 1
                    lay = Layer(n_in, n_out, relu, False, w.reshape(-1), mu=momentum,
                                nesterov=nesterov, dtype=dtype)
                    lay.mask = mk.reshape(-1)
                    layers.append(lay)
                else:
                    layers.append(
                        Layer(n_in, n_out, relu, True, v, rp, ci, momentum, nesterov, dtype))
        m = cls(layers)
        m.streams = st
        return m

    def parameters(self):
        """(name, array) in the reference's naming (train.py:227-238): layer i
        counts activation layers too."""
        out, idx = [], 0
        for lay in self.layers:
            if lay.sparse:
                out += [(f"layer{idx}.values", lay.values), (f"layer{idx}.bias", lay.bias)]
            else:
                out += [(f"layer{idx}.weights", lay.W), (f"layer{idx}.bias", lay.bias)]
            idx += 2 if lay.relu else 1
        return out

    def fingerprint(self) -> str:
        h = hashlib.sha256()
        for name, arr in self.parameters():
            h.update(name.encode())
            h.update(np.ascontiguousarray(arr).tobytes())
        return h.hexdigest()

    def forward(self, x):
        self._cache = []
        for lay in self.layers:
            if lay.sparse:
                y = spmm(lay.row_ptr, lay.col_idx, lay.values, x)
            else:
                y = lay.W @ x
            y += lay.bias[:, None]
            self._cache.append((x, y if lay.relu else None))
            x = np.maximum(y, 0) if lay.relu else y
        return x

    @staticmethod
    def softmax_ce_grad(y, t):
        z = y - y.max(axis=0, keepdims=True)
        e = np.exp(z)
        return e / e.sum(axis=0, keepdims=True) - t

    @staticmethod
    def softmax_ce_loss(y, t):
        z = y - y.max(axis=0, keepdims=True)
        log_norm = np.log(np.exp(z).sum(axis=0))
        return float(np.sum(log_norm - (z * t).sum(axis=0)))

    def backward(self, d):
        grads = []
        for lay, (x, ypre) in zip(reversed(self.layers), reversed(self._cache)):
            if lay.relu:
                d = d * (ypre > 0)
            if lay.sparse:
                g = sddmm(lay.row_ptr, lay.col_idx, d, x)
                gb = d.sum(axis=1)
                d = spmm_t(lay.row_ptr, lay.col_idx, lay.values, lay.n_in, d)
            else:
                g = (d @ x.T).reshape(-1)
                if lay.mask is not None:  # nn.py:255-256
                    g *= lay.mask
                gb = d.sum(axis=1)
                d = lay.W.T @ d
            grads.append((g, gb))
        return list(reversed(grads))

    def optimize(self, grads, eta):
        for lay, (g, gb) in zip(self.layers, grads):
            T = lay.values.dtype.type
            if lay.sparse:  # nn.py:189-193 (Nesterov default) / 194-197
                axpby(lay.mu, lay.vel, 1.0, g)
                if lay.nesterov:
                    axpby(1.0, lay.values, -eta * lay.mu, lay.vel)
                    axpby(1.0, lay.values, -eta, g)
                else:
                    axpby(1.0, lay.values, -eta, lay.vel)
            else:  # _step_vector on the dense weights (nn.py:118-131, 260-264)
                if lay.mask is not None:
                    lay.vel *= lay.mask
                self._step_vector(lay.values, g, lay.vel, lay, eta, T)
                if lay.mask is not None:
                    lay.values *= lay.mask
            self._step_vector(lay.bias, gb, lay.vbias, lay, eta, T)

    @staticmethod
    def _step_vector(param, grad, vel, lay, eta, T):
        vel *= T(lay.mu)
        vel += grad
        if lay.nesterov:
            param += T(-eta * lay.mu) * vel
            param += T(-eta) * grad
        else:
            param += T(-eta) * vel

    def step(self, xb, tb, eta, divisor=None):
        """One batch of the reference loop body (train.py:398-401); returns the
        summed batch loss of the forward pass (nn.py:397-408)."""
        y = self.forward(xb)
        loss = self.softmax_ce_loss(y, tb)
        d = self.softmax_ce_grad(y, tb) / (divisor or xb.shape[1])
        self.optimize(self.backward(d), eta)
        return loss

    def train(self, x, t, epochs, batch, schedule, shuffle=True, step_hook=None):
        """sgd_train's epoch loop (train.py:357-423) without evaluation."""
        n = x.shape[1]
        rng = self.streams("shuffle")
        idx = np.arange(n)
        for ep in range(epochs):
            if shuffle:
                rng.shuffle(idx)
            eta = schedule(ep, epochs)
            for k in range(n // batch):
                b = idx[k * batch:(k + 1) * batch]
                loss = self.step(x[:, b], t[:, b], eta)
                if step_hook:
                    step_hook(ep, k, loss)
        return self


def multistep(base_lr, milestones=(0.5, 0.75), gamma=0.1):
    def sched(epoch, total):
        passed = sum(1 for m in milestones if epoch >= int(m * total))
        return base_lr * gamma**passed
    return sched


def rel_err(actual, expected) -> float:
    """The reference tests' metric (pkg/tests/conftest.py:46-53)."""
    a = np.asarray(actual, dtype=np.float64)
    e = np.asarray(expected, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - e) / np.maximum(1.0, np.abs(e))))


os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

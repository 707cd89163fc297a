"""Device-resident CSR types and the four validated sparse operators.

Mirrors the reference operator layer pkg/src/sparsemlp/tensor_core.py (same
names, argument meaning, validation and exception types) with the storage moved
to B200 HBM and the arithmetic moved to the sm_100a kernels behind the C ABI
(include/sparsemlp_b200.h):

    spmm              Y = S @ B          _kernels.py:25-37   -> smb_spmm
    spmm_transposed   Y = S.T @ B        _kernels.py:40-59   -> smb_spmm_t (CSC index)
    sddmm             S = (A @ B.T) | P  _kernels.py:62-75   -> smb_sddmm
    sparse_combine    S = a*S + b*T      _kernels.py:78-83   -> smb_axpby

All four are bit-identical to the reference kernels for identical inputs
(ascending accumulation order, multiply and add rounded separately).

Array interop: dense operands may be numpy arrays (copied to the device, the
result copied back and returned as numpy, like the reference) or CUDA torch
tensors (no copies; results are CUDA tensors).  Index arrays are int32 and
values float32 or float64 (tensor_core.py:25-26, 170-171).  There is no CPU
fallback: without the CUDA library or a GPU every op raises DeviceError.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import DeviceError, InvalidArgumentError

_INDEX_LIMIT = 2**31

__all__ = [
    "CsrMatrix",
    "SparsityPattern",
    "spmm",
    "spmm_transposed",
    "sddmm",
    "sparse_combine",
    "csr_from_dense",
    "csr_to_dense",
    "dense_matmul",
    "row_sums",
    "add_bias",
    "hadamard",
    "set_num_threads",
    "get_num_threads",
    "max_num_threads",
    "warmup_kernels",
    "device",
    "to_numpy",
]

_NP_TO_TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}
_TORCH_TO_NP = {torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64)}


# ---------------------------------------------------------------------------
# device / stream helpers
# ---------------------------------------------------------------------------
def device() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def dtype_code(dt) -> int:
    dt = np.dtype(_TORCH_TO_NP.get(dt, dt)) if not isinstance(dt, np.dtype) else dt
    if dt == np.float32:
        return _lib.SMB_F32
    if dt == np.float64:
        return _lib.SMB_F64
    raise InvalidArgumentError(f"values must be float32 or float64, got {dt}")


def to_numpy(x):
    """Host numpy copy of a tensor / CsrMatrix values (identity for numpy)."""
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def _index_tensor(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=torch.int32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(device())


def _values_tensor(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        if a.dtype not in _TORCH_TO_NP:
            raise InvalidArgumentError(f"values must be float32 or float64, got {a.dtype}")
        return a.to(device()).contiguous()
    arr = np.ascontiguousarray(a)
    if arr.dtype not in (np.float32, np.float64):
        raise InvalidArgumentError(f"values must be float32 or float64, got {arr.dtype}")
    return torch.from_numpy(arr).to(device())


def _host_len(a) -> int:
    return int(a.shape[0]) if hasattr(a, "shape") else len(a)


def _check_index_range(nrows, ncols, nnz):
    if nrows < 0 or ncols < 0:
        raise InvalidArgumentError("matrix dimensions must be non-negative")
    if nrows >= _INDEX_LIMIT or ncols >= _INDEX_LIMIT or nnz >= _INDEX_LIMIT:
        raise InvalidArgumentError("dimensions and nnz must stay below 2**31 (32-bit indices)")


# ---------------------------------------------------------------------------
# pattern / matrix types
# ---------------------------------------------------------------------------
class _PatternHandle:
    """Owner of the C-side smb_pattern (CSC index + tile index)."""

    __slots__ = ("h", "__weakref__")

    def __init__(self, h):
        self.h = h

    def __del__(self):
        h, self.h = self.h, None
        if h and _lib._lib is not None:
            try:
                _lib._lib.smb_pattern_destroy(h)
            except Exception:
                pass


class SparsityPattern:
    """The fixed nonzero structure shared by a weight matrix, its gradient and
    its momentum buffer (tensor_core.py:97-152), resident on the GPU together
    with its CSC transpose index."""

    __slots__ = ("nrows", "ncols", "row_ptr", "col_idx", "_handle", "_host")

    def __init__(self, nrows, ncols, row_ptr, col_idx, validate: bool = True):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        nnz = _host_len(col_idx)
        _check_index_range(self.nrows, self.ncols, nnz)
        if _host_len(row_ptr) != self.nrows + 1:
            raise InvalidArgumentError(f"row_ptr must have length nrows+1={self.nrows + 1}")
        host = None
        if isinstance(row_ptr, np.ndarray) and isinstance(col_idx, np.ndarray):
            host = (
                np.ascontiguousarray(row_ptr, dtype=np.int32),
                np.ascontiguousarray(col_idx, dtype=np.int32),
            )
        self._host = host
        self.row_ptr = _index_tensor(row_ptr)
        self.col_idx = _index_tensor(col_idx)
        out = C.c_void_p()
        _lib.call(
            "smb_pattern_create",
            ptr(self.row_ptr),
            ptr(self.col_idx),
            self.nrows,
            self.ncols,
            nnz,
            1 if validate else 0,
            stream_ptr(),
            C.byref(out),
        )
        self._handle = _PatternHandle(out.value)

    @property
    def handle(self) -> int:
        return self._handle.h

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def validate(self) -> None:
        SparsityPattern(self.nrows, self.ncols, self.row_ptr, self.col_idx, validate=True)

    def host_arrays(self):
        """(row_ptr, col_idx) as host int32 numpy arrays (cached)."""
        if self._host is None:
            self._host = (to_numpy(self.row_ptr), to_numpy(self.col_idx))
        return self._host

    def csc(self):
        """(col_ptr, row_idx, perm) device copies of the CSC transpose index."""
        dev = self.row_ptr.device
        col_ptr = torch.empty(self.ncols + 1, dtype=torch.int32, device=dev)
        row_idx = torch.empty(self.nnz, dtype=torch.int32, device=dev)
        perm = torch.empty(self.nnz, dtype=torch.int32, device=dev)
        _lib.call("smb_pattern_csc", self.handle, ptr(col_ptr), ptr(row_idx), ptr(perm),
                  stream_ptr())
        return col_ptr, row_idx, perm

    def row_indices(self) -> torch.Tensor:
        counts = (self.row_ptr[1:] - self.row_ptr[:-1]).to(torch.int64)
        rows = torch.arange(self.nrows, dtype=torch.int32, device=self.row_ptr.device)
        return torch.repeat_interleave(rows, counts)

    def with_values(self, values) -> "CsrMatrix":
        return CsrMatrix._from_pattern(self, _values_tensor(values))

    def zeros(self, dtype=np.float32) -> "CsrMatrix":
        tdt = _NP_TO_TORCH[np.dtype(dtype)]
        return CsrMatrix._from_pattern(
            self, torch.zeros(self.nnz, dtype=tdt, device=self.row_ptr.device)
        )

    def dense_mask(self, dtype=np.float32) -> torch.Tensor:
        tdt = _NP_TO_TORCH[np.dtype(dtype)]
        mask = torch.zeros((self.nrows, self.ncols), dtype=tdt, device=self.row_ptr.device)
        if self.nnz:
            mask[self.row_indices().long(), self.col_idx.long()] = 1
        return mask

    def __eq__(self, other):
        if not isinstance(other, SparsityPattern):
            return NotImplemented
        return (
            self.nrows == other.nrows
            and self.ncols == other.ncols
            and torch.equal(self.row_ptr, other.row_ptr)
            and torch.equal(self.col_idx, other.col_idx)
        )

    __hash__ = None

    def __repr__(self):
        return f"SparsityPattern({self.nrows}x{self.ncols}, nnz={self.nnz})"


class CsrMatrix:
    """Compressed sparse row matrix with float32 or float64 values on the GPU.

    Zero-valued stored entries are kept: the pattern is fixed capacity.  The
    index arrays (and their CSC transpose index) live in the shared
    SparsityPattern (tensor_core.py:155-216).
    """

    __slots__ = ("_pattern", "values")

    def __init__(self, nrows, ncols, row_ptr, col_idx, values, validate: bool = True):
        vals = _values_tensor(values)
        pat = SparsityPattern(nrows, ncols, row_ptr, col_idx, validate=validate)
        if vals.shape[0] != pat.nnz or vals.dim() != 1:
            raise InvalidArgumentError("values and col_idx must have equal length")
        self._pattern = pat
        self.values = vals

    @classmethod
    def _from_pattern(cls, pattern: SparsityPattern, values: torch.Tensor) -> "CsrMatrix":
        if values.dim() != 1 or values.shape[0] != pattern.nnz:
            raise InvalidArgumentError("values and col_idx must have equal length")
        obj = cls.__new__(cls)
        obj._pattern = pattern
        obj.values = values
        return obj

    nrows = property(lambda self: self._pattern.nrows)
    ncols = property(lambda self: self._pattern.ncols)
    row_ptr = property(lambda self: self._pattern.row_ptr)
    col_idx = property(lambda self: self._pattern.col_idx)

    @property
    def nnz(self) -> int:
        return self._pattern.nnz

    @property
    def shape(self):
        return self._pattern.shape

    @property
    def dtype(self) -> np.dtype:
        return _TORCH_TO_NP[self.values.dtype]

    @property
    def pattern(self) -> SparsityPattern:
        return self._pattern

    def validate(self) -> None:
        self._pattern.validate()
        if self.values.shape[0] != self._pattern.nnz:
            raise InvalidArgumentError("values and col_idx must have equal length")

    def copy(self) -> "CsrMatrix":
        return CsrMatrix._from_pattern(self._pattern, self.values.clone())

    def same_structure(self, other: "CsrMatrix") -> bool:
        if self._pattern is other._pattern:
            return True
        return self._pattern == other._pattern

    def to_dense(self) -> torch.Tensor:
        return csr_to_dense(self)

    def __repr__(self):
        return f"CsrMatrix({self.nrows}x{self.ncols}, nnz={self.nnz}, dtype={self.dtype})"


# ---------------------------------------------------------------------------
# dense operand plumbing
# ---------------------------------------------------------------------------
def _check_dense(name, arr, dtype):
    """-> (device tensor [rows, n] with unit column stride, is_host_input)."""
    dtype = np.dtype(dtype)
    if isinstance(arr, torch.Tensor):
        if arr.dim() != 2:
            raise InvalidArgumentError(f"{name} must be a 2-D ndarray")
        if _TORCH_TO_NP.get(arr.dtype) != dtype:
            raise InvalidArgumentError(f"{name} must have dtype {dtype}, got {arr.dtype}")
        t = arr.to(device())
        if t.shape[1] > 1 and t.stride(1) != 1 or t.stride(0) < t.shape[1]:
            t = t.contiguous()
        return t, False
    if not isinstance(arr, np.ndarray) or arr.ndim != 2:
        raise InvalidArgumentError(f"{name} must be a 2-D ndarray")
    if arr.dtype != dtype:
        raise InvalidArgumentError(f"{name} must have dtype {dtype}, got {arr.dtype}")
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device()), True


def _ld(t: torch.Tensor) -> int:
    return int(t.stride(0)) if t.shape[0] > 1 else max(int(t.shape[1]), int(t.stride(0)), 1)


def _ret(t: torch.Tensor, host: bool):
    return to_numpy(t) if host else t


# ---------------------------------------------------------------------------
# the four operators
# ---------------------------------------------------------------------------
def spmm(s: CsrMatrix, dense, bias=None, relu: bool = False):
    """Sparse-times-dense product S @ B -> (s.nrows, B.cols)  (tensor_core.py:227-240).

    Optional fused epilogue: ``+ bias[:, None]`` (nn.py:173) and ReLU
    (nn.py:86-87).  Rows of S without nonzeros yield zero (or bias) rows.
    """
    d, host = _check_dense("dense operand", dense, s.dtype)
    if s.ncols != d.shape[0]:
        raise InvalidArgumentError(
            f"dimension mismatch: S is {s.nrows}x{s.ncols}, B has {d.shape[0]} rows"
        )
    n = int(d.shape[1])
    b = None
    if bias is not None:
        b = _values_tensor(bias).to(s.values.dtype)
        if b.shape != (s.nrows,):
            raise InvalidArgumentError(f"bias must have shape ({s.nrows},)")
    out = torch.empty((s.nrows, n), dtype=s.values.dtype, device=d.device)
    if s.nrows and n:
        _lib.call(
            "smb_spmm_p", dtype_code(s.dtype), s.pattern.handle, ptr(s.values), ptr(d), _ld(d),
            n, ptr(b), _lib.SMB_EPI_RELU if relu else _lib.SMB_EPI_NONE, ptr(out), _ld(out),
            stream_ptr(),
        )
    return _ret(out, host)


def spmm_transposed(s: CsrMatrix, dense, mask=None):
    """Transposed product S.T @ B -> (s.ncols, B.cols) without materialising S.T
    (tensor_core.py:243-255), through the pattern's CSC index.  Optional fused
    ``* (mask > 0)`` (ReLU.backward of the layer below, nn.py:89-91)."""
    d, host = _check_dense("dense operand", dense, s.dtype)
    if s.nrows != d.shape[0]:
        raise InvalidArgumentError(
            f"dimension mismatch: S is {s.nrows}x{s.ncols}, B has {d.shape[0]} rows"
        )
    n = int(d.shape[1])
    mk = None
    if mask is not None:
        mk, _ = _check_dense("mask", mask, s.dtype)
        if tuple(mk.shape) != (s.ncols, n):
            raise InvalidArgumentError("mask must have the output's shape")
    out = torch.zeros((s.ncols, n), dtype=s.values.dtype, device=d.device)
    if s.ncols and n:
        _lib.call(
            "smb_spmm_t", dtype_code(s.dtype), s.pattern.handle, ptr(s.values), ptr(d), _ld(d), n,
            ptr(mk), _ld(mk) if mk is not None else 0, ptr(out), _ld(out), stream_ptr(),
        )
    return _ret(out, host)


def sddmm(pattern: SparsityPattern, a, b, out: CsrMatrix | None = None) -> CsrMatrix:
    """Sampled dense-dense product (A @ B.T) on the pattern (tensor_core.py:258-288).

    value(i, j) = dot(A[i, :], B[j, :]) for each stored (i, j); the dense
    product is never formed.  With ``out`` its values are overwritten in place.
    """
    if isinstance(pattern, CsrMatrix):
        pattern = pattern.pattern
    a_dt = _TORCH_TO_NP[a.dtype] if isinstance(a, torch.Tensor) else np.asarray(a).dtype
    b_dt = _TORCH_TO_NP[b.dtype] if isinstance(b, torch.Tensor) else np.asarray(b).dtype
    if a_dt != b_dt:
        raise InvalidArgumentError("A and B must share a dtype")
    ad, _ = _check_dense("A", a, a_dt)
    bd, _ = _check_dense("B", b, a_dt)
    if ad.shape[0] != pattern.nrows or bd.shape[0] != pattern.ncols:
        raise InvalidArgumentError(
            f"dimension mismatch: pattern is {pattern.nrows}x{pattern.ncols}, "
            f"A has {ad.shape[0]} rows, B has {bd.shape[0]} rows"
        )
    if ad.shape[1] != bd.shape[1]:
        raise InvalidArgumentError("A and B must have the same number of columns")
    if out is None:
        out = pattern.zeros(dtype=a_dt)
    elif out.dtype != a_dt or out.nnz != pattern.nnz:
        raise InvalidArgumentError("out matrix does not match pattern/dtype")
    if pattern.nnz:
        n = int(ad.shape[1])
        _lib.call(
            "smb_sddmm", dtype_code(a_dt), pattern.handle, ptr(ad), _ld(ad), ptr(bd), _ld(bd), n,
            ptr(out.values), stream_ptr(),
        )
    return out


def sparse_combine(alpha: float, s: CsrMatrix, beta: float, t: CsrMatrix, checked: bool = True):
    """In-place S = alpha*S + beta*T on raw value arrays (tensor_core.py:291-306);
    alpha and beta are cast to the value dtype first (tensor_core.py:304-305)."""
    if s.dtype != t.dtype:
        raise InvalidArgumentError("S and T must share a dtype")
    if checked and not s.same_structure(t):
        raise InvalidArgumentError("S and T must have identical sparsity structure")
    if s.nnz:
        _lib.call(
            "smb_axpby", dtype_code(s.dtype), float(alpha), ptr(s.values), float(beta),
            ptr(t.values), s.nnz, stream_ptr(),
        )
    return s


# ---------------------------------------------------------------------------
# helpers (not on the hot path)
# ---------------------------------------------------------------------------
def csr_from_dense(dense, dtype=None) -> CsrMatrix:
    """Compress a dense matrix, dropping exact zeros (tensor_core.py:309-329)."""
    if isinstance(dense, torch.Tensor):
        dense = to_numpy(dense)
    if not isinstance(dense, np.ndarray) or dense.ndim != 2:
        raise InvalidArgumentError("expected a 2-D ndarray")
    if dtype is None:
        dtype = dense.dtype if dense.dtype in (np.float32, np.float64) else np.float32
    dense = np.ascontiguousarray(dense, dtype=dtype)
    nrows, ncols = dense.shape
    _check_index_range(nrows, ncols, 0)
    rows, cols = np.nonzero(dense)
    row_ptr = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=nrows), out=row_ptr[1:])
    return CsrMatrix(
        nrows, ncols, row_ptr.astype(np.int32), cols.astype(np.int32), dense[rows, cols],
        validate=False,
    )


def csr_to_dense(s: CsrMatrix) -> torch.Tensor:
    out = torch.zeros((s.nrows, s.ncols), dtype=s.values.dtype, device=s.values.device)
    if s.nnz:
        out[s.pattern.row_indices().long(), s.col_idx.long()] = s.values
    return out


def dense_matmul(a, b, transpose_a: bool = False, transpose_b: bool = False):
    """Dense product with optional transposes (fp32/fp64 cuBLAS, TF32 off)."""
    host = isinstance(a, np.ndarray) and isinstance(b, np.ndarray)
    at = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))
    bt = b if isinstance(b, torch.Tensor) else torch.from_numpy(np.asarray(b))
    if at.dim() != 2 or bt.dim() != 2:
        raise InvalidArgumentError("operands must be 2-D")
    left = at.T if transpose_a else at
    right = bt.T if transpose_b else bt
    if left.shape[1] != right.shape[0]:
        raise InvalidArgumentError(f"dimension mismatch: {tuple(left.shape)} @ {tuple(right.shape)}")
    with _no_tf32():
        out = left.to(device()) @ right.to(device())
    return _ret(out, host)


class _no_tf32:
    def __enter__(self):
        self.prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False

    def __exit__(self, *exc):
        torch.backends.cuda.matmul.allow_tf32 = self.prev


def row_sums(dense):
    """Row sums in numpy's pairwise order (tensor_core.py:353-356), on the GPU."""
    if isinstance(dense, torch.Tensor):
        if dense.dim() != 2:
            raise InvalidArgumentError("expected a 2-D ndarray")
        dt = _TORCH_TO_NP.get(dense.dtype)
        if dt is None:
            raise InvalidArgumentError(f"unsupported dtype {dense.dtype}")
    else:
        dense = np.asarray(dense)
        if dense.ndim != 2:
            raise InvalidArgumentError("expected a 2-D ndarray")
        dt = dense.dtype if dense.dtype in (np.float32, np.float64) else np.dtype(np.float64)
        dense = dense.astype(dt, copy=False)
    d, host = _check_dense("dense", dense, dt)
    out = torch.empty(d.shape[0], dtype=d.dtype, device=d.device)
    if d.shape[0]:
        _lib.call("smb_row_sums", dtype_code(dt), ptr(d), d.shape[0], d.shape[1], _ld(d),
                  ptr(out), stream_ptr())
    return _ret(out, host)


def add_bias(dense, bias):
    """Add a length-m bias vector to every column of an m x n matrix."""
    if dense.ndim != 2 or bias.ndim != 1 or bias.shape[0] != dense.shape[0]:
        raise InvalidArgumentError(
            f"bias of length {tuple(bias.shape)} does not broadcast over {tuple(dense.shape)}"
        )
    return dense + bias[:, None]


def hadamard(a, b):
    if tuple(a.shape) != tuple(b.shape):
        raise InvalidArgumentError(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    return a * b


# Thread-count API of the reference (tensor_core.py:48-68).  GPU results never
# depend on a host thread count; these remain for drop-in compatibility.
_THREADS = 1


def set_num_threads(n: int) -> None:
    global _THREADS
    if not 1 <= int(n) <= max_num_threads():
        raise InvalidArgumentError(f"thread count must be in [1, {max_num_threads()}], got {n}")
    _THREADS = int(n)


def get_num_threads() -> int:
    return _THREADS


def max_num_threads() -> int:
    import os

    return max(8, os.cpu_count() or 1)


def warmup_kernels(dtypes=(np.float32,)) -> None:
    """Load the library and launch every operator once (tensor_core.py:374-382)."""
    for dt in dtypes:
        s = csr_from_dense(np.array([[1.0, 0.0], [0.5, 2.0]], dtype=dt))
        d = torch.ones((2, 2), dtype=_NP_TO_TORCH[np.dtype(dt)], device=device())
        spmm(s, d)
        spmm_transposed(s, d)
        sddmm(s.pattern, d, d)
        sparse_combine(1.0, s, 0.0, s.copy())
    torch.cuda.synchronize()

"""ctypes binding of the C ABI declared in include/sparsemlp_b200.h.

This is the only place Python touches native code.  There is deliberately no
CPU fallback: if the shared library cannot be loaded (or no GPU is visible when
an op runs) the call raises ``DeviceError``.  Status codes map onto the
reference's exception types (errors.py): SMB_ERR_INVALID -> InvalidArgumentError,
SMB_ERR_STATE -> StateError, SMB_ERR_CUDA -> DeviceError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import DeviceError, InvalidArgumentError, StateError

# SMB_LIB overrides the library file (tuning experiments load alternative builds)
LIB_PATH = Path(os.environ.get("SMB_LIB") or Path(__file__).resolve().parent / "libsparsemlp_b200.so")

SMB_OK, SMB_ERR_INVALID, SMB_ERR_STATE, SMB_ERR_CUDA = 0, 1, 2, 3
SMB_F32, SMB_F64 = 0, 1
SMB_EPI_NONE, SMB_EPI_RELU = 0, 1
SMB_OPT_NONE, SMB_OPT_GD, SMB_OPT_MOMENTUM, SMB_OPT_NESTEROV = 0, 1, 2, 3
SMB_HINT_CONCURRENT = 0x100  # OR-ed into opt_kind of smb_sddmm_update_into

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int
_u64 = C.c_uint64
_f64 = C.c_double

# name -> (restype, argtypes); mirrors include/sparsemlp_b200.h one to one
SIGNATURES = {
    "smb_abi_version": (_i32, []),
    "smb_last_error": (C.c_char_p, []),
    "smb_launch_count": (_u64, []),
    "smb_spmm": (_i32, [_i32, _p, _p, _p, _i64, _i64, _p, _i64, _i64, _p, _i32, _p, _i64, _p]),
    "smb_pattern_create": (_i32, [_p, _p, _i64, _i64, _i64, _i32, _p, C.POINTER(_p)]),
    "smb_pattern_destroy": (_i32, [_p]),
    "smb_pattern_csc": (_i32, [_p, _p, _p, _p, _p]),
    "smb_spmm_t": (_i32, [_i32, _p, _p, _p, _i64, _i64, _p, _i64, _p, _i64, _p]),
    "smb_spmm_t_csc": (_i32, [_i32, _p, _p, _p, _i64, _i64, _p, _i64, _p, _i64, _p]),
    "smb_values_to_csc": (_i32, [_i32, _p, _p, _p, _p]),
    "smb_spmm_p": (_i32, [_i32, _p, _p, _p, _i64, _i64, _p, _i32, _p, _i64, _p]),
    "smb_sddmm": (_i32, [_i32, _p, _p, _i64, _p, _i64, _i64, _p, _p]),
    "smb_axpby": (_i32, [_i32, _f64, _p, _f64, _p, _i64, _p]),
    "smb_sddmm_update": (
        _i32,
        [_i32, _p, _p, _i64, _p, _i64, _i64, _p, _p, _p, _p, _p, _p, _i32, _f64, _f64, _p],
    ),
    "smb_spmm_t_bias": (
        _i32,
        [_i32, _p, _p, _p, _i64, _i64, _p, _i64, _p, _i64, _p, _p, _p, _i32, _f64, _f64, _p],
    ),
    "smb_bias_grad_update": (_i32, [_i32, _p, _i64, _i64, _i64, _p, _p, _p, _i32, _f64, _f64, _p]),
    "smb_softmax_ce_workspace_bytes": (C.c_size_t, [_i64]),
    "smb_softmax_ce_step": (
        _i32,
        [_i32, _p, _i64, _p, _i64, _i64, _i64, _f64, _p, _i64, _p, _p, _p, _p, _i32, _f64, _f64,
         _p, _i32, _p, _p],
    ),
    "smb_sddmm_update_into": (
        _i32,
        [_i32, _p, _p, _i64, _p, _i64, _i64, _p, _p, _p, _p, _p, _p, _p, _i32, _f64, _f64, _p],
    ),
    "smb_optimizer_step": (_i32, [_i32, _p, _p, _p, _i64, _i32, _f64, _f64, _p]),
    "smb_dense_backward_input": (
        _i32, [_i32, _p, _i64, _i64, _i64, _p, _i64, _i64, _p, _i64, _p, _i64, _p]),
    "smb_dense_grad_update": (
        _i32, [_i32, _p, _i64, _i64, _p, _i64, _i64, _i64, _p, _i64, _p, _p, _i32, _f64, _f64,
               _p]),
    "smb_dense_forward_workspace_bytes": (C.c_size_t, [_i64, _i64, _i64]),
    "smb_dense_forward_small": (
        _i32, [_i32, _p, _i64, _i64, _i64, _p, _i64, _i64, _p, _p, _i64, _p, _p]),
    "smb_optimizer_step_multi": (_i32, [_i32, _p, _i32, _i64, _i32, _f64, _f64, _p]),
    "smb_masked_optimizer_step": (_i32, [_i32, _p, _p, _p, _p, _i64, _i32, _f64, _f64, _p]),
    "smb_row_sums": (_i32, [_i32, _p, _i64, _i64, _i64, _p, _p]),
    "smb_softmax_ce_grad": (
        _i32,
        [_i32, _p, _i64, _p, _i64, _i64, _i64, _f64, _p, _i64, _p, _p],
    ),
    "smb_relu": (_i32, [_i32, _p, _i64, _i64, _i64, _p, _i64, _p]),
    "smb_relu_backward": (_i32, [_i32, _p, _i64, _p, _i64, _i64, _i64, _p, _i64, _p]),
    "smb_gather_columns": (_i32, [_i32, _p, _i64, _i64, _p, _p, _i64, _i64, _p, _i64, _p]),
    "smb_step_counter_advance": (_i32, [_p, _i32, _p]),
    "smb_gather_columns_ahead": (_i32, [_i32, _p, _i64, _i64, _p, _p, _i32, _i32, _i64, _p, _i64,
                                        _p]),
    "smb_xavier_pcg64": (_i32, [_i32, _u64, _u64, _u64, _u64, _u64, _i64, _f64, _p, _p]),
    "smb_sample_pattern": (_i32, [_i64, _i64, _i64, _u64, _u64, _p, _p, _p]),
    "smb_philox_u64": (_u64, [_u64, _u64, _u64]),
    "smb_chain_plan_create": (_i32, [_i32, _p, _p, _i64, _i64, C.POINTER(_p)]),
    "smb_chain_plan_destroy": (_i32, [_p]),
    "smb_chain_plan_info": (_i32, [_p, _p]),
    "smb_chain_plan_profile": (_i32, [_p, _p]),
    "smb_chain_workspace_bytes": (C.c_size_t, [_i64]),
    "smb_chain_refresh": (_i32, [_p, _i32, _p, _p]),
    "smb_chain_run": (_i32, [_p, _p, _p, _p, _p, _i64, _f64, _p, _p, _p]),
}

_lock = threading.Lock()
_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building first if the .so is absent or stale) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_missing and os.environ.get("SMB_NO_BUILD") != "1":
            from . import build as _build

            try:
                if _build.needs_build():
                    _build.build()
            except Exception as exc:  # toolchain missing: only fatal if no prebuilt .so
                if not LIB_PATH.exists():
                    raise DeviceError(f"cannot build {LIB_PATH.name}: {exc}") from exc
        if not LIB_PATH.exists():
            raise DeviceError(f"CUDA library {LIB_PATH} is missing; run __graft_entry__.build()")
        try:
            lib = C.CDLL(str(LIB_PATH))
        except OSError as exc:
            raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.smb_abi_version() != 1:
            raise DeviceError("libsparsemlp_b200 ABI version mismatch")
        _lib = lib
        return lib


def check(status: int, what: str = "") -> None:
    if status == SMB_OK:
        return
    msg = load().smb_last_error().decode(errors="replace") or what
    if status == SMB_ERR_INVALID:
        raise InvalidArgumentError(msg)
    if status == SMB_ERR_STATE:
        raise StateError(msg)
    raise DeviceError(msg)


def call(name: str, *args) -> None:
    """Call an smb_* entry point and raise on a non-zero status."""
    check(getattr(load(), name)(*args), name)


def launch_count() -> int:
    return int(load().smb_launch_count())

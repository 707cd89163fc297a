"""Model archives: one NPY file per tensor plus manifest.json, schema 1.0.

The on-disk format is the reference's (pkg/src/sparsemlp/data_io.py:250-535:
file names ``layerNN_<tensor>.npy``, manifest keys, the exception types and
messages callers match on), so archives move both ways between the reference
and this package -- pattern injection into the oracle, checkpoint hand-off,
on-disk size claims.  The implementation is table-driven: each layer kind
has a codec that lists its manifest fields and tensors once, and the same
table drives both writing and reading.  Parameters live in HBM: saving copies
each tensor to the host once; loading uploads them and rebuilds the device
CSR pattern (validated on the GPU with the reference's messages).
"""

from __future__ import annotations

import ast
import json
import os
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .errors import DatasetIOError, FormatError, InvalidArgumentError
from .nn import (
    ActivationLayer,
    DenseLinearLayer,
    SparseLinearLayer,
    activation_from_name,
    optimizer_from_dict,
)
from .sparsity import Rng
from .tensor_core import SparsityPattern, csr_from_dense
from .train import Sequential

__all__ = [
    "save_npy",
    "load_npy",
    "save_model",
    "load_model",
    "SizeReport",
    "model_size_report",
    "archive_weight_file_bytes",
]

SCHEMA_VERSION = "1.0"
LIBRARY_VERSION = "0.1.0"  # the reference package version this archive format matches
_ARCHIVE_DTYPES = (np.dtype(np.float32), np.dtype(np.float64), np.dtype(np.int32))
_MAGIC = b"\x93NUMPY"


# ---------------------------------------------------------------------------
# NPY tensors (data_io.py:255-280 semantics)
# ---------------------------------------------------------------------------
def save_npy(path, arr) -> None:
    """Write one tensor; float32 / float64 / int32 only, never pickled."""
    a = arr.detach().cpu().numpy() if isinstance(arr, torch.Tensor) else np.asarray(arr)
    a = np.ascontiguousarray(a)
    if a.dtype not in _ARCHIVE_DTYPES:
        raise InvalidArgumentError(f"unsupported archive dtype {a.dtype}")
    with open(path, "wb") as fh:
        np.save(fh, a, allow_pickle=False)


def _read_npy_header(fh, path):
    """(dtype, fortran_order, shape) from an NPY v1/v2/v3 header."""
    if fh.read(6) != _MAGIC:
        raise FormatError(f"{path}: bad NPY magic bytes")
    ver = fh.read(2)
    if len(ver) != 2 or ver[0] not in (1, 2, 3):
        raise FormatError(f"{path}: corrupt NPY header (version {ver!r})")
    size_fmt = "<H" if ver[0] == 1 else "<I"
    raw = fh.read(struct.calcsize(size_fmt))
    if len(raw) != struct.calcsize(size_fmt):
        raise FormatError(f"{path}: corrupt NPY header (truncated)")
    (hlen,) = struct.unpack(size_fmt, raw)
    text = fh.read(hlen)
    try:
        header = ast.literal_eval(text.decode("latin1" if ver[0] < 3 else "utf8"))
        dtype = np.dtype(header["descr"])
        shape = tuple(int(s) for s in header["shape"])
        fortran = bool(header["fortran_order"])
    except Exception as exc:  # malformed dict / missing keys / bad descr
        raise FormatError(f"{path}: corrupt NPY header ({exc})") from exc
    if dtype.hasobject:
        raise FormatError(f"{path}: corrupt NPY header (object arrays are not allowed)")
    return dtype, fortran, shape


def load_npy(path, expect_dtype=None, expect_shape=None) -> np.ndarray:
    """Read one tensor, checking magic, header, dtype and shape."""
    path = Path(path)
    if not path.is_file():
        raise DatasetIOError(f"missing tensor file: {path}")
    with open(path, "rb") as fh:
        dtype, fortran, shape = _read_npy_header(fh, path)
        count = int(np.prod(shape, dtype=np.int64))
        body = fh.read(count * dtype.itemsize)
    if len(body) != count * dtype.itemsize:
        raise FormatError(f"{path}: corrupt NPY header (payload shorter than its shape)")
    arr = np.frombuffer(body, dtype=dtype, count=count).reshape(shape, order="F" if fortran else "C")
    if expect_dtype is not None and arr.dtype != np.dtype(expect_dtype):
        raise FormatError(f"{path}: dtype {arr.dtype}, manifest says {expect_dtype}")
    if expect_shape is not None and arr.shape != tuple(expect_shape):
        raise FormatError(f"{path}: shape {arr.shape}, manifest says {tuple(expect_shape)}")
    return np.array(arr)  # owned, writable


# ---------------------------------------------------------------------------
# layer codecs: one table entry per manifest "kind"
# ---------------------------------------------------------------------------
class _Codec:
    """describe(layer) -> (manifest fields, [(tensor key, array)]);
    build(entry, fetch) -> layer, with fetch(key, dtype, shape) reading the
    tensor file the entry's "files" map names for `key`."""

    kind = ""
    layer_type = None


class _SparseCodec(_Codec):
    kind, layer_type = "sparse", SparseLinearLayer

    def describe(self, layer):
        w = layer.weights
        fields = {"n_in": layer.n_in, "n_out": layer.n_out, "nnz": w.nnz,
                  "density": layer.density, "optimizer": layer.optimizer.to_dict()}
        return fields, [("values", w.values), ("col_idx", w.col_idx), ("row_ptr", w.row_ptr),
                        ("bias", layer.bias)]

    def build(self, entry, fetch, dtype):
        n_in, n_out, nnz = entry["n_in"], entry["n_out"], entry["nnz"]
        values = fetch("values", dtype, (nnz,))
        col_idx = fetch("col_idx", np.int32, (nnz,))
        row_ptr = fetch("row_ptr", np.int32, (n_out + 1,))
        bias = fetch("bias", dtype, (n_out,))
        try:
            pattern = SparsityPattern(n_out, n_in, row_ptr, col_idx)
        except InvalidArgumentError as exc:
            raise FormatError(f"invalid CSR structure in archive: {exc}") from exc
        return SparseLinearLayer(pattern, values, bias, optimizer_from_dict(entry["optimizer"]))


class _DenseCodec(_Codec):
    """Dense layer; a masked-dense baseline layer stores its mask as a CSR
    pattern (mask_col_idx / mask_row_ptr)."""

    kind, layer_type = "dense", DenseLinearLayer

    def describe(self, layer):
        fields = {"n_in": layer.n_in, "n_out": layer.n_out, "density": layer.density,
                  "masked": layer.mask is not None, "optimizer": layer.optimizer.to_dict()}
        tensors = [("weights", layer.weights), ("bias", layer.bias)]
        if layer.mask is not None:
            csr = csr_from_dense(layer.mask)
            tensors += [("mask_col_idx", csr.col_idx), ("mask_row_ptr", csr.row_ptr)]
        return fields, tensors

    def build(self, entry, fetch, dtype):
        n_in, n_out = entry["n_in"], entry["n_out"]
        weights = fetch("weights", dtype, (n_out, n_in))
        bias = fetch("bias", dtype, (n_out,))
        mask = None
        if entry.get("masked"):
            col_idx = fetch("mask_col_idx", np.int32, None)
            row_ptr = fetch("mask_row_ptr", np.int32, (n_out + 1,))
            try:
                mask = SparsityPattern(n_out, n_in, row_ptr, col_idx).dense_mask(dtype)
            except InvalidArgumentError as exc:
                raise FormatError(f"invalid mask structure in archive: {exc}") from exc
        return DenseLinearLayer(weights, bias, optimizer_from_dict(entry["optimizer"]), mask=mask)


class _ActivationCodec(_Codec):
    kind, layer_type = "activation", ActivationLayer

    def describe(self, layer):
        return {"fn": layer.fn.name}, []

    def build(self, entry, fetch, dtype):
        return ActivationLayer(activation_from_name(entry["fn"]))


_CODECS = [_SparseCodec(), _DenseCodec(), _ActivationCodec()]
_BY_KIND = {c.kind: c for c in _CODECS}
# kinds the reference writes that are not on the B200 training path
_OFF_PATH_KINDS = ("batchnorm", "dropout")


def _codec_for_layer(layer) -> _Codec:
    for c in _CODECS:
        if isinstance(layer, c.layer_type):
            return c
    raise InvalidArgumentError(f"cannot serialize layer {type(layer).__name__}")


# ---------------------------------------------------------------------------
# model archives (data_io.py:359-455 format)
# ---------------------------------------------------------------------------
def save_model(model, dir_path) -> dict:
    """Write a compiled model to ``dir_path``; returns the manifest."""
    model._require_compiled()
    root = Path(dir_path)
    root.mkdir(parents=True, exist_ok=True)
    entries = []
    for i, layer in enumerate(model.layers):
        codec = _codec_for_layer(layer)
        fields, tensors = codec.describe(layer)
        files = {key: f"layer{i:02d}_{key}.npy" for key, _ in tensors}
        for key, arr in tensors:
            save_npy(root / files[key], arr)
        entries.append({"kind": codec.kind, **fields, "files": files})
    manifest = {"schema_version": SCHEMA_VERSION, "library_version": LIBRARY_VERSION,
                "input_size": model.input_size, "batch_size": model.batch_size,
                "dtype": np.dtype(model.dtype).name, "layers": entries}
    (root / "manifest.json").write_text(json.dumps(manifest, indent=1))
    return manifest


def _read_manifest(root: Path) -> dict:
    path = root / "manifest.json"
    if not path.is_file():
        raise DatasetIOError(f"missing manifest: {path}")
    try:
        manifest = json.loads(path.read_text())
    except json.JSONDecodeError as exc:
        raise FormatError(f"{path}: invalid JSON ({exc})") from exc
    major = str(manifest.get("schema_version", "")).split(".")[0]
    if major != SCHEMA_VERSION.split(".")[0]:
        raise FormatError(
            f"unsupported archive schema version {str(manifest.get('schema_version', ''))!r}")
    return manifest


def load_model(dir_path, seed: int = 0) -> Sequential:
    """Rebuild a model from an archive onto the GPU; parameters reload
    bit-identically."""
    root = Path(dir_path)
    manifest = _read_manifest(root)
    dtype = np.dtype(manifest["dtype"])
    model = Sequential()
    model.rng = Rng(seed)
    model.rng.stream("dropout")  # the stream the reference reserves for dropout layers
    for entry in manifest["layers"]:
        kind = entry["kind"]
        codec = _BY_KIND.get(kind)
        if codec is None:
            if kind in _OFF_PATH_KINDS:
                raise FormatError(f"layer kind {kind!r} is not on the B200 training path")
            raise FormatError(f"unknown layer kind {kind!r} in manifest")
        files = entry.get("files", {})

        def fetch(key, want_dtype, want_shape, files=files):
            return load_npy(root / files[key], want_dtype, want_shape)

        model.layers.append(codec.build(entry, fetch, dtype))
    model.input_size = manifest["input_size"]
    model.batch_size = manifest["batch_size"]
    model.dtype = dtype
    widths = [l.n_out for l in model.layers if isinstance(l, (SparseLinearLayer, DenseLinearLayer))]
    model.output_size = widths[-1] if widths else model.input_size
    model.compiled = True
    return model


# ---------------------------------------------------------------------------
# size accounting (data_io.py:458-531)
# ---------------------------------------------------------------------------
@dataclass
class SizeReport:
    """Bytes needed to store the model's tensors, no file headers."""

    layers: list
    weight_bytes: int
    bias_bytes: int
    other_bytes: int

    @property
    def total_bytes(self) -> int:
        return self.weight_bytes + self.bias_bytes + self.other_bytes

    def to_dict(self):
        return {"layers": self.layers, "weight_bytes": self.weight_bytes,
                "bias_bytes": self.bias_bytes, "other_bytes": self.other_bytes,
                "total_bytes": self.total_bytes}


def _layer_bytes(layer):
    """(kind, stored weights, weight bytes, bias bytes) of a linear layer:
    sparse = values + int32 col_idx + int32 row_ptr, dense = m * k values."""
    b = layer.bias.element_size() * layer.n_out
    if isinstance(layer, SparseLinearLayer):
        z = layer.weights.nnz
        return "sparse", z, layer.weights.values.element_size() * z + 4 * z + 4 * (layer.n_out + 1), b
    z = layer.n_in * layer.n_out
    return "dense", z, layer.weights.element_size() * z, b


def model_size_report(model) -> SizeReport:
    model._require_compiled()
    rows = []
    for i, layer in enumerate(model.layers):
        if isinstance(layer, (SparseLinearLayer, DenseLinearLayer)):
            kind, z, w, b = _layer_bytes(layer)
            rows.append({"index": i, "kind": kind, "nnz": z, "weight_bytes": w, "bias_bytes": b})
    return SizeReport(layers=rows, weight_bytes=sum(r["weight_bytes"] for r in rows),
                      bias_bytes=sum(r["bias_bytes"] for r in rows), other_bytes=0)


_WEIGHT_FILE_KEYS = ("values", "col_idx", "row_ptr", "weights")


def archive_weight_file_bytes(dir_path) -> int:
    """On-disk bytes of the weight tensor files of an archive."""
    root = Path(dir_path)
    manifest = json.loads((root / "manifest.json").read_text())
    return sum(os.path.getsize(root / fname) for entry in manifest["layers"]
               for key, fname in entry.get("files", {}).items() if key in _WEIGHT_FILE_KEYS)

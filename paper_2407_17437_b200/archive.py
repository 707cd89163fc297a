"""Model archives: one NPY file per tensor plus manifest.json, schema 1.0.

Drop-in for the reference's archive I/O (pkg/src/sparsemlp/data_io.py:250-535):
same file names (``layerNN_values.npy`` ...), manifest keys, validation and
exception types, so archives move both ways between the reference and this
package (pattern injection into the oracle, checkpoint hand-off, on-disk size
claims).  Parameters live in HBM: ``save_model`` copies each tensor to the
host once, ``load_model`` uploads them and rebuilds the device CSR pattern
(validated on the GPU with the reference's messages).
"""

from __future__ import annotations

import json
import os
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
from .tensor_core import SparsityPattern, csr_from_dense, to_numpy
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


def _host(arr) -> np.ndarray:
    return np.ascontiguousarray(to_numpy(arr) if isinstance(arr, torch.Tensor) else arr)


def save_npy(path, arr) -> None:
    """data_io.py:255-259: float32 / float64 / int32 only, no pickles."""
    a = _host(arr)
    if a.dtype not in (np.float32, np.float64, np.int32):
        raise InvalidArgumentError(f"unsupported archive dtype {a.dtype}")
    with open(path, "wb") as fh:
        np.save(fh, a, allow_pickle=False)


def load_npy(path, expect_dtype=None, expect_shape=None) -> np.ndarray:
    """data_io.py:262-280: magic / header / dtype / shape checks."""
    path = Path(path)
    if not path.is_file():
        raise DatasetIOError(f"missing tensor file: {path}")
    with open(path, "rb") as fh:
        if fh.read(6) != b"\x93NUMPY":
            raise FormatError(f"{path}: bad NPY magic bytes")
        fh.seek(0)
        try:
            arr = np.load(fh, allow_pickle=False)
        except ValueError as exc:
            raise FormatError(f"{path}: corrupt NPY header ({exc})") from exc
    if expect_dtype is not None and arr.dtype != np.dtype(expect_dtype):
        raise FormatError(f"{path}: dtype {arr.dtype}, manifest says {expect_dtype}")
    if expect_shape is not None and arr.shape != tuple(expect_shape):
        raise FormatError(f"{path}: shape {arr.shape}, manifest says {tuple(expect_shape)}")
    return arr


def _entry(i: int, layer):
    """(manifest entry, {file name: tensor}) of one layer (data_io.py:283-356)."""
    prefix = f"layer{i:02d}"
    if isinstance(layer, SparseLinearLayer):
        files = {k: f"{prefix}_{k}.npy" for k in ("values", "col_idx", "row_ptr", "bias")}
        entry = {"kind": "sparse", "n_in": layer.n_in, "n_out": layer.n_out,
                 "nnz": layer.weights.nnz, "density": layer.density,
                 "optimizer": layer.optimizer.to_dict(), "files": files}
        tensors = {files["values"]: layer.weights.values, files["col_idx"]: layer.weights.col_idx,
                   files["row_ptr"]: layer.weights.row_ptr, files["bias"]: layer.bias}
        return entry, tensors
    if isinstance(layer, DenseLinearLayer):
        files = {"weights": f"{prefix}_weights.npy", "bias": f"{prefix}_bias.npy"}
        tensors = {files["weights"]: layer.weights, files["bias"]: layer.bias}
        if layer.mask is not None:  # the mask is stored as a CSR pattern
            mask_csr = csr_from_dense(layer.mask)
            files["mask_col_idx"] = f"{prefix}_mask_col_idx.npy"
            files["mask_row_ptr"] = f"{prefix}_mask_row_ptr.npy"
            tensors[files["mask_col_idx"]] = mask_csr.col_idx
            tensors[files["mask_row_ptr"]] = mask_csr.row_ptr
        entry = {"kind": "dense", "n_in": layer.n_in, "n_out": layer.n_out,
                 "density": layer.density, "masked": layer.mask is not None,
                 "optimizer": layer.optimizer.to_dict(), "files": files}
        return entry, tensors
    if isinstance(layer, ActivationLayer):
        return {"kind": "activation", "fn": layer.fn.name, "files": {}}, {}
    raise InvalidArgumentError(f"cannot serialize layer {type(layer).__name__}")


def save_model(model, dir_path) -> dict:
    """Write a compiled model to ``dir_path`` (data_io.py:359-380); returns the manifest."""
    model._require_compiled()
    out = Path(dir_path)
    out.mkdir(parents=True, exist_ok=True)
    layers = []
    for i, layer in enumerate(model.layers):
        entry, tensors = _entry(i, layer)
        for name, arr in tensors.items():
            save_npy(out / name, arr)
        layers.append(entry)
    manifest = {"schema_version": SCHEMA_VERSION, "library_version": LIBRARY_VERSION,
                "input_size": model.input_size, "batch_size": model.batch_size,
                "dtype": np.dtype(model.dtype).name, "layers": layers}
    with open(out / "manifest.json", "w") as fh:
        json.dump(manifest, fh, indent=1)
    return manifest


def load_model(dir_path, seed: int = 0) -> Sequential:
    """Rebuild a model from an archive onto the GPU; parameters reload
    bit-identically (data_io.py:383-455)."""
    root = Path(dir_path)
    manifest_path = root / "manifest.json"
    if not manifest_path.is_file():
        raise DatasetIOError(f"missing manifest: {manifest_path}")
    with open(manifest_path) as fh:
        try:
            manifest = json.load(fh)
        except json.JSONDecodeError as exc:
            raise FormatError(f"{manifest_path}: invalid JSON ({exc})") from exc
    version = str(manifest.get("schema_version", ""))
    if version.split(".")[0] != SCHEMA_VERSION.split(".")[0]:
        raise FormatError(f"unsupported archive schema version {version!r}")
    dtype = np.dtype(manifest["dtype"])

    model = Sequential()
    model.rng = Rng(seed)
    model.rng.stream("dropout")  # reserved like the reference (data_io.py:400)
    for entry in manifest["layers"]:
        kind = entry["kind"]
        files = entry.get("files", {})
        if kind == "sparse":
            n_in, n_out, nnz = entry["n_in"], entry["n_out"], entry["nnz"]
            values = load_npy(root / files["values"], dtype, (nnz,))
            col_idx = load_npy(root / files["col_idx"], np.int32, (nnz,))
            row_ptr = load_npy(root / files["row_ptr"], np.int32, (n_out + 1,))
            bias = load_npy(root / files["bias"], dtype, (n_out,))
            try:
                pattern = SparsityPattern(n_out, n_in, row_ptr, col_idx)
            except InvalidArgumentError as exc:
                raise FormatError(f"invalid CSR structure in archive: {exc}") from exc
            layer = SparseLinearLayer(pattern, values, bias,
                                      optimizer_from_dict(entry["optimizer"]))
        elif kind == "dense":
            n_in, n_out = entry["n_in"], entry["n_out"]
            weights = load_npy(root / files["weights"], dtype, (n_out, n_in))
            bias = load_npy(root / files["bias"], dtype, (n_out,))
            mask = None
            if entry.get("masked"):
                col_idx = load_npy(root / files["mask_col_idx"], np.int32)
                row_ptr = load_npy(root / files["mask_row_ptr"], np.int32, (n_out + 1,))
                try:
                    mask = SparsityPattern(n_out, n_in, row_ptr, col_idx).dense_mask(dtype)
                except InvalidArgumentError as exc:
                    raise FormatError(f"invalid mask structure in archive: {exc}") from exc
            layer = DenseLinearLayer(weights, bias, optimizer_from_dict(entry["optimizer"]),
                                     mask=mask)
        elif kind == "activation":
            layer = ActivationLayer(activation_from_name(entry["fn"]))
        elif kind in ("batchnorm", "dropout"):
            raise FormatError(f"layer kind {kind!r} is not on the B200 training path")
        else:
            raise FormatError(f"unknown layer kind {kind!r} in manifest")
        model.layers.append(layer)

    model.input_size = manifest["input_size"]
    model.batch_size = manifest["batch_size"]
    model.dtype = dtype
    sizes = [l.n_out for l in model.layers if isinstance(l, (SparseLinearLayer, DenseLinearLayer))]
    model.output_size = sizes[-1] if sizes else model.input_size
    model.compiled = True
    return model


@dataclass
class SizeReport:
    """Bytes needed to store the model's tensors, no file headers (data_io.py:458-482)."""

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


def model_size_report(model) -> SizeReport:
    """data_io.py:485-515: sparse = values + col_idx + row_ptr, dense = m*k."""
    model._require_compiled()
    layers, wt, bt = [], 0, 0
    for i, layer in enumerate(model.layers):
        if isinstance(layer, SparseLinearLayer):
            item = layer.weights.values.element_size()
            z = layer.weights.nnz
            w = item * z + 4 * z + 4 * (layer.n_out + 1)
            b = layer.bias.element_size() * layer.n_out
            layers.append({"index": i, "kind": "sparse", "nnz": z, "weight_bytes": w,
                           "bias_bytes": b})
        elif isinstance(layer, DenseLinearLayer):
            w = layer.weights.element_size() * layer.n_in * layer.n_out
            b = layer.bias.element_size() * layer.n_out
            layers.append({"index": i, "kind": "dense", "nnz": layer.n_in * layer.n_out,
                           "weight_bytes": w, "bias_bytes": b})
        else:
            continue
        wt += w
        bt += b
    return SizeReport(layers=layers, weight_bytes=wt, bias_bytes=bt, other_bytes=0)


def archive_weight_file_bytes(dir_path) -> int:
    """On-disk bytes of the weight tensor files of an archive (data_io.py:518-531)."""
    root = Path(dir_path)
    with open(root / "manifest.json") as fh:
        manifest = json.load(fh)
    total = 0
    for entry in manifest["layers"]:
        for key, fname in entry.get("files", {}).items():
            if key in ("values", "col_idx", "row_ptr", "weights"):
                total += os.path.getsize(root / fname)
    return total

"""Datasets for the training path.

``Dataset`` mirrors the reference container (data_io.py:62-72: feature-major
Xtrain [features, N] float32, one-hot Ttrain [classes, N]).  ``synthetic_dataset``
is the seeded N(0,1) stand-in for CIFAR-10 that BASELINE.json / SURVEY.md 8(d)
specify (3072 features, 10 classes, per-feature standardised, uniform labels,
all from one seed); both the reference arm and this package are fed the same
arrays.  ``DeviceDataset`` is the HBM-resident copy the fused step gathers from:
stored sample-major [N, features] so the per-step batch gather reads whole
contiguous samples (replaces train.py:395-396 + tensor_core.py:224).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import InvalidArgumentError
from .tensor_core import device

__all__ = ["Dataset", "synthetic_dataset", "DeviceDataset", "one_hot"]


@dataclass
class Dataset:
    Xtrain: np.ndarray
    Ttrain: np.ndarray
    Xtest: np.ndarray | None = None
    Ttest: np.ndarray | None = None

    def __post_init__(self):
        if self.Xtrain.shape[1] != self.Ttrain.shape[1]:
            raise InvalidArgumentError("Xtrain and Ttrain must have the same number of columns")


def one_hot(labels: np.ndarray, classes: int) -> np.ndarray:
    t = np.zeros((classes, labels.shape[0]), dtype=np.float32)
    t[labels, np.arange(labels.shape[0])] = 1.0
    return t


def synthetic_dataset(seed: int = 0, n_samples: int = 50_000, features: int = 3072,
                      classes: int = 10) -> Dataset:
    """Seeded synthetic stand-in for CIFAR-10:
    X ~ N(0,1) float32 [features, N] standardised per feature, labels uniform."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((features, n_samples), dtype=np.float32)
    mean = x.mean(axis=1, keepdims=True)
    std = x.std(axis=1, keepdims=True)
    std[std == 0] = 1.0
    x = ((x - mean) / std).astype(np.float32)
    labels = rng.integers(0, classes, n_samples)
    return Dataset(Xtrain=np.ascontiguousarray(x), Ttrain=one_hot(labels, classes))


class DeviceDataset:
    """HBM-resident training split, sample-major: X [N, F], T [N, C] float32."""

    def __init__(self, dataset: Dataset, dtype=torch.float32):
        dev = device()
        self.n_samples = int(dataset.Xtrain.shape[1])
        self.features = int(dataset.Xtrain.shape[0])
        self.classes = int(dataset.Ttrain.shape[0])
        self.X = torch.from_numpy(np.ascontiguousarray(dataset.Xtrain.T)).to(dev, dtype)
        self.T = torch.from_numpy(np.ascontiguousarray(dataset.Ttrain.T)).to(dev, dtype)

    @property
    def nbytes(self) -> int:
        return self.X.numel() * self.X.element_size() + self.T.numel() * self.T.element_size()

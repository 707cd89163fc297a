"""Experiment configuration, model builder and weight fingerprint.

Drop-in for the config/builder part of pkg/src/sparsemlp/bench.py:
``ExperimentConfig`` (bench.py:72-118), the density -> lr table
(bench.py:51-69), ``build_model`` (bench.py:127-151: ER plan, saturated layers
become Dense, every layer Momentum(0.9, nesterov=True) by default, ReLU on all
but the last layer) and ``weights_fingerprint`` (bench.py:197-203: SHA-256 over
every parameter's name and raw bytes in layer order).
"""

from __future__ import annotations

import hashlib
from dataclasses import asdict, dataclass, field

import numpy as np

from .errors import ConfigurationError
from .nn import Momentum, ReLU
from .sparsity import er_densities, layer_pairs_from_chain
from .tensor_core import to_numpy
from .train import Dense, MaskedDense, MultiStepSchedule, Sequential, Sparse

__all__ = [
    "TABLE_LR_DEFAULTS",
    "default_learning_rate",
    "ExperimentConfig",
    "build_model",
    "weights_fingerprint",
]

TABLE_LR_DEFAULTS = {
    1.0: 0.01, 0.5: 0.01, 0.2: 0.01, 0.1: 0.03, 0.05: 0.03, 0.01: 0.1, 0.005: 0.1, 0.001: 0.1,
}


def default_learning_rate(density: float) -> float:
    """Exact table match, else the nearest table density in log space."""
    if density in TABLE_LR_DEFAULTS:
        return TABLE_LR_DEFAULTS[density]
    keys = sorted(TABLE_LR_DEFAULTS)
    nearest = min(keys, key=lambda k: abs(np.log10(k) - np.log10(density)))
    return TABLE_LR_DEFAULTS[nearest]


@dataclass
class ExperimentConfig:
    layer_dims: list = field(default_factory=lambda: [3072, 1024, 512, 10])
    density: float = 1.0
    backend: str = "sparse"
    epochs: int = 10
    batch_size: int = 100
    lr: float | None = None
    lr_milestones: tuple = (0.5, 0.75)
    lr_gamma: float = 0.1
    momentum: float = 0.9
    nesterov: bool = True
    seed: int = 0
    dataset: str = "synthetic"
    threads: int | None = None
    out: str | None = None
    eval_metrics: bool = True
    shuffle: bool = True
    augment: bool = False
    # B200 additions (no reference counterpart): data-parallel world size the
    # batch is sharded over (sgd_train's process_group must match) and the
    # CUDA device the model lives on
    world_size: int = 1
    device: str = "cuda"

    def __post_init__(self):
        if self.world_size < 1 or self.batch_size % self.world_size:
            raise ConfigurationError(
                f"batch_size {self.batch_size} must be divisible by world_size {self.world_size}")
        if not 0.0 < self.density <= 1.0:
            raise ConfigurationError(f"density must be in (0, 1], got {self.density}")
        if self.backend not in ("sparse", "masked"):
            raise ConfigurationError(
                f"backend must be 'sparse' or 'masked', got {self.backend!r}")
        if len(self.layer_dims) < 2:
            raise ConfigurationError("layer_dims needs input and output sizes at least")

    def resolved_lr(self) -> float:
        return self.lr if self.lr is not None else default_learning_rate(self.density)

    def schedule(self):
        return MultiStepSchedule(self.resolved_lr(), self.lr_milestones, self.lr_gamma)

    def to_dict(self) -> dict:
        d = asdict(self)
        d["lr"] = self.resolved_lr()
        d["lr_milestones"] = list(self.lr_milestones)
        return d


def build_model(config: ExperimentConfig, large_patterns: bool = False,
                pattern_sampler: str = "host"):
    """ER plan -> Sequential of Sparse (backend "sparse") or MaskedDense
    (backend "masked") layers, Dense where the density saturates, compiled
    with the config's seed (bench.py:127-151).  Returns (model, plan)."""
    plan = er_densities(layer_pairs_from_chain(config.layer_dims), config.density)
    model = Sequential()
    last = len(plan.layer_dims) - 1
    for i, ((_, n_out), dens, nnz) in enumerate(
        zip(plan.layer_dims, plan.layer_densities, plan.layer_nnz)
    ):
        act = ReLU() if i < last else None
        opt = Momentum(config.momentum, nesterov=config.nesterov)
        if dens >= 1.0:
            model.add(Dense(n_out, activation=act, optimizer=opt))
        elif config.backend == "sparse":
            model.add(Sparse(n_out, dens, activation=act, optimizer=opt, nnz=nnz))
        else:
            model.add(MaskedDense(n_out, dens, activation=act, optimizer=opt, nnz=nnz))
    import torch

    dev = torch.device(config.device)
    if dev.type != "cuda":
        raise ConfigurationError(f"the B200 path runs on CUDA devices, got {config.device!r}")
    with torch.cuda.device(dev.index if dev.index is not None else torch.cuda.current_device()):
        model.compile(input_size=config.layer_dims[0], batch_size=config.batch_size,
                      seed=config.seed, large_patterns=large_patterns,
                      pattern_sampler=pattern_sampler)
    return model, plan


def weights_fingerprint(model) -> str:
    """SHA-256 over every parameter tensor's name and raw bytes, in layer order."""
    digest = hashlib.sha256()
    for name, arr in model.parameters():
        digest.update(name.encode())
        digest.update(np.ascontiguousarray(to_numpy(arr)).tobytes())
    return digest.hexdigest()

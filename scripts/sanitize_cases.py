"""Small workloads that launch every kernel family of the library once or a few
times, for compute-sanitizer (memcheck / racecheck / synccheck) runs:

* the fused training step (PDL launches, side streams, gather kernels,
  softmax step, row-sum / bias kernels, CSC value copies) at the config-2
  shape with B=1024, eager (no CUDA graph, so every launch is visible);
* a config-4-like wide step (3072-8192-8192-10, many-wave SDDMM tiles:
  sddmm_warp_kernel; dense output layer: split-K forward, dense_t, dense_grad);
* the data-parallel step structure (force_dp: gradients into the flat buffer,
  per-layer update launches);
* config-3 single kernels (8192^2, d=0.01, B=128) and an L2-sliced SpMM
  (30000^2, B=600: several rows per CTA, column slices);
* batch-1 inference (row_spmv_kernel).

Usage: compute-sanitizer --tool <tool> python scripts/sanitize_cases.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr


def fused_steps(chain, density, B, steps=2, force_dp=False):
    data = smb.synthetic_dataset(seed=1, n_samples=B * (steps + 1), features=chain[0])
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=density, seed=2,
                                                    batch_size=B))
    st = smb.FusedTrainStep(model, B, use_graph=False, force_dp=force_dp)
    st.attach_dataset(smb.DeviceDataset(data))
    st.set_epoch(np.arange(B * (steps + 1)))
    for _ in range(steps):
        st.step(0.01)
    torch.cuda.synchronize()
    print(f"fused {chain} d={density} B={B} dp={force_dp}: loss {st.loss_value():.4f}", flush=True)
    return model


def kernels(n, d, B):
    nnz = int(d * n * n)
    pat = smb.sample_pattern(n, n, nnz, smb.Rng(0).stream("pattern"))
    dev = torch.device("cuda")
    vals = torch.randn(nnz, device=dev)
    vel = torch.zeros_like(vals)
    X = torch.randn(n, B, device=dev)
    dY = torch.randn(n, B, device=dev)
    out = torch.empty(n, B, device=dev)
    s = stream_ptr()
    _lib.call("smb_spmm_p", 0, pat.handle, ptr(vals), ptr(X), B, B, None, 0, ptr(out), B, s)
    _lib.call("smb_spmm_t", 0, pat.handle, ptr(vals), ptr(dY), B, B, ptr(X), B, ptr(out), B, s)
    _lib.call("smb_sddmm_update", 0, pat.handle, ptr(dY), B, ptr(X), B, B, ptr(vals), ptr(vel),
              None, None, None, None, _lib.SMB_OPT_NESTEROV, 0.9, 1e-3, s)
    torch.cuda.synchronize()
    print(f"kernels n={n} d={d} B={B}: ok", flush=True)


def main():
    torch.cuda.set_device(0)
    model = fused_steps([3072, 1024, 512, 10], 0.01, 1024)
    fused_steps([3072, 1024, 512, 10], 0.01, 100, force_dp=True)
    fused_steps([3072, 8192, 8192, 10], 0.01, 256)
    kernels(8192, 0.01, 128)
    kernels(30000, 0.0005, 600)
    sess = smb.InferenceSession(model, batch=1, use_graph=False)
    x = np.random.default_rng(0).standard_normal((3072, 1)).astype(np.float32)
    sess(x)
    torch.cuda.synchronize()
    print("inference: ok", flush=True)


if __name__ == "__main__":
    main()

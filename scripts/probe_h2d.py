"""Host->device copy bandwidth of the e2e batch (12.6 MB fp32) from pinned
memory: one stream vs the copy split over 2 / 4 streams."""
import sys
import time

sys.path.insert(0, ".")
import torch

import os
try:  # the GPU's NUMA-local cores, as bench.py binds them
    import pynvml
    pynvml.nvmlInit()
    pynvml.nvmlDeviceSetCpuAffinity(pynvml.nvmlDeviceGetHandleByIndex(0))
except Exception as exc:  # (affinity is an optimisation)
    print("no NVML affinity:", exc)
x = torch.randn(3072, 1024).pin_memory()
d = torch.empty(3072, 1024, device="cuda")
for nst in (1, 2, 3, 4, 8):
    sts = [torch.cuda.Stream() for _ in range(nst)]
    rows = 3072 // nst
    for _ in range(3):
        for i, s in enumerate(sts):
            with torch.cuda.stream(s):
                d[i * rows:(i + 1) * rows].copy_(x[i * rows:(i + 1) * rows], non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 50
    for _ in range(reps):
        for i, s in enumerate(sts):
            with torch.cuda.stream(s):
                d[i * rows:(i + 1) * rows].copy_(x[i * rows:(i + 1) * rows], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"streams={nst}: {x.numel() * 4 * reps / dt / 1e9:.1f} GB/s", flush=True)

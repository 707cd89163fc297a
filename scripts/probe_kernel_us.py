"""Per-kernel graph-timed durations (KernelTimer) of one fused step, plus the
step time back to back.  usage: [SMB_LIB=...] python scripts/probe_kernel_us.py [LAYERS D B]"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2407_17437_b200 as smb
from paper_2407_17437_b200.engine import KernelTimer

L = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3072,1024,512,10").split(",")]
D = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
data = smb.synthetic_dataset(seed=0, n_samples=8 * B, features=L[0], classes=L[-1])
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=L, density=D, batch_size=B),
                          large_patterns=any(a * b >= 2**31 for a, b in zip(L[:-1], L[1:])))
st = smb.FusedTrainStep(model, B)
st.attach_dataset(smb.DeviceDataset(data))
st.set_epoch(np.arange(8 * B))
for _ in range(5):
    st.step(0.01)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(100):
    st.step(0.01)
e.record()
e.synchronize()
out = KernelTimer().kernel_durations(st, 0.01)
tag = os.path.basename(os.environ.get("SMB_LIB", "current"))
print(tag, f"step {s.elapsed_time(e) * 10:.1f} us",
      {k: round(1e3 * ms / c, 2) for k, (c, ms) in out.items()}, flush=True)

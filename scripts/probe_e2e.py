"""e2e (train_batch from pinned host batches) at the config-2 point: host wall
time per call, device time per step, and the same loop with the step replaced
by nothing (copies only)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2407_17437_b200 as smb

B, L = 1024, [3072, 1024, 512, 10]
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=L, density=0.01, batch_size=B))
import os
st = smb.FusedTrainStep(model, B, chain=os.environ.get("E2E_CHAIN", "1") == "1")
rng = np.random.default_rng(0)
xs = [torch.from_numpy(rng.standard_normal((L[0], B), dtype=np.float32)).pin_memory() for _ in range(4)]
t = np.zeros((10, B), np.float32)
t[rng.integers(0, 10, B), np.arange(B)] = 1
ts = [torch.from_numpy(t.copy()).pin_memory() for _ in range(4)]
loss = torch.empty(1, dtype=torch.float64).pin_memory()
for i in range(5):
    st.train_batch(xs[i % 4], ts[i % 4], 0.01, loss)
torch.cuda.synchronize()
N = 100
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
h0 = time.perf_counter()
for i in range(N):
    st.train_batch(xs[i % 4], ts[i % 4], 0.01, loss)
h1 = time.perf_counter()
e.record()
e.synchronize()
h2 = time.perf_counter()
print(f"host enqueue {1e6 * (h1 - h0) / N:.1f} us/call, wall {1e6 * (h2 - h0) / N:.1f} us/step, "
      f"device {1e3 * s.elapsed_time(e) / N:.1f} us/step -> {B * N / (s.elapsed_time(e) / 1e3):.3e} samples/s")

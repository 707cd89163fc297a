#!/bin/bash
# config-2 fused step, back-to-back replays, with the next-batch gather launched
# at the step start or at the end of the backward (the default)
for p in start end; do
  SMB_PREFETCH_AT=$p python - <<'PY'
import sys, os; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
B = 1024
data = smb.synthetic_dataset(seed=0, n_samples=16384, features=3072)
dd = smb.DeviceDataset(data)
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=0.01, batch_size=B, lr=0.01))
st = smb.FusedTrainStep(model, B); st.attach_dataset(dd); st.set_epoch(np.arange(16384))
for _ in range(6): st.step(0.01)
torch.cuda.synchronize()
res = []
for rep in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(400): st.step(0.01)
    e.record(); e.synchronize(); res.append(s.elapsed_time(e) * 1e3 / 400)
print(os.environ["SMB_PREFETCH_AT"], ["%.2f" % r for r in res])
PY
done

"""One eager fused training step on a BASELINE config inside the NVTX range
"prof", for ncu captures (--nvtx --nvtx-include "prof/"); the kernel tags of
that step, in launch order, go to <tags_file> (the C-ABI calls the step makes,
minus the step counter / optimizer launches the profile regex skips).

usage: python scripts/ncu_step.py [layers] [density] [batch] [warmup] [tags_file]
"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2407_17437_b200 as smb

layers = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3072,1024,512,10").split(",")]
density = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
warm = int(sys.argv[4]) if len(sys.argv) > 4 else 3
tags_file = sys.argv[5] if len(sys.argv) > 5 else None
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=layers, density=density,
                                                batch_size=batch, lr=0.01),
                           large_patterns=any(a * b >= 2**31 for a, b in zip(layers[:-1], layers[1:])))
n = max(8192, 2 * batch)
data = smb.synthetic_dataset(seed=0, n_samples=n, features=layers[0], classes=layers[-1])
st = smb.FusedTrainStep(model, batch, use_graph=False)
st.attach_dataset(smb.DeviceDataset(data))
st.set_epoch(np.arange(n))
for _ in range(warm):
    st.step(0.01)
torch.cuda.synchronize()
with torch.cuda.nvtx.range("prof"):
    st.step(0.01)
    torch.cuda.synchronize()


class _Rec:
    def __init__(self):
        self.calls = []


rec = _Rec()
st.timer = rec
st.step(0.01)
torch.cuda.synchronize()
st.timer = None
# C-ABI calls that launch two kernels (both match the profile regex)
TWO = {"smb_dense_forward_small": (".part", ".sum")}
tags = []
for t, name, _ in rec.calls:
    if t.startswith(("counter", "update")) or name == "smb_step_counter_advance":
        continue
    tags += [t + suf for suf in TWO[name]] if name in TWO else [t]
if tags_file:
    open(tags_file, "w").write(",".join(tags))
print("ok", len(tags), "tags")

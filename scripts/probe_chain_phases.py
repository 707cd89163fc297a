"""Phase timestamps of the column-chain kernel (smb_chain_plan_profile):
per CTA, %globaltimer at the kernel's checkpoints of one graph-replayed
config-2 step, printed relative to the earliest CTA start (median and max
over CTAs)."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib

B = int(os.environ.get("TL_B", "1024"))
layers = [int(x) for x in os.environ.get("TL_LAYERS", "3072,1024,512,10").split(",")]
d = float(os.environ.get("TL_D", "0.01"))
data = smb.synthetic_dataset(seed=0, n_samples=8 * B, features=layers[0], classes=layers[-1])
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=layers, density=d, batch_size=B, lr=0.01))
st = smb.FusedTrainStep(model, B)
info = st.chain_info()
print("chain", info)
ctas = info["cluster"] * info["groups"]
buf = torch.zeros(ctas * 32, dtype=torch.int64, device="cuda")
_lib.call("smb_chain_plan_profile", st._chain.h, buf.data_ptr())
st.attach_dataset(smb.DeviceDataset(data))
st.set_epoch(np.arange(8 * B))
for _ in range(8):
    st.step(0.01)
torch.cuda.synchronize()
a = buf.view(ctas, 32).cpu().numpy().astype(np.int64)
dbg = a[:, 20:32]
n = int((a[0, :20] > 0).sum())
a = a[:, :n]
t0 = a[:, 0].min()
rel = (a - t0) / 1000.0
labels = ["start", "staged", "a0 in"]
print(f"{'stamp':>6} {'min':>8} {'median':>8} {'max':>8}  (us from the first CTA start)")
for j in range(n):
    print(f"{j:6d} {rel[:, j].min():8.2f} {np.median(rel[:, j]):8.2f} {rel[:, j].max():8.2f}")
print("forward-last rows of warp 0, CTA 0 (us from its phase start):",
      [round((x - dbg[0, 0]) / 1000.0, 2) for x in dbg[0] if x > 0])
print("trip counts:", os.environ.get("TL_X", ""))

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
n = int((a[0] > 0).sum())
d = (a[:, 1:n] - a[:, :n - 1]) / 1965.0  # SM cycles -> us at the 1965 MHz boost clock
cum = (a[:, :n] - a[:, :1]) / 1965.0
print(f"{'stamp':>6} {'d median':>9} {'d max':>8} {'cum median':>11} {'cum max':>8}  (us, per CTA, SM clock)")
for j in range(1, n):
    print(f"{j:6d} {np.median(d[:, j - 1]):9.2f} {d[:, j - 1].max():8.2f} {np.median(cum[:, j]):11.2f} {cum[:, j].max():8.2f}")

"""One eager fused training step on a BASELINE config, for ncu captures.

usage: python scripts/ncu_step.py [layers] [density] [batch] [steps]
"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2407_17437_b200 as smb

layers = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3072,1024,512,10").split(",")]
density = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=layers, density=density,
                                                batch_size=batch, lr=0.01))
n = max(8192, 2 * batch)
data = smb.synthetic_dataset(seed=0, n_samples=n, features=layers[0], classes=layers[-1])
st = smb.FusedTrainStep(model, batch, use_graph=False)
st.attach_dataset(smb.DeviceDataset(data))
st.set_epoch(np.arange(n))
for _ in range(steps):
    st.step(0.01)
torch.cuda.synchronize()
print("ok")

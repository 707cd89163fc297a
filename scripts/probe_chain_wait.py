import sys, time, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
B = 1024
layers = [3072, 1024, 512, 10]
data = smb.synthetic_dataset(seed=0, n_samples=4 * B, features=layers[0], classes=layers[-1])
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=layers, density=0.01, batch_size=B, lr=0.01))
st = smb.FusedTrainStep(model, B, use_graph=False)
st.attach_dataset(smb.DeviceDataset(data))
st.set_epoch(np.arange(4 * B))
torch.cuda.synchronize()
print("setup ok", flush=True)
st.step(0.01)
torch.cuda.synchronize()
print("first step ok", flush=True)
st.step(0.01)
print("enqueued", flush=True)
time.sleep(3)
# read the plan's flags through a side stream
lib = _lib.load()
s = torch.cuda.Stream()
print("query main:", torch.cuda.current_stream().query(), flush=True)
for k, s_ in st._sides.items():
    print(k, s_.query(), flush=True)
torch.cuda.synchronize()
print("done", flush=True)

"""Kernel timeline of the graph-replayed config-2 step (torch.profiler / CUPTI
kernel records: start, duration, stream of every kernel inside the replays).
Prints the kernels of one steady-state step relative to its first kernel."""
import json, os, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_17437_b200 as smb

B = int(os.environ.get("TL_B", "1024"))
layers = [int(x) for x in os.environ.get("TL_LAYERS", "3072,1024,512,10").split(",")]
d = float(os.environ.get("TL_D", "0.01"))
data = smb.synthetic_dataset(seed=0, n_samples=8 * B, features=layers[0], classes=layers[-1])
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=layers, density=d, batch_size=B, lr=0.01))
st = smb.FusedTrainStep(model, B)
st.attach_dataset(smb.DeviceDataset(data))
st.set_epoch(np.arange(8 * B))
for _ in range(6):
    st.step(0.01)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(6):
        st.step(0.01)
    torch.cuda.synchronize()
path = "gpurun_out/timeline.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
print("kernels", len(ev))
def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("smb::", "")
    return n[:70]
t0 = ev[0]["ts"]
per = len(ev) // 6
for i, e in enumerate(ev):
    if i % per == 0:
        print("----")
    print(f"{e['ts'] - t0:8.2f} {e['ts'] + e['dur'] - t0:8.2f} {e['dur']:7.2f} s{e['args'].get('stream')} {short(e['name'])}")

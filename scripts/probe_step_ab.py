"""Back-to-back fused steps on a given chain (A/B of env-switched variants).
usage: python scripts/probe_step_ab.py LAYERS DENSITY BATCH"""
import sys, os; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
L = [int(x) for x in sys.argv[1].split(',')]; d = float(sys.argv[2]); B = int(sys.argv[3])
data = smb.synthetic_dataset(seed=0, n_samples=max(8192, 2 * B), features=L[0], classes=L[-1])
dd = smb.DeviceDataset(data)
large = any(a * b >= 2**31 for a, b in zip(L[:-1], L[1:]))
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=L, density=d, batch_size=B, lr=0.01), large_patterns=large)
st = smb.FusedTrainStep(model, B); st.attach_dataset(dd); st.set_epoch(np.arange(data.Xtrain.shape[1]))
for _ in range(5): st.step(0.01)
torch.cuda.synchronize()
res = []
for rep in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50): st.step(0.01)
    e.record(); e.synchronize(); res.append(s.elapsed_time(e) * 1e3 / 50)
print(os.environ.get("SMB_DENSE_T", "1"), sys.argv[1:], ["%.1f" % r for r in res])

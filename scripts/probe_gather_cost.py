"""Critical-path cost of the device batch gather: back-to-back graph replays of
the config-2 step with gather vs on a pre-filled input slot (no gather)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
B = 1024
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=0.01,
                                                batch_size=B, lr=0.01))
data = smb.synthetic_dataset(seed=0, n_samples=16384, features=3072)
st = smb.FusedTrainStep(model, B)
st.attach_dataset(smb.DeviceDataset(data))
st.set_epoch(np.arange(16384))
def run(gather, n=500):
    for _ in range(5): st.step(0.01, gather=gather)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): st.step(0.01, gather=gather)
    e.record(); e.synchronize()
    return s.elapsed_time(e) * 1e3 / n
for _ in range(2):
    print("with gather %.2f us/step, no gather %.2f us/step" % (run(True), run(False)))

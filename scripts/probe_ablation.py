"""Critical-path ablation of the config-2 fused step: back-to-back graph
replays with one kernel tag skipped at a time (timing only -- the numbers a
skipped step computes are meaningless)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import engine
import os
B = int(os.environ.get("ABL_B", "1024"))
LAYERS = [int(x) for x in os.environ.get("ABL_LAYERS", "3072,1024,512,10").split(",")]
DENS = float(os.environ.get("ABL_D", "0.01"))
STEPS = int(os.environ.get("ABL_STEPS", "400"))
data = smb.synthetic_dataset(seed=0, n_samples=16384 if B >= 1024 else 4096, features=LAYERS[0],
                             classes=LAYERS[-1])
ddata = smb.DeviceDataset(data)
orig = engine.FusedTrainStep._call

def time_with(skip):
    def patched(self, tag, name, *args):
        if tag in skip:
            return
        return orig(self, tag, name, *args)
    engine.FusedTrainStep._call = patched
    try:
        large = any(a * b >= 2**31 for a, b in zip(LAYERS[:-1], LAYERS[1:]))
        model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=LAYERS, density=DENS,
                                                        batch_size=B, lr=0.01),
                                   large_patterns=large)
        st = smb.FusedTrainStep(model, B)
        st.attach_dataset(ddata)
        st.set_epoch(np.arange(data.Xtrain.shape[1]))
        for _ in range(6): st.step(0.01)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(STEPS): st.step(0.01)
        e.record(); e.synchronize()
        return s.elapsed_time(e) * 1e3 / STEPS
    finally:
        engine.FusedTrainStep._call = orig

base = time_with(set())
print(f"baseline {base:.2f} us/step")
if os.environ.get("ABL_ONLY_BASE") == "1":
    sys.exit(0)
nl = len(LAYERS) - 1
tags = (["gather", "gather_t"] + [f"spmm[{i}]" for i in range(nl)] + ["softmax_ce"]
        + [f"spmm_t[{i}]" for i in range(nl - 1, 0, -1)] + [f"dense_t[{nl - 1}]"]
        + [f"sddmm_update[{i}]" for i in range(nl)] + [f"bias[{i}]" for i in range(nl)])
for t in tags:
    v = time_with({t})
    print(f"skip {t:18s} {v:8.2f} us/step  (saves {base - v:6.2f})")
v = time_with({t for t in tags if t.startswith("sddmm")})
print(f"skip all sddmm       {v:8.2f} us/step  (saves {base - v:6.2f})")
v = time_with(set(tags))
print(f"skip everything      {v:8.2f} us/step")

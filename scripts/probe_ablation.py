"""Critical-path ablation of the config-2 fused step: back-to-back graph
replays with one kernel tag skipped at a time (timing only -- the numbers a
skipped step computes are meaningless)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import engine
import os
B = int(os.environ.get("ABL_B", "1024"))
data = smb.synthetic_dataset(seed=0, n_samples=16384 if B >= 1024 else 4096, features=3072)
ddata = smb.DeviceDataset(data)
orig = engine.FusedTrainStep._call

def time_with(skip):
    def patched(self, tag, name, *args):
        if tag in skip:
            return
        return orig(self, tag, name, *args)
    engine.FusedTrainStep._call = patched
    try:
        model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10],
                                                        density=0.01, batch_size=B, lr=0.01))
        st = smb.FusedTrainStep(model, B, fuse_logits=os.environ.get("ABL_FUSE_LOGITS") == "1")
        st.attach_dataset(ddata)
        st.set_epoch(np.arange(data.Xtrain.shape[1]))
        for _ in range(6): st.step(0.01)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(400): st.step(0.01)
        e.record(); e.synchronize()
        return s.elapsed_time(e) * 1e3 / 400
    finally:
        engine.FusedTrainStep._call = orig

base = time_with(set())
print(f"baseline {base:.2f} us/step")
tags = ["gather", "gather_t", "spmm[0]", "spmm[1]", "spmm[2]", "softmax_ce", "spmm_t[2]",
        "spmm_t[1]", "sddmm_update[0]", "sddmm_update[1]", "sddmm_update[2]"]
for t in tags:
    v = time_with({t})
    print(f"skip {t:18s} {v:8.2f} us/step  (saves {base - v:6.2f})")
v = time_with({"sddmm_update[0]", "sddmm_update[1]", "sddmm_update[2]"})
print(f"skip all sddmm       {v:8.2f} us/step  (saves {base - v:6.2f})")
v = time_with(set(tags))
print(f"skip everything      {v:8.2f} us/step")

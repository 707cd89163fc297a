"""Scratch timing: per-kernel CUDA-event times of the fused step (eager) and
graph-replay step time, for a few configs.  Not a bench number."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2407_17437_b200 as smb
from paper_2407_17437_b200.engine import KernelTimer

def run(chain, dens, B, n_samples=20000, steps=20):
    model, plan = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=dens, batch_size=B, lr=0.01))
    data = smb.synthetic_dataset(seed=0, n_samples=n_samples, features=chain[0])
    st = smb.FusedTrainStep(model, B)
    st.attach_dataset(smb.DeviceDataset(data))
    st.set_epoch(np.random.default_rng(0).permutation(n_samples))
    for _ in range(3): st.step(0.01)
    torch.cuda.synchronize()
    t = KernelTimer(); st.timer = t; st.use_graph = False
    for _ in range(steps):
        KernelTimer.hold_gpu()
        st.step(0.01)
    summ = t.summary(); st.timer = None; st.use_graph = True
    tot = 0
    print(f"== chain={chain} d={dens} B={B} nnz={plan.layer_nnz}")
    for k, (c, ms) in sorted(summ.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k:18s} {1000*ms/c:9.2f} us"); tot += ms / c
    print(f"   sum of kernels   {1000*tot:9.2f} us")
    for _ in range(3): st.step(0.01)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps): st.step(0.01)
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / steps
    print(f"   graph step       {1000*ms:9.2f} us  -> {B/ms*1e3:,.0f} samples/s")

run([3072,1024,512,10], 0.01, 100)
run([3072,1024,512,10], 0.01, 1024)
run([3072,1024,512,10], 0.1, 1024)
run([3072,8192,8192,8192,10], 0.01, 1024, n_samples=8192, steps=10)

"""Config-2 step time (back to back and with the L2 flush of bench.py) under
monkeypatched engine variants, plus the CUPTI kernel timeline of one
replayed baseline step.  usage: python scripts/probe_cfg2_variants.py"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib

B, L, D = 1024, [3072, 1024, 512, 10], 0.01
data = smb.synthetic_dataset(seed=0, n_samples=20480, features=L[0], classes=L[-1])
dd = smb.DeviceDataset(data)
flush = torch.empty(512 * 2**20 // 4, device="cuda")
sink = torch.empty((), device="cuda")


def run(tag, lab=None, **kw):
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=L, density=D, batch_size=B))
    st = smb.FusedTrainStep(model, B, **kw)
    for k, v in (lab or {}).items():
        setattr(st, k, v)
    st.attach_dataset(dd)
    st.set_epoch(np.arange(20480))
    for _ in range(6):
        st.step(0.01)
    torch.cuda.synchronize()
    b2b = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(100):
            st.step(0.01)
        e.record()
        e.synchronize()
        b2b.append(s.elapsed_time(e) * 10)
    fl = []
    for i in range(40):
        flush.fill_(float(i))
        torch.sum(flush, 0, out=sink)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        st.step(0.01)
        e.record()
        e.synchronize()
        fl.append(s.elapsed_time(e) * 1e3)
    print(f"{tag:28s} b2b {min(b2b):6.1f} us  flushed {np.median(fl):6.1f} us", flush=True)
    return st


def timeline(st, steps=4):
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            st.step(0.01)
        torch.cuda.synchronize()
    path = "gpurun_out/timeline.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    per = len(ev) // steps
    ev = ev[-per:]
    t0 = ev[0]["ts"]
    for e in ev:
        n = e["name"].replace("(anonymous namespace)::", "").replace("smb::", "")[:60]
        print(f"{e['ts'] - t0:8.2f} {e['ts'] + e['dur'] - t0:8.2f} {e['dur']:7.2f} "
              f"s{e['args'].get('stream')} {n}")


if __name__ == "__main__":
    st = run("baseline")
    st2 = run("sddmm at end", lab={"_lab_sddmm_at_end": True})
    hint = _lib.SMB_HINT_CONCURRENT
    _lib.SMB_HINT_CONCURRENT = 0
    st3 = run("sddmm at end, no hint", lab={"_lab_sddmm_at_end": True})
    _lib.SMB_HINT_CONCURRENT = hint
    timeline(st2)

"""A/B of the SDDMM staging variants on the benchmarked shapes: bit-exact
against the oracle, then graph-timed (20 launches, L2-hot like the step).
usage: SMB_SDDMM_TMA=<stages|0> python scripts/lab_sddmm_tma.py"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr
from oracle import oracle as O

O.build()
O.set_threads(os.cpu_count() or 1)
tag = os.path.basename(os.environ.get("SMB_LIB", "current"))
SHAPES = [(8192, 8192, 0.0084, 1024), (8192, 3072, 0.0154, 1024),
          (8192, 8192, 0.001, 512), (8192, 8192, 0.001, 2048), (8192, 8192, 0.01, 128),
          (8192, 8192, 0.01, 512), (8192, 8192, 0.1, 512),
          (65536, 65536, 0.000587, 512), (65536, 3072, 0.00656, 512),
          (1024, 3072, 0.0078, 1024)]
if os.environ.get("LAB_SMALL"):
    SHAPES = [(1024, 3072, 0.0078, 1024), (512, 1024, 0.0175, 1024), (10, 512, 0.609, 1024),
              (1024, 3072, 0.0078, 100), (512, 1024, 0.0175, 100)]
for (m, k, d, B) in SHAPES:
    nnz = int(round(d * m * k))
    pat = smb.sample_pattern(m, k, nnz, smb.Rng(0).stream("pattern"), large=m * k >= 2**31)
    rng = np.random.default_rng(1)
    dev = "cuda"
    vals = torch.from_numpy(rng.standard_normal(nnz).astype(np.float32)).to(dev)
    vel = torch.zeros_like(vals)
    X = torch.randn(k, B, device=dev)
    dY = torch.randn(m, B, device=dev)
    g = torch.empty_like(vals)
    out = torch.empty_like(vals)

    def launch():
        _lib.call("smb_sddmm_update_into", 0, pat.handle, ptr(dY), B, ptr(X), B, B, ptr(vals),
                  ptr(out), ptr(vel), None, None, None, None, 3, 0.9, 1e-4, stream_ptr())

    _lib.call("smb_sddmm", 0, pat.handle, ptr(dY), B, ptr(X), B, B, ptr(g), stream_ptr())
    torch.cuda.synchronize()
    ok = "-"
    if nnz * B <= 2e9:
        rp, ci = pat.host_arrays()
        ref = O.sddmm(rp, ci, dY.cpu().numpy(), X.cpu().numpy())
        ok = "bit-exact" if np.array_equal(ref.view(np.int32), g.cpu().numpy().view(np.int32)) else "MISMATCH"
    launch()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=cs):
        for _ in range(20):
            launch()
    torch.cuda.current_stream().wait_stream(cs)
    gr.replay()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        gr.replay()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3 / 20)
    us = min(ts)
    print(f"{tag} {m}x{k} d={d} B={B} nnz={nnz}: {us:8.2f} us  {nnz * B / us / 1e6:6.2f} Tpairs/s  {ok}",
          flush=True)

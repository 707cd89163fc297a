"""Time smb_backward_fused against smb_spmm_t + smb_sddmm_update_into on one
8192 x 8192 layer (config 3 / config 4 shapes), warm L2, GPU held.
usage: python scripts/probe_bwd_fused.py [density] [B]"""
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr
d = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01
B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
n = 8192
nnz = int(round(d * n * n))
pat = smb.sample_pattern(n, n, nnz, smb.Rng(0).stream("pattern"))
vals = torch.randn(nnz, device="cuda"); vel = torch.zeros_like(vals); w2 = torch.empty_like(vals)
X = torch.randn(n, B, device="cuda"); dY = torch.randn(n, B, device="cuda")
out = torch.empty(n, B, device="cuda")
def sep():
    st = stream_ptr()
    _lib.call("smb_spmm_t", 0, pat.handle, ptr(vals), ptr(dY), B, B, ptr(X), B, ptr(out), B, st)
    _lib.call("smb_sddmm_update_into", 0, pat.handle, ptr(dY), B, ptr(X), B, B, ptr(vals), ptr(w2),
              ptr(vel), None, None, None, None, 3, 0.9, 1e-6, st)
def fused():
    _lib.call("smb_backward_fused", 0, pat.handle, ptr(dY), B, ptr(X), B, B, 1, ptr(out), B,
              ptr(vals), ptr(w2), ptr(vel), None, 3, 0.9, 1e-6, stream_ptr())
def timeit(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(5_000_000)
    s.record()
    for _ in range(reps): f()
    e.record(); e.synchronize()
    return s.elapsed_time(e) * 1e3 / reps
print(f"d={d} B={B} nnz={nnz}: separate {timeit(sep):.1f} us, fused {timeit(fused):.1f} us")

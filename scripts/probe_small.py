"""Probe the small config-2 kernels: softmax-CE step (10 x 1024) and the
last-layer SDDMM+update (10 x 512, 3117 nnz), B=1024, warm L2."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr
B = 1024
y = torch.randn(10, B, device="cuda"); t = torch.zeros(10, B, device="cuda"); t[torch.randint(0, 10, (B,)), torch.arange(B)] = 1
dy = torch.empty(10, B, device="cuda"); loss = torch.zeros(1, dtype=torch.float64, device="cuda")
bias = torch.zeros(10, device="cuda"); vb = torch.zeros(10, device="cuda")
ws = torch.zeros(int(_lib.load().smb_softmax_ce_workspace_bytes(B)), dtype=torch.uint8, device="cuda")
pat = smb.sample_pattern(10, 512, 3117, smb.Rng(0).stream("pattern"))
vals = torch.randn(pat.nnz, device="cuda"); vel = torch.zeros_like(vals)
A = torch.rand(512, B, device="cuda")
def sm():
    _lib.call("smb_softmax_ce_step", 0, ptr(y), B, ptr(t), B, 10, B, float(B), ptr(dy), B, ptr(loss), ptr(bias), ptr(vb), None, 3, 0.9, 0.01, None, 0, ptr(ws), stream_ptr())
def sd():
    _lib.call("smb_sddmm_update", 0, pat.handle, ptr(dy), B, ptr(A), B, B, ptr(vals), ptr(vel), None, None, None, None, 3, 0.9, 0.01, stream_ptr())
for f, name in ((sm, "softmax_step"), (sd, "sddmm_update 10x512")):
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): f()
    e.record(); e.synchronize()
    print("%s: %.2f us" % (name, s.elapsed_time(e) * 1e3 / 20))

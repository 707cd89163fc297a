"""Probe: the config-2 last layer (10 x 512, 3117 nnz) SpMM at B=1024, warm L2."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr
m, k, B = 10, 512, 1024
pat = smb.sample_pattern(m, k, 3117, smb.Rng(0).stream("pattern"))
vals = torch.randn(pat.nnz, device="cuda")
X = torch.randn(k, B, device="cuda"); out = torch.empty(m, B, device="cuda")
def run():
    _lib.call("smb_spmm", 0, ptr(pat.row_ptr), ptr(pat.col_idx), ptr(vals), m, k, ptr(X), B, B, None, 0, ptr(out), B, stream_ptr())
for _ in range(3): run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): run()
e.record(); e.synchronize()
print("spmm 10x512 B=1024: %.2f us" % (s.elapsed_time(e) * 1e3 / 20))

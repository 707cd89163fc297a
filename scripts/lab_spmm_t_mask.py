"""Transposed SpMM with / without the fused ReLU mask vs the forward SpMM on
the config-5 hidden layer (65536^2, d=0.000587, B=512), graph-timed."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr

m = k = 65536
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
nnz = 2521658
rp, ci = smb.sparsity.sample_pattern_large_host(m, k, nnz, smb.Rng(1).stream("pattern"))
pat = smb.SparsityPattern(m, k, rp, ci, validate=False)
dev = "cuda"
vals = torch.randn(nnz, device=dev)
vcsc = torch.empty_like(vals)
_lib.call("smb_values_to_csc", 0, pat.handle, ptr(vals), ptr(vcsc), stream_ptr())
X = torch.randn(k, B, device=dev).relu_()
dY = torch.randn(m, B, device=dev)
out = torch.empty(k, B, device=dev)


def timeit(fn, reps=20):
    fn()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(reps):
            fn()
    torch.cuda.current_stream().wait_stream(cs)
    g.replay()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3 / reps)
    return min(ts)


fwd = timeit(lambda: _lib.call("smb_spmm_p", 0, pat.handle, ptr(vals), ptr(X), B, B, None, 0,
                               ptr(out), B, stream_ptr()))
t_mask = timeit(lambda: _lib.call("smb_spmm_t_csc", 0, pat.handle, ptr(vcsc), ptr(dY), B, B,
                                  ptr(X), B, ptr(out), B, stream_ptr()))
t_nomask = timeit(lambda: _lib.call("smb_spmm_t_csc", 0, pat.handle, ptr(vcsc), ptr(dY), B, B,
                                    None, 0, ptr(out), B, stream_ptr()))
print(f"B={B}: spmm {fwd:.1f} us, spmm_t+mask {t_mask:.1f} us, spmm_t {t_nomask:.1f} us")

# the same product through the forward kernel on W^T stored as CSR
cp = torch.empty(k + 1, dtype=torch.int32, device=dev)
ri = torch.empty(nnz, dtype=torch.int32, device=dev)
_lib.call("smb_pattern_csc", pat.handle, ptr(cp), ptr(ri), None, stream_ptr())
patT = smb.SparsityPattern(k, m, cp, ri, validate=False)
out2 = torch.empty(k, B, device=dev)
t_fwdT = timeit(lambda: _lib.call("smb_spmm_p", 0, patT.handle, ptr(vcsc), ptr(dY), B, B, None, 0,
                                  ptr(out2), B, stream_ptr()))
_lib.call("smb_spmm_t_csc", 0, pat.handle, ptr(vcsc), ptr(dY), B, B, None, 0, ptr(out), B,
          stream_ptr())
torch.cuda.synchronize()
print(f"B={B}: forward kernel on W^T (CSR) {t_fwdT:.1f} us, equal: {torch.equal(out, out2)}")

# order / buffer swap check: the two launches alternate and swap outputs
for rep in range(2):
    a = timeit(lambda: _lib.call("smb_spmm_p", 0, patT.handle, ptr(vcsc), ptr(dY), B, B, None, 0,
                                 ptr(out), B, stream_ptr()))
    b = timeit(lambda: _lib.call("smb_spmm_t_csc", 0, pat.handle, ptr(vcsc), ptr(dY), B, B, None,
                                 0, ptr(out2), B, stream_ptr()))
    print(f"rep {rep}: forward kernel on W^T -> out {a:.1f} us, spmm_t_csc -> out2 {b:.1f} us")
ri2 = pat.col_ptr_dev if hasattr(pat, "col_ptr_dev") else None
print("pattern handle fields equal:",
      bool(torch.equal(cp, cp)), "nnz", nnz)

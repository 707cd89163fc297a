"""Where the transposed SpMM's extra time goes at the config-4 hidden shape
(8192 x 8192, ER d = 0.00839, B = 1024), graph-timed: the CSC kernel with
values through perm (+/- the ReLU mask) against the CSR kernel run on the
transposed pattern (no perm, no mask)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr

import os
B, n, nnz = 1024, 8192, 562878
if os.environ.get("CFG") == "5":  # config-5 hidden layer
    B, n, nnz = 512, 65536, 2521658
    from paper_2407_17437_b200.sparsity import sample_pattern_large_host
    rp_, ci_ = sample_pattern_large_host(n, n, nnz, np.random.default_rng(0))
    pat = smb.SparsityPattern(n, n, rp_, ci_)
else:
    pat = smb.sample_pattern(n, n, nnz, smb.Rng(0).stream("pattern"))
rp, ci = pat.host_arrays()
# W^T in CSR = W in CSC (rows of W^T ascending per column: stable sort)
order = np.argsort(ci, kind="stable")
rows = np.repeat(np.arange(n, dtype=np.int32), np.diff(rp))
rpt = np.zeros(n + 1, np.int32); np.cumsum(np.bincount(ci, minlength=n), out=rpt[1:])
patT = smb.SparsityPattern(n, n, rpt, rows[order].astype(np.int32))
dev = torch.device("cuda")
vals = torch.randn(nnz, device=dev)
valsT = vals[torch.from_numpy(order).to(dev)].contiguous()
dY = torch.randn(n, B, device=dev)
mask = torch.randn(n, B, device=dev).relu_()
out = torch.empty(n, B, device=dev)


def timed(f, reps=20, replays=5):
    f(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream(); cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=cs):
        for _ in range(reps): f()
    torch.cuda.current_stream().wait_stream(cs)
    g.replay()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(replays): g.replay()
    e.record(); e.synchronize()
    return s.elapsed_time(e) * 1e3 / (reps * replays)


r = {}
r["spmm_t perm+mask"] = timed(lambda: _lib.call("smb_spmm_t", 0, pat.handle, ptr(vals), ptr(dY), B, B, ptr(mask), B, ptr(out), B, stream_ptr()))
r["spmm_t perm"] = timed(lambda: _lib.call("smb_spmm_t", 0, pat.handle, ptr(vals), ptr(dY), B, B, None, 0, ptr(out), B, stream_ptr()))
r["csr on W^T (no perm, no mask)"] = timed(lambda: _lib.call("smb_spmm_p", 0, patT.handle, ptr(valsT), ptr(dY), B, B, None, 0, ptr(out), B, stream_ptr()))
r["csr forward on W"] = timed(lambda: _lib.call("smb_spmm_p", 0, pat.handle, ptr(vals), ptr(dY), B, B, None, 0, ptr(out), B, stream_ptr()))
for k, v in r.items():
    print(f"{k:32s} {v:8.2f} us")

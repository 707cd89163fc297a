"""One forward-kernel launch on W^T (CSR) and one smb_spmm_t_csc launch on the
config-5 hidden layer (65536^2, B=512) for an ncu side-by-side."""
import sys

sys.path.insert(0, ".")
import torch

import paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr

m = k = 65536
B = 512
nnz = 2521658
rp, ci = smb.sparsity.sample_pattern_large_host(m, k, nnz, smb.Rng(1).stream("pattern"))
pat = smb.SparsityPattern(m, k, rp, ci, validate=False)
vals = torch.randn(nnz, device="cuda")
vcsc = torch.empty_like(vals)
_lib.call("smb_values_to_csc", 0, pat.handle, ptr(vals), ptr(vcsc), stream_ptr())
dY = torch.randn(m, B, device="cuda")
out = torch.empty(k, B, device="cuda")
cp = torch.empty(k + 1, dtype=torch.int32, device="cuda")
ri = torch.empty(nnz, dtype=torch.int32, device="cuda")
_lib.call("smb_pattern_csc", pat.handle, ptr(cp), ptr(ri), None, stream_ptr())
patT = smb.SparsityPattern(k, m, cp, ri, validate=False)
torch.cuda.synchronize()
_lib.call("smb_spmm_p", 0, patT.handle, ptr(vcsc), ptr(dY), B, B, None, 0, ptr(out), B,
          stream_ptr())
_lib.call("smb_spmm_t_csc", 0, pat.handle, ptr(vcsc), ptr(dY), B, B, None, 0, ptr(out), B,
          stream_ptr())
torch.cuda.synchronize()

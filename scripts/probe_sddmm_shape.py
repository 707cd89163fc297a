"""Launch the SDDMM + update on one layer shape a few times (for ncu captures).
usage: python scripts/probe_sddmm_shape.py M K DENSITY BATCH [REPS]"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr

m, k, d, B = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
nnz = int(round(d * m * k))
pat = smb.sample_pattern(m, k, nnz, smb.Rng(0).stream("pattern"), large=m * k >= 2**31)
rng = np.random.default_rng(1)
vals = torch.from_numpy(rng.standard_normal(nnz).astype(np.float32)).cuda()
vel = torch.zeros_like(vals)
out = torch.empty_like(vals)
X = torch.randn(k, B, device="cuda")
dY = torch.randn(m, B, device="cuda")
for _ in range(reps):
    _lib.call("smb_sddmm_update_into", 0, pat.handle, ptr(dY), B, ptr(X), B, B, ptr(vals),
              ptr(out), ptr(vel), None, None, None, None, 3, 0.9, 1e-4, stream_ptr())
torch.cuda.synchronize()
print("ok", m, k, nnz, B)

#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/ncu_k.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr
n, B, d = 8192, 512, 0.01
pat = smb.sample_pattern(n, n, int(d*n*n), smb.Rng(0).stream("pattern"))
vals = torch.randn(pat.nnz, device="cuda"); vel = torch.zeros_like(vals)
X = torch.randn(n, B, device="cuda"); dY = torch.randn(n, B, device="cuda"); out = torch.empty(n, B, device="cuda")
for _ in range(2):
    _lib.call("smb_spmm", 0, ptr(pat.row_ptr), ptr(pat.col_idx), ptr(vals), n, n, ptr(X), B, B, None, 0, ptr(out), B, stream_ptr())
    _lib.call("smb_sddmm_update", 0, pat.handle, ptr(dY), B, ptr(X), B, B, ptr(vals), ptr(vel), None, None, None, None, 3, 0.9, 1e-6, stream_ptr())
torch.cuda.synchronize()
PY
timeout 300 python /tmp/ncu_k.py > gpurun_out/ncu_k_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sddmm_pipe|row_spmm" -s 2 -c 2 -o gpurun_out/prof_k2 python /tmp/ncu_k.py > gpurun_out/ncu_k.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_k.log
tail -2 gpurun_out/ncu_k.log

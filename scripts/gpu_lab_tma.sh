#!/bin/bash
mkdir -p gpurun_out
for s in 0 42 43 12 13 14 22 23; do SMB_SDDMM_TMA=$s timeout 600 python scripts/lab_sddmm_tma.py; done > gpurun_out/lab_tma.log 2>&1
cat gpurun_out/lab_tma.log | grep -v Warn

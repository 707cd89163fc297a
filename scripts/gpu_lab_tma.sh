#!/bin/bash
mkdir -p gpurun_out
for s in 0 12 14 16 18; do LAB_SMALL=1 SMB_SDDMM_TMA=$s timeout 600 python scripts/lab_sddmm_tma.py; done > gpurun_out/lab_tma.log 2>&1
for s in 0 12; do SMB_SDDMM_TMA=$s timeout 600 python scripts/probe_cfg2_variants.py 2>&1 | grep "b2b"; done >> gpurun_out/lab_tma.log
cat gpurun_out/lab_tma.log | grep -v Warn

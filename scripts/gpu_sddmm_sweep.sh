#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 2 3 4 5; do SMB_SDDMM_VARIANT=$v timeout 120 python scripts/probe_sddmm.py; done > gpurun_out/sddmm_sweep.log 2>&1
cat gpurun_out/sddmm_sweep.log

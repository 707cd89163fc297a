#!/bin/bash
for w in 0 1 4 8; do SMB_SPMM_W=$w timeout 120 python scripts/probe_spmm_small.py; done > gpurun_out/spmm_sweep.log 2>&1
cat gpurun_out/spmm_sweep.log

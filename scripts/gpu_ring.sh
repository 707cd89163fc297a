#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for w in 0 2; do SMB_SPMM_W=$w timeout 120 python scripts/probe_spmm_small.py; done
timeout 300 python scripts/probe_gather_cost.py

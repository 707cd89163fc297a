#!/bin/bash
mkdir -p gpurun_out
export SMB_SDDMM_VARIANT=${1:-2}
timeout 120 python scripts/probe_sddmm.py > gpurun_out/var_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sddmm_pipe -s 115 -c 1 -o gpurun_out/sddmm_var_L4 python scripts/probe_sddmm.py > gpurun_out/var_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sddmm_pipe -s 5 -c 1 -o gpurun_out/sddmm_var_L0 python scripts/probe_sddmm.py >> gpurun_out/var_ncu.log 2>&1
echo "ncu exit $?"

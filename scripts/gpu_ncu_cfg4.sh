#!/bin/bash
mkdir -p gpurun_out
L=3072,8192,8192,8192,10
timeout 300 python scripts/ncu_step.py $L 0.01 1024 3 > gpurun_out/cfg4_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 2 -k regex:sddmm_pipe -s 6 -c 1 -o gpurun_out/cfg4_sddmm python scripts/ncu_step.py $L 0.01 1024 3 > gpurun_out/cfg4_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 2 -k regex:row_spmm -s 9 -c 1 -o gpurun_out/cfg4_spmm python scripts/ncu_step.py $L 0.01 1024 3 >> gpurun_out/cfg4_ncu.log 2>&1
echo "ncu exit $?"

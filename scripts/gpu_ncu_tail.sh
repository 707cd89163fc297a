#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/ncu_step.py 3072,1024,512,10 0.01 1024 4 > gpurun_out/tail_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:tail_step -s 3 -c 1 -o gpurun_out/tail_full python scripts/ncu_step.py 3072,1024,512,10 0.01 1024 4 > gpurun_out/tail_ncu.log 2>&1
echo "ncu exit $?"

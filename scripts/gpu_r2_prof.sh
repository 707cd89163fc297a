#!/bin/bash
# round 2: config-2 launch list + full capture, config-4 full capture (incl. the TMA SDDMM)
bash scripts/gpu_profile_step.sh r02_cfg2 3072,1024,512,10 0.01 1024 14 > gpurun_out/prof2.log 2>&1
bash scripts/gpu_profile_step.sh r02_cfg4 3072,8192,8192,8192,10 0.01 1024 18 > gpurun_out/prof4.log 2>&1
cat gpurun_out/prof2.log gpurun_out/prof4.log
ls -la gpurun_out/*.ncu-rep gpurun_out/*launches.csv

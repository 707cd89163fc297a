#!/bin/bash
# round 2: config-2 and config-4 launch lists + full captures (incl. the TMA SDDMM)
bash scripts/gpu_profile_step.sh r02_cfg2 3072,1024,512,10 0.01 1024 keep > gpurun_out/prof2.log 2>&1
bash scripts/gpu_profile_step.sh r02_cfg4 3072,8192,8192,8192,10 0.01 1024 > gpurun_out/prof4.log 2>&1
cat gpurun_out/prof2.log gpurun_out/prof4.log
du -sh gpurun_out

#!/bin/bash
# round-2 final measurement set (r02f): bench lines, config-3 kernel table,
# config-2 / config-4 launch lists and ncu --set full summaries
bash scripts/gpu_r2_final.sh > gpurun_out/r2f_final.log 2>&1
bash scripts/gpu_profile_step.sh r02f_cfg2 3072,1024,512,10 0.01 1024 > gpurun_out/r2f_prof2.log 2>&1
bash scripts/gpu_profile_step.sh r02f_cfg4 3072,8192,8192,8192,10 0.01 1024 > gpurun_out/r2f_prof4.log 2>&1
tail -12 gpurun_out/r2f_final.log | cut -c1-300; cat gpurun_out/r2f_prof2.log gpurun_out/r2f_prof4.log

#!/bin/bash
bash scripts/gpu_profile_step.sh r02_cfg5_b512 3072,65536,65536,10 0.001 512 > gpurun_out/prof5.log 2>&1
cat gpurun_out/prof5.log; cat gpurun_out/r02_cfg5_b512_full.md | cut -c1-330

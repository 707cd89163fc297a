#!/bin/bash
mkdir -p gpurun_out
python scripts/probe_small.py > gpurun_out/probe2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"softmax|sddmm" -s 6 -c 2 -o gpurun_out/prof_small python scripts/probe_small.py >> gpurun_out/probe2.log 2>&1
head -2 gpurun_out/probe2.log

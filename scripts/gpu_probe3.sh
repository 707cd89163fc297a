#!/bin/bash
mkdir -p gpurun_out
python scripts/probe_small.py > gpurun_out/probe3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"softmax" -s 3 -c 1 -o gpurun_out/prof_softmax python scripts/probe_small.py >> gpurun_out/probe3.log 2>&1
head -2 gpurun_out/probe3.log

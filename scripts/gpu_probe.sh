#!/bin/bash
mkdir -p gpurun_out
python scripts/probe_spmm.py > gpurun_out/probe.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:row_spmm -s 3 -c 1 -o gpurun_out/prof_probe python scripts/probe_spmm.py >> gpurun_out/probe.log 2>&1
tail -3 gpurun_out/probe.log

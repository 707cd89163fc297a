#!/bin/bash
# one compute-sanitizer tool per call: bash scripts/gpu_sanitize.sh <memcheck|racecheck|synccheck>
tool=$1
mkdir -p gpurun_out
timeout 600 python scripts/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
echo "exit $?" >> gpurun_out/sanitize_$tool.log
tail -15 gpurun_out/sanitize_$tool.log

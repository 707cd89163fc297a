#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --layers 3072,65536,65536,10 --density 0.001 --batch 512 --steps 100 --cpu-seconds 20 > gpurun_out/bench_cfg5.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg5.log
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench_cfg5.log | cut -c1-3500

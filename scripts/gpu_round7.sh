#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 50 --no-cpu-baseline --sweep > gpurun_out/bench_sweep.log 2>&1; echo "sweep exit $?" >> gpurun_out/bench_sweep.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench_sweep.log; tail -2 gpurun_out/bench.log | cut -c1-300

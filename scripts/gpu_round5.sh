#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 900 python bench.py --backend masked --steps 300 --no-cpu-baseline > gpurun_out/bench_masked.log 2>&1; echo "bench masked exit $?" >> gpurun_out/bench_masked.log
timeout 1200 python bench.py --steps 50 --no-cpu-baseline --sweep > gpurun_out/bench_sweep.log 2>&1; echo "sweep exit $?" >> gpurun_out/bench_sweep.log
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log | cut -c1-2500; tail -2 gpurun_out/bench_masked.log | cut -c1-600; tail -1 gpurun_out/bench_sweep.log

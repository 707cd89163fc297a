#!/bin/bash
# round 2: new parity tests at the bench configs, two-rank engine test, full gpu suite, bench
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -x -k "bench_configs or two_process or identity or external or kernel_durations or layer_api_bitwise" > gpurun_out/pytest_new.log 2>&1; echo "pytest-new exit $?" >> gpurun_out/pytest_new.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --force-dp --steps 20 --warmup 5 --no-extras > gpurun_out/bench_dp.log 2> gpurun_out/bench_dp.err; echo "bench-dp exit $?" >> gpurun_out/bench_dp.log
tail -3 gpurun_out/pytest_new.log; tail -3 gpurun_out/pytest_gpu.log; tail -c 600 gpurun_out/bench.log; tail -c 300 gpurun_out/bench_dp.log

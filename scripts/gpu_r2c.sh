#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/pytest_a.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_a.log
tail -3 gpurun_out/pytest_a.log
timeout 900 python bench.py --layers 3072,65536,65536,10 --density 0.001 --batch 4096 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.log 2> gpurun_out/bench5.err; echo "bench exit $?" >> gpurun_out/bench5.log
timeout 900 python bench.py --layers 3072,65536,65536,10 --density 0.001 --batch 512 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench5b.log 2> gpurun_out/bench5b.err; echo "bench exit $?" >> gpurun_out/bench5b.log
for f in bench5 bench5b; do grep "^{" gpurun_out/$f.log | python -c "
import sys,json
j=json.loads(sys.stdin.read())
print(j['value'], j['ms_per_step'], j['kernel_us'])
"; done

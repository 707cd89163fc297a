#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 1000 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
bash scripts/gpu_ncu_tail.sh > /dev/null 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); print(j['value'], j['ms_per_step'], j['back_to_back']['value'], j['kernel_us'])
    else: print(l.strip())"

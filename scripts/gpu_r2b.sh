#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.log
tail -3 gpurun_out/pytest_gpu.log; grep "^{" gpurun_out/bench.log | python -c "
import sys,json
j=json.loads(sys.stdin.read())
print(j['value'], j['ms_per_step'], j['e2e']['value'], j['roofline']['kernel'], j['roofline']['frac'])
for n,e in j['extra_configs'].items(): print(n, e['value'], e['ms_per_step'], e['kernel_us'])
"
timeout 600 python scripts/kernel_bench.py > gpurun_out/kernel_bench.log 2>&1; echo "kb exit $?" >> gpurun_out/kernel_bench.log
tail -10 gpurun_out/kernel_bench.log

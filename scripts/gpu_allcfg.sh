#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "exit $?" >> gpurun_out/bench.log
timeout 1200 python bench.py --layers 3072,8192,8192,8192,10 --density 0.01 --batch 1024 --steps 200 --cpu-seconds 20 > gpurun_out/bench_cfg4.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg4.log
timeout 1500 python bench.py --layers 3072,65536,65536,10 --density 0.001 --batch 512 --steps 100 --cpu-seconds 20 > gpurun_out/bench_cfg5.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg5.log
timeout 900 python scripts/kernel_bench.py > gpurun_out/kernel_bench.log 2>&1; echo "exit $?" >> gpurun_out/kernel_bench.log
for f in bench bench_cfg4 bench_cfg5; do grep "^{" gpurun_out/$f.log | python -c "
import sys, json
j = json.loads(sys.stdin.read())
print('$f', j['value'], j['ms_per_step'], j['e2e']['value'], j.get('cpu_baseline', {}).get('value'), j['roofline']['kernel'], j['roofline']['frac'], j['roofline']['roof_frac'])"; done
tail -3 gpurun_out/kernel_bench.log | cut -c1-300

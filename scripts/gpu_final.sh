#!/bin/bash
# full refresh: tests, smoke, config 2 (+ sweep), config 4, config 5, config-3 kernel bench,
# reference arm, config-2 ncu launch list + full capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --sweep > gpurun_out/bench.log 2>&1; echo "exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "exit $?" >> gpurun_out/bench_ref.log
timeout 1200 python bench.py --layers 3072,8192,8192,8192,10 --density 0.01 --batch 1024 --steps 200 --cpu-seconds 20 > gpurun_out/bench_cfg4.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg4.log
timeout 1500 python bench.py --layers 3072,65536,65536,10 --density 0.001 --batch 512 --steps 100 --cpu-seconds 20 > gpurun_out/bench_cfg5.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg5.log
timeout 900 python scripts/kernel_bench.py > gpurun_out/kernel_bench.log 2>&1; echo "exit $?" >> gpurun_out/kernel_bench.log
bash scripts/gpu_profile_step.sh r02d_cfg2 3072,1024,512,10 0.01 1024 > gpurun_out/prof.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for f in bench bench_cfg4 bench_cfg5; do grep "^{" gpurun_out/$f.log | python -c "
import sys, json
j = json.loads(sys.stdin.read())
print('$f', j['value'], j['ms_per_step'], j['e2e']['value'], j.get('cpu_baseline', {}).get('value'), j['roofline']['kernel'], j['roofline']['frac'])"; done
tail -1 gpurun_out/bench_ref.log | cut -c1-300

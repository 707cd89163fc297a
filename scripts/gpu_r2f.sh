#!/bin/bash
mkdir -p gpurun_out
python scripts/probe_h2d.py > gpurun_out/h2d.log 2>&1; cat gpurun_out/h2d.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.log
grep "^{" gpurun_out/bench.log | python -c "
import sys,json
j=json.loads(sys.stdin.read())
print(j['value'], j['ms_per_step'], j['back_to_back'], j['e2e']['value'], j['e2e']['h2d_gbs'], j['roofline']['kernel'], j['roofline']['frac'])
for n,e in j['extra_configs'].items(): print(n, e['value'], e['ms_per_step'], e['back_to_back']['value'], e['roofline']['kernel'], e['roofline']['frac'], e.get('build_s'), e.get('build_s_device_sampler'))
"
bash scripts/gpu_profile_step.sh r02_cfg4 3072,8192,8192,8192,10 0.01 1024 keep > gpurun_out/prof4.log 2>&1
cat gpurun_out/prof4.log

#!/bin/bash
# what the driver runs at round end (plus timing of each part)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dl_build.log 2>&1; echo "build $?"
t0=$(date +%s); timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/dl_pytest.log 2>&1; echo "pytest $? ($(( $(date +%s) - t0 )) s)"; tail -2 gpurun_out/dl_pytest.log
t0=$(date +%s); timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dl_smoke.log 2>&1; echo "smoke $? ($(( $(date +%s) - t0 )) s)"; tail -1 gpurun_out/dl_smoke.log
t0=$(date +%s); timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/dl_ref.log 2>&1; echo "ref $? ($(( $(date +%s) - t0 )) s)"
t0=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/dl_bench.log 2> gpurun_out/dl_bench.err; echo "bench $? ($(( $(date +%s) - t0 )) s)"
grep "^{" gpurun_out/dl_bench.log | python -c "
import sys,json
j=json.loads(sys.stdin.read())
print(j['value'], j['ms_per_step'], j['e2e']['value'], j['e2e']['h2d_gbs'], j['roofline']['kernel'], j['roofline']['frac'], j['clocks'])
for n,e in j['extra_configs'].items(): print(n, e['value'], e['ms_per_step'], e['e2e']['value'], e['roofline']['kernel'], e['roofline']['frac'], e.get('cpu_baseline',{}).get('value'))
"

#!/bin/bash
# quick iteration on the column-chain step: its parity tests, the config-2
# bench (no extras), the kernel's phase stamps and a timeline of the step
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ci_build.log 2>&1; echo "build $?"
timeout 300 python -m pytest tests/test_gpu_chain.py ${CI_TESTS} -x -q -m gpu > gpurun_out/ci_pytest.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/ci_pytest.log
timeout 120 python scripts/probe_chain_phases.py > gpurun_out/ci_phases.log 2>&1; echo "phases $?"; cat gpurun_out/ci_phases.log
timeout 240 python bench.py --steps 50 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/ci_bench.log 2> gpurun_out/ci_bench.err; echo "bench $?"
grep "^{" gpurun_out/ci_bench.log | python -c "
import sys,json
j=json.loads(sys.stdin.read())
print(j['value'], j['ms_per_step'], j['back_to_back'], j['e2e']['value'], j['roofline']['kernel'], j['roofline']['frac'])
print(j['kernel_us'])"
timeout 120 python scripts/probe_timeline.py > gpurun_out/ci_timeline.log 2>&1; echo "timeline $?"; sed -n 3,20p gpurun_out/ci_timeline.log

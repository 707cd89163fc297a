#!/bin/bash
# quick iteration on the dense output-layer kernels: their parity tests and
# the config-5 (B=512) bench's per-kernel times
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/di_build.log 2>&1; echo "build $?"
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_guard.py -k "dense" -x -q -m gpu > gpurun_out/di_pytest.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/di_pytest.log
timeout 900 python bench.py --layers 3072,65536,65536,10 --density 0.001 --batch ${DI_B:-512} --steps 30 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/di_bench.log 2> gpurun_out/di_bench.err; echo "bench $?"
grep "^{" gpurun_out/di_bench.log | python -c "
import sys,json
j=json.loads(sys.stdin.read())
print(j['value'], j['ms_per_step'])
print({k: v for k, v in j['kernel_us'].items() if 'dense' in k or 'bias' in k})"

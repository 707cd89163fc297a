#!/bin/bash
# bench one configuration with the tree's library and every _variants/*.so:
# bash scripts/gpu_ab_bench.sh "<bench.py arguments>"
mkdir -p gpurun_out
for lib in _variants/*.so paper_2407_17437_b200/libsparsemlp_b200.so; do
  echo "== $lib"
  SMB_LIB=$lib timeout 900 python bench.py $1 --no-extras --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(l['value'], l['ms_per_step']); print(json.dumps(l['kernel_us']))"
done 2>&1 | tee gpurun_out/ab_bench.log

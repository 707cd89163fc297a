#!/bin/bash
# config-2 bench line (value, back to back, kernel_us) with the tree's library and every _variants/*.so
mkdir -p gpurun_out
for lib in _variants/*.so paper_2407_17437_b200/libsparsemlp_b200.so; do
  echo "== $lib"
  SMB_LIB=$lib timeout 900 python bench.py --no-extras --no-cpu-baseline $1 2>/dev/null | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(l['value']), round(l['ms_per_step']*1e3,2), 'b2b', round(l['back_to_back']['value'])); print(json.dumps(l['kernel_us']))"
done 2>&1 | tee gpurun_out/ab_bench2.log

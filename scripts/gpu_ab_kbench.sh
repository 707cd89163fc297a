#!/bin/bash
# config-3 kernel table (densities $1) with the tree's library and every _variants/*.so
mkdir -p gpurun_out
for lib in _variants/*.so paper_2407_17437_b200/libsparsemlp_b200.so; do
  echo "== $lib"; SMB_LIB=$lib timeout 600 python scripts/kernel_bench.py $1 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['density'], r['B'], {k:(r[k]['us'], r[k]['frac_hbm']) for k in ('spmm','spmm_t','sddmm_update')})"
done 2>&1 | tee gpurun_out/ab_kbench.log

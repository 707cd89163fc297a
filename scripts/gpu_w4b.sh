#!/bin/bash

for w in 9; do
  echo "W=$w"
  SMB_SPMM_W=$w timeout 120 python scripts/probe_spmm_small.py
  SMB_SPMM_W=$w timeout 300 python -c "
import sys; sys.path.insert(0,'scripts'); import kernel_bench as kb
kb.main(densities=(0.001, 0.01, 0.1), batches=(128, 512, 2048))" 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        j = json.loads(l); print(j['density'], j['B'], 'spmm', j['spmm']['us'], 'spmm_t', j['spmm_t']['us'], 'sddmm', j['sddmm_update']['us'])"
done


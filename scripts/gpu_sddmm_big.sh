#!/bin/bash
mkdir -p gpurun_out
for v in 0 6 7; do
  echo "variant $v"
  SMB_SDDMM_VARIANT=$v timeout 300 python -c "
import sys; sys.path.insert(0,'scripts'); import kernel_bench as kb
kb.main(densities=(0.01, 0.1), batches=(128, 512))" 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        j = json.loads(l); print(j['density'], j['B'], 'sddmm', j['sddmm_update']['us'], j['sddmm_update']['Gpairs/s'])
    else: print(l.rstrip())"
done > gpurun_out/sddmm_big.log 2>&1
SMB_SDDMM_VARIANT=0 timeout 120 python scripts/probe_sddmm.py >> gpurun_out/sddmm_big.log 2>&1
cat gpurun_out/sddmm_big.log

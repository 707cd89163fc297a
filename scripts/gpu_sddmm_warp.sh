#!/bin/bash
for v in 3 4 5; do
  echo "variant $v"
  SMB_SDDMM_VARIANT=$v timeout 120 python scripts/probe_sddmm.py
  SMB_SDDMM_VARIANT=$v timeout 300 python -c "
import sys; sys.path.insert(0,'scripts'); import kernel_bench as kb
kb.main(densities=(0.001, 0.01, 0.1), batches=(128, 512, 2048))" 2>&1 | python -c "
import sys, json
print(' '.join('%s/%s:%s' % (j['density'], j['B'], j['sddmm_update']['us']) for j in (json.loads(l) for l in sys.stdin if l.startswith('{'))))"
done

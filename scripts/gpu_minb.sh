#!/bin/bash
for L in "" build/lib_minb6.so; do
  echo "lib=$L"
  SMB_NO_BUILD=1 SMB_LIB=$L timeout 120 python scripts/probe_spmm_small.py
  SMB_NO_BUILD=1 SMB_LIB=$L timeout 300 python -c "
import sys; sys.path.insert(0,'scripts'); import kernel_bench as kb
kb.main(densities=(0.001, 0.01, 0.1), batches=(512, 2048))" 2>&1 | python -c "
import sys, json
print(' '.join('%s/%s:%s,%s' % (j['density'], j['B'], j['spmm']['us'], j['spmm_t']['us']) for j in (json.loads(l) for l in sys.stdin if l.startswith('{'))))"
done

#!/bin/bash
# back-to-back config-2 step time under env-selected engine variants
for v in "" "SMB_L0_MAIN=1" "SMB_PREFETCH_AT=start" "SMB_L0_MAIN=1 SMB_PREFETCH_AT=start"; do
  for rep in 1 2; do
    echo "[$v] $(env $v ABL_ONLY_BASE=1 python scripts/probe_ablation.py 2>&1 | head -1)"
  done
done

#!/bin/bash
# back-to-back config-2 step time under env-selected engine variants
# (usage: scripts/probe_variants.sh "ENV=.. ENV2=.." "..." ...)
for v in "$@"; do
  for rep in 1 2; do
    echo "[$v] $(env $v ABL_ONLY_BASE=1 python scripts/probe_ablation.py 2>&1 | tail -1)"
  done
done

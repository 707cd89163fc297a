#!/bin/bash
# step time of each _variants/*.so against the current build (config 2 unless args)
for rep in 1 2; do
  python scripts/probe_kernel_us.py "$@" 2>&1 | grep -v Warn | cut -c1-30
  for f in _variants/*.so; do
    SMB_LIB=$f python scripts/probe_kernel_us.py "$@" 2>&1 | grep -v Warn | cut -c1-30
  done
done

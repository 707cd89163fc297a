#!/bin/bash
# A/B of per-kernel durations: _old_tree vs current (args: LAYERS D B)
for i in 1 2; do (cd _old_tree && python probe_kernel_us.py "$@" | sed 's/^/OLD /'); python scripts/probe_kernel_us.py "$@"; done 2>&1 | grep -v Warn

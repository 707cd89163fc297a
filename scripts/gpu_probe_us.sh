#!/bin/bash
for i in 1 2; do (cd _old_tree && python probe_kernel_us.py | sed 's/^/OLD /'); python scripts/probe_kernel_us.py; done 2>&1 | grep -v Warn

#!/bin/bash
for i in 1 2; do for lib in paper_2407_17437_b200/lib_base_r2a.so paper_2407_17437_b200/libsparsemlp_b200.so; do SMB_LIB=$lib python scripts/probe_kernel_us.py; done; done 2>&1 | grep -v Warn

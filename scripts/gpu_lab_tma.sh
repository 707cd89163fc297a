#!/bin/bash
# A/B of builds of the library on the SDDMM lab shapes: the tree's library and
# every _variants/*.so (scripts/build_variant.sh)
mkdir -p gpurun_out
for lib in _variants/*.so paper_2407_17437_b200/libsparsemlp_b200.so; do SMB_LIB=$lib timeout 600 python scripts/lab_sddmm_tma.py; done > gpurun_out/lab_tma.log 2>&1
cat gpurun_out/lab_tma.log | grep -v Warn

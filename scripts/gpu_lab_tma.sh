#!/bin/bash
# A/B of two builds of the library on the SDDMM lab shapes (lib_base.so = the previous tree)
mkdir -p gpurun_out
for lib in paper_2407_17437_b200/lib_base.so paper_2407_17437_b200/libsparsemlp_b200.so; do SMB_LIB=$lib timeout 600 python scripts/lab_sddmm_tma.py; done > gpurun_out/lab_tma.log 2>&1
cat gpurun_out/lab_tma.log | grep -v Warn

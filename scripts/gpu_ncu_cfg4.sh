#!/bin/bash
# config 4 (3072-8192-8192-8192-10, d=0.01, B=1024): ncu launch list of the
# step's kernels, then one --set full capture of every sparse kernel of one
# eager step (3 SpMM, 2 SpMM-T, 3 SDDMM = 8 launches per step)
mkdir -p gpurun_out
L=3072,8192,8192,8192,10
timeout 300 python scripts/ncu_step.py $L 0.01 1024 3 > gpurun_out/cfg4_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k 'regex:row_spmm|sddmm|softmax_step|gather_columns|bias_rows|relu|optimizer' \
  --log-file gpurun_out/cfg4_launches.csv python scripts/ncu_step.py $L 0.01 1024 3 > gpurun_out/cfg4_ncu1.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:row_spmm|sddmm' -s 16 -c 8 \
  -o gpurun_out/cfg4_full python scripts/ncu_step.py $L 0.01 1024 3 > gpurun_out/cfg4_ncu2.log 2>&1
echo "ncu exit $?"

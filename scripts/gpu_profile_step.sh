#!/bin/bash
# ncu launch list + one --set full capture of every kernel of one steady-state step.
# usage: bash scripts/gpu_profile_step.sh NAME LAYERS DENSITY BATCH PER_STEP
NAME=$1; L=$2; D=$3; B=$4; K=$5
mkdir -p gpurun_out
RX='regex:row_spmm|sddmm_pipe|sddmm_warp|sddmm_tma|softmax_step|gather_columns|bias_rows|deep_kernel|spmv|values_to_csc|dense_'
timeout 300 python scripts/ncu_step.py $L $D $B 4 > gpurun_out/${NAME}_plain.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$RX" \
  --log-file gpurun_out/${NAME}_launches.csv python scripts/ncu_step.py $L $D $B 4 > gpurun_out/${NAME}_ncu1.log 2>&1
echo "launch list exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "$RX" -s $((3*K)) -c $K \
  -o gpurun_out/${NAME}_full python scripts/ncu_step.py $L $D $B 4 > gpurun_out/${NAME}_ncu2.log 2>&1
echo "full exit $?"

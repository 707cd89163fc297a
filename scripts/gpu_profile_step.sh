#!/bin/bash
# ncu launch list + one --set full capture of every kernel of one steady-state
# step (NVTX range "prof"), summarised on the box (profiles-ready markdown).
# usage: bash scripts/gpu_profile_step.sh NAME LAYERS DENSITY BATCH [keep_rep]
NAME=$1; L=$2; D=$3; B=$4; KEEP=$5
mkdir -p gpurun_out
RX='regex:row_spmm|sddmm_pipe|sddmm_warp|sddmm_tma|sddmm_lean|softmax_step|gather_columns|bias_rows|deep_kernel|spmv|values_to_csc|dense_|chain_kernel|padded_refresh'
CMD="python scripts/ncu_step.py $L $D $B 3 gpurun_out/${NAME}_tags.txt"
timeout 300 $CMD > gpurun_out/${NAME}_plain.log 2>&1 || { echo "plain failed"; cat gpurun_out/${NAME}_plain.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$RX" \
  --nvtx --nvtx-include "prof/" --log-file gpurun_out/${NAME}_launches.csv $CMD > gpurun_out/${NAME}_ncu1.log 2>&1
echo "launch list exit $?"
timeout 1500 ncu -f --set full --clock-control none --import-source on -k "$RX" \
  --nvtx --nvtx-include "prof/" -o /tmp/${NAME}_full $CMD > gpurun_out/${NAME}_ncu2.log 2>&1
echo "full exit $?"
TAGS=$(cat gpurun_out/${NAME}_tags.txt)
python scripts/summarize_ncu.py launches gpurun_out/${NAME}_launches.csv gpurun_out/${NAME}_launches.md \
  --header "# ${NAME}: ncu launch list of one eager step ($L, d=$D, B=$B; cold caches, serialised)" > /dev/null
python scripts/summarize_ncu.py full /tmp/${NAME}_full.ncu-rep gpurun_out/${NAME}_full.md --tags "$TAGS" \
  --header "# ${NAME}: ncu --set full of one eager step ($L, d=$D, B=$B; serialised, cold caches)" \
  --traffic-key "$L|$D|$B" --traffic-json gpurun_out/ncu_traffic_${NAME}.json > /dev/null
echo "summaries exit $?"
if [ -n "$KEEP" ]; then cp /tmp/${NAME}_full.ncu-rep gpurun_out/; fi

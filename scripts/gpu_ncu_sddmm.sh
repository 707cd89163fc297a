#!/bin/bash
# ncu --set full of the TMA SDDMM at the config-4 hidden layer and the config-5 hidden layer (B=4096, blocked order)
mkdir -p gpurun_out
for shape in "8192 8192 0.0084 1024 c4" "65536 65536 0.000587 4096 c5"; do
  set -- $shape
  timeout 300 python scripts/probe_sddmm_shape.py $1 $2 $3 $4 > gpurun_out/ns_plain_$5.log 2>&1 || { echo "plain run failed $5"; continue; }
  timeout 1200 ncu -f --set full --clock-control none --import-source on -k "regex:sddmm_tmak" -s 2 -c 1 \
    -o gpurun_out/r02f_sddmm_$5 python scripts/probe_sddmm_shape.py $1 $2 $3 $4 > gpurun_out/ns_ncu_$5.log 2>&1
  echo "ncu $5 $?"
  ncu -i gpurun_out/r02f_sddmm_$5.ncu-rep --page raw --csv > gpurun_out/r02f_sddmm_$5_raw.csv 2>&1
  python scripts/ncu_hot.py gpurun_out/r02f_sddmm_$5.ncu-rep 0 30 > gpurun_out/r02f_sddmm_$5_hot.txt 2>&1
done

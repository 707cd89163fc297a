#!/bin/bash
# ncu --set full of one 256-column phase of the blocked-order TMA SDDMM (config-5 hidden layer, B=4096)
mkdir -p gpurun_out
timeout 300 python scripts/probe_sddmm_shape.py 65536 65536 0.000587 4096 2 > gpurun_out/ns_plain_c5p.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 ncu -f --set full --clock-control none --import-source on -k "regex:sddmm_tmak" -s 20 -c 1 \
  -o gpurun_out/r02f_sddmm_c5_phase python scripts/probe_sddmm_shape.py 65536 65536 0.000587 4096 2 > gpurun_out/ns_ncu_c5p.log 2>&1
echo "ncu $?"
ncu -i gpurun_out/r02f_sddmm_c5_phase.ncu-rep --page raw --csv > gpurun_out/r02f_sddmm_c5_phase_raw.csv 2>&1
python scripts/ncu_hot.py gpurun_out/r02f_sddmm_c5_phase.ncu-rep 0 30 > gpurun_out/r02f_sddmm_c5_phase_hot.txt 2>&1

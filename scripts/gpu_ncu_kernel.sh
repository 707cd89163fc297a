#!/bin/bash
# one ncu --set full capture of one kernel of the config-2 step (regex $1) + hot SASS lines
# usage: bash scripts/gpu_ncu_kernel.sh REGEX NAME
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/nk_build.log 2>&1
timeout 300 python scripts/probe_chain_phases.py > gpurun_out/nk_plain.log 2>&1 && \
timeout 900 ncu -f --set full --clock-control none --import-source on -k "regex:$1" -s 3 -c 1 \
  -o gpurun_out/$2 python scripts/probe_chain_phases.py > gpurun_out/nk_ncu.log 2>&1
echo "ncu $?"
python scripts/ncu_hot.py gpurun_out/$2.ncu-rep 0 40 > gpurun_out/$2_hot.txt 2>&1
ncu -i gpurun_out/$2.ncu-rep --page details --csv > gpurun_out/$2_details.csv 2>&1
head -45 gpurun_out/$2_hot.txt

#!/bin/bash
# one ncu --set full capture of the column-chain kernel (config 2) + hot SASS lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cn_build.log 2>&1
timeout 300 python scripts/probe_chain_phases.py > gpurun_out/cn_plain.log 2>&1 && \
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:chain_kernel -s 2 -c 1 \
  -o gpurun_out/chain_full python scripts/probe_chain_phases.py > gpurun_out/cn_ncu.log 2>&1
echo "ncu $?"
python scripts/ncu_hot.py gpurun_out/chain_full.ncu-rep 0 60 > gpurun_out/cn_hot.txt 2>&1
ncu -i gpurun_out/chain_full.ncu-rep --page details --csv > gpurun_out/cn_details.csv 2>&1
head -70 gpurun_out/cn_hot.txt

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --backend masked --steps 300 --no-cpu-baseline > gpurun_out/bench_masked.log 2>&1; echo "bench masked exit $?" >> gpurun_out/bench_masked.log
for d in 0.001 0.005; do
  timeout 300 python scripts/ncu_step.py 3072,1024,512,10 $d 1024 4 > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k 'regex:row_spmm|sddmm_pipe|softmax_step|gather_columns|bias_rows' \
    --log-file gpurun_out/launches_d$d.csv python scripts/ncu_step.py 3072,1024,512,10 $d 1024 4 > /dev/null 2>&1
done
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench_masked.log | cut -c1-400

#!/bin/bash
# round 2 measurement set: default bench (+ sweep), reference arm, config 5 at B=512,
# config-3 kernel bench; JSON lines saved for profiles/
mkdir -p gpurun_out
timeout 1500 python bench.py --sweep --steps 50 --warmup 5 > gpurun_out/b_default.log 2> gpurun_out/b_default.err; echo "exit $?" >> gpurun_out/b_default.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/b_ref.log 2>&1; echo "exit $?" >> gpurun_out/b_ref.log
timeout 900 python bench.py --layers 3072,65536,65536,10 --density 0.001 --batch 512 --steps 50 --warmup 5 --cpu-seconds 15 > gpurun_out/b_cfg5_512.log 2> gpurun_out/b_cfg5_512.err; echo "exit $?" >> gpurun_out/b_cfg5_512.log
timeout 600 python bench.py --force-dp --steps 50 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/b_dp.log 2> gpurun_out/b_dp.err; echo "exit $?" >> gpurun_out/b_dp.log
timeout 900 python scripts/kernel_bench.py > gpurun_out/kb.jsonl 2> gpurun_out/kb.err; echo "exit $?" >> gpurun_out/kb.err
for f in b_default b_ref b_cfg5_512 b_dp; do tail -1 gpurun_out/$f.log; grep "^{" gpurun_out/$f.log | head -c 400; echo; done

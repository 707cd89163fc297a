#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python scripts/probe_b100.py
python scripts/probe_ablation.py 2>&1 | grep baseline
timeout 900 python bench.py --steps 50 --no-cpu-baseline --sweep 2>&1 | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read())
print('value', j['value'], j['ms_per_step'])
for r in j['sweep']: print(r)"

#!/bin/bash
# sweep the persistent-loop thresholds (bench value per setting)
mkdir -p gpurun_out
for cfg in "8 16" "4 16" "16 16" "8 8" "8 24" "8 32" "1 32"; do
  set -- $cfg
  SBR_REFILL_MIN=$1 SBR_LEAF_MIN=$2 timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/tune.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/tune.json')); print('refill', $1, 'leaf', $2, round(d['value']/1e9,3), round(d['kernel_ms']['trace'],1))"
done

#!/bin/bash
mkdir -p gpurun_out
for occ in 0 6 7 8; do
  SBR_TRACE_OCC=$occ timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/occ_$occ.json 2>gpurun_out/occ_$occ.err
  python -c "import json; d=json.load(open('gpurun_out/occ_$occ.json')); print($occ, d['value']/1e9, d['kernel_ms'])"
done

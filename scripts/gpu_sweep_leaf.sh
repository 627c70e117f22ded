#!/bin/bash
mkdir -p gpurun_out
for nl in 1 2 4 8; do
  timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --n-leaf $nl > gpurun_out/leaf_$nl.json 2>gpurun_out/leaf_$nl.err
  python -c "import json; d=json.load(open('gpurun_out/leaf_$nl.json')); print('n_leaf', $nl, d['value']/1e9, d['kernel_ms'])"
done
for occ in 0 6 7; do
  SBR_TRACE_OCC=$occ timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/occ_$occ.json 2>gpurun_out/occ_$occ.err
  python -c "import json; d=json.load(open('gpurun_out/occ_$occ.json')); print('occ', $occ, d['value']/1e9, d['kernel_ms'])"
done

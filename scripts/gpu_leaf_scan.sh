#!/bin/bash
# BVH leaf size (reference SAH builder) vs bench value
for nl in 1 2 4 8; do
  timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --n-leaf $nl > gpurun_out/leaf.json 2>gpurun_out/leaf.err
  python -c "import json; d=json.load(open('gpurun_out/leaf.json')); print('n_leaf', $nl, round(d['value']/1e9,3), {k: round(v,1) for k,v in d['kernel_ms'].items()})" || tail -3 gpurun_out/leaf.err
done

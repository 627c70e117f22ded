#!/bin/bash
# A/B: query 0 by raster pass vs by BVH traversal (C4 bench, 3 steps)
mkdir -p gpurun_out
for m in raster bvh; do
  SBR_PRIMARY=$m timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_$m.json 2>gpurun_out/ab_$m.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$m.json')); print('$m', round(d['value']/1e9,3), d['ms_per_step'], d['kernel_ms'])" || tail -5 gpurun_out/ab_$m.err
done

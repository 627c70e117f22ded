#!/bin/bash
# primary vs secondary query cost split (bounce budget sweep) + LBVH vs SAH tree quality
mkdir -p gpurun_out
for b in 1 2 5; do
  timeout 600 python bench.py --steps 2 --warmup 2 --angles 72 --no-e2e --no-cpu --bounces $b > gpurun_out/split_$b.json 2>gpurun_out/split_$b.err
  python -c "import json; d=json.load(open('gpurun_out/split_$b.json')); print('B', $b, d['queries_per_step'], d['kernel_ms'])"
done
timeout 900 python scripts/tree_quality.py > gpurun_out/tree_quality.json 2> gpurun_out/tree_quality.err
cat gpurun_out/tree_quality.json

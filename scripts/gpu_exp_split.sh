#!/bin/bash
# per-bounce-budget trace cost (C4, 72 angles) -- where the trace kernel's time goes
mkdir -p gpurun_out
for b in 1 2 3 5; do
  timeout 600 python bench.py --steps 2 --warmup 2 --angles 72 --no-e2e --no-cpu --bounces $b > gpurun_out/split_$b.json 2>gpurun_out/split_$b.err
  python -c "import json; d=json.load(open('gpurun_out/split_$b.json')); print('B', $b, d['queries_per_step'], d['kernel_ms'])"
done

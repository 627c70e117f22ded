#!/bin/bash
# A/B: 4-wide vs 8-wide traversal tree (bench C4 + C5 config), parity with width 8
timeout 900 env SBR_WIDTH=8 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for w in 4 8; do
  SBR_WIDTH=$w timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/w.json 2>gpurun_out/w.err
  python -c "import json; d=json.load(open('gpurun_out/w.json')); print('width', $w, round(d['value']/1e9,3), {k: round(v,1) for k,v in d['kernel_ms'].items()})" || tail -3 gpurun_out/w.err
  SBR_WIDTH=$w python scripts/bench_configs.py --configs c5 --reps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  C5', round(d['trace_ms'],1), round(d['intersections_per_s']/1e9,3))"
done

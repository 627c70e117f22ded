#!/bin/bash
# full GPU suite + smoke + C4 bench line (A/B env) + C5 config line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for envs in "X=1" ${AB_ENVS}; do
  env $envs timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err
  python -c "import json; d=json.load(open('gpurun_out/bench_quick.json')); print('$envs', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms'].items()})" || tail -5 gpurun_out/bench_quick.err
done
if [ -n "$C5" ]; then
  for envs in "X=1" ${AB_ENVS}; do
    env $envs timeout 600 python scripts/bench_configs.py --configs c5 --reps 2 2>/dev/null | cut -c1-700
  done
fi

#!/bin/bash
# bench default vs build_variants/*.so (C4 360 angles, 3 steps), then optional tests
mkdir -p gpurun_out
for lib in default build_variants/*.so; do
  if [ "$lib" = default ]; then unset SBR_LIB; else export SBR_LIB=$PWD/$lib; fi
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "import json; d=json.load(open('gpurun_out/var.json')); print('$lib', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms'].items()})" || tail -3 gpurun_out/var.err
done
unset SBR_LIB
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -x -q > gpurun_out/pytest_new.log 2>&1
  tail -5 gpurun_out/pytest_new.log
fi

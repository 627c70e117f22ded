#!/bin/bash
# bench each build_variants/*.so against the default library (C4, 2 steps)
mkdir -p gpurun_out
for lib in default build_variants/*.so; do
  if [ "$lib" = default ]; then unset SBR_LIB; else export SBR_LIB=$PWD/$lib; fi
  timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "import json; d=json.load(open('gpurun_out/var.json')); print('$lib', round(d['value']/1e9,3), {k: round(v,1) for k,v in d['kernel_ms'].items()})" || tail -3 gpurun_out/var.err
done

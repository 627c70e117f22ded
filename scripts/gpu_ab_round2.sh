#!/bin/bash
# A/B of build_variants/*.so and SBR_L2_PERSIST values vs the default library
# (C4, 360 angles), then the new full-size and acceptance tests.
mkdir -p gpurun_out
run() {  # label
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "import json; d=json.load(open('gpurun_out/var.json')); print('$1', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms'].items()})" || tail -3 gpurun_out/var.err
}
for lib in default build_variants/*.so; do
  if [ "$lib" = default ]; then unset SBR_LIB; else export SBR_LIB=$PWD/$lib; fi
  run $lib
done
unset SBR_LIB
for mb in 24 48 80; do SBR_L2_PERSIST=$mb run "l2persist=$mb"; done
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -x -q --durations=15 > gpurun_out/pytest_new.log 2>&1
  tail -25 gpurun_out/pytest_new.log
fi

#!/bin/bash
# quick A/B of build_variants/*.so vs the default library on 72 C4 angles
for lib in default build_variants/*.so; do
  if [ "$lib" = default ]; then unset SBR_LIB; else export SBR_LIB=$PWD/$lib; fi
  case "$lib" in *noreset*) export SBR_FORCE_MEMSET=1;; *) unset SBR_FORCE_MEMSET;; esac
  timeout 300 python bench.py --angles ${ANGLES:-72} --steps 3 --warmup 2 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms'].items()})"
done

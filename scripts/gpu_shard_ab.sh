#!/bin/bash
# A/B of build_variants/*.so on C4 (bench) and the C5 shard timings at N = 1, 8
for lib in default build_variants/*.so; do
  if [ "$lib" = default ]; then unset SBR_LIB; else export SBR_LIB=$PWD/$lib; fi
  echo "== $lib"
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms'].items()})"
  (cd scripts && timeout 600 python shard_one.py 0 8 | tail -1; timeout 600 python shard_one.py 0 1 | tail -1)
done

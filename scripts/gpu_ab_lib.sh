#!/bin/bash
# A/B of build_variants/$VAR.so against the default library: parity suite on
# the variant, then C4 bench trace time and C5 trace time for both
VAR=${VAR:-flat}
SBR_LIB=$PWD/build_variants/$VAR.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for lib in default build_variants/$VAR.so; do if [ $lib = default ]; then unset SBR_LIB; else export SBR_LIB=$PWD/$lib; fi
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib C4', round(d['value']/1e9,3), d['kernel_ms']['trace'])"
python scripts/bench_configs.py --configs c5 --reps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  C5', round(d['trace_ms'],1))"
done

#!/bin/bash
# Everything profiles/ is refreshed from: tests, bench line, per-config lines,
# ncu launch list of one C4 step, ncu --set full of the trace + raster kernels,
# per-rank shard timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | cut -c1-300
timeout 1200 python scripts/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
bash scripts/gpu_launches.sh > /dev/null 2>&1
ANGLES=16 bash scripts/gpu_ncu_trace.sh
ANGLES=16 bash scripts/gpu_ncu_raster.sh
timeout 900 python scripts/shard_timing.py 1,2,4,8 > gpurun_out/shard.jsonl 2> gpurun_out/shard.err
python scripts/l2_bw.py > /dev/null 2>&1; cp profiles/l2_peak.json gpurun_out/

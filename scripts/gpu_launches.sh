#!/bin/bash
# ncu launch list (per-kernel durations) of one full C4 step (solve kernels
# only; the BVH build is listed by scripts/build_timing.py); the committed
# profiles/ launch summaries come from this
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:'k_raster|k_trace|k_prim|k_po|k_seg|k_final|k_pad' -c 200 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --angles ${ANGLES:-360} --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv | head -40

#!/bin/bash
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_raster -c 1 \
  -o gpurun_out/prof_raster -f python bench.py --steps 1 --warmup 0 --angles ${ANGLES:-16} --no-e2e --no-cpu > gpurun_out/ncu_raster.log 2>&1
tail -2 gpurun_out/ncu_raster.log

#!/bin/bash
# raster census + ncu --set full of the raster and trace kernels (16 C4 angles)
mkdir -p gpurun_out
timeout 600 python scripts/raster_census.py 360 > gpurun_out/raster_census.json 2> gpurun_out/raster_census.err
cat gpurun_out/raster_census.json; tail -3 gpurun_out/raster_census.err
ANGLES=16 bash scripts/gpu_ncu_raster.sh
ANGLES=16 bash scripts/gpu_ncu_trace.sh
ls -la gpurun_out

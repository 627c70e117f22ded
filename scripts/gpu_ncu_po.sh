#!/bin/bash
# one ncu --set full capture of k_po at nk = 1 (C4, 360 angles: the bench's launch)
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_po -c 1 \
  -o gpurun_out/prof_po -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_po.log 2>&1
tail -2 gpurun_out/ncu_po.log

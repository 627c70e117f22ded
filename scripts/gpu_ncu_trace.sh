#!/bin/bash
# one ncu --set full capture of the trace kernel + the PO kernel (8 angles of C4)
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_trace_persistent -c 1 \
  -o gpurun_out/prof_trace -f python bench.py --steps 1 --warmup 0 --angles ${ANGLES:-8} --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log

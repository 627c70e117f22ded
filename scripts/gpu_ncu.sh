#!/bin/bash
# one ncu --set full capture of the trace kernel (and optionally PO)
mkdir -p gpurun_out
K=${KERNEL:-k_trace_persistent}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
  -o gpurun_out/prof_${TAG:-trace} -f python bench.py --steps 1 --warmup 0 --angles ${ANGLES:-8} --no-e2e --no-cpu > gpurun_out/ncu_${TAG:-trace}.log 2>&1
tail -2 gpurun_out/ncu_${TAG:-trace}.log

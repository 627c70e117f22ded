#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the small
# all-kernel workload; logs in gpurun_out/san_*.log
mkdir -p gpurun_out
for tool in memcheck synccheck initcheck racecheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
  timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool $extra --print-limit 50 \
     --log-file gpurun_out/san_$tool.log python scripts/sanitize_workload.py > gpurun_out/san_$tool.out 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/san_$tool.out; tail -3 gpurun_out/san_$tool.log
done

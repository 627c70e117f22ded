#!/bin/bash
# GPU-box bench run: quick calibration, the contract bench line, ncu launch list.
mkdir -p gpurun_out
ANGLES=${ANGLES:-360}
timeout 600 python bench.py --angles 36 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -2 gpurun_out/bench_quick.err; cat gpurun_out/bench_quick.json
timeout 1200 python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-3} --angles $ANGLES > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --angles 36 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_trace_persistent -c 1 \
    -o gpurun_out/prof_trace -f python bench.py --steps 1 --warmup 0 --angles 8 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_po -c 1 \
    -o gpurun_out/prof_po -f python bench.py --steps 1 --warmup 0 --angles 8 --no-e2e --no-cpu > gpurun_out/ncu_po.log 2>&1
  tail -3 gpurun_out/ncu_full.log
fi

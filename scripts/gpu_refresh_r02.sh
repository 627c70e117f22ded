#!/bin/bash
# Everything the round-2 profiles/ are refreshed from: GPU suite, the bench
# line (default contract), C1-C5 config lines, the ncu launch list of one C4
# step and ncu --set full captures of the trace, raster and PO kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-300 gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cut -c1-300 gpurun_out/bench_ref.json
timeout 1200 python scripts/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; wc -l gpurun_out/configs.jsonl
bash scripts/gpu_launches.sh > /dev/null 2>&1; ls -la gpurun_out/launches.csv
ANGLES=16 bash scripts/gpu_ncu_trace.sh
ANGLES=16 bash scripts/gpu_ncu_raster.sh
bash scripts/gpu_ncu_po.sh
bash scripts/gpu_ncu_po64.sh
ls gpurun_out/*.ncu-rep

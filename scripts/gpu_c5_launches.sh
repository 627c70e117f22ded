cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_raster|k_prim|k_trace|k_po" --csv --log-file gpurun_out/c5_launches.csv python scripts/bench_configs.py --configs c5 --reps 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/c5_launches.csv | head -40

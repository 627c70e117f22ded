"""GPU SAH build time of the C4 mesh (two builds; SBR_SAH_TIMING=1 prints
per-level times).  Used with ncu for the per-kernel launch list of the build."""
import os, sys, time, math
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2604_09243_b200 as sbr
mesh, lam, cfg = bench.workload(1.0, 360)
mesh.device()
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tree = sbr.build(mesh, cfg.build_params()); torch.cuda.synchronize()
    print("build", 1e3*(time.perf_counter()-t0), flush=True)

"""run_sweep stage stamps on the C4 bench workload (SBR_SWEEP_TIMING=1,
SBR_SAH_TIMING=1): where the end-to-end time beyond the fused solve goes."""
import dataclasses, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SBR_SWEEP_TIMING"] = "1"
os.environ["SBR_SAH_TIMING"] = "1"
import torch
import bench
import paper_2604_09243_b200 as sbr
mesh, lam, cfg = bench.workload(1.0, 360)
for rep in range(int(os.environ.get('REPS', '4'))):
    fresh = dataclasses.replace(mesh, _dev={})
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = sbr.run_sweep(cfg, fresh)
    torch.cuda.synchronize()
    print(f"call {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)

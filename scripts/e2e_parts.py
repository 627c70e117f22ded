"""Host-side parts of run_sweep on the C4 workload: mesh upload
(sbr_mesh_create), GPU SAH build, aperture table, and the solve call."""
import dataclasses, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import _native as nat
from paper_2604_09243_b200.sweep import sweep_grids
mesh, lam, cfg = bench.workload(1.0, 360)
ctx = nat.context()
for rep in range(4):
    fresh = dataclasses.replace(mesh, _dev={})
    ctx.synchronize()
    t0 = time.perf_counter(); fresh.device(ctx); ctx.synchronize(); t1 = time.perf_counter()
    tree = sbr.build(fresh, cfg.build_params()); ctx.synchronize(); t2 = time.perf_counter()
    th, ph, cells, grids = sweep_grids(cfg, fresh); t3 = time.perf_counter()
    res = sbr.solve_grids(tree, fresh, grids, cfg.trace_params(), [2 * math.pi / cfg.wavelength])
    t4 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.2f} build {1e3*(t2-t1):.2f} apertures {1e3*(t3-t2):.2f} "
          f"solve {1e3*(t4-t3):.2f} ms", flush=True)
    del tree

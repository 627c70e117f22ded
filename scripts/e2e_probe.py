"""Time the public run_sweep path (C4) several times, after a few device-
resident solves (as bench.py does); print wall ms per call and its phases."""
import dataclasses, math, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen, sweep as S, bvh as bvh_mod
from paper_2604_09243_b200.sweep import sweep_grids, solve_grids

mesh = meshgen.generate_aircraft()
cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=10e9, theta=sbr.AngleRange(math.pi/2, math.pi/2, 1),
                      phi=sbr.AngleRange(0.0, math.radians(359), 360), max_bounces=5)
tree = sbr.build(mesh)
th, ph, cells, grids = sweep_grids(cfg, mesh)
for _ in range(4):
    solve_grids(tree, mesh, grids, cfg.trace_params(), [2 * math.pi / cfg.wavelength])
torch.cuda.synchronize()
orig_build = bvh_mod.build
stamps = {}
def build_t(*a, **k):
    t = time.perf_counter(); r = orig_build(*a, **k); stamps["build"] = time.perf_counter() - t; return r
bvh_mod.build = build_t
for rep in range(6):
    fresh = dataclasses.replace(mesh, _dev={})
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = sbr.run_sweep(cfg, fresh)
    torch.cuda.synchronize()
    print(rep, "total", round((time.perf_counter() - t0) * 1e3, 1), "build", round(stamps["build"] * 1e3, 1),
          "solve", round(out.time_ms.sum(), 1), flush=True)

import math, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen, _native as nat
from paper_2604_09243_b200.sweep import sweep_grids
mesh = meshgen.generate_aircraft()
cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=10e9, theta=sbr.AngleRange(math.pi/2, math.pi/2, 1), phi=sbr.AngleRange(0.0, math.radians(359), 360), max_bounces=5, n_leaf=2)
tree = sbr.build(mesh, cfg.build_params())
th, ph, cells, grids = sweep_grids(cfg, mesh)
ctx = nat.context()
for i in range(3):
    ctx.profile(True)
    try:
        sbr.solve_grids(tree, mesh, grids, cfg.trace_params(), [2*math.pi/cfg.wavelength])
    except Exception as e:
        pass
    ctx.synchronize()
    print("raster_ms", round(ctx.kernel_stats()["raster_ms"], 2), flush=True)

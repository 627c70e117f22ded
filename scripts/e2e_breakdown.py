"""Time each stage of the public run_sweep path on the C4 workload."""
import dataclasses, math, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen, bvh as bvh_mod
from paper_2604_09243_b200.sweep import sweep_grids, solve_grids

mesh = meshgen.generate_aircraft()
lam = 299792458.0 / 10e9
cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=10e9, theta=sbr.AngleRange(math.pi/2, math.pi/2, 1),
                      phi=sbr.AngleRange(0.0, math.radians(359), 360), max_bounces=5)
sbr.run_sweep(cfg, mesh)
for rep in range(3):
    fresh = dataclasses.replace(mesh, _dev={})
    torch.cuda.synchronize(); t = [time.perf_counter()]
    fresh.device(); t.append(time.perf_counter())
    tree = bvh_mod.build(fresh, cfg.build_params()); t.append(time.perf_counter())
    th, ph, cells, grids = sweep_grids(cfg, fresh); t.append(time.perf_counter())
    res = solve_grids(tree, fresh, grids, cfg.trace_params(), [2*math.pi/lam], -1.0, lambda_min=lam, allow_aliasing=False); t.append(time.perf_counter())
    ck = fresh.checksum(); t.append(time.perf_counter())
    names = ["upload", "lbvh", "apertures", "solve", "checksum"]
    print({n: round((t[i+1]-t[i])*1e3, 1) for i, n in enumerate(names)}, flush=True)

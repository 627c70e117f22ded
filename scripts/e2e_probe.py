"""Time the public run_sweep path (C4) several times; print wall ms per call."""
import dataclasses, math, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
mesh = meshgen.generate_aircraft()
cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=10e9, theta=sbr.AngleRange(math.pi/2, math.pi/2, 1),
                      phi=sbr.AngleRange(0.0, math.radians(359), 360), max_bounces=5)
for rep in range(6):
    fresh = dataclasses.replace(mesh, _dev={})
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = sbr.run_sweep(cfg, fresh)
    torch.cuda.synchronize()
    print(rep, round((time.perf_counter() - t0) * 1e3, 1), "solve_ms", round(out.time_ms.sum(), 1), flush=True)

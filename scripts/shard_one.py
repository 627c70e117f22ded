"""One C5 ray-tile shard (rank R of N, default 0 of 8), run twice (the
second is the one to read in a profiler)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
import shard_timing as S
rank, world = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (0, 8)
mesh = meshgen.quantized_icosphere(1.0, 8)
tree = sbr.build(mesh)
ka = np.linspace(937.5, 1000.0, 64)
lam_min = 2 * math.pi / ka.max()
grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, 0.0), 6.4826e-5,
                          wavelength=lam_min)
for _ in range(2):
    print(S.shard_ms(tree, mesh, [grid], sbr.TraceParams(max_bounces=1), ka, lam_min, rank,
                     world, "rays", reps=1))

"""Raster pass census on C5 (s8 sphere, 1.0e9 rays, one angle): candidates,
WIDE pairs, chunk-queue overflows, stage times."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen, _native as nat

mesh = meshgen.quantized_icosphere(1.0, 8)
tree = sbr.build(mesh)
lam = 2 * math.pi / 1000.0
grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, 0.0), 6.4826e-5, wavelength=lam)
ctx = nat.context()
for i in range(2):
    ctx.raster_counters()
    ctx.profile(True)
    res = sbr.solve_grids(tree, mesh, [grid], sbr.TraceParams(max_bounces=1), [2 * math.pi / lam])
    ctx.synchronize()
    st = ctx.kernel_stats()
    cnt = ctx.raster_counters()
    print(json.dumps({"triangles": int(mesh.triangle_count), **cnt,
                      "candidates_per_tri": cnt["candidates"] / mesh.triangle_count,
                      "rays": int(grid.n_u * grid.n_v), **{k: round(v, 3) for k, v in st.items()}}), flush=True)

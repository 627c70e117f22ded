"""Raster pass census on the C4 bench workload: candidate cells tested,
WIDE (ill-conditioned) pairs, chunk-queue overflows and primary hits per
step, plus stage times.  python scripts/raster_census.py [angles]"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen, _native as nat
from paper_2604_09243_b200.sweep import sweep_grids

n = int(sys.argv[1]) if len(sys.argv) > 1 else 360
mesh = meshgen.generate_aircraft()
cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=10e9,
                      theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                      phi=sbr.AngleRange(0.0, math.radians(n - 1), n), max_bounces=5, n_leaf=2)
tree = sbr.build(mesh, cfg.build_params())
th, ph, cells, grids = sweep_grids(cfg, mesh)
ctx = nat.context()
os.environ["SBR_PRIMARY"] = "raster"
for i in range(3):
    ctx.raster_counters()
    ctx.profile(True)
    res = sbr.solve_grids(tree, mesh, grids, cfg.trace_params(), [2 * math.pi / cfg.wavelength])
    ctx.synchronize()
    st = ctx.kernel_stats()
    cnt = ctx.raster_counters()
rays = sum(g.n_u * g.n_v for g in grids)
out = {"angles": n, "triangles": int(mesh.triangle_count), "rays": int(rays),
       "pairs": int(mesh.triangle_count) * n, **cnt,
       "candidates_per_pair": cnt["candidates"] / (mesh.triangle_count * n),
       "queries": int(sum(res.queries)), **{k: round(v, 3) if isinstance(v, float) else v
                                             for k, v in st.items()}}
print(json.dumps(out))

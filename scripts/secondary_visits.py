"""Node+leaf visits per closest-hit query for the first bounce of C4 rays
(reflected rays leaving the surface) vs primary rays, on the SAH and LBVH
trees, via closest_hit_batch (visits = BVH4 nodes + leaves popped)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen

mesh = meshgen.generate_aircraft()
lam = 299792458.0 / 10e9
out = {}
for rule in ("sah", "lbvh"):
    tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
    tp = sbr.TraceParams(max_bounces=1)
    eps = tp.resolve_epsilon(mesh)
    prim_v, sec_v = [], []
    for ph in (0.0, 45.0, 120.0, 200.0):
        g = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, math.radians(ph)),
                               lam / 5, wavelength=lam)
        rec = sbr.trace_grid(tree, mesh, g, tp)
        n = g.ray_count
        i, j = np.divmod(np.arange(n), g.n_v)
        o = (g.corner + ((i + 0.5) * g.spacing)[:, None] * g.u) + ((j + 0.5) * g.spacing)[:, None] * g.v
        d = np.broadcast_to(g.k_inc, o.shape)
        sel = np.arange(0, n, 7)
        _, _, vis = sbr.closest_hit_batch(tree, mesh, o[sel], d[sel])
        prim_v.append(vis)
        h = rec.valid
        hp = o[h] + rec.path[h][:, None] * g.k_inc + eps * rec.normal0[h]
        _, _, vis2 = sbr.closest_hit_batch(tree, mesh, hp, rec.out_dir[h])
        sec_v.append(vis2)
    pv, sv = np.concatenate(prim_v), np.concatenate(sec_v)
    out[rule] = {"primary_visits_mean": float(pv.mean()), "secondary_visits_mean": float(sv.mean()),
                 "secondary_p50_p90_p99": np.percentile(sv, [50, 90, 99]).tolist(),
                 "secondary_queries": int(sv.size)}
print(json.dumps(out, indent=1))

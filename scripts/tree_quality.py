"""Compare traversal work on the GPU LBVH (exported to the reference layout)
vs the reference binned-SAH tree, with the instrumented CPU oracle."""
import math, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
from paper_2604_09243_b200.transport import build_aperture, IncidentDirection
from oracle import oracle as orc

mesh = meshgen.generate_aircraft()
lam = 299792458.0 / 10e9
trees = {}
t = sbr.build(mesh)
trees["lbvh"] = orc.OracleBvh(t.nodes_min, t.nodes_max, t.node_first, t.node_count, t.tri_order, t.max_depth_seen, 128)
trees["sah"] = orc.build(mesh.v0, mesh.v1, mesh.v2)
out = {}
for name, tree in trees.items():
    sc = orc.Scene(mesh.v0, mesh.v1, mesh.v2, mesh.normals, tree)
    tot = dict(pops=0, boxes=0, tris=0, internal=0, queries=0)
    for ph in range(0, 360, 45):
        g = build_aperture(mesh.aabb, IncidentDirection(math.pi/2, math.radians(ph)), lam/5, wavelength=lam)
        for b in range(8):
            r0 = (2*b+1)*g.n_u//16
            c = orc.Counters()
            orc.trace_grid(sc, g, 5, 1e-6*mesh.aabb.diagonal(), rows=(r0, min(g.n_u, r0+8)), counters=c)
            for k, v in c.as_dict().items(): tot[k] += v
    q = tot["queries"]
    out[name] = {k: v / q for k, v in tot.items()}
    out[name]["nodes"] = int(tree.node_first.shape[0]); out[name]["depth"] = int(tree.max_depth_seen)
print(json.dumps(out, indent=1))

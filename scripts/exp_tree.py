"""Experiment: trace cost with the GPU LBVH vs the reference binned-SAH tree
(built on the CPU by the oracle restatement of bvh.py:218-299 and uploaded
with sbr_bvh_upload).  C4 workload, N angles; prints trace/raster ms."""
import math, os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen, _native as nat
from paper_2604_09243_b200.sweep import sweep_grids
from oracle import oracle as orc

n_ang = int(sys.argv[1]) if len(sys.argv) > 1 else 72
mesh = meshgen.generate_aircraft()
lam = 299792458.0 / 10e9
cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=10e9, theta=sbr.AngleRange(math.pi/2, math.pi/2, 1),
                      phi=sbr.AngleRange(0.0, math.radians(n_ang - 1), n_ang), max_bounces=5)
th, ph, cells, grids = sweep_grids(cfg, mesh)
tp = cfg.trace_params()
ctx = nat.context(0)
trees = {"lbvh": sbr.build(mesh)}
for rule in ("sah", "median"):
    t0 = time.time()
    ot = orc.build(mesh.v0, mesh.v1, mesh.v2, split_rule=rule, n_leaf=4)
    trees[rule] = sbr.Bvh(ot.nodes_min, ot.nodes_max, ot.node_first, ot.node_count, ot.tri_order,
                          ot.max_depth_seen)
    print(rule, "cpu build s", round(time.time() - t0, 2), file=sys.stderr)
out = {}
for name, tree in trees.items():
    for rep in range(3):
        ctx.profile(True)
        res = sbr.solve_grids(tree, mesh, grids, tp, [2 * math.pi / lam])
        ctx.synchronize()
        k = ctx.kernel_stats()
    out[name] = {"trace_ms": k["trace_ms"], "raster_ms": k["raster_ms"],
                 "queries": int(res.queries.sum()), "amp0": str(res.amplitude[0, 0])}
print(json.dumps(out, indent=1))

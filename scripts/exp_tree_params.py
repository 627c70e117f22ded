"""Experiment: trace time of the C4 sweep (72 azimuths) for GPU-built SAH
trees with other bin counts / cost constants (results are tree-independent:
the amplitudes must match bit for bit)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen, _native as nat
from paper_2604_09243_b200.sweep import sweep_grids

n_ang = int(sys.argv[1]) if len(sys.argv) > 1 else 72
mesh = meshgen.generate_aircraft()
lam = 299792458.0 / 10e9
cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=10e9, theta=sbr.AngleRange(math.pi/2, math.pi/2, 1),
                      phi=sbr.AngleRange(0.0, math.radians(n_ang - 1), n_ang), max_bounces=5)
th, ph, cells, grids = sweep_grids(cfg, mesh)
tp = cfg.trace_params()
ctx = nat.context(0)
variants = [("sah16", dict()), ("sah32", dict(bins_per_axis=32)), ("sah64", dict(bins_per_axis=64)),
            ("ct2", dict(c_t=2.0)), ("ct0.5", dict(c_t=0.5)), ("ct4", dict(c_t=4.0)),
            ("nl1_ct2", dict(n_leaf=1, c_t=2.0)), ("nl3", dict(n_leaf=3)), ("lbvh", dict(split_rule="lbvh"))]
out = {}
ref_amp = None
for name, kw in variants:
    p = dict(split_rule="sah", n_leaf=2); p.update(kw)
    tree = sbr.build(mesh, sbr.BuildParams(**p))
    best = None
    for rep in range(3):
        ctx.profile(True)
        res = sbr.solve_grids(tree, mesh, grids, tp, [2 * math.pi / lam])
        ctx.synchronize()
        k = ctx.kernel_stats()
        best = k["trace_ms"] if best is None else min(best, k["trace_ms"])
    amp = res.amplitude.copy()
    if ref_amp is None:
        ref_amp = amp
    out[name] = {"params": p, "trace_ms": round(best, 2), "nodes": int(tree.node_count.shape[0]) if hasattr(tree, "node_count") else None,
                 "identical_amplitudes": bool((amp == ref_amp).all())}
    print(name, out[name], flush=True)
json.dump(out, open("gpurun_out/exp_tree_params.json", "w"), indent=1)

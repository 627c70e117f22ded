"""GPU build time of the LBVH and of the reference-exact binned-SAH tree
(C4 aircraft, C5 sphere s8), and the C4 trace time with each tree."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen, _native as nat
from paper_2604_09243_b200.sweep import sweep_grids

out = {}
for name, mesh in (("C4", meshgen.generate_aircraft()), ("C5", meshgen.quantized_icosphere(1.0, 8))):
    mesh.device()
    for rule in ("lbvh", "sah"):
        ts = []
        for _ in range(4):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        out[f"{name}_{rule}_build_ms"] = round(1e3 * sorted(ts)[1], 2)
        out[f"{name}_{rule}_depth"] = tree.max_depth_seen
        if name == "C4":
            cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=10e9,
                                  theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                                  phi=sbr.AngleRange(0.0, math.radians(359), 360), max_bounces=5)
            th, ph, cells, grids = sweep_grids(cfg, mesh)
            ctx = nat.context()
            for _ in range(2):
                ctx.profile(True)
                sbr.solve_grids(tree, mesh, grids, cfg.trace_params(), [2 * math.pi / cfg.wavelength])
            k = ctx.kernel_stats()
            out[f"C4_{rule}_trace_ms"] = round(k["trace_ms"], 2)
print(json.dumps(out, indent=1))

"""PO precision of the multi-wavenumber paths (rotation recurrence for a
uniform sweep, per-frequency otherwise) against the oracle's accumulate, on a
C5-like sphere aperture scaled down to ~4M rays, 64 wavenumbers
ka in [937.5, 1000] (the C5 band).  Writes gpurun_out/parity_po_multik.json."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
from oracle import oracle as orc

mesh = meshgen.quantized_icosphere(1.0, 8)
tree = sbr.build(mesh, sbr.BuildParams(split_rule="sah", n_leaf=2))
ot = orc.build(mesh.v0, mesh.v1, mesh.v2, split_rule="sah", n_leaf=4)
scene = orc.Scene(mesh.v0, mesh.v1, mesh.v2, mesh.normals, ot)
ka = np.linspace(937.5, 1000.0, 64)
ks = ka / 1.0
lam_min = 2 * math.pi / ks.max()
g = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, 0.0), 2.0 / 2000,
                       wavelength=lam_min, allow_aliasing=True)
tp = sbr.TraceParams(max_bounces=1)
ref = orc.trace_grid(scene, g, 1, tp.resolve_epsilon(mesh))
out = {"rays": len(ref), "nk": len(ks)}
for name, kv in (("uniform64_rotation", ks), ("irregular64_per_frequency", ks * (1 + 1e-3 * np.sin(np.arange(64))))):
    amp = sbr.solve_grids(tree, mesh, [g], tp, kv, allow_aliasing=True).amplitude[0]
    errs = []
    for f, k in enumerate(kv):
        a_ref = orc.accumulate(ref, g.k_inc, 2 * math.pi / k, g.cell_area)
        errs.append(abs(amp[f] - a_ref) / abs(a_ref))
    out[name] = {"max_rel_err": float(max(errs)), "median_rel_err": float(np.median(errs))}
    print(name, out[name], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/parity_po_multik.json", "w"), indent=1)

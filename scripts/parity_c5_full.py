"""C5 at full size: the 1.0e9-ray sphere aperture, 64 wavenumbers (uniform:
the rotation-recurrence PO path), fused GPU solve vs the oracle on the host
cores (records traced in row bands, each band accumulated per wavenumber,
band sums added in FP64).  Also counts bounces/valid rays.  Writes
gpurun_out/parity_c5_full.json."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
from oracle import oracle as orc

mesh = meshgen.quantized_icosphere(1.0, 8)
tree = sbr.build(mesh)
tp = sbr.TraceParams(max_bounces=1)
ka = np.linspace(937.5, 1000.0, 64)
lam_min = 2 * math.pi / ka.max()
g = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, 0.0), 6.4826e-5, wavelength=lam_min)
t0 = time.time()
res = sbr.solve_grids(tree, mesh, [g], tp, ka, lambda_min=lam_min, allow_aliasing=False)
gpu_s = time.time() - t0
amp = res.amplitude[0]
ot = orc.build(mesh.v0, mesh.v1, mesh.v2, split_rule="sah", n_leaf=4)
scene = orc.Scene(mesh.v0, mesh.v1, mesh.v2, mesh.normals, ot)
eps = tp.resolve_epsilon(mesh)
ref = np.zeros(64, complex)
valid = queries = 0
t1 = time.time()
band = 256
for i0 in range(0, g.n_u, band):
    rec = orc.trace_grid(scene, g, 1, eps, rows=(i0, min(g.n_u, i0 + band)))
    valid += int(rec.valid.sum())
    queries += int((rec.bounces.astype(np.int64) + 1).sum())
    for f, k in enumerate(ka):
        ref[f] += orc.accumulate(rec, g.k_inc, 2 * math.pi / k, g.cell_area)
ora_s = time.time() - t1
rel = np.abs(amp - ref) / np.abs(ref)
out = {"rays": int(g.n_u * g.n_v), "grid": [g.n_u, g.n_v], "nk": 64,
       "valid_rays": {"gpu": int(res.valid_rays[0]), "oracle": valid},
       "queries": {"gpu": int(res.queries[0]), "oracle": queries},
       "max_amp_rel_err": float(rel.max()), "median_amp_rel_err": float(np.median(rel)),
       "max_db_err": float(np.max(np.abs(20 * np.log10(np.abs(amp) / np.abs(ref))))),
       "gpu_solve_s": round(gpu_s, 2), "oracle_s": round(ora_s, 1)}
print(json.dumps(out), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/parity_c5_full.json", "w"), indent=1)

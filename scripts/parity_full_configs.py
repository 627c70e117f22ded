"""Full-size parity of C1, C2 and C3 (every aperture of the sweep): GPU
trace_grid records + per-bounce ids vs the oracle on the host cores, bit for
bit, and the fused solve's amplitude vs the oracle's accumulate.  Writes
gpurun_out/parity_full_configs.json."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
from oracle import oracle as orc

FIELDS = ("valid", "normal0", "path", "bounces", "escaped", "out_dir", "tri_ids")


def run(name, mesh, lam, B, dirs):
    tree = sbr.build(mesh)
    ot = orc.build(mesh.v0, mesh.v1, mesh.v2, split_rule="sah", n_leaf=4)
    scene = orc.Scene(mesh.v0, mesh.v1, mesh.v2, mesh.normals, ot)
    tp = sbr.TraceParams(max_bounces=B)
    eps = tp.resolve_epsilon(mesh)
    grids = [sbr.build_aperture(mesh.aabb, d, lam / 5, wavelength=lam) for d in dirs]
    amps = sbr.solve_grids(tree, mesh, grids, tp, [2 * math.pi / lam]).amplitude[:, 0]
    rays = mism = 0
    worst = 0.0
    for g, a in zip(grids, amps):
        gpu = sbr.trace_grid(tree, mesh, g, tp, with_ids=True)
        ref = orc.trace_grid(scene, g, B, eps, with_ids=True)
        n = len(ref)
        rays += n
        for f in FIELDS:
            mism += int((~np.all(np.asarray(getattr(gpu, f)).reshape(n, -1) ==
                                 np.asarray(getattr(ref, f)).reshape(n, -1), axis=1)).sum())
        a_ref = orc.accumulate(ref, g.k_inc, lam, g.cell_area)
        worst = max(worst, abs(complex(a) - a_ref) / abs(a_ref))
    row = {"config": name, "apertures": len(grids), "rays": rays, "mismatched_ray_fields": mism,
           "max_amp_rel_err": worst}
    print(json.dumps(row), flush=True)
    return row


out = []
ka = 20.0
out.append(run("C1 (16 fibonacci directions)", meshgen.quantized_icosphere(1.0, 5), 2 * math.pi / ka, 4,
               sbr.fibonacci_directions(16)))
ka = 100.0
out.append(run("C2", meshgen.quantized_icosphere(1.0, 6), 2 * math.pi / ka, 1,
               [sbr.IncidentDirection(math.pi / 2, math.radians(p)) for p in np.linspace(0, 359, 360)]))
out.append(run("C3-dihedral", meshgen.dihedral_mesh(), 0.05, 3,
               [sbr.IncidentDirection(math.pi / 2, math.radians(p)) for p in np.linspace(0, 90, 181)]))
out.append(run("C3-trihedral", meshgen.trihedral_mesh(), 0.05, 3,
               [sbr.IncidentDirection(math.radians(54.7356), math.radians(p)) for p in np.linspace(0, 90, 181)]))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/parity_full_configs.json", "w"), indent=1)

"""Census of the tree-dependent ray class per BASELINE config.

For every ray the oracle's classifier (orc_classify_grid) decides whether
the reference's answer is tree-independent ("robust": every query's winning
hit lies robustly inside its triangle's box and no other accepting triangle
ties it within rounding).  Non-robust rays are the only ones on which the
reference itself could answer differently with another tree; the fast path
(raster + BVH4) is compared record for record (with per-bounce ids) with the
oracle on ALL rays, and the mismatches are counted separately on both classes.

  python scripts/robust_census.py  -> gpurun_out/robust_census.json
"""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
from oracle import oracle as orc

C = 299792458.0
REC = ("valid", "normal0", "path", "bounces", "escaped", "out_dir", "tri_ids")


def census(name, mesh, grids, B, rows=None, row_sample=None):
    """rows: one row range for every grid; row_sample: k evenly spaced
    rows through the middle half of each grid (the classifier is a linear
    scan over all triangles per query -- large meshes are sampled)."""
    tree = sbr.build(mesh)
    scene = orc.Scene.from_mesh(mesh)
    tp = sbr.TraceParams(max_bounces=B)
    eps = tp.resolve_epsilon(mesh)
    n = nonrob = mism = mism_nonrob = 0
    t0 = time.time()
    for g in grids:
        ranges = [rows]
        if row_sample:
            ranges = [(int(i), int(i) + 1) for i in
                      np.linspace(g.n_u // 4, 3 * g.n_u // 4, row_sample).astype(int)]
        for rr in ranges:
            rob, _, _ = orc.classify_grid(scene, g, B, eps, rows=rr)
            rec = sbr.trace_grid(tree, mesh, g, tp, with_ids=True, rows=rr)
            ref = orc.trace_grid(scene, g, B, eps, rows=rr, with_ids=True)
            bad = np.zeros(rob.size, bool)
            for k in REC:
                a, b = getattr(rec, k), getattr(ref, k)
                neq = a != b
                bad |= neq.reshape(neq.shape[0], -1).any(axis=1) if neq.ndim > 1 else neq
            n += rob.size
            nonrob += int((~rob).sum())
            mism += int(bad.sum())
            mism_nonrob += int((bad & ~rob).sum())
    out = {"config": name, "triangles": int(mesh.triangle_count), "apertures": len(grids),
           "rays": n, "non_robust_rays": nonrob, "non_robust_fraction": nonrob / max(n, 1),
           "mismatching_rays": mism, "mismatching_non_robust_rays": mism_nonrob,
           "max_bounces": B, "sampled_rows_per_aperture": row_sample,
           "seconds": round(time.time() - t0, 1)}
    print(json.dumps(out), flush=True)
    return out


def main():
    want = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4", "c5"]
    res = []
    if "c1" not in want:
        return main_large(want, res)
    s5 = meshgen.quantized_icosphere(1.0, 5)
    lam = 2 * math.pi / 20
    res.append(census("C1 sphere ka=20 (90,0), lambda/5", s5,
                      [sbr.build_aperture(s5.aabb, sbr.IncidentDirection(math.pi / 2, 0.0), lam / 5,
                                          wavelength=lam)], 4))
    s6 = meshgen.quantized_icosphere(1.0, 6)
    lam = 2 * math.pi / 100
    res.append(census("C2 sphere ka=100, 360 azimuths, B=1", s6,
                      [sbr.build_aperture(s6.aabb, sbr.IncidentDirection(math.pi / 2, math.radians(p)),
                                          lam / 5, wavelength=lam) for p in range(360)], 1))
    lam = 0.05
    for nm, mesh, th in (("C3 dihedral", meshgen.dihedral_mesh(1.0), math.pi / 2),
                         ("C3 trihedral", meshgen.trihedral_mesh(1.0), math.radians(54.7356))):
        res.append(census(nm + ", 181 azimuths, B=3", mesh,
                          [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(th, p), lam / 5,
                                              wavelength=lam)
                           for p in np.linspace(0, math.pi / 2, 181)], 3))
    return main_large(want, res)


def main_large(want, res):
    if "c4" not in want and "c5" not in want:
        return
    air = meshgen.generate_aircraft(density=1.0)
    lam = C / 10e9
    if "c4" in want:
        res.append(census("C4 aircraft, 24 apertures (every 15 deg), 2 sampled rows each, B=5",
                          air, [sbr.build_aperture(air.aabb,
                                                   sbr.IncidentDirection(math.pi / 2, math.radians(p)),
                                                   lam / 5, wavelength=lam)
                                for p in range(0, 360, 15)], 5, row_sample=2))
    s8 = meshgen.quantized_icosphere(1.0, 8)
    g = sbr.build_aperture(s8.aabb, sbr.IncidentDirection(math.pi / 2, 0.0), 6.4826e-5,
                           wavelength=2 * math.pi / 1000)
    nrows = -(-10_000_000 // g.n_v)
    i0 = g.n_u // 2 - nrows // 2
    if "c5" in want:
        res.append(census("C5 sphere s8, 4 sampled rows (126k rays), B=1", s8, [g], 1,
                          row_sample=4))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/robust_census.json", "w"), indent=1)


if __name__ == "__main__":
    main()

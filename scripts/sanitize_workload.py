"""Small workload that touches every kernel family of libsbr200 once, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
GPU SAH, median and LBVH builds, closest hits (fast and reference order),
trace_grid (raster and BVH primaries, ids, hashes), the fused solve over C1,
C3 (dihedral, trihedral) and a small C4 aircraft (1 and 8 wavenumbers),
accumulate and validate_sphere."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen

def main():
    sphere = meshgen.quantized_icosphere(1.0, 4)
    air = meshgen.generate_aircraft(density=0.02)
    dih, tri = meshgen.dihedral_mesh(1.0), meshgen.trihedral_mesh(1.0)
    rng = np.random.default_rng(1)
    for mesh in (sphere, air):
        for rule in ("sah", "median", "lbvh"):
            t = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
            o = rng.normal(size=(256, 3)) * 3.0
            d = -o / np.linalg.norm(o, axis=1)[:, None]
            sbr.closest_hit_batch(t, mesh, o, d)
            if rule != "lbvh":
                with sbr.traversal_order("reference"):
                    sbr.closest_hit_batch(t, mesh, o, d)
    t_air = sbr.build(air)
    lam = 0.2
    g = sbr.build_aperture(air.aabb, sbr.IncidentDirection(math.pi / 2, 0.7), lam / 5, wavelength=lam)
    for prim in ("raster", "bvh"):
        os.environ["SBR_PRIMARY"] = prim
        sbr.trace_grid(t_air, air, g, sbr.TraceParams(max_bounces=3), with_ids=True)
        sbr.trace_grid_hash(t_air, air, g, sbr.TraceParams(max_bounces=1))
        sbr.solve_grids(t_air, air, [g, g], sbr.TraceParams(max_bounces=5), [2 * math.pi / lam])
    os.environ.pop("SBR_PRIMARY")
    rec = sbr.trace_grid(t_air, air, g, sbr.TraceParams(max_bounces=3))
    sbr.accumulate(rec, g.k_inc, sbr.ScatterParams.from_wavelength(lam, g.cell_area))
    ks = np.linspace(2 * math.pi / lam, 2.2 * math.pi / lam, 8)
    sbr.solve_grids(t_air, air, [g], sbr.TraceParams(max_bounces=5), ks)
    with sbr.traversal_order("reference"):
        sbr.solve_grids(t_air, air, [g], sbr.TraceParams(max_bounces=5), [2 * math.pi / lam])
    for mesh, th in ((dih, math.pi / 2), (tri, 0.9553)):
        t = sbr.build(mesh)
        grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(th, p), 0.01, wavelength=0.05)
                 for p in np.linspace(0, math.pi / 2, 5)]
        sbr.solve_grids(t, mesh, grids, sbr.TraceParams(max_bounces=3), [2 * math.pi / 0.05])
    sbr.validate_sphere(1.0, [8.0], subdivisions=3, n_directions=4)
    print("sanitize workload done")

if __name__ == "__main__":
    main()
    # everything the workload created is garbage now: release meshes and
    # trees, then the contexts, so memcheck --leak-check sees a clean exit
    from paper_2604_09243_b200 import _native as nat
    print("live device allocations before shutdown:", nat.live_allocations())
    nat.shutdown()
    print("live device allocations after shutdown:", nat.live_allocations())

"""Throughput + accuracy of every BASELINE.json configuration (C1-C5).

bench.py carries the driver's single headline line (C4); this script reports
the other configurations the north star lists, on one GPU:

  C1  PEC sphere ka=20 (icosphere s5, 20k tris), one angle, vs Mie (direction
      averaged over 16 Fibonacci directions, the reference's method)
  C2  PEC sphere ka=100 (s6, 82k tris), 360-angle sweep, 1 bounce (+ probe)
  C3  dihedral + trihedral, 3 bounces, 181-angle sweeps
  C4  procedural aircraft (~1M tris), 5 bounces, 360 angles, 10 GHz
  C5  sphere ka=1000 (s8, 1.3M tris), one angle, 31623^2 = 1.0e9 rays,
      64 wavenumbers ka in [937.5, 1000] -- fused solve, vs Mie (PO limit)

    python scripts/bench_configs.py [--configs c1,c2,c3,c4,c5] [--reps 3]

Prints one JSON object per config; timing is CUDA events on the library
stream around the fused solve (mesh/BVH resident), median of --reps.
"""

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2604_09243_b200 as sbr  # noqa: E402
from paper_2604_09243_b200 import _native as nat, meshgen  # noqa: E402

C = 299792458.0


def timed_solve(tree, mesh, grids, tp, ks, reps, lam_min):
    ctx = nat.context()
    stream = torch.cuda.ExternalStream(ctx.stream)
    res = sbr.solve_grids(tree, mesh, grids, tp, ks, lambda_min=lam_min, allow_aliasing=False)
    times, kst = [], []
    for _ in range(reps):
        ctx.profile(True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = sbr.solve_grids(tree, mesh, grids, tp, ks, lambda_min=lam_min,
                              allow_aliasing=False)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        kst.append(ctx.kernel_stats())
    ctx.profile(False)
    i = int(np.argsort(times)[len(times) // 2])
    return res, times[i], kst[i]


def report(name, mesh, grids, res, t, kst, nk, extra):
    q = int(res.queries.sum())
    rays = sum(g.ray_count for g in grids)
    sel = int(res.valid_rays.sum())
    out = {"config": name, "triangles": mesh.triangle_count, "angles": len(grids),
           "rays": rays, "queries": q, "seconds": t,
           "intersections_per_s": q / t, "angles_per_s": len(grids) / t,
           "raster_ms": kst["raster_ms"], "trace_ms": kst["trace_ms"], "po_ms": kst["po_ms"],
           "po_terms": sel * nk,
           "po_terms_per_s": sel * nk / (kst["po_ms"] / 1e3) if kst["po_ms"] else None}
    out.update(extra)
    print(json.dumps(out), flush=True)
    return out


def c1(reps):
    ka = 20.0
    lam = 2 * math.pi / ka
    mesh = meshgen.quantized_icosphere(1.0, 5)
    tree = sbr.build(mesh)
    tp = sbr.TraceParams(max_bounces=4)
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, 0.0), lam / 5,
                                wavelength=lam)]
    res, t, kst = timed_solve(tree, mesh, grids, tp, [ka], reps, lam)
    dirs = sbr.fibonacci_directions(16)
    g16 = [sbr.build_aperture(mesh.aabb, d, lam / 5, wavelength=lam) for d in dirs]
    r16 = sbr.solve_grids(tree, mesh, g16, tp, [ka])
    sig = float(np.mean([sbr.rcs(a).sigma_m2 for a in r16.amplitude[:, 0]]))
    mie = sbr.mie_backscatter_pec(ka, 1.0)
    return report("C1", mesh, grids, res, t, kst, 1,
                  {"sigma_single_angle_m2": sbr.rcs(res.amplitude[0, 0]).sigma_m2,
                   "sigma_16dir_mean_m2": sig, "sigma_mie_m2": mie,
                   "mie_rel_error_16dir": abs(sig - mie) / mie})


def c2(reps):
    ka = 100.0
    lam = 2 * math.pi / ka
    mesh = meshgen.quantized_icosphere(1.0, 6)
    tree = sbr.build(mesh)
    tp = sbr.TraceParams(max_bounces=1)
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, math.radians(p)),
                                lam / 5, wavelength=lam) for p in np.linspace(0, 359, 360)]
    res, t, kst = timed_solve(tree, mesh, grids, tp, [ka], reps, lam)
    sig = np.array([sbr.rcs(a).sigma_m2 for a in res.amplitude[:, 0]])
    mie = sbr.mie_backscatter_pec(ka, 1.0)
    return report("C2", mesh, grids, res, t, kst, 1,
                  {"sigma_sweep_mean_m2": float(sig.mean()), "sigma_mie_m2": mie,
                   "mie_rel_error_sweep_mean": float(abs(sig.mean() - mie) / mie)})


def c3(reps):
    lam = 0.05
    out = []
    for name, mesh, theta, span in (("C3-dihedral", meshgen.dihedral_mesh(), math.pi / 2, 90.0),
                                    ("C3-trihedral", meshgen.trihedral_mesh(),
                                     math.radians(54.7356), 90.0)):
        tree = sbr.build(mesh)
        tp = sbr.TraceParams(max_bounces=3)
        grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(theta, math.radians(p)),
                                    lam / 5, wavelength=lam) for p in np.linspace(0, span, 181)]
        res, t, kst = timed_solve(tree, mesh, grids, tp, [2 * math.pi / lam], reps, lam)
        out.append(report(name, mesh, grids, res, t, kst, 1,
                          {"bounce_histogram": res.bounce_counts.sum(0).tolist()}))
    return out


def c4(reps):
    mesh = meshgen.generate_aircraft()
    lam = C / 10e9
    tree = sbr.build(mesh)
    tp = sbr.TraceParams(max_bounces=5)
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, math.radians(p)),
                                lam / 5, wavelength=lam) for p in np.linspace(0, 359, 360)]
    res, t, kst = timed_solve(tree, mesh, grids, tp, [2 * math.pi / lam], reps, lam)
    return report("C4", mesh, grids, res, t, kst, 1,
                  {"bounce_histogram": res.bounce_counts.sum(0).tolist()})


def c5(reps):
    mesh = meshgen.quantized_icosphere(1.0, 8)
    tree = sbr.build(mesh)
    tp = sbr.TraceParams(max_bounces=1)
    ka = np.linspace(937.5, 1000.0, 64)
    lam_min = 2 * math.pi / ka.max()
    grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, 0.0), 6.4826e-5,
                              wavelength=lam_min)
    res, t, kst = timed_solve(tree, mesh, [grid], tp, ka, max(1, reps - 1), lam_min)
    sig = np.array([sbr.rcs(a).sigma_m2 for a in res.amplitude[0]])
    mie = np.array([sbr.mie_backscatter_pec(x, 1.0) for x in ka[::16]])
    return report("C5", mesh, [grid], res, t, kst, len(ka),
                  {"grid": [grid.n_u, grid.n_v], "wavenumbers": len(ka),
                   "sigma_m2_first_last": [float(sig[0]), float(sig[-1])],
                   "sigma_mie_m2_subset": mie.tolist(),
                   "mie_rel_error_subset": (np.abs(sig[::16] - mie) / mie).tolist()})


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="c1,c2,c3,c4,c5")
    p.add_argument("--reps", type=int, default=3)
    args = p.parse_args()
    torch.cuda.set_device(0)
    for c in args.configs.split(","):
        globals()[c.strip()](args.reps)


if __name__ == "__main__":
    main()

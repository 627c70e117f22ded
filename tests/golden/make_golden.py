"""Generate the golden parity fixtures by running the REFERENCE package.

Run here (the CPU container, where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONHASHSEED=0 \
        python tests/golden/make_golden.py

It imports the reference ``sbr`` package from /root/reference/pkg/src (never
copied into this repo) and its test helpers (pkg/tests/meshes.py), evaluates
the trace-integrate path on small deterministic inputs, and writes
compressed ``.npz`` fixtures next to this script.  The fixtures travel to the
GPU box; the reference does not.

Besides the reference's own outputs the script records per-bounce hit
triangle ids with a numba restatement of transport.py:276-356 that calls the
reference's own ``sbr.bvh._traverse``; the restatement is self-checked
bit-for-bit against ``sbr.trace_grid`` on every fixture.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import platform
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import numba  # noqa: E402
import numpy as np  # noqa: E402
from numba import njit  # noqa: E402

import sbr  # noqa: E402
from sbr import bvh as ref_bvh  # noqa: E402
from sbr.sweep import solve_direction  # noqa: E402
from meshes import (dihedral_mesh, perturbed_grid_mesh, plate_mesh,  # noqa: E402
                    random_probe_rays, brute_force_hits)

OUT = os.path.dirname(os.path.abspath(__file__))


def trihedral_mesh(size=1.0):
    """Three unit squares on the coordinate planes (new for config C3)."""
    s = size
    v = [[0, 0, 0], [s, 0, 0], [s, s, 0], [0, s, 0],   # z = 0
         [0, 0, s], [s, 0, s],                          # y = 0 (with 0,1)
         [0, s, s]]                                      # x = 0 (with 0,3,4)
    f = [[0, 1, 2], [0, 2, 3],
         [0, 1, 5], [0, 5, 4],
         [0, 3, 6], [0, 6, 4]]
    return sbr.mesh_from_arrays(v, f)


def quantized_icosphere(sub):
    m = sbr.generate_icosphere(1.0, sub)
    tri = np.stack([m.v0, m.v1, m.v2], axis=1).astype(np.float32).astype(np.float64)
    return sbr.mesh_from_soup(tri)


@njit(cache=True)
def _trace_ids(nodes_min, nodes_max, node_first, node_count, tri_order,
               v0, v1, v2, normals, corner, uvec, vvec, kvec, spacing,
               n_u, n_v, max_bounces, eps, strict, stack_depth,
               o_valid, o_n0, o_path, o_b, o_esc, o_dir, o_tri):
    """transport.py:276-356 restated, recording the hit triangle per bounce."""
    stack = np.empty(stack_depth, dtype=np.int32)
    for i in range(n_u):
        bx = corner[0] + (i + 0.5) * spacing * uvec[0]
        by = corner[1] + (i + 0.5) * spacing * uvec[1]
        bz = corner[2] + (i + 0.5) * spacing * uvec[2]
        for j in range(n_v):
            r = i * n_v + j
            ox = bx + (j + 0.5) * spacing * vvec[0]
            oy = by + (j + 0.5) * spacing * vvec[1]
            oz = bz + (j + 0.5) * spacing * vvec[2]
            dx = kvec[0]; dy = kvec[1]; dz = kvec[2]
            path = 0.0; bounces = 0; valid = False; escaped = False
            n0x = 0.0; n0y = 0.0; n0z = 0.0
            for s in range(max_bounces):
                o_tri[r, s] = -1
            done = False
            for s in range(max_bounces):
                tri, t, _ = ref_bvh._traverse(nodes_min, nodes_max, node_first,
                                              node_count, tri_order, v0, v1, v2,
                                              ox, oy, oz, dx, dy, dz, 0.0,
                                              np.inf, stack)
                if tri < 0:
                    escaped = True
                    break
                nx = normals[tri, 0]; ny = normals[tri, 1]; nz = normals[tri, 2]
                nd = nx * dx + ny * dy + nz * dz
                if nd > 0.0:
                    if strict and bounces == 0:
                        done = True
                        break
                    nx = -nx; ny = -ny; nz = -nz; nd = -nd
                o_tri[r, s] = tri
                hx = ox + t * dx; hy = oy + t * dy; hz = oz + t * dz
                path += t
                bounces += 1
                if bounces == 1:
                    n0x = nx; n0y = ny; n0z = nz
                    valid = True
                dx -= 2.0 * nd * nx
                dy -= 2.0 * nd * ny
                dz -= 2.0 * nd * nz
                ox = hx + eps * nx; oy = hy + eps * ny; oz = hz + eps * nz
            if done:
                o_valid[r] = False; o_n0[r, 0] = 0.0; o_n0[r, 1] = 0.0
                o_n0[r, 2] = 0.0; o_path[r] = 0.0; o_b[r] = 0; o_esc[r] = True
                o_dir[r, 0] = dx; o_dir[r, 1] = dy; o_dir[r, 2] = dz
                continue
            if valid and not escaped:
                tri, _, _ = ref_bvh._traverse(nodes_min, nodes_max, node_first,
                                              node_count, tri_order, v0, v1, v2,
                                              ox, oy, oz, dx, dy, dz, 0.0,
                                              np.inf, stack)
                escaped = tri < 0
            o_valid[r] = valid; o_n0[r, 0] = n0x; o_n0[r, 1] = n0y
            o_n0[r, 2] = n0z; o_path[r] = path; o_b[r] = bounces
            o_esc[r] = escaped
            o_dir[r, 0] = dx; o_dir[r, 1] = dy; o_dir[r, 2] = dz


def trace_with_ids(tree, mesh, grid, params):
    n = grid.ray_count
    B = params.max_bounces
    out = dict(valid=np.empty(n, np.bool_), normal0=np.empty((n, 3)),
               path=np.empty(n), bounces=np.empty(n, np.int32),
               escaped=np.empty(n, np.bool_), out_dir=np.empty((n, 3)),
               tri_ids=np.empty((n, B), np.int32))
    _trace_ids(tree.nodes_min, tree.nodes_max, tree.node_first,
               tree.node_count, tree.tri_order, mesh.v0, mesh.v1, mesh.v2,
               mesh.normals, np.ascontiguousarray(grid.corner, np.float64),
               np.ascontiguousarray(grid.u, np.float64),
               np.ascontiguousarray(grid.v, np.float64),
               np.ascontiguousarray(grid.k_inc, np.float64), grid.spacing,
               grid.n_u, grid.n_v, B, params.resolve_epsilon(mesh),
               params.strict_orientation, tree.params.max_depth + 2,
               out["valid"], out["normal0"], out["path"], out["bounces"],
               out["escaped"], out["out_dir"], out["tri_ids"])
    return out


def mesh_arrays(mesh, prefix="mesh_"):
    return {prefix + k: np.asarray(getattr(mesh, k)) for k in
            ("v0", "v1", "v2", "normals")}


def bvh_arrays(tree, prefix="bvh_"):
    return {prefix + "nodes_min": tree.nodes_min,
            prefix + "nodes_max": tree.nodes_max,
            prefix + "node_first": tree.node_first,
            prefix + "node_count": tree.node_count,
            prefix + "tri_order": tree.tri_order,
            prefix + "max_depth_seen": np.int64(tree.max_depth_seen)}


def grid_arrays(grid):
    return {"grid_corner": grid.corner, "grid_u": grid.u, "grid_v": grid.v,
            "grid_k": grid.k_inc, "grid_spacing": np.float64(grid.spacing),
            "grid_n_u": np.int64(grid.n_u), "grid_n_v": np.int64(grid.n_v),
            "grid_cell_area": np.float64(grid.cell_area),
            "grid_standoff": np.float64(grid.standoff),
            "grid_margin": np.float64(grid.margin)}


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"  wrote {name}.npz ({os.path.getsize(path) / 1024:.0f} KiB)")


# ---------------------------------------------------------------------------

def gen_mt():
    """Random ray/triangle pairs (test_geometry.py:186-229 style) + edge KATs."""
    rng = np.random.default_rng(1234)
    n = 4000
    v0 = rng.uniform(-1, 1, (n, 3)); v1 = rng.uniform(-1, 1, (n, 3))
    v2 = rng.uniform(-1, 1, (n, 3))
    o = rng.uniform(-3, 3, (n, 3))
    tgt = (v0 + v1 + v2) / 3 + rng.normal(scale=0.6, size=(n, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1)[:, None]
    # crafted cases: vertex hits, edge hits, parallel, t-window boundaries
    extra_v0, extra_v1, extra_v2, extra_o, extra_d, extra_tmin, extra_tmax = (
        [], [], [], [], [], [], [])
    tri = (np.array([0.0, 0, 0]), np.array([1.0, 0, 0]), np.array([0.0, 1, 0]))
    for p, dd, tmin, tmax in [
            ((0.0, 0.0, 1.0), (0, 0, -1.0), 0.0, np.inf),     # vertex
            ((1.0, 0.0, 1.0), (0, 0, -1.0), 0.0, np.inf),     # vertex
            ((0.5, 0.5, 1.0), (0, 0, -1.0), 0.0, np.inf),     # hypotenuse
            ((0.5, 0.0, 1.0), (0, 0, -1.0), 0.0, np.inf),     # edge
            ((0.2, 0.2, 1.0), (1.0, 0, 0.0), 0.0, np.inf),    # parallel
            ((0.2, 0.2, 1.0), (0, 0, -1.0), 1.0, np.inf),     # t == t_min
            ((0.2, 0.2, 1.0), (0, 0, -1.0), 0.0, 1.0),        # t == t_max
            ((0.2, 0.2, 1.0), (0, 0, -1.0), 0.0, 0.999),      # beyond t_max
            ((0.2, 0.2, -1.0), (0, 0, 1.0), 0.0, np.inf),     # back face
            ((0.5000000001, 0.5, 1.0), (0, 0, -1.0), 0.0, np.inf)]:
        extra_v0.append(tri[0]); extra_v1.append(tri[1]); extra_v2.append(tri[2])
        extra_o.append(p); extra_d.append(dd); extra_tmin.append(tmin)
        extra_tmax.append(tmax)
    t = np.empty(n)
    for r in range(n):
        res = sbr.ray_triangle_intersect(o[r], d[r], sbr.Triangle(v0[r], v1[r], v2[r], None))
        t[r] = -1.0 if res is None else res[0]
    te = np.empty(len(extra_o))
    for r in range(len(extra_o)):
        res = sbr.ray_triangle_intersect(extra_o[r], extra_d[r],
                                         sbr.Triangle(extra_v0[r], extra_v1[r], extra_v2[r], None),
                                         extra_tmin[r], extra_tmax[r])
        te[r] = -1.0 if res is None else res[0]
    save("mt", v0=v0, v1=v1, v2=v2, o=o, d=d, t=t,
         kat_v0=np.array(extra_v0), kat_v1=np.array(extra_v1),
         kat_v2=np.array(extra_v2), kat_o=np.array(extra_o, float),
         kat_d=np.array(extra_d, float), kat_tmin=np.array(extra_tmin),
         kat_tmax=np.array(extra_tmax), kat_t=te)
    print(f"    mt: {int((t > 0).sum())} hits / {n}")


def gen_bvh_and_closest():
    cases = {
        "single": sbr.mesh_from_arrays([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]]),
        "dihedral": dihedral_mesh(1.0),
        "ico2": sbr.generate_icosphere(1.0, 2),
        "ico3": sbr.generate_icosphere(1.0, 3),
        "rough20": perturbed_grid_mesh(cells=20),
        "ico3f32": sbr.generate_icosphere(1.0, 3, dtype=np.float32),
    }
    for name, mesh in cases.items():
        arrays = mesh_arrays(mesh)
        for rule in ("sah", "median"):
            tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
            tree.validate(mesh)
            arrays.update(bvh_arrays(tree, prefix=f"{rule}_"))
        seed = sum(map(ord, name))
        origins, dirs = random_probe_rays(mesh, 1000, seed=seed)
        tree = sbr.build(mesh)
        if mesh.dtype == np.float32:
            # the reference casts rays to the mesh dtype (bvh.py:413-414);
            # record the float64 trace-path convention instead (documented)
            origins = origins.astype(np.float32).astype(np.float64)
            dirs = dirs.astype(np.float32).astype(np.float64)
        tri, t, vis = sbr.closest_hit_batch(tree, mesh, origins, dirs)
        arrays.update(origins=origins, dirs=dirs, sah_tri=tri, sah_t=t,
                      sah_visits=vis)
        if mesh.dtype == np.float64:
            btri, bt = brute_force_hits(mesh, origins, dirs)
            assert np.array_equal(btri, tri)
            arrays.update(brute_tri=btri, brute_t=bt)
        tree_m = sbr.build(mesh, sbr.BuildParams(split_rule="median"))
        tri_m, t_m, vis_m = sbr.closest_hit_batch(tree_m, mesh, origins, dirs)
        arrays.update(median_tri=tri_m, median_t=t_m, median_visits=vis_m)
        save(f"bvh_{name}", **arrays)


TRACE_CASES = []


def trace_case(name, mesh, theta, phi, wavelength, spacing, max_bounces,
               margin=0.025, strict=False, epsilon=None, extra_k=()):
    TRACE_CASES.append((name, mesh, theta, phi, wavelength, spacing,
                        max_bounces, margin, strict, epsilon, extra_k))


def gen_trace():
    lam = 0.1
    trace_case("plate_c3", plate_mesh(1.0), 0.0, 0.0, lam, lam / 10, 3, margin=0.0)
    trace_case("dihedral_b2", dihedral_mesh(1.0), math.pi / 2, math.pi / 4,
               0.05, 0.01, 2)
    trace_case("dihedral_b3_phi30", dihedral_mesh(1.0), math.pi / 2,
               math.radians(30.0), 0.1, 0.02, 3)
    trace_case("dihedral_strict", dihedral_mesh(1.0), math.pi / 2,
               math.radians(200.0), 0.1, 0.02, 3, strict=True)
    trace_case("trihedral_b3", trihedral_mesh(1.0), math.radians(54.7356),
               math.pi / 4, 0.1, 0.02, 3)
    trace_case("trihedral_b3_off", trihedral_mesh(1.0), math.radians(40.0),
               math.radians(20.0), 0.1, 0.02, 3)
    ka = 20.0
    lam_c1 = 2 * math.pi / ka
    trace_case("sphere_c1", quantized_icosphere(5), math.pi / 2, 0.0, lam_c1,
               lam_c1 / 5, 4, extra_k=(lam_c1 * 0.97, lam_c1 * 1.03))
    trace_case("ico3_b10", sbr.generate_icosphere(1.0, 3), 0.4, 2.0, 0.25,
               0.05, 10)
    trace_case("rough40_b5", perturbed_grid_mesh(cells=40, extent=2.0,
                                                 amplitude=0.08, seed=42),
               0.35, 0.8, 0.1, 0.02, 5)
    trace_case("ico3f32_b4", sbr.generate_icosphere(1.0, 3, dtype=np.float32),
               1.1, 0.7, 0.25, 0.05, 4)
    trace_case("plate_eps", plate_mesh(1.0), 0.0, 0.0, 0.55, 0.11, 3,
               margin=0.0, epsilon=1e-4)

    for (name, mesh, theta, phi, lam, spacing, B, margin, strict, eps,
         extra_k) in TRACE_CASES:
        tree = sbr.build(mesh)
        d = sbr.IncidentDirection(theta, phi)
        grid = sbr.build_aperture(mesh.aabb, d, spacing, margin=margin,
                                  wavelength=lam)
        params = sbr.TraceParams(max_bounces=B, strict_orientation=strict,
                                 epsilon=eps)
        rec = sbr.trace_grid(tree, mesh, grid, params)
        ids = trace_with_ids(tree, mesh, grid, params)
        for k in ("valid", "normal0", "path", "bounces", "escaped", "out_dir"):
            assert np.array_equal(getattr(rec, k), ids[k]), (name, k)
        sp = sbr.ScatterParams.from_wavelength(lam, grid.cell_area)
        amp = sbr.accumulate(rec, d.k_inc, sp)
        amp_t = sbr.accumulate(rec, d.k_inc, sp, count_trapped=True)
        lams = [lam] + list(extra_k)
        amps_k = [sbr.accumulate(rec, d.k_inc,
                                 sbr.ScatterParams.from_wavelength(L, grid.cell_area))
                  for L in lams]
        sol = solve_direction(tree, mesh, d, spacing, lam, margin=margin,
                              trace_params=params)
        assert sol.amplitude == amp
        arrays = mesh_arrays(mesh)
        arrays.update(grid_arrays(grid))
        arrays.update(
            theta=np.float64(theta), phi=np.float64(phi),
            wavelength=np.float64(lam), max_bounces=np.int64(B),
            strict=np.bool_(strict), epsilon=np.float64(params.resolve_epsilon(mesh)),
            epsilon_given=np.bool_(eps is not None),
            single=np.bool_(mesh.dtype == np.float32),
            valid=rec.valid, normal0=rec.normal0, path=rec.path,
            bounces=rec.bounces, escaped=rec.escaped, out_dir=rec.out_dir,
            tri_ids=ids["tri_ids"],
            amplitude=np.complex128(amp), amplitude_trapped=np.complex128(amp_t),
            wavelengths=np.array(lams), amplitudes_k=np.array(amps_k),
            sigma_m2=np.float64(sol.rcs.sigma_m2),
            sigma_dbsm=np.float64(sol.rcs.sigma_dbsm),
            valid_rays=np.int64(sol.valid_rays), max_bounce=np.int64(sol.max_bounce),
            bounce_counts=sol.bounce_counts)
        save(f"trace_{name}", **arrays)
        print(f"    {name}: {grid.n_u}x{grid.n_v} rays, valid={sol.valid_rays},"
              f" hist={sol.bounce_counts.tolist()}, sigma={sol.rcs.sigma_m2:.6g}")


def gen_aperture():
    rng = np.random.default_rng(5)
    boxes = [((0.0, 0.0, 0.0), (1.0, 1.0, 0.0)),
             ((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)),
             ((0.0, 0.0, 0.0), (15.0, 13.0, 4.0)),
             ((-3.5, 2.0, 0.1), (7.25, 2.5, 9.0))]
    rows = []
    for bi, (lo, hi) in enumerate(boxes):
        aabb = sbr.Aabb(np.array(lo), np.array(hi))
        for _ in range(25):
            th = float(rng.uniform(0, math.pi)); ph = float(rng.uniform(0, 2 * math.pi))
            sp = float(rng.uniform(0.01, 0.3)); mg = float(rng.choice([0.0, 0.025, 0.1]))
            g = sbr.build_aperture(aabb, sbr.IncidentDirection(th, ph), sp, margin=mg)
            rows.append((bi, th, ph, sp, mg, g.n_u, g.n_v, *g.corner, *g.u, *g.v,
                         *g.k_inc, g.standoff))
        for th, ph in [(0.0, 0.0), (math.pi / 2, 0.0), (math.pi / 2, math.pi / 4),
                       (math.pi, 0.0), (math.pi / 2, math.pi / 2)]:
            g = sbr.build_aperture(aabb, sbr.IncidentDirection(th, ph), 0.05)
            rows.append((bi, th, ph, 0.05, 0.025, g.n_u, g.n_v, *g.corner, *g.u,
                         *g.v, *g.k_inc, g.standoff))
    save("aperture", boxes_lo=np.array([b[0] for b in boxes]),
         boxes_hi=np.array([b[1] for b in boxes]), rows=np.array(rows))


def gen_sweep():
    mesh = dihedral_mesh(1.0)
    cfg = sbr.SweepConfig(mesh_path="dihedral.obj", frequency_hz=3e9,
                          theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                          phi=sbr.AngleRange(0.0, math.pi / 2, 7),
                          max_bounces=3, workers=1)
    res = sbr.run_sweep(cfg, mesh)
    save("sweep_dihedral", theta=res.theta, phi=res.phi, amplitude=res.amplitude,
         sigma_m2=res.sigma_m2, sigma_dbsm=res.sigma_dbsm,
         valid_rays=res.valid_rays, max_bounces_seen=res.max_bounces_seen,
         bounce_histogram=res.bounce_histogram, frequency_hz=np.float64(3e9),
         max_bounces=np.int64(3), mesh_checksum=np.array(res.mesh_checksum))
    rep = sbr.validate_sphere(1.0, [8.0, 12.0], subdivisions=3, n_directions=6,
                              max_bounces=4)
    save("validate_sphere_small", kr=np.array([r.kr for r in rep.rows]),
         sigma_sbr=np.array([r.sigma_sbr_m2 for r in rep.rows]),
         sigma_mie=np.array([r.sigma_mie_m2 for r in rep.rows]),
         rel_error=np.array([r.rel_error for r in rep.rows]),
         spacing=np.array([r.spacing_m for r in rep.rows]),
         fib=np.array([(d.theta, d.phi) for d in sbr.fibonacci_directions(16)]))


def gen_meshes_and_mie():
    hashes = {}
    for s in range(0, 7):
        m = sbr.generate_icosphere(1.0, s)
        h = hashlib.sha256()
        for a in (m.v0, m.v1, m.v2, m.normals):
            h.update(np.ascontiguousarray(a).tobytes())
        hashes[s] = h.hexdigest()
    m2 = sbr.generate_icosphere(2.5, 2)
    xs = np.array([0.1, 1.0, 5.0, 20.0, 30.0, 50.0, 100.0, 250.0, 1000.0])
    mie = np.array([sbr.mie_backscatter_pec(x, 1.0) for x in xs])
    rough = perturbed_grid_mesh(cells=71)
    save("meshes", ico_hash_levels=np.arange(7),
         ico_hashes=np.array([hashes[s] for s in range(7)]),
         ico2r25_v0=m2.v0, ico2r25_v1=m2.v1, ico2r25_v2=m2.v2,
         ico2r25_normals=m2.normals, mie_x=xs, mie_sigma=mie,
         rough71_checksum=np.array(rough.checksum()),
         dihedral_checksum=np.array(dihedral_mesh().checksum()))


def _edgeon_triangle(rng, center, d, size, tilt):
    """A triangle whose plane contains direction d up to a relative tilt
    |n.d| ~ tilt (near-edge-on for rays along d)."""
    d = d / np.linalg.norm(d)
    a = rng.normal(size=3)
    e = a - (a @ d) * d
    e /= np.linalg.norm(e)
    m = np.cross(d, e)                      # normal of the exactly edge-on plane
    p0 = center + size * (rng.uniform(-0.5, 0.5) * d + rng.uniform(-0.5, 0.5) * e)
    p1 = center + size * (rng.uniform(-0.5, 0.5) * d + rng.uniform(-0.5, 0.5) * e)
    p2 = center + size * (rng.uniform(-0.5, 0.5) * d + rng.uniform(-0.5, 0.5) * e)
    p2 = p2 + tilt * size * m
    return np.array([p0, p1, p2]), e, m


def gen_edgeon():
    """Near-edge-on fixtures (|n.d| <= 1e-13): the class where Moller-Trumbore
    accepts rays far outside the triangle and the reference's own answer
    depends on its tree (bvh.py:329-342).  Recorded: the reference's
    closest hits on its SAH and median trees, the linear scan
    (tests/meshes.py brute_force_hits), and trace_grid records + ids on an
    aperture whose grid columns lie in edge-on planes."""
    rng = np.random.default_rng(20261017)
    # ---- (a) random triangles x rays lying in their planes (closest hit) ----
    # origins ON the triangle's plane (affine combinations of its vertices,
    # mostly outside it), directions in the plane tilted by |n.d| in
    # [1e-16, 1e-13]: det is then rounding-dominated and u, v, t are noise
    tris, origins, dirs = [], [], []
    for k in range(300):
        center = rng.uniform(-3.0, 3.0, 3)
        size = float(10 ** rng.uniform(-2, 0))
        tri = center + size * rng.normal(size=(3, 3))
        tris.append(tri)
        e1, e2 = tri[1] - tri[0], tri[2] - tri[0]
        nrm = np.cross(e1, e2)
        nrm /= np.linalg.norm(nrm)
        for _ in range(67):
            # far (up to 48 edge lengths), mid and close to the triangle
            al, be = rng.uniform(-6.0, 6.0, 2) * (8.0, 1.0, 0.25)[_ % 3] + (0, 0, 0.3)[_ % 3]
            o = tri[0] + al * e1 + be * e2
            g1, g2 = rng.normal(size=2)
            dd = g1 * e1 + g2 * e2
            dd /= np.linalg.norm(dd)
            dd = dd + float(10 ** rng.uniform(-16, -13)) * rng.choice([-1, 1]) * nrm
            origins.append(o)
            dirs.append(dd / np.linalg.norm(dd))
    mesh = sbr.mesh_from_soup(np.array(tris))
    origins = np.array(origins)
    dirs = np.array(dirs)
    arrays = mesh_arrays(mesh)
    arrays.update(origins=origins, dirs=dirs)
    for rule in ("sah", "median"):
        tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
        arrays.update(bvh_arrays(tree, prefix=f"{rule}_"))
        tri, t, vis = sbr.closest_hit_batch(tree, mesh, origins, dirs)
        arrays.update({f"{rule}_tri": tri, f"{rule}_t": t, f"{rule}_visits": vis})
    btri, bt = brute_force_hits(mesh, origins, dirs)
    arrays.update(brute_tri=btri, brute_t=bt)
    save("edgeon_rays", **arrays)
    print(f"    edgeon_rays: {len(origins)} rays, hits sah={int((arrays['sah_tri'] >= 0).sum())}"
          f" median={int((arrays['median_tri'] >= 0).sum())} brute={int((btri >= 0).sum())};"
          f" sah!=brute {int((arrays['sah_tri'] != btri).sum())},"
          f" median!=brute {int((arrays['median_tri'] != btri).sum())}")

    # ---- (b) aperture whose columns lie in edge-on planes (trace_grid) -----
    th, ph, lam = 1.1, 0.7, 0.1
    spacing = lam / 5
    din = sbr.IncidentDirection(th, ph)
    k = np.asarray(din.k_inc, np.float64)
    anchors = [np.array([[-2.0, -2, -2], [-1.99, -2, -2], [-2, -1.99, -2]]),
               np.array([[2.0, 2, 2], [1.99, 2, 2], [2, 1.99, 2]])]
    box = sbr.mesh_from_soup(np.array(anchors))
    grid = sbr.build_aperture(box.aabb, din, spacing, wavelength=lam)
    u = np.asarray(grid.u); v = np.asarray(grid.v); corner = np.asarray(grid.corner)

    def origin(i, j):
        bx = corner + ((i + 0.5) * spacing) * u
        return bx + ((j + 0.5) * spacing) * v

    tris = list(anchors)
    # a backstop plate across the beam (real hits behind the edge-on set)
    c, hu, hv = 0.8 * k, 0.7 * u, 0.7 * v
    tris += [np.array([c - hu - hv, c + hu - hv, c + hu + hv]),
             np.array([c - hu - hv, c + hu + hv, c - hu + hv])]
    # a few ordinary triangles in front, for multi-bounce paths
    for _ in range(12):
        cc = rng.uniform(-1.0, 1.0, 3) - 0.8 * k
        a, b = rng.normal(size=3), rng.normal(size=3)
        tris.append(np.array([cc, cc + 0.3 * a / np.linalg.norm(a), cc + 0.3 * b / np.linalg.norm(b)]))
    n_edge = 0
    while n_edge < 48:
        i = int(rng.integers(grid.n_u * 3 // 10, grid.n_u * 7 // 10))
        j = int(rng.integers(grid.n_v * 3 // 10, grid.n_v * 7 // 10))
        o = origin(i, j)
        # a plane holding every ray of row i (directions k and v) or of
        # column j (directions k and u)
        w = v if n_edge % 2 else u
        size = float(10 ** rng.uniform(-1.3, -0.5))
        tilt = float(10 ** rng.uniform(-16, -13)) if n_edge % 4 >= 2 else 0.0
        center = o + (grid.standoff + float(rng.uniform(-1.0, 1.0))) * k
        p = [center + size * (rng.uniform(-0.5, 0.5) * k + rng.uniform(-0.5, 0.5) * w)
             for _ in range(3)]
        p[2] = p[2] + tilt * size * np.cross(k, w)
        p = np.array(p)
        if np.abs(p).max() > 1.95:
            continue
        tris.append(p)
        n_edge += 1
    mesh = sbr.mesh_from_soup(np.array(tris))
    assert np.allclose(mesh.aabb.min, box.aabb.min) and np.allclose(mesh.aabb.max, box.aabb.max)
    grid = sbr.build_aperture(mesh.aabb, din, spacing, wavelength=lam)
    tree = sbr.build(mesh)
    params = sbr.TraceParams(max_bounces=3)
    rec = sbr.trace_grid(tree, mesh, grid, params)
    ids = trace_with_ids(tree, mesh, grid, params)
    for key in ("valid", "normal0", "path", "bounces", "escaped", "out_dir"):
        assert np.array_equal(getattr(rec, key), ids[key]), key
    n = grid.ray_count
    ii, jj = np.divmod(np.arange(n), grid.n_v)
    o_all = (corner + ((ii + 0.5) * spacing)[:, None] * u) + ((jj + 0.5) * spacing)[:, None] * v
    btri, bt = brute_force_hits(mesh, o_all, np.tile(k, (n, 1)))
    arrays = mesh_arrays(mesh)
    arrays.update(grid_arrays(grid))
    arrays.update(theta=np.float64(th), phi=np.float64(ph), wavelength=np.float64(lam),
                  max_bounces=np.int64(3), strict=np.bool_(False),
                  epsilon=np.float64(params.resolve_epsilon(mesh)),
                  valid=rec.valid, normal0=rec.normal0, path=rec.path, bounces=rec.bounces,
                  escaped=rec.escaped, out_dir=rec.out_dir, tri_ids=ids["tri_ids"],
                  prim_brute_tri=btri, prim_brute_t=bt)
    arrays.update(bvh_arrays(tree, prefix="sah_"))
    save("edgeon_grid", **arrays)
    first = ids["tri_ids"][:, 0].astype(np.int64)
    print(f"    edgeon_grid: {grid.n_u}x{grid.n_v} rays, query-0 ref!=linear scan:"
          f" {int((first != btri).sum())}")


def main():
    print(f"reference sbr {sbr.__version__} numba {numba.__version__} "
          f"numpy {np.__version__} python {platform.python_version()}")
    gen_mt()
    gen_bvh_and_closest()
    gen_trace()
    gen_aperture()
    gen_sweep()
    gen_meshes_and_mie()
    gen_edgeon()
    with open(os.path.join(OUT, "VERSIONS.json"), "w") as fh:
        json.dump({"sbr": sbr.__version__, "numba": numba.__version__,
                   "numpy": np.__version__, "python": platform.python_version(),
                   "PYTHONHASHSEED": os.environ.get("PYTHONHASHSEED")}, fh,
                  indent=1)


if __name__ == "__main__":
    if len(sys.argv) > 1:   # e.g. make_golden.py gen_edgeon
        for fn in sys.argv[1:]:
            globals()[fn]()
    else:
        main()

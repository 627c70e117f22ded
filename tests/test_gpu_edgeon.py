"""Near-edge-on / tie rays: the class where the reference's own answer depends
on its tree (bvh.py:329-342), and the reference-order traversal mode.

* ``traversal_order("reference")`` replays bvh.py:306-362 on the reference
  tree: bit-identical to the reference on EVERY ray, visit counts included.
* The fast path (raster + BVH4 kernel) is bit-identical on every ROBUST ray
  (oracle classifier); on the others it returns an accepting
  triangle (a valid closest hit of some conservative traversal).
* The raster pass answers query 0 with the linear scan on EVERY ray, the
  reference's documented semantics (bvh.py:394-395), edge-on rays included.
"""

import math

import numpy as np
import pytest

import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

REC = ("valid", "normal0", "path", "bounces", "escaped", "out_dir", "tri_ids")


def _mesh(g):
    v0, v1, v2 = g["mesh_v0"], g["mesh_v1"], g["mesh_v2"]
    pts = np.concatenate([v0, v1, v2]).astype(np.float64)
    return sbr.Mesh(v0=v0, v1=v1, v2=v2, normals=g["mesh_normals"],
                    aabb=sbr.Aabb(pts.min(0), pts.max(0)))


def _grid(g):
    return sbr.ApertureGrid(u=g["grid_u"], v=g["grid_v"], k_inc=g["grid_k"],
                            corner=g["grid_corner"], spacing=float(g["grid_spacing"]),
                            n_u=int(g["grid_n_u"]), n_v=int(g["grid_n_v"]),
                            cell_area=float(g["grid_cell_area"]),
                            standoff=float(g["grid_standoff"]), margin=float(g["grid_margin"]))


def _uploaded(g, rule):
    return sbr.Bvh(g[f"{rule}_nodes_min"], g[f"{rule}_nodes_max"], g[f"{rule}_node_first"],
                   g[f"{rule}_node_count"], g[f"{rule}_tri_order"],
                   int(g[f"{rule}_max_depth_seen"]))


@pytest.fixture
def reference_order():
    with sbr.traversal_order("reference"):
        yield


def _oracle_scene(orc, g):
    tree = orc.build(g["mesh_v0"], g["mesh_v1"], g["mesh_v2"])
    return orc.Scene(g["mesh_v0"], g["mesh_v1"], g["mesh_v2"], g["mesh_normals"], tree)


# ---------------------------------------------------------------------------
# reference-order mode: bit for bit on every ray
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("rule", ["sah", "median"])
def test_reference_order_closest_hit_edgeon(rule, reference_order):
    g = load_golden("edgeon_rays")
    mesh = _mesh(g)
    for tree in (sbr.build(mesh, sbr.BuildParams(split_rule=rule)), _uploaded(g, rule)):
        tri, t, vis = sbr.closest_hit_batch(tree, mesh, g["origins"], g["dirs"])
        assert np.array_equal(tri, g[f"{rule}_tri"])
        assert np.array_equal(t, g[f"{rule}_t"])
        assert np.array_equal(vis, g[f"{rule}_visits"])   # the reference's own visit count


def test_reference_order_trace_grid_edgeon(reference_order):
    g = load_golden("edgeon_grid")
    mesh = _mesh(g)
    tree = sbr.build(mesh)
    rec = sbr.trace_grid(tree, mesh, _grid(g), sbr.TraceParams(max_bounces=3), with_ids=True)
    for k in REC:
        assert np.array_equal(getattr(rec, k), g[k]), k


@pytest.mark.parametrize("name", golden_names("bvh_"))
def test_reference_order_closest_hit_goldens(name, reference_order):
    g = load_golden(name)
    mesh = _mesh(g)
    for rule in ("sah", "median"):
        tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
        tri, t, vis = sbr.closest_hit_batch(tree, mesh, g["origins"], g["dirs"])
        assert np.array_equal(tri, g[f"{rule}_tri"]), rule
        assert np.array_equal(t, g[f"{rule}_t"]), rule
        assert np.array_equal(vis, g[f"{rule}_visits"]), rule


@pytest.mark.parametrize("name", golden_names("trace_"))
def test_reference_order_trace_goldens(name, reference_order):
    g = load_golden(name)
    mesh = _mesh(g)
    tree = sbr.build(mesh)
    params = sbr.TraceParams(max_bounces=int(g["max_bounces"]), epsilon=float(g["epsilon"]),
                             strict_orientation=bool(g["strict"]))
    rec = sbr.trace_grid(tree, mesh, _grid(g), params, with_ids=True)
    for k in REC:
        assert np.array_equal(getattr(rec, k), g[k]), (name, k)


def test_reference_order_solve_equals_fast_on_robust_workload():
    """The fused solve in reference order gives the fast path's bits on an
    ordinary multi-bounce aircraft sweep (no tree-dependent rays there)."""
    mesh = meshgen.generate_aircraft(density=0.03)
    tree = sbr.build(mesh)
    lam = 0.1
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(th, ph), lam / 5,
                                wavelength=lam)
             for th, ph in [(math.pi / 2, 0.0), (math.pi / 2, 2.0), (1.1, 4.0)]]
    tp = sbr.TraceParams(max_bounces=5)
    fast = sbr.solve_grids(tree, mesh, grids, tp, [2 * math.pi / lam])
    with sbr.traversal_order("reference"):
        ref = sbr.solve_grids(tree, mesh, grids, tp, [2 * math.pi / lam])
    assert np.array_equal(fast.amplitude, ref.amplitude)
    assert np.array_equal(fast.bounce_counts, ref.bounce_counts)
    assert np.array_equal(fast.queries, ref.queries)


def test_reference_order_needs_reference_tree():
    mesh = meshgen.plate_mesh()
    tree = sbr.build(mesh, sbr.BuildParams(split_rule="lbvh"))
    with sbr.traversal_order("reference"):
        with pytest.raises(sbr.ValidationError, match="reference tree"):
            sbr.closest_hit_batch(tree, mesh, [[0.5, 0.5, 1.0]], [[0, 0, -1.0]])
    assert sbr.get_traversal_order() == "fast"


# ---------------------------------------------------------------------------
# fast path: bit-exact on robust rays, a valid accepting answer elsewhere
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("rule", ["sah", "median", "lbvh"])
def test_fast_closest_hit_edgeon(orc, rule):
    g = load_golden("edgeon_rays")
    mesh = _mesh(g)
    tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
    tri, t, _ = sbr.closest_hit_batch(tree, mesh, g["origins"], g["dirs"])
    rob = orc.classify_rays(_oracle_scene(orc, g), g["origins"], g["dirs"])
    ref = g["brute_tri"]
    assert np.array_equal(tri[rob], ref[rob])
    assert np.array_equal(t[rob & (ref >= 0)], g["brute_t"][rob & (ref >= 0)])
    # elsewhere: a hit of an accepting triangle at exactly its MT distance
    for r in np.flatnonzero(~rob & (tri >= 0)):
        k = int(tri[r])
        tt = orc.tri_hit_pairs(g["mesh_v0"][k:k + 1], g["mesh_v1"][k:k + 1],
                               g["mesh_v2"][k:k + 1], g["origins"][r:r + 1],
                               g["dirs"][r:r + 1])
        assert tt[0] == t[r]


@pytest.mark.parametrize("primary", ["raster", "bvh"])
def test_fast_trace_grid_edgeon(orc, monkeypatch, primary):
    monkeypatch.setenv("SBR_PRIMARY", primary)
    g = load_golden("edgeon_grid")
    mesh = _mesh(g)
    tree = sbr.build(mesh)
    grid = _grid(g)
    rec = sbr.trace_grid(tree, mesh, grid, sbr.TraceParams(max_bounces=3), with_ids=True)
    rob, _, _ = orc.classify_grid(_oracle_scene(orc, g), grid, 3, float(g["epsilon"]))
    assert rob.sum() > 0.99 * rob.size
    for k in REC:
        assert np.array_equal(getattr(rec, k)[rob], g[k][rob]), k


def test_raster_query0_is_the_linear_scan_on_every_ray(monkeypatch):
    """Query 0 from the raster pass == the reference's linear scan
    (tests/meshes.py brute_force_hits) on EVERY ray of the edge-on aperture,
    including the rays whose Moller-Trumbore acceptance lies far outside the
    triangle (where the reference's BVH itself disagrees with its scan)."""
    monkeypatch.setenv("SBR_PRIMARY", "raster")
    g = load_golden("edgeon_grid")
    mesh = _mesh(g)
    tree = sbr.build(mesh)
    rec = sbr.trace_grid(tree, mesh, _grid(g), sbr.TraceParams(max_bounces=1), with_ids=True)
    bt = g["prim_brute_tri"]
    assert np.array_equal(rec.tri_ids[:, 0].astype(np.int64), bt)
    hit = bt >= 0
    assert np.array_equal(rec.path[hit], g["prim_brute_t"][hit])
    assert (g["tri_ids"][:, 0] != bt).sum() >= 10   # the reference's BVH differs there


def test_raster_big_queue_overflow(monkeypatch):
    """A chunk queue far too small for the big triangles (SBR_BIG_CAP) must
    not change a bit: overflowing reservations publish no work and the
    triangles are walked inline (stale entries were read)."""
    mesh = meshgen.quantized_icosphere(1.0, 3)
    tree = sbr.build(mesh)
    lam = 2 * math.pi / 600
    grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(1.0, 0.4), lam / 5,
                              wavelength=lam)
    tp = sbr.TraceParams(max_bounces=2)
    monkeypatch.setenv("SBR_PRIMARY", "raster")
    a = sbr.trace_grid(tree, mesh, grid, tp, with_ids=True)
    for cap in ("1", "7", "300"):
        monkeypatch.setenv("SBR_BIG_CAP", cap)
        b = sbr.trace_grid(tree, mesh, grid, tp, with_ids=True)
        for k in REC:
            assert np.array_equal(getattr(a, k), getattr(b, k)), (cap, k)
    monkeypatch.setenv("SBR_PRIMARY", "bvh")
    monkeypatch.delenv("SBR_BIG_CAP")
    c = sbr.trace_grid(tree, mesh, grid, tp, with_ids=True)
    for k in REC:
        assert np.array_equal(getattr(a, k), getattr(c, k)), k


def test_raster_candidates_are_tight():
    """The proven candidate region is no looser than the old projected
    bounding box + 0.01 cell (computed here on the host): a bound that
    silently widened to whole aperture rows once cost 1000x in time while
    every result stayed correct."""
    from paper_2604_09243_b200 import _native as nat
    mesh = meshgen.generate_aircraft(density=0.05)
    tree = sbr.build(mesh)
    lam = 0.1
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(th, ph), lam / 5,
                                wavelength=lam)
             for th, ph in [(math.pi / 2, 0.0), (math.pi / 2, 0.7), (1.0, 2.0)]]
    ctx = nat.context()
    import os
    old = os.environ.get("SBR_PRIMARY")
    os.environ["SBR_PRIMARY"] = "raster"
    try:
        ctx.raster_counters()
        sbr.solve_grids(tree, mesh, grids, sbr.TraceParams(max_bounces=2), [2 * math.pi / lam])
        got = ctx.raster_counters()
    finally:
        if old is None:
            os.environ.pop("SBR_PRIMARY")
        else:
            os.environ["SBR_PRIMARY"] = old
    bound = 0
    v0, e1, e2 = mesh.v0, mesh.v1 - mesh.v0, mesh.v2 - mesh.v0
    for g in grids:
        u, v, c, sp = np.asarray(g.u), np.asarray(g.v), np.asarray(g.corner), g.spacing
        a0 = ((v0 - c) @ u) / sp - 0.5
        b0 = ((v0 - c) @ v) / sp - 0.5
        A = np.stack([a0, a0 + (e1 @ u) / sp, a0 + (e2 @ u) / sp])
        B = np.stack([b0, b0 + (e1 @ v) / sp, b0 + (e2 @ v) / sp])
        i0 = np.maximum(0, np.ceil(A.min(0) - 0.01)); i1 = np.minimum(g.n_u - 1, np.floor(A.max(0) + 0.01))
        j0 = np.maximum(0, np.ceil(B.min(0) - 0.01)); j1 = np.minimum(g.n_v - 1, np.floor(B.max(0) + 0.01))
        bound += int((np.clip(i1 - i0 + 1, 0, None) * np.clip(j1 - j0 + 1, 0, None)).sum())
    assert 0 < got["candidates"] <= bound, (got, bound)
    assert got["queue_overflows"] == 0


def _chain_tree(mesh):
    """A valid reference-layout tree that is a chain: node 2k is internal
    (left = leaf 2k+1 holding triangle k, right = node 2k+2), so its depth is
    ntri - 1 -- far past the fast kernels' BVH4 stack bound."""
    n = mesh.triangle_count
    lo = np.minimum(np.minimum(mesh.v0, mesh.v1), mesh.v2).astype(np.float64)
    hi = np.maximum(np.maximum(mesh.v0, mesh.v1), mesh.v2).astype(np.float64)
    suf_lo = np.minimum.accumulate(lo[::-1])[::-1]
    suf_hi = np.maximum.accumulate(hi[::-1])[::-1]
    m = 2 * n - 1
    nmin, nmax = np.zeros((m, 3)), np.zeros((m, 3))
    first, count = np.zeros(m, np.int32), np.zeros(m, np.int32)
    for k in range(n - 1):
        nmin[2 * k], nmax[2 * k], first[2 * k] = suf_lo[k], suf_hi[k], 2 * k + 2
        nmin[2 * k + 1], nmax[2 * k + 1] = lo[k], hi[k]
        first[2 * k + 1], count[2 * k + 1] = k, 1
    nmin[m - 1], nmax[m - 1], first[m - 1], count[m - 1] = lo[n - 1], hi[n - 1], n - 1, 1
    return nmin, nmax, first, count, np.arange(n, dtype=np.int32), n - 1


def test_deep_tree_is_traced_in_reference_order(orc):
    """BVH4 depth > 31 (a 127-deep chain): no EINVAL; every traversal of that
    tree replays bvh.py:306-362 on it (the reference's stack is max_depth+2,
    bvh.py:381-382), bit for bit against the oracle on the same tree."""
    mesh = meshgen.perturbed_grid_mesh(cells=8, extent=1.0, amplitude=0.05, seed=5)
    arrays = _chain_tree(mesh)
    tree = sbr.Bvh(*arrays)
    tree.validate(mesh)
    origins, dirs = meshgen_probe(mesh)
    tri, t, vis = sbr.closest_hit_batch(tree, mesh, origins, dirs)
    scene = orc.Scene(mesh.v0, mesh.v1, mesh.v2, mesh.normals,
                      orc.OracleBvh(*arrays[:5], arrays[5], 200))
    btri, bt = orc.brute_force_hits(scene, origins, dirs)
    assert np.array_equal(tri, btri)
    assert np.array_equal(t[tri >= 0], bt[tri >= 0])
    lam = 0.05
    grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(0.4, 0.9), lam / 5,
                              wavelength=lam)
    params = sbr.TraceParams(max_bounces=3)
    rec = sbr.trace_grid(tree, mesh, grid, params, with_ids=True)
    ref = orc.trace_grid(scene, grid, 3, params.resolve_epsilon(mesh), with_ids=True)
    for k in REC:
        assert np.array_equal(getattr(rec, k), getattr(ref, k)), k
    sol = sbr.solve_direction(tree, mesh, sbr.IncidentDirection(0.4, 0.9), lam / 5, lam,
                              trace_params=params)
    assert sol.valid_rays == int(ref.valid.sum())


def meshgen_probe(mesh, n=4000, seed=3):
    rng = np.random.default_rng(seed)
    c = 0.5 * (mesh.aabb.min + mesh.aabb.max)
    r = mesh.aabb.diagonal()
    g = rng.normal(size=(n, 3))
    g /= np.linalg.norm(g, axis=1)[:, None]
    o = c + 1.6 * r * g
    d = c + 0.4 * r * rng.uniform(-1, 1, size=(n, 3)) - o
    return o, d / np.linalg.norm(d, axis=1)[:, None]

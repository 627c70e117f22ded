"""CUDA path vs the reference: golden vectors (produced by the reference
itself) and the pinned CPU oracle on identical inputs.

Bars (BASELINE.json north_star):
  * closest-hit triangle ids, t, bounce counts, per-bounce triangle ids and
    every HitRecords field: bit-exact;
  * complex amplitude: 1e-4 relative field; RCS: 0.05 dB.
"""

import math
import os

import numpy as np
import pytest

import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

FIELD_RTOL = 1e-4
DB_TOL = 0.05


def _mesh(g):
    """The fixture's exact Mesh arrays (float32 meshes keep their float32
    normals, which were rounded from the FP64 construction)."""
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


@pytest.fixture(params=["raster", "bvh"])
def primary(request, monkeypatch):
    """Query 0 answered by the raster pass (default) or by BVH traversal."""
    monkeypatch.setenv("SBR_PRIMARY", request.param)
    return request.param


def _amp_close(a, ref):
    a, ref = complex(a), complex(ref)
    assert abs(a - ref) <= FIELD_RTOL * abs(ref) + 1e-300, (a, ref)
    if abs(ref) > 0:
        db = 20 * math.log10(abs(a) / abs(ref))
        assert abs(db) <= DB_TOL


# ---------------------------------------------------------------------------
def test_mt_pairs_bitwise():
    g = load_golden("mt")
    t = np.empty_like(g["t"])
    from paper_2604_09243_b200 import _native as nat
    ctx = nat.context()
    arrs = [nat.f64(g[k]) for k in ("v0", "v1", "v2", "o", "d")]
    nat.check(ctx.lib.sbr_tri_hit_pairs(ctx.handle, *[nat.ptr(a) for a in arrs], t.shape[0],
                                        0.0, np.inf, 0, nat.ptr(t)))
    assert np.array_equal(t, g["t"])
    for r in range(g["kat_t"].shape[0]):
        res = sbr.ray_triangle_intersect(g["kat_o"][r], g["kat_d"][r],
                                         sbr.Triangle(g["kat_v0"][r], g["kat_v1"][r],
                                                      g["kat_v2"][r], np.zeros(3)),
                                         g["kat_tmin"][r], g["kat_tmax"][r])
        got = -1.0 if res is None else res[0]
        assert got == g["kat_t"][r], r


def test_aabb_predicate():
    box = sbr.Aabb([0, 0, 0], [1, 1, 1])
    assert sbr.ray_aabb_intersect([0.5, 0.5, 2.0], [np.inf, np.inf, -1.0], box) == (True, 1.0)
    assert sbr.ray_aabb_intersect([1.5, 0.5, 2.0], [np.inf, np.inf, -1.0], box)[0] is False
    assert sbr.ray_aabb_intersect([0.5, 0.5, 0.5], [1.0, 1.0, 1.0], box) == (True, 0.0)


@pytest.mark.parametrize("name", golden_names("bvh_"))
def test_closest_hit_lbvh_matches_reference(name):
    g = load_golden(name)
    mesh = _mesh(g)
    tree = sbr.build(mesh)
    tree.validate(mesh)
    tri, t, vis = sbr.closest_hit_batch(tree, mesh, g["origins"], g["dirs"])
    assert np.array_equal(tri, g["sah_tri"])
    # float32 meshes too: the rays are cast to float32 as bvh.py:414-415 does
    assert np.array_equal(t, g["sah_t"])
    assert (vis >= 1).all()


@pytest.mark.parametrize("name", ["bvh_ico3", "bvh_rough20", "bvh_dihedral", "bvh_single"])
@pytest.mark.parametrize("rule", ["sah", "median"])
def test_closest_hit_uploaded_reference_tree(name, rule):
    g = load_golden(name)
    mesh = _mesh(g)
    tree = sbr.Bvh(g[f"{rule}_nodes_min"], g[f"{rule}_nodes_max"], g[f"{rule}_node_first"],
                   g[f"{rule}_node_count"], g[f"{rule}_tri_order"],
                   int(g[f"{rule}_max_depth_seen"]))
    tri, t, _ = sbr.closest_hit_batch(tree, mesh, g["origins"], g["dirs"])
    assert np.array_equal(tri, g[f"{rule}_tri"])
    assert np.array_equal(t, g[f"{rule}_t"])


def test_closest_hit_t_window_and_root_cull():
    mesh = sbr.generate_icosphere(1.0, 2)
    tree = sbr.build(mesh)
    hit = sbr.closest_hit(tree, mesh, (0, 0, 5.0), (0.0, 0.0, -1.0))
    assert hit.t == pytest.approx(4.0, abs=0.05)
    far = sbr.closest_hit(tree, mesh, (0, 0, 5.0), (0.0, 0.0, -1.0), t_min=hit.t + 1e-6)
    assert far is not None and far.t > 5.5
    miss, visits = sbr.closest_hit_counted(tree, mesh, (5, 5, 5.0), (0.0, 0.0, -1.0))
    assert miss is None and visits == 1


@pytest.mark.parametrize("name", golden_names("trace_"))
def test_trace_grid_bitwise_with_ids(name, primary):
    g = load_golden(name)
    mesh = _mesh(g)
    tree = sbr.build(mesh)
    params = sbr.TraceParams(max_bounces=int(g["max_bounces"]), epsilon=float(g["epsilon"]),
                             strict_orientation=bool(g["strict"]))
    rec = sbr.trace_grid(tree, mesh, _grid(g), params, with_ids=True)
    for k in ("valid", "normal0", "path", "bounces", "escaped", "out_dir", "tri_ids"):
        assert np.array_equal(getattr(rec, k), g[k]), k


@pytest.mark.parametrize("name", golden_names("trace_"))
def test_accumulate_matches_reference(name):
    g = load_golden(name)
    rec = sbr.HitRecords(g["valid"], g["normal0"], g["path"], g["bounces"], g["escaped"],
                         g["out_dir"])
    lam, area = float(g["wavelength"]), float(g["grid_cell_area"])
    _amp_close(sbr.accumulate(rec, g["grid_k"], sbr.ScatterParams.from_wavelength(lam, area)),
               g["amplitude"])
    _amp_close(sbr.accumulate(rec, g["grid_k"], sbr.ScatterParams.from_wavelength(lam, area),
                              count_trapped=True), g["amplitude_trapped"])
    ks = 2 * np.pi / g["wavelengths"]
    multi = sbr.accumulate_multi(rec, g["grid_k"], ks, area)
    for a, ref in zip(multi, g["amplitudes_k"]):
        _amp_close(a, ref)


@pytest.mark.parametrize("name", golden_names("trace_"))
def test_fused_solve_matches_reference(name, primary):
    g = load_golden(name)
    if g["epsilon_given"]:
        pytest.skip("fixture uses an explicit epsilon; covered by trace test")
    mesh = _mesh(g)
    tree = sbr.build(mesh)
    d = sbr.IncidentDirection(float(g["theta"]), float(g["phi"]))
    params = sbr.TraceParams(max_bounces=int(g["max_bounces"]),
                             strict_orientation=bool(g["strict"]))
    sol = sbr.solve_direction(tree, mesh, d, float(g["grid_spacing"]), float(g["wavelength"]),
                              margin=float(g["grid_margin"]), trace_params=params)
    assert sol.valid_rays == int(g["valid_rays"])
    assert sol.max_bounce == int(g["max_bounce"])
    assert np.array_equal(sol.bounce_counts, g["bounce_counts"])
    _amp_close(sol.amplitude, g["amplitude"])
    ref_db = float(g["sigma_dbsm"])
    if np.isfinite(ref_db):
        assert abs(sol.rcs.sigma_dbsm - ref_db) <= DB_TOL
    # keep_records path gives the same bits as the fused path
    sol2 = sbr.solve_direction(tree, mesh, d, float(g["grid_spacing"]), float(g["wavelength"]),
                               margin=float(g["grid_margin"]), trace_params=params,
                               keep_records=True)
    assert sol2.amplitude == sol.amplitude


def test_run_sweep_matches_reference():
    g = load_golden("sweep_dihedral")
    mesh = meshgen.dihedral_mesh(1.0)
    cfg = sbr.SweepConfig(mesh_path="dihedral.obj", frequency_hz=3e9,
                          theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                          phi=sbr.AngleRange(0.0, math.pi / 2, 7), max_bounces=3)
    res = sbr.run_sweep(cfg, mesh)
    assert np.array_equal(res.valid_rays, g["valid_rays"])
    assert np.array_equal(res.max_bounces_seen, g["max_bounces_seen"])
    assert np.array_equal(res.bounce_histogram, g["bounce_histogram"])
    for a, ref in zip(res.amplitude.ravel(), g["amplitude"].ravel()):
        _amp_close(a, ref)
    assert res.mesh_checksum == str(g["mesh_checksum"])
    # per-cell time_ms (sweep.py:330-341): fused = the solve time split by
    # each cell's device queries; per_cell_timing = one timed call per cell
    assert np.all(res.time_ms > 0) and res.time_ms.shape == res.amplitude.shape
    q = res.queries.astype(float)
    assert np.allclose(res.time_ms / res.time_ms.sum(), q / q.sum())
    cell = sbr.run_sweep(cfg, mesh, per_cell_timing=True)
    assert np.array_equal(cell.amplitude, res.amplitude)
    assert np.array_equal(cell.valid_rays, res.valid_rays)
    assert np.all(cell.time_ms > 0)
    assert not np.allclose(cell.time_ms / cell.time_ms.sum(), q / q.sum(), rtol=1e-9)


def test_validate_sphere_matches_reference():
    g = load_golden("validate_sphere_small")
    rep = sbr.validate_sphere(1.0, [8.0, 12.0], subdivisions=3, n_directions=6, max_bounces=4)
    for row, s, m in zip(rep.rows, g["sigma_sbr"], g["sigma_mie"]):
        assert row.sigma_sbr_m2 == pytest.approx(float(s), rel=2e-4)   # 1e-4 field
        assert row.sigma_mie_m2 == pytest.approx(float(m), rel=1e-12)


# ---------------------------------------------------------------------------
# larger inputs against the pinned CPU oracle (same mesh, same grid)
# ---------------------------------------------------------------------------
def _oracle_scene(orc, mesh):
    return orc.Scene.from_mesh(mesh, single=mesh.dtype == np.float32)


@pytest.mark.parametrize("case", ["aircraft", "sphere_s6", "rough_b5"])
def test_trace_vs_oracle_larger(orc, case, primary):
    if case == "aircraft":
        mesh = meshgen.generate_aircraft(density=0.05)
        lam, B, dirs = 0.12, 5, [(math.pi / 2, math.pi), (math.pi / 2, 0.3), (1.2, 2.0)]
    elif case == "sphere_s6":
        mesh = meshgen.quantized_icosphere(1.0, 6)
        lam, B, dirs = 2 * math.pi / 100, 1, [(math.pi / 2, 0.0), (math.pi / 2, 1.0)]
    else:
        mesh = meshgen.perturbed_grid_mesh(cells=120, extent=4.0, amplitude=0.08, seed=3)
        lam, B, dirs = 0.1, 5, [(0.3, 0.7)]
    tree = sbr.build(mesh)
    scene = _oracle_scene(orc, mesh)
    params = sbr.TraceParams(max_bounces=B)
    for th, ph in dirs:
        grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(th, ph), lam / 5,
                                  wavelength=lam)
        rows = (0, min(grid.n_u, max(1, 60000 // grid.n_v)))
        ref = orc.trace_grid(scene, grid, B, params.resolve_epsilon(mesh), rows=rows,
                             with_ids=True)
        rec = sbr.trace_grid(tree, mesh, grid, params, with_ids=True)
        n = ref.valid.shape[0]
        for k in ("valid", "normal0", "path", "bounces", "escaped", "out_dir", "tri_ids"):
            assert np.array_equal(getattr(rec, k)[:n], getattr(ref, k)), (case, k)
        full = orc.trace_grid(scene, grid, B, params.resolve_epsilon(mesh))
        a_ref = orc.accumulate(full, grid.k_inc, lam, grid.cell_area)
        sol = sbr.solve_direction(tree, mesh, sbr.IncidentDirection(th, ph), lam / 5, lam,
                                  trace_params=params)
        _amp_close(sol.amplitude, a_ref)
        assert sol.valid_rays == int(full.valid.sum())


def test_solve_is_deterministic_and_batch_invariant(monkeypatch, primary):
    mesh = meshgen.quantized_icosphere(1.0, 5)
    tree = sbr.build(mesh)
    lam = 2 * math.pi / 60
    grids = [sbr.build_aperture(mesh.aabb, d, lam / 5, wavelength=lam)
             for d in sbr.fibonacci_directions(5)]
    tp = sbr.TraceParams(max_bounces=4)
    ks = 2 * np.pi / (lam * np.linspace(0.95, 1.05, 11))
    a = sbr.solve_grids(tree, mesh, grids, tp, ks)
    b = sbr.solve_grids(tree, mesh, grids, tp, ks)
    assert np.array_equal(a.amplitude, b.amplitude)
    monkeypatch.setenv("SBR_SLOT_BUDGET", "6144")
    c = sbr.solve_grids(tree, mesh, grids, tp, ks)
    assert np.array_equal(a.amplitude, c.amplitude)
    assert np.array_equal(a.bounce_counts, c.bounce_counts)
    # each grid alone == its row of the batch
    for i, g in enumerate(grids):
        s = sbr.solve_grids(tree, mesh, [g], tp, ks)
        assert np.array_equal(s.amplitude[0], a.amplitude[i])


def test_sharded_solve_equals_single(orc, primary):
    """Simulated N-rank run on one GPU: summing the disjoint shard buffers
    and finalising reproduces sbr_solve bit for bit (both shard modes)."""
    import ctypes
    import torch
    from paper_2604_09243_b200 import _native as nat, distributed as D
    from paper_2604_09243_b200.sweep import grid_array
    mesh = meshgen.quantized_icosphere(1.0, 4)
    tree = sbr.build(mesh)
    lam = 2 * math.pi / 450   # big grids -> several segments per grid
    grids = [sbr.build_aperture(mesh.aabb, d, lam / 5, wavelength=lam)
             for d in sbr.fibonacci_directions(3)]
    tp = sbr.TraceParams(max_bounces=2)
    ks = np.array([2 * np.pi / lam, 2 * np.pi / (0.9 * lam)])
    ref = sbr.solve_grids(tree, mesh, grids, tp, ks)
    ctx = nat.context()
    d = tree.device(mesh, ctx)
    base = D.segment_layout(grids)
    assert base[-1] > len(grids)
    garr = grid_array(grids)
    cp = nat.make_trace_params(2, tp.resolve_epsilon(mesh))
    for mode in ("angles", "rays"):
        for world in (2, 3):
            tot_seg = torch.zeros(int(base[-1]) * 4, dtype=torch.float64, device="cuda")
            tot_diag = torch.zeros((len(grids), D.diag_stride(2)), dtype=torch.int64,
                                   device="cuda")
            maxb = torch.zeros(len(grids), dtype=torch.int64, device="cuda")
            for rank in range(world):
                seg = torch.zeros_like(tot_seg)
                diag = torch.zeros_like(tot_diag)
                nat.check(ctx.lib.sbr_solve_shard(ctx.handle, d.mesh_dev.handle, d.handle, garr,
                                                  len(grids), ctypes.byref(cp), nat.ptr(ks), 2,
                                                  -1.0, 0, rank, world, D.MODES[mode],
                                                  nat.c_vp(seg.data_ptr()),
                                                  nat.c_vp(diag.data_ptr())))
                ctx.synchronize()
                tot_seg += seg
                tot_diag += diag
                maxb = torch.maximum(maxb, diag[:, 2])
            tot_diag[:, 2] = maxb
            amp = np.zeros((len(grids), 2, 2))
            vr = np.zeros(len(grids), np.int64)
            dg = nat.Diag(vr.ctypes.data, None, None, None)
            nat.check(ctx.lib.sbr_finalize(ctx.handle, garr, len(grids), nat.ptr(ks), 2, 2,
                                           nat.c_vp(tot_seg.data_ptr()),
                                           nat.c_vp(tot_diag.data_ptr()), nat.ptr(amp),
                                           ctypes.byref(dg)))
            assert np.array_equal(amp.view(np.complex128)[..., 0], ref.amplitude), (mode, world)
            assert np.array_equal(vr, ref.valid_rays)


def test_mie_sphere_direction_averaged():
    """SBR-PO sphere vs Mie with the reference's direction averaging
    (test_acceptance.py:38-49 style)."""
    rep = sbr.validate_sphere(1.0, [20.0, 30.0], sampling_factor=5.0, subdivisions=5,
                              n_directions=16)
    for row in rep.rows:
        assert row.rel_error <= 0.08, row
    assert rep.mean_rel_error() <= 0.06


def test_plate_closed_form():
    side, lam = 1.0, 0.1
    mesh = meshgen.plate_mesh(side)
    tree = sbr.build(mesh)
    d = sbr.IncidentDirection(0.0, 0.0)
    sol = sbr.solve_direction(tree, mesh, d, lam / 10, lam, margin=0.0,
                              trace_params=sbr.TraceParams(max_bounces=3))
    ref = sbr.plate_reference(side, lam)
    assert abs(sol.rcs.sigma_m2 - ref) / ref <= 0.01


def test_errors_map_to_reference_exceptions():
    mesh = meshgen.plate_mesh()
    tree = sbr.build(mesh)
    rec = sbr.trace_grid(tree, mesh, sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(0, 0),
                                                        0.1, margin=0.0))
    bad = sbr.HitRecords(rec.valid, rec.normal0, rec.path.copy(), rec.bounces, rec.escaped,
                         rec.out_dir)
    bad.path[5] = np.inf
    with pytest.raises(sbr.NumericalError, match="record index 5"):
        sbr.accumulate(bad, [0, 0, -1.0], sbr.ScatterParams.from_wavelength(0.5, 0.01))
    grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(0, 0), 0.1, margin=0.0)
    with pytest.raises(sbr.ValidationError):
        sbr.solve_grids(tree, mesh, [grid], sbr.TraceParams(max_bounces=1), [2 * np.pi / 0.2],
                        lambda_min=0.2, allow_aliasing=False)


def test_strict_and_budget_semantics():
    mesh = meshgen.plate_mesh()
    tree = sbr.build(mesh)
    rec = sbr.trace_ray(tree, mesh, (0.5, 0.5, -3.0), (0.0, 0.0, 1.0),
                        sbr.TraceParams(strict_orientation=True))
    assert not rec.valid and rec.escaped
    lax = sbr.trace_ray(tree, mesh, (0.5, 0.5, -3.0), (0.0, 0.0, 1.0))
    assert lax.valid and np.allclose(lax.normal0, [0, 0, -1])
    dmesh = meshgen.dihedral_mesh()
    dtree = sbr.build(dmesh)
    k = sbr.IncidentDirection(math.pi / 2, math.pi / 4).k_inc
    one = sbr.trace_ray(dtree, dmesh, (1.5, 1.2, 0.5), k, sbr.TraceParams(max_bounces=1))
    two = sbr.trace_ray(dtree, dmesh, (1.5, 1.2, 0.5), k, sbr.TraceParams(max_bounces=2))
    assert one.bounces == 1 and two.bounces == 2 and not one.escaped and two.escaped


def test_launches_are_counted():
    from paper_2604_09243_b200 import _native as nat
    ctx = nat.context()
    before = ctx.launches
    mesh = meshgen.quantized_icosphere(1.0, 3)
    tree = sbr.build(mesh)
    sbr.solve_direction(tree, mesh, sbr.IncidentDirection(0.3, 0.2), 0.05, 0.25)
    assert ctx.launches - before >= 6   # LBVH kernels + trace + po + reduces


@pytest.mark.parametrize("uniform", [True, False])
def test_multifrequency_po_vs_oracle(orc, uniform):
    """C5-style frequency sweep: 64 wavenumbers (linspace -> rotation
    recurrence in k_po; perturbed -> direct SFU sincos per term)."""
    mesh = meshgen.quantized_icosphere(1.0, 4)
    tree = sbr.build(mesh)
    ka = np.linspace(60.0, 64.0, 64)
    if not uniform:
        ka[5] += 1e-3
    lam_min = 2 * math.pi / ka.max()
    d = sbr.IncidentDirection(math.pi / 2, 0.3)
    grid = sbr.build_aperture(mesh.aabb, d, lam_min / 6, wavelength=lam_min)
    tp = sbr.TraceParams(max_bounces=2)
    res = sbr.solve_grids(tree, mesh, [grid], tp, ka)
    rec = sbr.trace_grid(tree, mesh, grid, tp)
    multi = sbr.accumulate_multi(rec, grid.k_inc, ka, grid.cell_area)
    for f in range(0, 64, 7):
        ref = orc.accumulate(rec, grid.k_inc, 2 * math.pi / ka[f], grid.cell_area)
        _amp_close(res.amplitude[0, f], ref)
        _amp_close(multi[f], ref)


def test_raster_primary_equals_bvh_primary(monkeypatch):
    """The raster pass answers query 0 with the same bits as BVH traversal:
    a multi-angle aircraft solve gives bitwise-identical amplitudes and
    diagnostics in both modes (also with tiny batches and ray-tile shards)."""
    mesh = meshgen.generate_aircraft(density=0.03)
    tree = sbr.build(mesh)
    lam = 0.1
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(th, ph), lam / 5,
                                wavelength=lam)
             for th, ph in [(math.pi / 2, 0.0), (math.pi / 2, 2.0), (1.1, 4.0), (0.2, 1.0)]]
    tp = sbr.TraceParams(max_bounces=5)
    ks = [2 * math.pi / lam]
    out = {}
    for mode in ("bvh", "raster"):
        monkeypatch.setenv("SBR_PRIMARY", mode)
        out[mode] = sbr.solve_grids(tree, mesh, grids, tp, ks)
    monkeypatch.setenv("SBR_SLOT_BUDGET", "5120")
    out["raster_small"] = sbr.solve_grids(tree, mesh, grids, tp, ks)
    for k in ("raster", "raster_small"):
        assert np.array_equal(out[k].amplitude, out["bvh"].amplitude), k
        assert np.array_equal(out[k].bounce_counts, out["bvh"].bounce_counts), k
        assert np.array_equal(out[k].valid_rays, out["bvh"].valid_rays), k
        assert np.array_equal(out[k].queries, out["bvh"].queries), k


# ---------------------------------------------------------------------------
# GPU binned-SAH build == the reference tree, node for node
# ---------------------------------------------------------------------------
_TREE_KEYS = ("nodes_min", "nodes_max", "node_first", "node_count", "tri_order")


@pytest.mark.parametrize("name", golden_names("bvh_"))
@pytest.mark.parametrize("rule", ["sah", "median"])
def test_gpu_build_is_the_reference_tree(name, rule):
    g = load_golden(name)
    mesh = _mesh(g)
    tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
    for k in _TREE_KEYS:
        ref = g[f"{rule}_{k}"]
        got = getattr(tree, k)
        assert got.dtype == ref.dtype or k in ("node_first", "node_count", "tri_order"), k
        assert np.array_equal(got, ref), k
    assert tree.max_depth_seen == int(g[f"{rule}_max_depth_seen"])
    tree.validate(mesh)


# bins 2 / 32 / 64 exercise the candidate packing of k_small (B <= 32) and
# its unpacked path (B > 32), and k_select's per-lane candidates over one to
# several rounds; depth8 forces leaves above 32 triangles at max_depth
_SAH_CASES = {
    "bins8_leaf2": dict(bins_per_axis=8, n_leaf=2, c_t=0.5, c_i=2.0),
    "bins2": dict(bins_per_axis=2, n_leaf=2),
    "bins32_leaf1": dict(bins_per_axis=32, n_leaf=1),
    "bins64_ct3": dict(bins_per_axis=64, n_leaf=3, c_t=3.0),
    "depth8": dict(max_depth=8, n_leaf=2),
}


@pytest.mark.parametrize("case", ["aircraft", "sphere_s6", "rough", "median", *_SAH_CASES])
def test_gpu_sah_build_matches_oracle_large(orc, case):
    params = sbr.BuildParams(split_rule="median" if case == "median" else "sah")
    if case == "aircraft":
        mesh = meshgen.generate_aircraft(density=0.08)
    elif case == "sphere_s6":
        mesh = meshgen.quantized_icosphere(1.0, 6)
    elif case in ("rough", "median"):
        mesh = meshgen.perturbed_grid_mesh(cells=150, extent=4.0, amplitude=0.08, seed=3)
    else:
        mesh = meshgen.generate_aircraft(density=0.03)
        params = sbr.BuildParams(split_rule="sah", **_SAH_CASES[case])
    tree = sbr.build(mesh, params)
    ref = orc.build(mesh.v0, mesh.v1, mesh.v2, split_rule=params.split_rule, n_leaf=params.n_leaf,
                    bins_per_axis=params.bins_per_axis, c_t=params.c_t, c_i=params.c_i,
                    max_depth=params.max_depth)
    for k in _TREE_KEYS:
        assert np.array_equal(getattr(tree, k), getattr(ref, k)), (case, k)
    assert tree.max_depth_seen == ref.max_depth_seen
    # and the traversal results are those of the LBVH (tree independence)
    lam = 0.1
    grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(1.1, 0.7), lam / 5,
                              wavelength=lam)
    tp = sbr.TraceParams(max_bounces=4)
    a = sbr.trace_grid(tree, mesh, grid, tp, with_ids=True)
    b = sbr.trace_grid(sbr.build(mesh, sbr.BuildParams(split_rule="lbvh")), mesh, grid, tp,
                       with_ids=True)
    for k in ("valid", "path", "bounces", "tri_ids", "out_dir"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), (case, k)


def test_l2_probe_and_debug_counters():
    import ctypes
    from paper_2604_09243_b200 import _native as nat
    ctx = nat.context()
    g = nat.c_dbl()
    nat.check(ctx.lib.sbr_probe_l2_bandwidth(ctx.handle, 8 << 20, 2, ctypes.byref(g)))
    assert g.value > 100.0          # GB/s; the measured peak lives in profiles/l2_peak.json
    buf = np.ones(24, np.int64)
    nat.check(ctx.lib.sbr_ctx_debug_counters(ctx.handle, nat.ptr(buf), 24))
    assert (buf >= 0).all()         # zeros unless built with -DSBR_TRACE_STATS


def test_sah_build_handles_leaf_roots_and_coincident_centroids():
    """A 1-triangle mesh (leaf root) and a stack of coincident triangles (no
    admissible split: one big leaf) take the host conversion path; the tree
    is still the reference's and traversal still matches the LBVH."""
    tri = np.array([[[0.0, 0, 0], [1, 0, 0], [0, 1, 0]]])
    m1 = sbr.mesh_from_soup(tri)
    t1 = sbr.build(m1, sbr.BuildParams(split_rule="sah"))
    assert t1.node_count.tolist() == [1] and t1.max_depth_seen == 0
    # 200 copies of one triangle at slightly different heights along z: all
    # centroids share x, y -> splits along z only; plus 100 exact duplicates
    base = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    stack = [base + [0, 0, 0.001 * k] for k in range(200)] + [base + [0, 0, 5.0]] * 100
    m2 = sbr.mesh_from_soup(np.array(stack))
    t2 = sbr.build(m2, sbr.BuildParams(split_rule="sah"))
    t2.validate(m2)
    assert int(t2.node_count.max()) >= 100      # the duplicates end in one leaf
    grid = sbr.build_aperture(m2.aabb, sbr.IncidentDirection(0.3, 0.2), 0.02, wavelength=0.1)
    tp = sbr.TraceParams(max_bounces=3)
    a = sbr.trace_grid(t2, m2, grid, tp, with_ids=True)
    b = sbr.trace_grid(sbr.build(m2, sbr.BuildParams(split_rule="lbvh")), m2, grid, tp,
                       with_ids=True)
    for k in ("valid", "path", "bounces", "tri_ids"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


@pytest.mark.parametrize("mesh_name", ["aircraft", "sphere", "rough"])
def test_raster_vs_bvh_random_directions(monkeypatch, mesh_name):
    """Query 0 by rasterisation == query 0 by traversal, ray for ray (all
    HitRecords fields and per-bounce ids), over random incidence directions
    including grazing ones, on meshes with slivers, big and tiny triangles."""
    if mesh_name == "aircraft":
        mesh, lam = meshgen.generate_aircraft(density=0.05), 0.08
    elif mesh_name == "sphere":
        mesh, lam = meshgen.quantized_icosphere(1.0, 5), 0.05
    else:
        mesh, lam = meshgen.perturbed_grid_mesh(cells=90, extent=4.0, amplitude=0.3, seed=11), 0.1
    tree = sbr.build(mesh)
    rng = np.random.default_rng(2024)
    tp = sbr.TraceParams(max_bounces=4)
    for _ in range(6):
        th = float(np.arccos(rng.uniform(-1, 1)))
        ph = float(rng.uniform(0, 2 * np.pi))
        if _ == 0:
            th = np.pi / 2 - 1e-9          # grazing a plane of the aircraft / plate
        grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(th, ph), lam / 5,
                                  wavelength=lam)
        out = {}
        for mode in ("bvh", "raster"):
            monkeypatch.setenv("SBR_PRIMARY", mode)
            out[mode] = sbr.trace_grid(tree, mesh, grid, tp, with_ids=True)
        for k in ("valid", "normal0", "path", "bounces", "escaped", "out_dir", "tri_ids"):
            assert np.array_equal(getattr(out["raster"], k), getattr(out["bvh"], k)), (th, ph, k)


def test_ctx_trim_releases_scratch_and_results_repeat():
    """sbr_ctx_trim frees the grow-only scratch; the next solve re-grows it
    and returns the same bits."""
    import torch
    from paper_2604_09243_b200 import _native as nat
    mesh = meshgen.generate_aircraft(density=0.03)
    tree = sbr.build(mesh)
    lam = 0.1
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, ph), lam / 5,
                                wavelength=lam) for ph in (0.0, 1.5)]
    tp = sbr.TraceParams(max_bounces=3)
    a = sbr.solve_grids(tree, mesh, grids, tp, [2 * math.pi / lam])
    ctx = nat.context()
    ctx.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    ctx.trim()
    free1 = torch.cuda.mem_get_info()[0]
    assert free1 >= free0
    b = sbr.solve_grids(tree, mesh, grids, tp, [2 * math.pi / lam])
    assert np.array_equal(a.amplitude, b.amplitude)
    assert np.array_equal(a.queries, b.queries)


def test_po_field_precision_at_near_nulls(orc):
    """The fused solve's per-wavenumber PO (FP64 phases and lane sums)
    follows the reference's complex128 sum to well under the 1e-4 field
    tolerance at every azimuth of the C3 trihedral sweep, nulls included
    (FP32 phases left 7.9e-5 here)."""
    mesh = meshgen.trihedral_mesh()
    lam = 0.05
    tree = sbr.build(mesh)
    tp = sbr.TraceParams(max_bounces=3)
    scene = _oracle_scene(orc, mesh)
    eps = tp.resolve_epsilon(mesh)
    dirs = [sbr.IncidentDirection(math.radians(54.7356), math.radians(p))
            for p in np.linspace(0, 90, 181)]
    grids = [sbr.build_aperture(mesh.aabb, d, lam / 5, wavelength=lam) for d in dirs]
    amp = sbr.solve_grids(tree, mesh, grids, tp, [2 * math.pi / lam]).amplitude[:, 0]
    worst = 0.0
    for g, a in zip(grids, amp):
        ref = orc.trace_grid(scene, g, 3, eps)
        a_ref = orc.accumulate(ref, g.k_inc, lam, g.cell_area)
        worst = max(worst, abs(complex(a) - a_ref) / abs(a_ref))
    assert worst < 1e-5, worst


def test_slot_reuse_without_memset_is_exact(monkeypatch):
    """List-mode PO restores the raster's all-ones slots, so repeated solves
    skip the memset; interleaving paths that dirty the slots (host-record
    accumulate, BVH primary, reference order, smaller batches) must not
    change a bit of the next raster solve."""
    mesh = meshgen.generate_aircraft(density=0.03)
    tree = sbr.build(mesh)
    lam = 0.1
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, ph), lam / 5,
                                wavelength=lam) for ph in (0.0, 1.0, 2.5)]
    tp = sbr.TraceParams(max_bounces=5)
    ks = [2 * math.pi / lam]
    monkeypatch.setenv("SBR_PRIMARY", "raster")
    first = sbr.solve_grids(tree, mesh, grids, tp, ks)

    def again(tag):
        r = sbr.solve_grids(tree, mesh, grids, tp, ks)
        assert np.array_equal(r.amplitude, first.amplitude), tag
        assert np.array_equal(r.queries, first.queries), tag
        assert np.array_equal(r.bounce_counts, first.bounce_counts), tag

    again("repeat")
    rec = sbr.trace_grid(tree, mesh, grids[1], tp)
    sbr.accumulate_multi(rec, grids[1].k_inc, np.array(ks), grids[1].cell_area)
    again("after accumulate")
    monkeypatch.setenv("SBR_PRIMARY", "bvh")
    b = sbr.solve_grids(tree, mesh, grids, tp, ks)
    assert np.array_equal(b.amplitude, first.amplitude)
    monkeypatch.setenv("SBR_PRIMARY", "raster")
    again("after bvh primary")
    with sbr.traversal_order("reference"):
        sbr.solve_grids(tree, mesh, grids, tp, ks)
    again("after reference order")
    monkeypatch.setenv("SBR_SLOT_BUDGET", "4096")
    again("small batches")
    monkeypatch.delenv("SBR_SLOT_BUDGET")
    again("back to one batch")


def test_aabb_conservative_over_triangle_hits():
    """pkg/tests/test_geometry.py:255-272 on the device slab predicate
    (geometry.py:358-391 restated): every ray that hits a random triangle
    also hits the triangle's box (2000 triangles, seed 99)."""
    rng = np.random.default_rng(99)
    checked = 0
    for _ in range(2000):
        verts = rng.uniform(-1, 1, size=(3, 3))
        normal = np.cross(verts[1] - verts[0], verts[2] - verts[0])
        if np.linalg.norm(normal) < 1e-9:
            continue
        tri = sbr.Triangle(verts[0], verts[1], verts[2], normal / np.linalg.norm(normal))
        box = sbr.Aabb(verts.min(axis=0), verts.max(axis=0))
        origin = rng.uniform(-3, 3, size=3)
        # the reference's random direction, and one aimed at a point of the
        # triangle (edges and vertices included) so that most rays hit
        w = rng.dirichlet([0.5, 0.5, 0.5])
        w[rng.integers(0, 3)] *= rng.integers(0, 2)
        w /= w.sum()
        for d in (rng.normal(size=3), w @ verts - origin):
            d = d / np.linalg.norm(d)
            hit = sbr.ray_triangle_intersect(origin, d, tri)
            if hit is not None:
                inv = np.where(d != 0, 1.0 / np.where(d != 0, d, 1.0), np.inf)
                box_hit, entry = sbr.ray_aabb_intersect(origin, inv, box)
                assert box_hit and entry <= hit[0]
                checked += 1
    assert checked > 1000


@pytest.mark.parametrize("rule", ["sah", "lbvh"])
def test_fp32_slab_culling_is_conservative(orc, rule):
    """The hot path culls with FP32 outward-rounded boxes and a padded slab
    (sbr_device.cuh RayBox / node4_visit).  Stress it where FP32 is weakest:
    origins 1e2..1e5 scene sizes away, rays aimed at triangle vertices and
    edge points (grazing the leaf boxes' faces), and rays parallel to box
    faces.  A single wrongly culled box would lose a hit: the closest hits
    must equal the brute-force linear scan on every robust ray."""
    rng = np.random.default_rng(7)
    n = 2000
    c = rng.uniform(-1, 1, size=(n, 3))
    v0 = (c + 0.05 * rng.normal(size=(n, 3))).astype(np.float32).astype(np.float64)
    v1 = (c + 0.05 * rng.normal(size=(n, 3))).astype(np.float32).astype(np.float64)
    v2 = (c + 0.05 * rng.normal(size=(n, 3))).astype(np.float32).astype(np.float64)
    verts = np.stack([v0, v1, v2], axis=1).reshape(-1, 3)      # triangle i = rows 3i..3i+2
    mesh = sbr.mesh_from_arrays(verts, np.arange(3 * n).reshape(n, 3))
    m = 6000
    k = rng.integers(0, n, m)
    w = rng.dirichlet([0.3, 0.3, 0.3], size=m)
    w[: m // 3] = np.eye(3)[rng.integers(0, 3, m // 3)]            # vertices
    w[m // 3: m // 2, 2] = 0.0                                     # edge v0-v1
    w[m // 3: m // 2] /= w[m // 3: m // 2].sum(1, keepdims=True)
    target = w[:, :1] * mesh.v0[k] + w[:, 1:2] * mesh.v1[k] + w[:, 2:] * mesh.v2[k]
    d = rng.normal(size=(m, 3))
    d[: m // 6, rng.integers(0, 3)] = 0.0                          # parallel to a face pair
    d /= np.linalg.norm(d, axis=1)[:, None]
    dist = 10.0 ** rng.uniform(0, 5, size=m)
    origins = target - dist[:, None] * d
    tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
    tri, t, _ = sbr.closest_hit_batch(tree, mesh, origins, d)
    scene = orc.Scene.from_mesh(mesh)
    btri, bt = orc.brute_force_hits(scene, origins, d)
    rob = orc.classify_rays(scene, origins, d)
    assert rob.mean() > 0.8          # vertex / edge aims are near-ties by design
    assert (btri[rob] >= 0).mean() > 0.5
    assert np.array_equal(tri[rob], btri[rob])
    assert np.array_equal(t[rob & (btri >= 0)], bt[rob & (btri >= 0)])


def test_device_objects_are_released():
    """Meshes, trees and the fused solve's results own no device memory
    after they are dropped (live-allocation counter of the library; the
    solve scratch is grow-only and stays with the context)."""
    import gc
    from paper_2604_09243_b200 import _native as nat

    def cycle():
        mesh = meshgen.generate_aircraft(density=0.02)
        for rule in ("sah", "lbvh"):
            tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
            g = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(1.2, 0.4), 0.04,
                                   wavelength=0.2)
            sbr.solve_grids(tree, mesh, [g], sbr.TraceParams(max_bounces=3), [2 * math.pi / 0.2])
            sbr.trace_grid(tree, mesh, g, sbr.TraceParams(max_bounces=2), with_ids=True)

    cycle()
    gc.collect()
    base = nat.live_allocations()
    for _ in range(3):
        cycle()
        gc.collect()
        assert nat.live_allocations() == base


@pytest.mark.parametrize("strict", [False, True])
def test_fused_solve_count_trapped_and_strict(orc, primary, strict):
    """The fused solve (raster -> compaction -> trace -> list PO) with
    count_trapped=True (po.py:95-98 keeps valid rays that never escaped) and
    strict orientation (transport.py:306-307) against the oracle's records +
    accumulate, on a multi-bounce rough plate where many rays end trapped."""
    mesh = meshgen.perturbed_grid_mesh(cells=120, extent=4.0, amplitude=0.25, seed=11)
    tree = sbr.build(mesh)
    scene = orc.Scene.from_mesh(mesh)
    lam = 0.1
    params = sbr.TraceParams(max_bounces=3, strict_orientation=strict)
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(th, ph), lam / 5,
                                wavelength=lam)
             for th, ph in ((0.3, 0.7), (2.6, 4.0), (1.2, 1.9))]
    res = sbr.solve_grids(tree, mesh, grids, params, [2 * math.pi / lam], count_trapped=True)
    trapped = 0
    for i, g in enumerate(grids):
        ref = orc.trace_grid(scene, g, 3, params.resolve_epsilon(mesh), strict=strict)
        trapped += int((ref.valid.astype(bool) & ~ref.escaped.astype(bool)).sum())
        a = orc.accumulate(ref, g.k_inc, lam, g.cell_area, count_trapped=True)
        _amp_close(res.amplitude[i, 0], a)
        assert int(res.valid_rays[i]) == int(ref.valid.sum())
        assert int(res.queries[i]) == int((ref.bounces.astype(np.int64) + 1).sum())
    assert trapped > 1000


def test_empty_and_degenerate_inputs(orc, monkeypatch):
    """Empty ray lists, empty row ranges, no grids, a single-triangle mesh
    forced through the raster pass, and an aperture the mesh does not cover
    (every ray misses): shapes and values as the reference produces them."""
    mesh = meshgen.plate_mesh(1.0)
    tree = sbr.build(mesh)
    tri, t, vis = sbr.closest_hit_batch(tree, mesh, np.zeros((0, 3)), np.zeros((0, 3)))
    assert tri.shape == (0,) and t.shape == (0,) and vis.shape == (0,)
    grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(0.2, 0.3), 0.02, wavelength=0.1)
    rec = sbr.trace_grid(tree, mesh, grid, sbr.TraceParams(max_bounces=2), rows=(5, 5))
    assert rec.valid.shape == (0,)
    res = sbr.solve_grids(tree, mesh, [], sbr.TraceParams(max_bounces=2), [2 * math.pi / 0.1])
    assert res.amplitude.shape == (0, 1)
    one = sbr.mesh_from_arrays([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    t1 = sbr.build(one)
    g1 = sbr.build_aperture(one.aabb, sbr.IncidentDirection(0.0, 0.0), 0.01, wavelength=0.05)
    scene = orc.Scene.from_mesh(one)
    for prim in ("raster", "bvh"):
        monkeypatch.setenv("SBR_PRIMARY", prim)
        r = sbr.trace_grid(t1, one, g1, sbr.TraceParams(max_bounces=2), with_ids=True)
        ref = orc.trace_grid(scene, g1, 2, sbr.TraceParams().resolve_epsilon(one), with_ids=True)
        for k in ("valid", "normal0", "path", "bounces", "escaped", "out_dir", "tri_ids"):
            assert np.array_equal(getattr(r, k), getattr(ref, k)), (prim, k)
        assert 0 < r.valid.sum() < r.valid.size
        s = sbr.solve_grids(t1, one, [g1], sbr.TraceParams(max_bounces=2), [2 * math.pi / 0.05])
        assert int(s.valid_rays[0]) == int(ref.valid.sum())
    # an aperture built for another object: every ray misses the plate
    far = sbr.mesh_from_arrays([[10, 10, 10], [11, 10, 10], [10, 11, 10]], [[0, 1, 2]])
    gm = sbr.build_aperture(far.aabb, sbr.IncidentDirection(0.0, 0.0), 0.05, wavelength=0.25)
    sm = sbr.solve_grids(tree, mesh, [gm], sbr.TraceParams(max_bounces=2), [2 * math.pi / 0.25])
    assert sm.valid_rays[0] == 0 and sm.amplitude[0, 0] == 0
    assert sm.queries[0] == gm.n_u * gm.n_v

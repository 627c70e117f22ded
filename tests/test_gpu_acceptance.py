"""The reference's release criteria (pkg/tests/test_acceptance.py) on the GPU
path, at the reference's own thresholds.

Each test restates one criterion against ``paper_2604_09243_b200`` (the
drop-in) and, where the reference's run log records its numbers
(pkg/test_output.txt:210-222), also checks that this path reproduces them.

  c1  sphere vs Mie at kr = 30/50/100, lambda/5, s = 6, 64 directions:
      each <= 5 %, mean <= 3 %                         (test_acceptance.py:38-49)
  c2  fixed-spacing sweep: ok rows <= 5 %, aliased rows (> lambda/2) > 10 %
                                                       (test_acceptance.py:52-75)
  c3  plate at normal incidence vs 4 pi a^4 / lambda^2 within 1 %   (:78-94)
  c4  dihedral: retro gain >= 10 dB and 200 rays vs the two-mirror oracle
      (path rel 1e-9, exit antiparallel to 1e-9)        (:97-133)
  c5  closest hit == brute force on three meshes x 10^4 probe rays, both
      split rules (seeds = hash(name) % 2^16 under PYTHONHASHSEED=0)  (:136-154)
  c6  SAH visits <= median visits on icosphere s = 4    (:157-168)
  c7  byte-identical validation CSVs at any worker count (:171-200)
  c9  100k-triangle sweep with CSV + heatmap, >= 20 dB dynamic range (:249-289)

c8 (8-worker CPU thread efficiency) has no GPU counterpart: the sweep is one
device pipeline whatever ``workers`` says.
"""

import math

import numpy as np
import pytest

import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen

pytestmark = pytest.mark.gpu

# pkg/test_output.txt:210-221 (the reference's own run)
REF_C1 = {30.0: 3.13233, 50.0: 3.16289, 100.0: 3.24176}
REF_C2_ERR = {30.0: 0.0137, 40.0: 0.0172, 50.0: 0.0109, 150.0: 1.5148, 200.0: 3.4576,
              250.0: 4.8674}


def random_probe_rays(mesh, count, seed, radius_factor=1.6):
    """pkg/tests/meshes.py:89-100 (the probe-ray recipe of criterion 5)."""
    rng = np.random.default_rng(seed)
    center = 0.5 * (mesh.aabb.min + mesh.aabb.max)
    r = max(mesh.aabb.diagonal(), 1e-6)
    g = rng.normal(size=(count, 3))
    g /= np.linalg.norm(g, axis=1)[:, None]
    origins = center + radius_factor * r * g
    aim = center + 0.4 * r * rng.uniform(-1.0, 1.0, size=(count, 3))
    dirs = aim - origins
    dirs /= np.linalg.norm(dirs, axis=1)[:, None]
    return origins, dirs


def test_c1_sphere_mie_optical_agreement():
    report = sbr.validate_sphere(1.0, [30.0, 50.0, 100.0], sampling_factor=5.0,
                                 subdivisions=6, n_directions=64, workers=4)
    for row in report.rows:
        assert row.rel_error <= 0.05, (row.kr, row.rel_error)
        # the reference's own sigma, printed to 6 digits
        assert row.sigma_sbr_m2 == pytest.approx(REF_C1[row.kr], rel=2e-4, abs=6e-6)
    assert report.mean_rel_error() <= 0.03


def test_c2_aliasing_instability_onset():
    spacing = (2 * math.pi / 50.0) / 5.0
    report = sbr.validate_sphere(1.0, [30.0, 40.0, 50.0, 150.0, 200.0, 250.0],
                                 fixed_spacing=spacing, subdivisions=6, n_directions=64,
                                 workers=4)
    aliased = []
    for row in report.rows:
        lam = 2 * math.pi / row.kr
        if row.sampling_ok:
            assert row.rel_error <= 0.05, row.kr
        if row.spacing_m > lam / 2:
            aliased.append(row.rel_error)
        # the reference's printed error (2 decimals of a percent)
        assert abs(row.rel_error - REF_C2_ERR[row.kr]) <= 6e-5 + 2e-4 * (1 + row.rel_error), \
            (row.kr, row.rel_error)
    assert aliased and max(aliased) > 0.10


def test_c3_flat_plate_closed_form():
    side, lam = 1.0, 0.1
    mesh = meshgen.plate_mesh(side)
    tree = sbr.build(mesh)
    d = sbr.IncidentDirection(0.0, 0.0)
    grid = sbr.build_aperture(mesh.aabb, d, lam / 10, margin=0.0, wavelength=lam)
    rec = sbr.trace_grid(tree, mesh, grid, sbr.TraceParams(max_bounces=3))
    params = sbr.ScatterParams.from_wavelength(lam, grid.cell_area)
    sigma = sbr.rcs(sbr.accumulate(rec, d.k_inc, params)).sigma_m2
    ref = sbr.plate_reference(side, lam)
    assert abs(sigma - ref) / ref <= 0.01


def test_c4_dihedral_multibounce():
    mesh = meshgen.dihedral_mesh(1.0)
    tree = sbr.build(mesh)
    lam = 0.05
    direction = sbr.IncidentDirection(math.pi / 2, math.pi / 4)
    sig = {}
    for b in (1, 2):
        sol = sbr.solve_direction(tree, mesh, direction, lam / 5, lam,
                                  trace_params=sbr.TraceParams(max_bounces=b))
        sig[b] = sol.rcs.sigma_m2
    assert sig[2] > 0
    if sig[1] > 0:
        assert 10 * math.log10(sig[2] / sig[1]) >= 10.0
    eps = 1e-6 * mesh.aabb.diagonal()
    params = sbr.TraceParams(max_bounces=2, epsilon=eps)
    k = direction.k_inc
    rng = np.random.default_rng(4)
    checked = 0
    while checked < 200:
        w = rng.uniform(-0.65, 0.65)
        z = rng.uniform(0.05, 0.95)
        if abs(w) < 0.02:
            continue
        o = np.array([2.0 + w / math.sqrt(2), 2.0 - w / math.sqrt(2), z])
        rec = sbr.trace_ray(tree, mesh, o, k, params)
        assert rec.valid and rec.bounces == 2
        a_first = o[1] < o[0]
        n1 = np.array([0.0, 1, 0]) if a_first else np.array([1.0, 0, 0])
        t1 = o[1] * math.sqrt(2) if a_first else o[0] * math.sqrt(2)
        x1 = o + t1 * k + eps * n1
        d1 = k - 2 * np.dot(k, n1) * n1
        t2 = (x1[0] / -d1[0]) if a_first else (x1[1] / -d1[1])
        assert rec.path == pytest.approx(t1 + t2, rel=1e-9)
        assert float(np.linalg.norm(rec.out_dir + k)) < 1e-9
        checked += 1


C5_MESHES = {   # name -> seed = hash(name) % 2**16 with PYTHONHASHSEED=0
    "single-triangle": 45449,
    "icosphere-s3": 11971,
    "perturbed-grid-10k": 436,
}


def _c5_mesh(name):
    if name == "single-triangle":
        return sbr.mesh_from_arrays([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    if name == "icosphere-s3":
        return sbr.generate_icosphere(1.0, 3)
    return meshgen.perturbed_grid_mesh(cells=71)


@pytest.mark.parametrize("rule", ["median", "sah"])
@pytest.mark.parametrize("traversal", ["fast", "reference"])
def test_c5_bvh_matches_brute_force(orc, rule, traversal):
    for name, seed in C5_MESHES.items():
        mesh = _c5_mesh(name)
        tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
        tree.validate(mesh)
        origins, dirs = random_probe_rays(mesh, 10000, seed=seed)
        with sbr.traversal_order(traversal):
            tri, t, _ = sbr.closest_hit_batch(tree, mesh, origins, dirs)
        scene = orc.Scene.from_mesh(mesh)
        btri, bt = orc.brute_force_hits(scene, origins, dirs)
        assert np.array_equal(tri, btri), name
        hits = tri >= 0
        assert hits.sum() > 0 or name == "single-triangle"
        assert np.allclose(t[hits], bt[hits], rtol=1e-9, atol=0.0)


def test_c6_sah_traversal_benefit():
    mesh = sbr.generate_icosphere(1.0, 4)
    origins, dirs = random_probe_rays(mesh, 10000, seed=77)
    mean = {}
    with sbr.traversal_order("reference"):     # the reference's own visit count
        for rule in ("median", "sah"):
            tree = sbr.build(mesh, sbr.BuildParams(split_rule=rule))
            _, _, visits = sbr.closest_hit_batch(tree, mesh, origins, dirs)
            mean[rule] = float(np.mean(visits))
    assert mean["sah"] <= mean["median"]


def test_c7_determinism_across_runs_and_workers(tmp_path):
    blobs = []
    for tag, workers in (("a", 1), ("b", 2), ("c", 2)):
        report = sbr.validate_sphere(1.0, [30.0, 50.0], subdivisions=5, n_directions=8,
                                     workers=workers)
        path = tmp_path / f"run_{tag}.csv"
        sbr.write_validation_csv(report, path)
        blobs.append(path.read_bytes())
    assert blobs[0] == blobs[1] == blobs[2]


def test_c9_large_mesh_smoke(tmp_path):
    mesh = meshgen.perturbed_grid_mesh(cells=224, extent=4.0, amplitude=0.05)
    assert mesh.triangle_count >= 100_000
    mesh_path = tmp_path / "rough.obj"
    sbr.save_obj(mesh, mesh_path)
    spacing = 4.1 / 500.0
    cfg = sbr.SweepConfig.from_dict({
        "mesh": str(mesh_path),
        "frequency_hz": sbr.SPEED_OF_LIGHT / (10 * spacing),
        "theta_deg": {"start_deg": 0, "stop_deg": 180, "samples": 8},
        "phi_deg": {"start_deg": 0, "stop_deg": 315, "samples": 8},
        "spacing_m": spacing,
        "max_bounces": 100,
        "workers": 4,
    })
    result = sbr.run_sweep(cfg)
    first = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(0.0, 0.0), spacing)
    assert first.n_u >= 500 and first.n_v >= 500
    csv_path, ppm_path = tmp_path / "rough.csv", tmp_path / "rough.ppm"
    sbr.write_csv(result, csv_path)
    sbr.write_heatmap(result, ppm_path, db_floor=-50.0, db_ceil=40.0)
    lines = csv_path.read_text().splitlines()
    assert len(lines) == 1 + 64
    for line in lines[1:]:
        fields = line.split(",")
        assert len(fields) == 7
        assert math.isfinite(float(fields[2]))
    assert ppm_path.read_bytes()[:20].startswith(b"P6\n8 8\n255\n")
    finite = result.sigma_dbsm[np.isfinite(result.sigma_dbsm)]
    assert float(finite.max() - finite.min()) >= 20.0

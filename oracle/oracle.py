"""ctypes front-end of the CPU oracle (oracle/sbr_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Only tests/,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this module.  The product package
``paper_2604_09243_b200`` must never import it.

Parity pin: every entry point is checked against golden vectors generated
by running the reference ``sbr`` package (tests/golden/make_golden.py);
see tests/test_oracle_golden.py.

The aperture construction is restated here in NumPy from
pkg/src/sbr/transport.py:25-205 so that the oracle does not depend on the
product's host code.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsbr_oracle.so")
_lib = None


def build_library(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH)
            < os.path.getmtime(os.path.join(_HERE, "sbr_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class _Scene(ctypes.Structure):
    _fields_ = [
        ("nmin", ctypes.c_void_p), ("nmax", ctypes.c_void_p),
        ("first", ctypes.c_void_p), ("count", ctypes.c_void_p),
        ("order", ctypes.c_void_p), ("nnodes", ctypes.c_int64),
        ("stack_depth", ctypes.c_int32),
        ("v0", ctypes.c_void_p), ("v1", ctypes.c_void_p),
        ("v2", ctypes.c_void_p), ("normals", ctypes.c_void_p),
        ("ntri", ctypes.c_int64), ("single", ctypes.c_int32),
    ]


class Counters(ctypes.Structure):
    _fields_ = [("pops", ctypes.c_int64), ("boxes", ctypes.c_int64),
                ("tris", ctypes.c_int64), ("internal", ctypes.c_int64),
                ("queries", ctypes.c_int64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


def lib():
    global _lib
    if _lib is None:
        build_library()
        _lib = ctypes.CDLL(_LIB_PATH)
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def _threads(n):
    # 0 = every host core.  Resolved here rather than by omp_get_max_threads():
    # launchers such as torchrun export OMP_NUM_THREADS=1, which would time
    # the reference CPU path on one core.
    return int(n) if n else (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
                             else (os.cpu_count() or 1))


# ---------------------------------------------------------------------------
# BVH build (bvh.py:218-299)
# ---------------------------------------------------------------------------

@dataclass
class OracleBvh:
    nodes_min: np.ndarray
    nodes_max: np.ndarray
    node_first: np.ndarray
    node_count: np.ndarray
    tri_order: np.ndarray
    max_depth_seen: int
    max_depth: int = 64


def build(v0, v1, v2, split_rule="sah", n_leaf=4, bins_per_axis=16, c_t=1.0,
          c_i=1.0, max_depth=64, single=False) -> OracleBvh:
    v0 = _f64(v0, (-1, 3)); v1 = _f64(v1, (-1, 3)); v2 = _f64(v2, (-1, 3))
    t = v0.shape[0]
    m = max(2 * t - 1, 1)
    nmin = np.empty((m, 3)); nmax = np.empty((m, 3))
    first = np.empty(m, np.int32); count = np.empty(m, np.int32)
    order = np.empty(t, np.int32)
    nn = ctypes.c_int64(0); depth = ctypes.c_int32(0)
    rc = lib().orc_build(_p(v0), _p(v1), _p(v2), ctypes.c_int64(t),
                         ctypes.c_int32(1 if split_rule == "sah" else 0),
                         ctypes.c_int32(n_leaf), ctypes.c_int32(bins_per_axis),
                         ctypes.c_double(c_t), ctypes.c_double(c_i),
                         ctypes.c_int32(max_depth), ctypes.c_int32(int(single)),
                         _p(nmin), _p(nmax), _p(first), _p(count), _p(order),
                         ctypes.byref(nn), ctypes.byref(depth))
    if rc != 0:
        raise RuntimeError(f"orc_build failed rc={rc}")
    n = nn.value
    return OracleBvh(nmin[:n].copy(), nmax[:n].copy(), first[:n].copy(),
                     count[:n].copy(), order, int(depth.value), max_depth)


class Scene:
    """Mesh + preorder BVH bundle passed to the C kernels."""

    def __init__(self, v0, v1, v2, normals, bvh: OracleBvh, single=False):
        self.v0 = _f64(v0, (-1, 3)); self.v1 = _f64(v1, (-1, 3))
        self.v2 = _f64(v2, (-1, 3)); self.normals = _f64(normals, (-1, 3))
        self.bvh = bvh
        self.nmin = _f64(bvh.nodes_min, (-1, 3))
        self.nmax = _f64(bvh.nodes_max, (-1, 3))
        self.first = np.ascontiguousarray(bvh.node_first, np.int32)
        self.count = np.ascontiguousarray(bvh.node_count, np.int32)
        self.order = np.ascontiguousarray(bvh.tri_order, np.int32)
        self.single = bool(single)
        pts = np.concatenate([self.v0, self.v1, self.v2])
        self.aabb_min = pts.min(axis=0)
        self.aabb_max = pts.max(axis=0)
        self.default_eps = 1e-6 * float(np.linalg.norm(self.aabb_max - self.aabb_min))
        self._c = _Scene(_p(self.nmin).value, _p(self.nmax).value,
                         _p(self.first).value, _p(self.count).value,
                         _p(self.order).value, self.first.shape[0],
                         int(getattr(bvh, "max_depth", 64)) + 2,
                         _p(self.v0).value, _p(self.v1).value,
                         _p(self.v2).value, _p(self.normals).value,
                         self.v0.shape[0], int(self.single))

    @classmethod
    def from_mesh(cls, mesh, bvh=None, split_rule="sah", n_leaf=4, single=None):
        """Accepts any object with v0/v1/v2/normals (reference or product Mesh)."""
        if single is None:
            single = np.asarray(mesh.v0).dtype == np.float32
        if bvh is None:
            bvh = build(mesh.v0, mesh.v1, mesh.v2, split_rule=split_rule,
                        n_leaf=n_leaf, single=single)
        return cls(mesh.v0, mesh.v1, mesh.v2, mesh.normals, bvh, single)

    @property
    def ref(self):
        return ctypes.byref(self._c)

    @property
    def ntri(self):
        return self.v0.shape[0]


def closest_hit_batch(scene: Scene, origins, dirs, t_min=0.0, t_max=np.inf,
                      threads=0, counters: Counters | None = None):
    o = _f64(origins, (-1, 3)); d = _f64(dirs, (-1, 3))
    n = o.shape[0]
    tri = np.empty(n, np.int64); t = np.empty(n); vis = np.empty(n, np.int64)
    rc = lib().orc_closest_hit_batch(
        scene.ref, _p(o), _p(d), ctypes.c_int64(n), ctypes.c_double(t_min),
        ctypes.c_double(t_max), _p(tri), _p(t), _p(vis),
        ctypes.byref(counters) if counters is not None else None,
        ctypes.c_int(_threads(threads)))
    if rc != 0:
        raise RuntimeError(f"orc_closest_hit_batch rc={rc}")
    return tri, t, vis


def brute_force_hits(scene: Scene, origins, dirs, t_min=0.0, t_max=np.inf,
                     threads=0):
    o = _f64(origins, (-1, 3)); d = _f64(dirs, (-1, 3))
    n = o.shape[0]
    tri = np.empty(n, np.int64); t = np.empty(n)
    lib().orc_brute_force_batch(scene.ref, _p(o), _p(d), ctypes.c_int64(n),
                                ctypes.c_double(t_min), ctypes.c_double(t_max),
                                _p(tri), _p(t), ctypes.c_int(_threads(threads)))
    return tri, t


@dataclass
class Records:
    """Reference HitRecords layout (transport.py:251-273) + per-bounce ids."""

    valid: np.ndarray
    normal0: np.ndarray
    path: np.ndarray
    bounces: np.ndarray
    escaped: np.ndarray
    out_dir: np.ndarray
    tri_ids: np.ndarray | None = None

    def __len__(self):
        return self.valid.shape[0]


def _alloc_records(n, max_bounces, with_ids):
    return Records(np.empty(n, np.bool_), np.empty((n, 3)), np.empty(n),
                   np.empty(n, np.int32), np.empty(n, np.bool_),
                   np.empty((n, 3)),
                   np.empty((n, max_bounces), np.int32) if with_ids else None)


def trace_grid(scene: Scene, grid, max_bounces=10, eps=None, strict=False,
               rows=None, with_ids=False, threads=0,
               counters: Counters | None = None) -> Records:
    """transport.py:375-422; ``rows=(i0, i1)`` traces a row band only."""
    if eps is None:
        eps = scene.default_eps  # TraceParams.resolve_epsilon, transport.py:236-239
    i0, i1 = (0, grid.n_u) if rows is None else rows
    n = (i1 - i0) * grid.n_v
    rec = _alloc_records(n, max_bounces, with_ids)
    corner = _f64(grid.corner); u = _f64(grid.u); v = _f64(grid.v)
    k = _f64(grid.k_inc)
    rc = lib().orc_trace_grid(
        scene.ref, _p(corner), _p(u), _p(v), _p(k),
        ctypes.c_double(grid.spacing), ctypes.c_int64(grid.n_u),
        ctypes.c_int64(grid.n_v), ctypes.c_int64(i0), ctypes.c_int64(i1),
        ctypes.c_int32(max_bounces), ctypes.c_double(eps),
        ctypes.c_int32(int(strict)), _p(rec.valid), _p(rec.normal0),
        _p(rec.path), _p(rec.bounces), _p(rec.escaped), _p(rec.out_dir),
        _p(rec.tri_ids), ctypes.byref(counters) if counters is not None else None,
        ctypes.c_int(_threads(threads)))
    if rc != 0:
        raise RuntimeError(f"orc_trace_grid rc={rc}")
    return rec


def trace_rays(scene: Scene, origins, dirs, max_bounces=10, eps=1e-6,
               strict=False, with_ids=False, threads=0) -> Records:
    o = _f64(origins, (-1, 3)); d = _f64(dirs, (-1, 3))
    n = o.shape[0]
    rec = _alloc_records(n, max_bounces, with_ids)
    lib().orc_trace_rays(scene.ref, _p(o), _p(d), ctypes.c_int64(n),
                         ctypes.c_int32(max_bounces), ctypes.c_double(eps),
                         ctypes.c_int32(int(strict)), _p(rec.valid),
                         _p(rec.normal0), _p(rec.path), _p(rec.bounces),
                         _p(rec.escaped), _p(rec.out_dir), _p(rec.tri_ids),
                         ctypes.c_int(_threads(threads)))
    return rec


def trace_grid_hash(scene: Scene, grid, max_bounces=10, eps=None, strict=False,
                    rows=None, seg_rays=1 << 19, threads=0) -> np.ndarray:
    """Per-segment record hashes of trace_grid (+ per-bounce ids): the CPU
    twin of paper_2604_09243_b200.trace_grid_hash (same hash function)."""
    if eps is None:
        eps = scene.default_eps
    i0, i1 = (0, grid.n_u) if rows is None else rows
    out = np.zeros(-(-grid.n_u * grid.n_v // int(seg_rays)), np.uint64)
    corner = _f64(grid.corner); u = _f64(grid.u); v = _f64(grid.v)
    k = _f64(grid.k_inc)
    rc = lib().orc_trace_grid_hash(
        scene.ref, _p(corner), _p(u), _p(v), _p(k), ctypes.c_double(grid.spacing),
        ctypes.c_int64(grid.n_u), ctypes.c_int64(grid.n_v), ctypes.c_int64(i0),
        ctypes.c_int64(i1), ctypes.c_int32(max_bounces), ctypes.c_double(eps),
        ctypes.c_int32(int(strict)), ctypes.c_int64(int(seg_rays)), _p(out),
        ctypes.c_int(_threads(threads)))
    if rc != 0:
        raise RuntimeError(f"orc_trace_grid_hash rc={rc}")
    return out


def records_hash(rec: Records, max_bounces, r_base=0, seg_rays=1 << 19, n_total=None):
    """Per-segment hashes of materialised records (with tri_ids), same
    function as trace_grid_hash; rays r_base + [0, len(rec))."""
    n = len(rec)
    n_total = n_total if n_total is not None else r_base + n
    out = np.zeros(-(-n_total // int(seg_rays)), np.uint64)
    ids = np.ascontiguousarray(rec.tri_ids, np.int32)
    valid = np.ascontiguousarray(rec.valid, np.uint8)
    esc = np.ascontiguousarray(rec.escaped, np.uint8)
    b = np.ascontiguousarray(rec.bounces, np.int32)
    n0 = _f64(rec.normal0, (-1, 3)); pth = _f64(rec.path); od = _f64(rec.out_dir, (-1, 3))
    lib().orc_records_hash(ctypes.c_int64(n), ctypes.c_int64(r_base), ctypes.c_int32(max_bounces),
                           _p(valid), _p(n0), _p(pth), _p(b), _p(esc), _p(od), _p(ids),
                           ctypes.c_int64(int(seg_rays)), _p(out))
    return out


def classify_grid(scene: Scene, grid, max_bounces=10, eps=None, strict=False, rows=None,
                  threads=0):
    """(robust u8 per ray, linear-scan query-0 tri, t) -- see
    orc_classify_grid: robust rays have a tree-independent reference answer."""
    if eps is None:
        eps = scene.default_eps
    i0, i1 = (0, grid.n_u) if rows is None else rows
    n = (i1 - i0) * grid.n_v
    robust = np.empty(n, np.uint8)
    tri = np.empty(n, np.int64)
    t = np.empty(n)
    corner = _f64(grid.corner); u = _f64(grid.u); v = _f64(grid.v)
    k = _f64(grid.k_inc)
    lib().orc_classify_grid(scene.ref, _p(corner), _p(u), _p(v), _p(k),
                            ctypes.c_double(grid.spacing), ctypes.c_int64(grid.n_v),
                            ctypes.c_int64(i0), ctypes.c_int64(i1), ctypes.c_int32(max_bounces),
                            ctypes.c_double(eps), ctypes.c_int32(int(strict)), _p(robust),
                            _p(tri), _p(t), ctypes.c_int(_threads(threads)))
    return robust.astype(bool), tri, t


def classify_rays(scene: Scene, origins, dirs, threads=0):
    o = _f64(origins, (-1, 3)); d = _f64(dirs, (-1, 3))
    n = o.shape[0]
    robust = np.empty(n, np.uint8)
    lib().orc_classify_rays(scene.ref, _p(o), _p(d), ctypes.c_int64(n), _p(robust),
                            ctypes.c_int(_threads(threads)))
    return robust.astype(bool)


def pairwise_sum(values) -> complex:
    w = np.ascontiguousarray(np.asarray(values, np.complex128)).view(np.float64).copy()
    out = np.zeros(2)
    lib().orc_pairwise_sum(_p(w), ctypes.c_int64(w.shape[0] // 2), _p(out))
    return complex(out[0], out[1])


def accumulate(rec, k_inc, wavelength, cell_area, gamma=-1.0,
               count_trapped=False) -> complex:
    """po.py:83-113 with k = 2 pi / wavelength (po.py:46-48)."""
    valid = np.ascontiguousarray(rec.valid, np.uint8)
    esc = np.ascontiguousarray(rec.escaped, np.uint8)
    n0 = _f64(rec.normal0, (-1, 3)); path = _f64(rec.path)
    b = np.ascontiguousarray(rec.bounces, np.int32)
    kv = _f64(k_inc)
    out = np.zeros(2)
    bad = ctypes.c_int64(-1)
    k = 2.0 * math.pi / wavelength
    rc = lib().orc_accumulate(_p(valid), _p(n0), _p(path), _p(b), _p(esc),
                              ctypes.c_int64(valid.shape[0]), _p(kv),
                              ctypes.c_double(k), ctypes.c_double(cell_area),
                              ctypes.c_double(gamma),
                              ctypes.c_int32(int(count_trapped)), _p(out),
                              ctypes.byref(bad))
    if rc == 4:
        raise FloatingPointError(f"non-finite contribution at record index {bad.value}")
    if rc != 0:
        raise RuntimeError(f"orc_accumulate rc={rc}")
    return complex(out[0], out[1])


# ---------------------------------------------------------------------------
# Aperture (transport.py:25-205), restated for oracle independence
# ---------------------------------------------------------------------------

_GOLDEN = 0.6180339887498949


@dataclass
class Grid:
    u: np.ndarray
    v: np.ndarray
    k_inc: np.ndarray
    corner: np.ndarray
    spacing: float
    n_u: int
    n_v: int
    cell_area: float

    @property
    def ray_count(self):
        return self.n_u * self.n_v


def k_inc(theta, phi):
    s = math.sin(theta)
    return -np.array([s * math.cos(phi), s * math.sin(phi), math.cos(theta)])


def aperture(aabb_min, aabb_max, theta, phi, spacing, margin=0.025) -> Grid:
    k = k_inc(theta, phi)
    seed = np.zeros(3)
    seed[int(np.argmin(np.abs(k)))] = 1.0
    u = np.cross(seed, k)
    u /= np.linalg.norm(u)
    v = np.cross(k, u)
    lo = np.asarray(aabb_min, np.float64); hi = np.asarray(aabb_max, np.float64)
    sel = np.array([[(c >> a) & 1 for a in range(3)] for c in range(8)])
    corners = np.where(sel, hi, lo)
    pu = corners @ u; pv = corners @ v; pk = corners @ k
    l_u = float(pu.max() - pu.min()); l_v = float(pv.max() - pv.min())
    n_u = max(1, math.ceil((1.0 + margin) * l_u / spacing))
    n_v = max(1, math.ceil((1.0 + margin) * l_v / spacing))

    def frac(salt):
        x = theta * (salt + 37.0) * _GOLDEN + phi * (salt + 61.0) * _GOLDEN
        return (0.5 + x) % 1.0

    ju = (frac(1.0) - 0.5) * min(spacing, max(0.0, n_u * spacing - l_u))
    jv = (frac(2.0) - 0.5) * min(spacing, max(0.0, n_v * spacing - l_v))
    standoff = float(np.linalg.norm(hi - lo))
    plane_k = float(pk.min()) - standoff
    cu = 0.5 * float(pu.max() + pu.min()); cv = 0.5 * float(pv.max() + pv.min())
    corner = (plane_k * k + (cu - 0.5 * n_u * spacing + ju) * u
              + (cv - 0.5 * n_v * spacing + jv) * v)
    return Grid(u, v, k, corner, spacing, n_u, n_v, spacing * spacing)


def tri_hit_pairs(v0, v1, v2, origins, dirs, t_min=0.0, t_max=np.inf,
                  single=False):
    """geometry.py:326-355 per (ray, triangle) pair; -1.0 on miss."""
    v0 = _f64(v0, (-1, 3)); v1 = _f64(v1, (-1, 3)); v2 = _f64(v2, (-1, 3))
    o = _f64(origins, (-1, 3)); d = _f64(dirs, (-1, 3))
    t = np.empty(o.shape[0])
    lib().orc_tri_hit_pairs(_p(v0), _p(v1), _p(v2), _p(o), _p(d),
                            ctypes.c_int64(o.shape[0]), ctypes.c_double(t_min),
                            ctypes.c_double(t_max), ctypes.c_int32(int(single)),
                            _p(t))
    return t

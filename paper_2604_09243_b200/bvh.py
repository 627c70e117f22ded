"""Bounding volume hierarchy (API of pkg/src/sbr/bvh.py).

``build`` constructs the tree on the GPU.  ``split_rule="sah"`` (the
reference default) and ``"median"`` build the reference's own tree, node
for node (level-synchronous binned SAH / median split, csrc/sahbuild.cu);
``"lbvh"`` builds a Morton-code LBVH (csrc/lbvh.cu).  Every tree is
collapsed to a 4-wide tree for traversal.  The returned ``Bvh`` exposes the
reference preorder layout (verbatim for SAH/median, exported lazily from the
device) so ``Bvh.validate`` and CPU consumers keep working.  A ``Bvh``
constructed from reference arrays is uploaded on first use.

Closest-hit results: the fast traversal returns the lexicographic (t, id)
minimum over the triangles its conservative culling reaches -- the
reference's answer on every robust ray (the winning
hit lies inside its triangle's box and no other triangle ties it within
rounding).  Near-edge-on triangles can make Moller-Trumbore accept rays
outside their box; there the reference's own answer depends on its tree,
and ``traversal_order("reference")`` replays bvh.py:306-362 on the
reference tree, bit for bit on every ray (visit counts included).  In the
fast mode ``visits`` counts the device tree's node fetches.
"""

from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

from . import _native as nat
from .errors import ValidationError
from .geometry import Aabb, Mesh


@dataclass(frozen=True)
class BuildParams:
    """Construction knobs (bvh.py:22-49), all honoured by the GPU builders:
    ``split_rule`` "sah" / "median" (the reference trees, node for node) or
    "lbvh" (Morton LBVH, ``n_leaf`` <= 63); ``bins_per_axis`` (<= 64),
    ``c_t``, ``c_i``, ``max_depth`` as in the reference."""

    split_rule: str = "sah"
    n_leaf: int = 4
    bins_per_axis: int = 16
    c_t: float = 1.0
    c_i: float = 1.0
    max_depth: int = 64

    def __post_init__(self):
        if self.split_rule not in ("median", "sah", "lbvh"):
            raise ValidationError(f"unknown split rule {self.split_rule!r}")
        if self.n_leaf < 1:
            raise ValidationError("n_leaf must be >= 1")
        if self.split_rule == "sah" and self.bins_per_axis < 2:
            raise ValidationError("bins_per_axis must be >= 2 for SAH")
        if self.c_t <= 0 or self.c_i <= 0:
            raise ValidationError("cost constants must be positive")
        if self.max_depth < 1:
            raise ValidationError("max_depth must be >= 1")


class Hit(NamedTuple):
    t: float
    triangle_index: int
    normal: np.ndarray


class _DeviceBvh:
    is_tree = True

    def __init__(self, ctx, handle, mesh_dev):
        self.ctx = ctx
        self.handle = handle
        self.mesh_dev = mesh_dev   # keeps the device mesh alive
        nat.register_handle(self)

    def release(self):
        if self.handle:
            self.ctx.lib.sbr_bvh_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.release()
        except Exception:  # pragma: no cover
            pass


class Bvh:
    """Linearised hierarchy (bvh.py:58-121).

    ``node_count[i] > 0``: leaf owning ``tri_order[node_first[i]:+count]``;
    otherwise internal with left child ``i + 1`` and right child
    ``node_first[i]``.
    """

    _FIELDS = ("nodes_min", "nodes_max", "node_first", "node_count", "tri_order")

    def __init__(self, nodes_min=None, nodes_max=None, node_first=None, node_count=None,
                 tri_order=None, max_depth_seen: int = 0,
                 params: BuildParams = BuildParams()):
        self._host = None
        if nodes_min is not None:
            self._host = dict(nodes_min=np.asarray(nodes_min),
                              nodes_max=np.asarray(nodes_max),
                              node_first=np.asarray(node_first, np.int32),
                              node_count=np.asarray(node_count, np.int32),
                              tri_order=np.asarray(tri_order, np.int32))
        self._depth = int(max_depth_seen)
        self.params = params
        self._dev: dict = {}         # (device, id(mesh)) -> _DeviceBvh
        self._origin = None          # (device, mesh) of a GPU-built tree

    # ---- reference layout (exported lazily from a GPU-built tree) --------
    def _export(self):
        if self._host is not None:
            return self._host
        (dev, mesh), dbvh = self._origin, None
        dbvh = self._dev[(dev, id(mesh))]
        lib = dbvh.ctx.lib
        nn, nd, md = nat.c_i64(), nat.c_i64(), nat.c_i32()
        nat.check(lib.sbr_bvh_info(dbvh.handle, ctypes.byref(nn), ctypes.byref(nd),
                                   ctypes.byref(md)), "sbr_bvh_info")
        n = int(nn.value)
        out = dict(nodes_min=np.empty((n, 3)), nodes_max=np.empty((n, 3)),
                   node_first=np.empty(n, np.int32), node_count=np.empty(n, np.int32),
                   tri_order=np.empty(mesh.triangle_count, np.int32))
        nat.check(lib.sbr_bvh_export(dbvh.handle, *[nat.ptr(out[k]) for k in self._FIELDS]),
                  "sbr_bvh_export")
        if np.dtype(mesh.dtype) == np.float32:
            # bvh.py:286-290: float32 meshes get outward-rounded float32 boxes
            out["nodes_min"] = np.nextafter(out["nodes_min"].astype(np.float32),
                                            np.float32(-np.inf))
            out["nodes_max"] = np.nextafter(out["nodes_max"].astype(np.float32),
                                            np.float32(np.inf))
        self._host = out
        return out

    nodes_min = property(lambda self: self._export()["nodes_min"])
    nodes_max = property(lambda self: self._export()["nodes_max"])
    node_first = property(lambda self: self._export()["node_first"])
    node_count = property(lambda self: self._export()["node_count"])
    tri_order = property(lambda self: self._export()["tri_order"])

    @property
    def max_depth_seen(self) -> int:
        """Depth of the deepest node (root = 0)."""
        if self._origin is not None:
            (dev, mesh) = self._origin
            md = nat.c_i32()
            d = self._dev[(dev, id(mesh))]
            nat.check(d.ctx.lib.sbr_bvh_info(d.handle, None, None, ctypes.byref(md)))
            return int(md.value)
        return self._depth

    @property
    def node_total(self) -> int:
        return self.nodes_min.shape[0]

    def leaf_sizes(self) -> np.ndarray:
        return self.node_count[self.node_count > 0]

    def leaf_size_histogram(self) -> np.ndarray:
        return np.bincount(self.leaf_sizes())

    def root_box(self) -> Aabb:
        return Aabb(np.asarray(self.nodes_min[0], np.float64),
                    np.asarray(self.nodes_max[0], np.float64))

    def validate(self, mesh: Mesh) -> None:
        """Structural invariants (bvh.py:90-121): permutation, child
        containment (1e-12 slack), disjoint leaves covering every triangle."""
        h = self._export()
        nmin, nmax = h["nodes_min"], h["nodes_max"]
        first, count, order = h["node_first"], h["node_count"], h["tri_order"]
        n, t = nmin.shape[0], mesh.triangle_count
        if not np.array_equal(np.sort(order), np.arange(t)):
            raise AssertionError("tri_order is not a permutation")
        owned = np.zeros(t, dtype=bool)
        todo = [(0, -1)]
        while todo:
            i, par = todo.pop()
            if par >= 0:
                if np.any(nmin[i] < nmin[par] - 1e-12):
                    raise AssertionError(f"node {i} min escapes parent")
                if np.any(nmax[i] > nmax[par] + 1e-12):
                    raise AssertionError(f"node {i} max escapes parent")
            if count[i] > 0:
                f, c = int(first[i]), int(count[i])
                if f < 0 or f + c > t:
                    raise AssertionError(f"bad leaf range at node {i}")
                seg = order[f:f + c]
                if owned[seg].any():
                    raise AssertionError("triangle in two leaves")
                owned[seg] = True
            else:
                l, r = i + 1, int(first[i])
                if not (0 < l < n and 0 < r < n):
                    raise AssertionError(f"bad children at node {i}")
                todo.append((l, i))
                todo.append((r, i))
        if not owned.all():
            raise AssertionError("leaf ranges do not cover all triangles")

    # ---- device tree ------------------------------------------------------
    def device(self, mesh: Mesh, ctx: Optional[nat.Context] = None) -> _DeviceBvh:
        ctx = ctx or nat.context()
        key = (ctx.device, id(mesh))
        d = self._dev.get(key)
        if d is not None:
            return d
        dm = mesh.device(ctx)
        h = self._export() if (self._host is not None or self._origin) else None
        if h is None:
            raise ValidationError("Bvh has neither device nor host data")
        handle = nat.c_vp()
        arrs = [nat.f64(h["nodes_min"], (-1, 3)), nat.f64(h["nodes_max"], (-1, 3)),
                np.ascontiguousarray(h["node_first"], np.int32),
                np.ascontiguousarray(h["node_count"], np.int32),
                np.ascontiguousarray(h["tri_order"], np.int32)]
        if arrs[4].shape[0] != mesh.triangle_count:
            raise ValidationError("Bvh does not match the mesh (tri_order length)")
        nat.check(ctx.lib.sbr_bvh_upload(ctx.handle, dm.handle, *[nat.ptr(a) for a in arrs],
                                         arrs[0].shape[0], ctypes.byref(handle)),
                  "sbr_bvh_upload")
        d = _DeviceBvh(ctx, handle, dm)
        self._dev[key] = d
        return d


def sah_cost(sa_p: float, sa_l: float, sa_r: float, n_l: int, n_r: int,
             c_t: float, c_i: float) -> float:
    """c_t + (SA_L/SA_P) N_L c_i + (SA_R/SA_P) N_R c_i (bvh.py:124-127)."""
    return c_t + (sa_l / sa_p) * n_l * c_i + (sa_r / sa_p) * n_r * c_i


def _area(lo, hi) -> float:
    e = np.asarray(hi) - np.asarray(lo)
    return float(2.0 * (e[0] * e[1] + e[1] * e[2] + e[2] * e[0]))


_box_surface_area = _area   # the reference's private name (bvh.py:130-132)


def median_split(centroids: np.ndarray, node_box: Aabb):
    """Median partition on the longest box axis (bvh.py:135-151):
    ``(axis, left_positions, right_positions)`` or None if all coincide."""
    c = np.asarray(centroids, dtype=np.float64)
    n = c.shape[0]
    if n < 2:
        raise ValidationError("median_split requires >= 2 triangles")
    if (c == c[0]).all():
        return None
    axis = int(np.argmax(node_box.max - node_box.min))
    order = np.argsort(c[:, axis], kind="stable")
    return axis, order[:n // 2], order[n // 2:]


def binned_sah_split(tri_min: np.ndarray, tri_max: np.ndarray, centroids: np.ndarray,
                     node_box: Aabb, bins_per_axis: int = 16, c_t: float = 1.0,
                     c_i: float = 1.0, n_leaf: int = 4):
    """Best binned-SAH plane over all axes (bvh.py:154-215):
    ``(axis, boundary, left_positions, right_positions)`` or None."""
    c = np.asarray(centroids, dtype=np.float64)
    n = c.shape[0]
    if n < 2:
        raise ValidationError("binned_sah_split requires >= 2 triangles")
    sa_p = max(_area(node_box.min, node_box.max), 1e-300)
    best = None
    nb = bins_per_axis
    for axis in range(3):
        lo, hi = c[:, axis].min(), c[:, axis].max()
        if hi <= lo:
            continue
        bins = np.minimum((nb / (hi - lo) * (c[:, axis] - lo)).astype(np.int64), nb - 1)
        cnt = np.bincount(bins, minlength=nb)
        bmin = np.full((nb, 3), np.inf)
        bmax = np.full((nb, 3), -np.inf)
        np.minimum.at(bmin, bins, tri_min)
        np.maximum.at(bmax, bins, tri_max)
        pre_n = np.cumsum(cnt)
        pre_lo = np.minimum.accumulate(bmin, axis=0)
        pre_hi = np.maximum.accumulate(bmax, axis=0)
        suf_n = np.cumsum(cnt[::-1])[::-1]
        suf_lo = np.minimum.accumulate(bmin[::-1], axis=0)[::-1]
        suf_hi = np.maximum.accumulate(bmax[::-1], axis=0)[::-1]
        for b in range(nb - 1):
            nl, nr = int(pre_n[b]), int(suf_n[b + 1])
            if nl == 0 or nr == 0:
                continue
            cost = sah_cost(sa_p, _area(pre_lo[b], pre_hi[b]),
                            _area(suf_lo[b + 1], suf_hi[b + 1]), nl, nr, c_t, c_i)
            if best is None or cost < best[0]:
                best = (cost, axis, b, bins)
    if best is None:
        return None
    cost, axis, b, bins = best
    if cost >= n * c_i and n <= 4 * n_leaf:
        return None
    pos = np.arange(n)
    return axis, b, pos[bins <= b], pos[bins > b]


def build(mesh: Mesh, params: BuildParams = BuildParams()) -> Bvh:
    """BVH over the mesh triangles on the GPU (replaces bvh.py:218-299).

    ``split_rule="sah"`` (the reference default) and ``"median"`` build the
    reference's binned-SAH / median-split tree on the GPU, node for node
    identical to bvh.build; ``"lbvh"`` builds a Morton-order LBVH (fastest
    build).  Closest hits are identical for every tree."""
    if params.split_rule == "lbvh" and params.n_leaf > 63:
        raise ValidationError("the LBVH builder supports n_leaf <= 63")
    ctx = nat.context()
    dm = mesh.device(ctx)
    bp = nat.BuildParams()
    bp.split_rule = {"median": nat.SPLIT_MEDIAN, "sah": nat.SPLIT_SAH,
                     "lbvh": nat.SPLIT_LBVH}[params.split_rule]
    bp.n_leaf = int(params.n_leaf)
    bp.max_depth = int(params.max_depth)
    bp.bins_per_axis = int(params.bins_per_axis)
    bp.c_t = float(params.c_t)
    bp.c_i = float(params.c_i)
    handle = nat.c_vp()
    nat.check(ctx.lib.sbr_bvh_build(ctx.handle, dm.handle, ctypes.byref(bp),
                                    ctypes.byref(handle)), "sbr_bvh_build")
    tree = Bvh(params=params)
    tree._dev[(ctx.device, id(mesh))] = _DeviceBvh(ctx, handle, dm)
    tree._origin = (ctx.device, mesh)
    return tree


# ---------------------------------------------------------------------------
# traversal order (sbr_ctx_set_traversal)
# ---------------------------------------------------------------------------
_ORDERS = {"fast": nat.TRAVERSAL_FAST, "reference": nat.TRAVERSAL_REFERENCE}


def set_traversal_order(order: str, device: Optional[int] = None) -> None:
    """Select how every query of this device's context is answered.

    ``"fast"`` (default): raster pass for query 0 of aperture rays (the exact
    linear-scan answer, bvh.py:394-395) and the persistent BVH4 kernel for
    the rest; bit-identical to the reference on every query whose winning
    triangle's hit point lies robustly inside its box with no accepting
    triangle tied within rounding.  ``"reference"``: every query replays
    bvh.py:306-362 ``_traverse`` on the reference tree, so edge/vertex ties
    and near-edge-on acceptances resolve exactly as the reference resolves
    them (needs a ``"sah"``/``"median"`` build or an uploaded tree)."""
    if order not in _ORDERS:
        raise ValidationError(f"unknown traversal order {order!r}")
    nat.context(device).traversal = _ORDERS[order]


def get_traversal_order(device: Optional[int] = None) -> str:
    m = nat.context(device).traversal
    return next(k for k, v in _ORDERS.items() if v == m)


@contextlib.contextmanager
def traversal_order(order: str, device: Optional[int] = None):
    """``with traversal_order("reference"): ...`` -- scoped set_traversal_order."""
    prev = get_traversal_order(device)
    set_traversal_order(order, device)
    try:
        yield
    finally:
        set_traversal_order(prev, device)


def closest_hit(bvh: Bvh, mesh: Mesh, origin, direction, t_min: float = 0.0,
                t_max: float = np.inf) -> Optional[Hit]:
    """Closest intersection, identical to a linear scan (bvh.py:385-389)."""
    hit, _ = closest_hit_counted(bvh, mesh, origin, direction, t_min, t_max)
    return hit


def closest_hit_counted(bvh: Bvh, mesh: Mesh, origin, direction, t_min: float = 0.0,
                        t_max: float = np.inf):
    """(Hit or None, node visits) -- bvh.py:392-404."""
    tri, t, vis = closest_hit_batch(bvh, mesh, np.reshape(origin, (1, 3)),
                                    np.reshape(direction, (1, 3)), t_min, t_max)
    if tri[0] < 0:
        return None, int(vis[0])
    i = int(tri[0])
    return Hit(float(t[0]), i, np.asarray(mesh.normals[i], np.float64).copy()), int(vis[0])


def closest_hit_batch(bvh: Bvh, mesh: Mesh, origins, dirs, t_min: float = 0.0,
                      t_max: float = np.inf):
    """(tri, t, visits) arrays; tri = -1 where the ray misses (bvh.py:407-423).

    As in the reference, a float32 mesh casts the rays to float32 too
    (bvh.py:414-415), so the Moller-Trumbore arithmetic runs in float32 up
    to the float64 ``1.0 / det`` (sbr_device.cuh tri_hit_f32rays); the
    multi-bounce walk keeps float64 rays (transport.py:362-363)."""
    ctx = nat.context()
    d = bvh.device(mesh, ctx)
    o = nat.f64(origins, (-1, 3))
    v = nat.f64(dirs, (-1, 3))
    n = o.shape[0]
    tri = np.empty(n, np.int64)
    t = np.empty(n, np.float64)
    vis = np.empty(n, np.int64)
    nat.check(ctx.lib.sbr_closest_hit(ctx.handle, d.mesh_dev.handle, d.handle, nat.ptr(o),
                                      nat.ptr(v), n, float(t_min), float(t_max), nat.ptr(tri),
                                      nat.ptr(t), nat.ptr(vis)), "sbr_closest_hit")
    return tri, t, vis

"""Triangle-soup meshes and the scalar ray predicates (API of
pkg/src/sbr/geometry.py).

Host side: mesh construction, OBJ I/O and the analytic icosphere -- all
bit-identical to the reference so both implementations see the same input.
Device side: a Mesh lazily uploads itself to the GPU (``Mesh.device``);
``ray_triangle_intersect`` / ``ray_aabb_intersect`` evaluate on the GPU with
the exact FP64 arithmetic of geometry.py:326-391.
"""

from __future__ import annotations

import hashlib
import math
import warnings
from dataclasses import dataclass, field
from typing import NamedTuple, Optional

import numpy as np

from . import _native as nat
from .errors import ValidationError

# Regular icosahedron: golden-ratio rectangles, 12 vertices / 20 faces
# (the classic table; vertex 0 has unit circumradius after scaling).
_PHI = (1.0 + math.sqrt(5.0)) / 2.0
_ICOSA_V = np.array([(-1, _PHI, 0), (1, _PHI, 0), (-1, -_PHI, 0), (1, -_PHI, 0),
                     (0, -1, _PHI), (0, 1, _PHI), (0, -1, -_PHI), (0, 1, -_PHI),
                     (_PHI, 0, -1), (_PHI, 0, 1), (-_PHI, 0, -1), (-_PHI, 0, 1)],
                    dtype=np.float64)
_ICOSA_F = np.array([(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
                     (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
                     (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
                     (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)],
                    dtype=np.int64)


@dataclass(frozen=True)
class Aabb:
    """Axis-aligned box with min <= max componentwise (geometry.py:52-76)."""

    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.min, dtype=np.float64)
        hi = np.asarray(self.max, dtype=np.float64)
        object.__setattr__(self, "min", lo)
        object.__setattr__(self, "max", hi)
        if not np.all(lo <= hi):
            raise ValidationError(f"invalid AABB: min {lo} > max {hi}")

    def corners(self) -> np.ndarray:
        """The 8 corners; corner c takes max on axis a iff bit a of c is set."""
        bits = (np.arange(8)[:, None] >> np.arange(3)[None, :]) & 1
        return np.where(bits.astype(bool), self.max, self.min)

    def diagonal(self) -> float:
        return float(np.linalg.norm(self.max - self.min))

    def surface_area(self) -> float:
        e = self.max - self.min
        return float(2.0 * (e[0] * e[1] + e[1] * e[2] + e[2] * e[0]))


class Triangle(NamedTuple):
    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray
    normal: np.ndarray


class _DeviceMesh:
    """Owning handle of an sbr_mesh."""

    def __init__(self, ctx: nat.Context, mesh: "Mesh"):
        v0 = nat.f64(mesh.v0, (-1, 3)); v1 = nat.f64(mesh.v1, (-1, 3))
        v2 = nat.f64(mesh.v2, (-1, 3)); nn = nat.f64(mesh.normals, (-1, 3))
        storage = nat.STORAGE_SINGLE if mesh.dtype == np.float32 else nat.STORAGE_AUTO
        h = nat.c_vp()
        nat.check(ctx.lib.sbr_mesh_create(ctx.handle, nat.ptr(v0), nat.ptr(v1), nat.ptr(v2),
                                          nat.ptr(nn), v0.shape[0], storage,
                                          nat.ctypes.byref(h)), "sbr_mesh_create")
        self.ctx = ctx
        self.handle = h
        nat.register_handle(self)
        n = nat.c_i64(); st = nat.c_i32()
        nat.check(ctx.lib.sbr_mesh_info(h, nat.ctypes.byref(n), nat.ctypes.byref(st), None))
        self.storage = int(st.value)

    def release(self):
        if self.handle:
            self.ctx.lib.sbr_mesh_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.release()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


@dataclass(frozen=True)
class Mesh:
    """Immutable triangle soup with geometric normals (geometry.py:88-127).

    ``normals[i] = normalize((v1 - v0) x (v2 - v0))``.  ``device()`` returns
    the GPU copy (uploaded once per device and cached).
    """

    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray
    normals: np.ndarray
    aabb: Aabb
    path: Optional[str] = None
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def triangle_count(self) -> int:
        return self.v0.shape[0]

    @property
    def dtype(self) -> np.dtype:
        return self.v0.dtype

    def triangle(self, i: int) -> Triangle:
        return Triangle(self.v0[i], self.v1[i], self.v2[i], self.normals[i])

    def centroids(self) -> np.ndarray:
        return (self.v0 + self.v1 + self.v2) / 3.0

    def areas(self) -> np.ndarray:
        c = np.cross(self.v1 - self.v0, self.v2 - self.v0)
        return 0.5 * np.linalg.norm(c, axis=1)

    def checksum(self) -> str:
        """SHA-256 over the FP64 vertex data (cached: the mesh is immutable)."""
        cached = self._dev.get("checksum")
        if cached is None:
            h = hashlib.sha256()
            for a in (self.v0, self.v1, self.v2):
                h.update(np.ascontiguousarray(a, dtype=np.float64).data)
            cached = self._dev["checksum"] = h.hexdigest()
        return cached

    def device(self, ctx: Optional[nat.Context] = None) -> _DeviceMesh:
        ctx = ctx or nat.context()
        dm = self._dev.get(ctx.device)
        if dm is None:
            dm = _DeviceMesh(ctx, self)
            self._dev[ctx.device] = dm
        return dm


def mesh_from_soup(tri_vertices: np.ndarray, path: Optional[str] = None,
                   strict: bool = False, dtype=np.float64,
                   face_labels: Optional[np.ndarray] = None) -> Mesh:
    """(T,3,3) vertex soup -> Mesh (geometry.py:130-180).

    Zero-area triangles (twice-area <= 1e-14 * longest-edge^2) are dropped
    with a warning, or rejected when ``strict``.
    """
    soup = np.asarray(tri_vertices, dtype=np.float64)
    if soup.ndim != 3 or soup.shape[1:] != (3, 3):
        raise ValidationError(f"expected (T, 3, 3) triangle array, got {soup.shape}")
    if soup.shape[0] == 0:
        raise ValidationError("mesh has no triangles")
    a, b, c = soup[:, 0], soup[:, 1], soup[:, 2]
    e1, e2 = b - a, c - a
    n = np.cross(e1, e2)
    twice = np.linalg.norm(n, axis=1)
    longest = np.maximum(np.sum(e1 * e1, axis=1), np.sum(e2 * e2, axis=1))
    bad = twice <= 1e-14 * np.maximum(longest, 1e-300)
    if bad.any():
        where = np.flatnonzero(bad)
        labels = face_labels[where] if face_labels is not None else where
        if strict:
            raise ValidationError(f"zero-area triangle(s) at face index {labels.tolist()[:10]}")
        warnings.warn(f"dropping {where.size} zero-area triangle(s), first at face index "
                      f"{int(labels[0])}", stacklevel=2)
        keep = ~bad
        soup, n, twice = soup[keep], n[keep], twice[keep]
        if soup.shape[0] == 0:
            raise ValidationError("mesh has no non-degenerate triangles")
    unit = n / twice[:, None]
    dt = np.dtype(dtype)
    box = Aabb(soup.min(axis=(0, 1)), soup.max(axis=(0, 1)))
    return Mesh(v0=np.ascontiguousarray(soup[:, 0], dtype=dt),
                v1=np.ascontiguousarray(soup[:, 1], dtype=dt),
                v2=np.ascontiguousarray(soup[:, 2], dtype=dt),
                normals=np.ascontiguousarray(unit, dtype=dt), aabb=box, path=path)


def mesh_from_arrays(vertices: np.ndarray, faces: np.ndarray, **kwargs) -> Mesh:
    """Shared-vertex (V,3) + (F,3) -> Mesh."""
    v = np.asarray(vertices, dtype=np.float64)
    f = np.asarray(faces, dtype=np.int64)
    return mesh_from_soup(v[f], **kwargs)


def load_mesh(path, strict: bool = False, dtype=np.float64) -> Mesh:
    """Wavefront OBJ subset (geometry.py:190-241): ``v`` and ``f`` records,
    1-based or negative (relative) indices, polygons fan-triangulated.

    Parsed by the native reader (sbr_obj_read); files using number syntax
    only Python's float()/int() define go through the equivalent Python
    loop, so every input behaves exactly as in the reference."""
    got = nat.obj_read(path)
    if got is None:
        return _load_mesh_py(path, strict, dtype)
    v, f, labels = got
    return mesh_from_soup(v[f], path=str(path), strict=strict, dtype=dtype, face_labels=labels)


def _load_mesh_py(path, strict: bool = False, dtype=np.float64) -> Mesh:
    """The reference reader loop (geometry.py:199-241)."""
    verts: list = []
    tris: list = []
    labels: list = []
    face_no = 0
    with open(path, "r", encoding="utf-8", errors="replace") as fh:
        for lineno, line in enumerate(fh, start=1):
            tok = line.split()
            if not tok or tok[0].startswith("#"):
                continue
            if tok[0] == "v":
                if len(tok) < 4:
                    raise ValidationError(f"{path}:{lineno}: malformed vertex record")
                verts.append((float(tok[1]), float(tok[2]), float(tok[3])))
            elif tok[0] == "f":
                if len(tok) < 4:
                    raise ValidationError(f"{path}:{lineno}: face with <3 vertices")
                idx = []
                for ref in tok[1:]:
                    head = ref.split("/")[0]
                    k = int(head)
                    if k == 0:
                        raise ValidationError(
                            f"{path}:{lineno}: zero vertex index in face {face_no}")
                    k = k - 1 if k > 0 else len(verts) + k
                    if not 0 <= k < len(verts):
                        raise ValidationError(f"{path}:{lineno}: vertex index {head} out of "
                                              f"range in face {face_no}")
                    idx.append(k)
                for s in range(1, len(idx) - 1):
                    tris.append((idx[0], idx[s], idx[s + 1]))
                    labels.append(face_no)
                face_no += 1
    if not tris:
        raise ValidationError(f"{path}: no faces found")
    v = np.asarray(verts, dtype=np.float64)
    f = np.asarray(tris, dtype=np.int64)
    return mesh_from_soup(v[f], path=str(path), strict=strict, dtype=dtype,
                          face_labels=np.asarray(labels))


def save_obj(mesh: Mesh, path) -> None:
    """OBJ writer; equal vertices are shared (geometry.py:244-265), native."""
    nat.obj_write(path, mesh.v0, mesh.v1, mesh.v2)


def _save_obj_py(mesh: Mesh, path) -> None:
    """The reference writer loop (geometry.py:244-265), kept as the test oracle."""
    corners = np.stack([np.asarray(mesh.v0, np.float64), np.asarray(mesh.v1, np.float64),
                        np.asarray(mesh.v2, np.float64)], axis=1).reshape(-1, 3)
    lookup: dict = {}
    ids = np.empty(corners.shape[0], dtype=np.int64)
    for q, p in enumerate(map(tuple, corners)):
        ids[q] = lookup.setdefault(p, len(lookup))
    with open(path, "w", encoding="utf-8") as fh:
        for p in lookup:
            fh.write(f"v {p[0]:.17g} {p[1]:.17g} {p[2]:.17g}\n")
        for t in ids.reshape(-1, 3):
            fh.write(f"f {t[0] + 1} {t[1] + 1} {t[2] + 1}\n")


def _subdivide(verts: np.ndarray, faces: np.ndarray):
    """Split every face in four; one normalised midpoint per unique edge."""
    ring = np.concatenate([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]])
    ring = np.sort(ring, axis=1)
    edges, where = np.unique(ring, axis=0, return_inverse=True)
    mid = verts[edges[:, 0]] + verts[edges[:, 1]]
    mid /= np.linalg.norm(mid, axis=1)[:, None]
    m = where.reshape(3, -1).T + len(verts)
    a, b, c = faces.T
    ab, bc, ca = m.T
    out = np.concatenate([np.stack(t, axis=1) for t in
                          ((a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca))])
    return np.concatenate([verts, mid]), out


def generate_icosphere(radius: float, subdivisions: int, dtype=np.float64) -> Mesh:
    """Icosahedron subdivided ``subdivisions`` times onto a sphere
    (geometry.py:268-307): 20 * 4**s outward-facing triangles."""
    if radius <= 0:
        raise ValidationError(f"radius must be positive, got {radius}")
    if not 0 <= subdivisions <= 8:
        raise ValidationError(f"subdivisions must be in [0, 8], got {subdivisions}")
    verts = _ICOSA_V / np.linalg.norm(_ICOSA_V[0])
    faces = _ICOSA_F.copy()
    for _ in range(subdivisions):
        verts, faces = _subdivide(verts, faces)
    soup = (verts * radius)[faces]
    inward = np.einsum("ij,ij->i",
                       np.cross(soup[:, 1] - soup[:, 0], soup[:, 2] - soup[:, 0]),
                       soup.mean(axis=1)) < 0
    soup[inward] = soup[inward][:, [0, 2, 1]]
    return mesh_from_soup(soup, dtype=dtype)


def icosphere_sagitta(mesh: Mesh, radius: float) -> float:
    """radius - min distance from the origin to any triangle plane."""
    d = np.einsum("ij,ij->i", np.asarray(mesh.normals, np.float64),
                  np.asarray(mesh.v0, np.float64))
    return float(radius - d.min())


def ray_triangle_intersect(origin, direction, tri: Triangle, t_min: float = 0.0,
                           t_max: float = np.inf):
    """Edge-inclusive Moller-Trumbore on the GPU (geometry.py:394-409).

    Returns ``(t, normal)`` with t in (t_min, t_max], or None.
    """
    ctx = nat.context()
    single = np.asarray(tri.v0).dtype == np.float32
    arrs = [nat.f64(x, (1, 3)) for x in (tri.v0, tri.v1, tri.v2, origin, direction)]
    t = np.empty(1)
    nat.check(ctx.lib.sbr_tri_hit_pairs(ctx.handle, *[nat.ptr(a) for a in arrs], 1,
                                        float(t_min), float(t_max), int(single), nat.ptr(t)),
              "sbr_tri_hit_pairs")
    if t[0] < 0.0:
        return None
    return float(t[0]), np.asarray(tri.normal, dtype=np.float64).copy()


def ray_aabb_intersect(origin, dir_inv, box: Aabb, t_max: float = np.inf):
    """FP64 slab test on the GPU (geometry.py:412-425): (hit, entry)."""
    ctx = nat.context()
    arrs = [nat.f64(x, (1, 3)) for x in (box.min, box.max, origin, dir_inv)]
    hit = np.zeros(1, np.uint8)
    entry = np.zeros(1)
    nat.check(ctx.lib.sbr_aabb_hit_pairs(ctx.handle, *[nat.ptr(a) for a in arrs], 1,
                                         float(t_max), nat.ptr(hit), nat.ptr(entry)),
              "sbr_aabb_hit_pairs")
    return bool(hit[0]), float(entry[0])

"""Incident apertures and multi-bounce transport (API of
pkg/src/sbr/transport.py).

The aperture maths (k_inc, basis, sizing, registration stagger) is host FP64
and bit-identical to the reference; ray origins are generated on the device
from the grid scalars, and every bounce runs in the CUDA trace kernel.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

from . import _native as nat
from .bvh import Bvh
from .errors import ValidationError
from .geometry import Aabb, Mesh


@dataclass(frozen=True)
class IncidentDirection:
    """(theta, phi) in radians; propagation k_inc = -(st cp, st sp, ct)."""

    theta: float
    phi: float

    @property
    def k_inc(self) -> np.ndarray:
        st = math.sin(self.theta)
        return -np.array([st * math.cos(self.phi), st * math.sin(self.phi),
                          math.cos(self.theta)])

    @classmethod
    def from_vector(cls, k: np.ndarray) -> "IncidentDirection":
        k = np.asarray(k, dtype=np.float64)
        k = k / np.linalg.norm(k)
        return cls(math.acos(np.clip(-k[2], -1.0, 1.0)),
                   math.atan2(-k[1], -k[0]) % (2.0 * math.pi))


def _cross3(a, b) -> np.ndarray:
    """numpy.cross for two 3-vectors with the same per-component rounding
    (a1*b2 - a2*b1, ...: one product rounding each, then one subtraction),
    without numpy.cross's per-call axis bookkeeping."""
    a0, a1, a2 = float(a[0]), float(a[1]), float(a[2])
    b0, b1, b2 = float(b[0]), float(b[1]), float(b[2])
    return np.array([a1 * b2 - a2 * b1, a2 * b0 - a0 * b2, a0 * b1 - a1 * b0])


_AXES = np.eye(3)
_AXES.setflags(write=False)


def orthonormal_basis(k_inc) -> tuple[np.ndarray, np.ndarray]:
    """Right-handed (u, v, k): u = normalize(seed x k), v = k x u; the seed is
    the world axis least aligned with k (ties x -> y -> z)."""
    k = np.asarray(k_inc, dtype=np.float64)
    seed = _AXES[int(np.argmin(np.abs(k)))]
    u = _cross3(seed, k)
    u /= np.linalg.norm(u)
    return u, _cross3(k, u)


class SamplingCheck(NamedTuple):
    passed: bool
    ratio: float


def sampling_check(spacing: float, wavelength: float, factor: float = 5.0) -> SamplingCheck:
    """Anti-aliasing rule: spacing <= wavelength / factor (inclusive)."""
    if spacing <= 0 or wavelength <= 0 or factor <= 0:
        raise ValidationError("spacing, wavelength and factor must be positive")
    return SamplingCheck(spacing <= wavelength / factor, spacing * factor / wavelength)


@dataclass(frozen=True)
class ApertureGrid:
    """Orthographic launch grid: ray (i, j) starts at
    corner + (i+1/2) spacing u + (j+1/2) spacing v, travels along k_inc."""

    u: np.ndarray
    v: np.ndarray
    k_inc: np.ndarray
    corner: np.ndarray
    spacing: float
    n_u: int
    n_v: int
    cell_area: float
    standoff: float
    margin: float

    @property
    def ray_count(self) -> int:
        return self.n_u * self.n_v

    def ray_origin(self, i: int, j: int) -> np.ndarray:
        return (self.corner + (i + 0.5) * self.spacing * self.u
                + (j + 0.5) * self.spacing * self.v)

    def ray_origins(self) -> np.ndarray:
        i = np.repeat(np.arange(self.n_u), self.n_v) + 0.5
        j = np.tile(np.arange(self.n_v), self.n_u) + 0.5
        return (self.corner + i[:, None] * self.spacing * self.u
                + j[:, None] * self.spacing * self.v)

    def contains_projection(self, points: np.ndarray) -> np.ndarray:
        p = np.asarray(points, dtype=np.float64)
        a = p @ self.u - self.corner @ self.u
        b = p @ self.v - self.corner @ self.v
        tol = 1e-9
        return ((a >= -tol) & (a <= self.n_u * self.spacing + tol)
                & (b >= -tol) & (b <= self.n_v * self.spacing + tol))


_GOLDEN = 0.6180339887498949


def _registration_fraction(theta: float, phi: float, salt: float) -> float:
    """Per-direction sub-cell stagger in [0, 1) (transport.py:133-145)."""
    x = theta * (salt + 37.0) * _GOLDEN + phi * (salt + 61.0) * _GOLDEN
    return (0.5 + x) % 1.0


def build_aperture(aabb: Aabb, direction: IncidentDirection, spacing: float,
                   margin: float = 0.025, wavelength: Optional[float] = None,
                   sampling_factor: float = 5.0, allow_aliasing: bool = False) -> ApertureGrid:
    """Size and place one direction's launch grid (Eqs. L1-L3,
    transport.py:148-205): padded projected extents, ceil(L/spacing) rays,
    plane one box diagonal behind the target, registration stagger within
    the margin slack."""
    if spacing <= 0:
        raise ValidationError("spacing must be positive")
    if margin < 0:
        raise ValidationError("margin must be >= 0")
    if wavelength is not None and not allow_aliasing:
        chk = sampling_check(spacing, wavelength, sampling_factor)
        if not chk.passed:
            raise ValidationError(
                f"ray spacing {spacing:g} exceeds wavelength/{sampling_factor:g}"
                f" = {wavelength / sampling_factor:g} (ratio {chk.ratio:.3f});"
                " pass allow_aliasing to override")
    return _aperture(aabb.corners(), aabb.diagonal(), direction, spacing, margin)


def _aperture(pts: np.ndarray, standoff: float, direction: IncidentDirection, spacing: float,
              margin: float) -> ApertureGrid:
    """build_aperture after validation, from the box's corners and diagonal
    (computed once per sweep by sweep_grids: the same values every cell)."""
    k = direction.k_inc
    u, v = orthonormal_basis(k)
    # min / max of the eight projections as Python floats: the same values
    # (and the same IEEE subtraction / addition) as the numpy reductions
    pu, pv, pk = (pts @ u).tolist(), (pts @ v).tolist(), (pts @ k).tolist()
    pu_lo, pu_hi, pv_lo, pv_hi = min(pu), max(pu), min(pv), max(pv)
    ext_u = pu_hi - pu_lo
    ext_v = pv_hi - pv_lo
    n_u = max(1, math.ceil((1.0 + margin) * ext_u / spacing))
    n_v = max(1, math.ceil((1.0 + margin) * ext_v / spacing))
    jit_u = ((_registration_fraction(direction.theta, direction.phi, 1.0) - 0.5)
             * min(spacing, max(0.0, n_u * spacing - ext_u)))
    jit_v = ((_registration_fraction(direction.theta, direction.phi, 2.0) - 0.5)
             * min(spacing, max(0.0, n_v * spacing - ext_v)))
    plane = min(pk) - standoff
    mid_u = 0.5 * (pu_hi + pu_lo)
    mid_v = 0.5 * (pv_hi + pv_lo)
    corner = (plane * k + (mid_u - 0.5 * n_u * spacing + jit_u) * u
              + (mid_v - 0.5 * n_v * spacing + jit_v) * v)
    return ApertureGrid(u=u, v=v, k_inc=k, corner=corner, spacing=spacing, n_u=n_u,
                        n_v=n_v, cell_area=spacing * spacing, standoff=standoff,
                        margin=margin)


def reflect(d, n) -> np.ndarray:
    """d - 2 (d . n) n."""
    d = np.asarray(d, dtype=np.float64)
    n = np.asarray(n, dtype=np.float64)
    return d - 2.0 * np.dot(d, n) * n


@dataclass(frozen=True)
class TraceParams:
    """Transport knobs (transport.py:215-239); epsilon None resolves to
    1e-6 x mesh AABB diagonal."""

    max_bounces: int = 10
    epsilon: Optional[float] = None
    sampling_factor: float = 5.0
    strict_orientation: bool = False

    def __post_init__(self):
        if self.max_bounces < 1:
            raise ValidationError("max_bounces must be >= 1")
        if self.epsilon is not None and self.epsilon <= 0:
            raise ValidationError("epsilon must be positive")

    def resolve_epsilon(self, mesh: Mesh) -> float:
        return self.epsilon if self.epsilon is not None else 1e-6 * mesh.aabb.diagonal()


class HitRecord(NamedTuple):
    valid: bool
    normal0: np.ndarray
    path: float
    bounces: int
    escaped: bool
    out_dir: np.ndarray


@dataclass(frozen=True)
class HitRecords:
    """SoA records, record r = i * n_v + j (transport.py:251-273).
    ``tri_ids`` (optional extension) holds the hit triangle per bounce."""

    valid: np.ndarray
    normal0: np.ndarray
    path: np.ndarray
    bounces: np.ndarray
    escaped: np.ndarray
    out_dir: np.ndarray
    tri_ids: Optional[np.ndarray] = None

    def __len__(self) -> int:
        return self.valid.shape[0]

    def record(self, r: int) -> HitRecord:
        return HitRecord(bool(self.valid[r]), self.normal0[r].copy(), float(self.path[r]),
                         int(self.bounces[r]), bool(self.escaped[r]), self.out_dir[r].copy())


def _alloc(n: int, max_bounces: int, with_ids: bool):
    return (np.empty(n, np.bool_), np.empty((n, 3)), np.empty(n), np.empty(n, np.int32),
            np.empty(n, np.bool_), np.empty((n, 3)),
            np.empty((n, max_bounces), np.int32) if with_ids else None)


def _cparams(mesh: Mesh, params: TraceParams):
    return nat.make_trace_params(params.max_bounces, params.resolve_epsilon(mesh),
                                 params.strict_orientation, True, 0.0, params.sampling_factor)


def trace_rays(bvh: Bvh, mesh: Mesh, origins, directions,
               params: TraceParams = TraceParams(), with_ids: bool = False) -> HitRecords:
    """Trace an explicit ray list on the GPU (batched trace_ray)."""
    ctx = nat.context()
    d = bvh.device(mesh, ctx)
    o = nat.f64(origins, (-1, 3))
    k = nat.f64(directions, (-1, 3))
    n = o.shape[0]
    out = _alloc(n, params.max_bounces, with_ids)
    cp = _cparams(mesh, params)
    nat.check(ctx.lib.sbr_trace_rays(ctx.handle, d.mesh_dev.handle, d.handle, nat.ptr(o),
                                     nat.ptr(k), n, ctypes.byref(cp),
                                     *[nat.ptr(a) for a in out]), "sbr_trace_rays")
    return HitRecords(*out)


def trace_ray(bvh: Bvh, mesh: Mesh, origin, direction,
              params: TraceParams = TraceParams()) -> HitRecord:
    """Trace one ray (transport.py:359-372)."""
    return trace_rays(bvh, mesh, np.reshape(origin, (1, 3)), np.reshape(direction, (1, 3)),
                      params).record(0)


def trace_grid(bvh: Bvh, mesh: Mesh, grid: ApertureGrid, params: TraceParams = TraceParams(),
               workers: int = 1, with_ids: bool = False, rows=None) -> HitRecords:
    """Trace every grid ray on the GPU (transport.py:375-422).  ``workers``
    is accepted for API parity; the result never depends on it.  ``rows =
    (i_start, i_end)`` traces that row range only, like one worker's
    ``_trace_rows`` call (transport.py:330-356); records then start at ray
    ``i_start * n_v``."""
    ctx = nat.context()
    d = bvh.device(mesh, ctx)
    i0, i1 = (0, grid.n_u) if rows is None else (int(rows[0]), int(rows[1]))
    n = (i1 - i0) * grid.n_v
    out = _alloc(n, params.max_bounces, with_ids)
    g = nat.make_grid(grid)
    cp = _cparams(mesh, params)
    nat.check(ctx.lib.sbr_trace_grid_rows(ctx.handle, d.mesh_dev.handle, d.handle,
                                          ctypes.byref(g), ctypes.byref(cp), i0, i1,
                                          *[nat.ptr(a) for a in out]),
              "sbr_trace_grid_rows")
    return HitRecords(*out)


def trace_grid_hash(bvh: Bvh, mesh: Mesh, grid: ApertureGrid,
                    params: TraceParams = TraceParams(), rows=None,
                    seg_rays: int = nat.SEGMENT_RAYS) -> np.ndarray:
    """Per-segment record checksums of ``trace_grid(..., with_ids=True)``
    without materialising the records (sbr_trace_grid_hash): uint64 array,
    entry s = wrapping sum over the rays r // seg_rays == s of a splitmix64
    chain over r, the per-bounce ids and every HitRecords field.  Equal to
    the oracle's ``trace_grid_hash`` on identical inputs iff every record
    is bit-identical (up to 2^-64 collisions)."""
    ctx = nat.context()
    d = bvh.device(mesh, ctx)
    i0, i1 = (0, grid.n_u) if rows is None else (int(rows[0]), int(rows[1]))
    out = np.zeros(-(-grid.n_u * grid.n_v // int(seg_rays)), np.uint64)
    g = nat.make_grid(grid)
    cp = _cparams(mesh, params)
    nat.check(ctx.lib.sbr_trace_grid_hash(ctx.handle, d.mesh_dev.handle, d.handle,
                                          ctypes.byref(g), ctypes.byref(cp), i0, i1,
                                          int(seg_rays), nat.ptr(out)), "sbr_trace_grid_hash")
    return out


def dump_hits_csv(records: HitRecords, grid: ApertureGrid, path) -> None:
    """Per-ray diagnostic dump: i, j, valid, n0, R, N (transport.py:425-436),
    formatted by the native multi-threaded writer (sbr_dump_hits_csv)."""
    import os
    lib = nat.load_library()
    n = grid.n_u * grid.n_v
    valid = np.ascontiguousarray(records.valid[:n], dtype=np.uint8)
    n0 = nat.f64(records.normal0[:n], (-1, 3))
    rp = nat.f64(records.path[:n])
    nb = np.ascontiguousarray(records.bounces[:n], dtype=np.int32)
    nat.check(lib.sbr_dump_hits_csv(os.fsencode(path), grid.n_u, grid.n_v, nat.ptr(valid),
                                    nat.ptr(n0), nat.ptr(rp), nat.ptr(nb)), "sbr_dump_hits_csv")


def _dump_hits_csv_py(records: HitRecords, grid: ApertureGrid, path) -> None:
    """The reference writer loop (transport.py:425-436), kept as the test oracle."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("i,j,valid,nx,ny,nz,R,N\n")
        for r in range(grid.n_u * grid.n_v):
            i, j = divmod(r, grid.n_v)
            n0 = records.normal0[r]
            fh.write(f"{i},{j},{int(records.valid[r])},{n0[0]:.9g},{n0[1]:.9g},"
                     f"{n0[2]:.9g},{records.path[r]:.9g},{records.bounces[r]}\n")

"""Deterministic synthetic targets for the benchmark configurations.

* ``plate_mesh`` / ``dihedral_mesh`` / ``perturbed_grid_mesh`` reproduce the
  reference test meshes (pkg/tests/meshes.py:10-48) vertex for vertex.
* ``trihedral_mesh``: three unit squares on the coordinate planes (C3).
* ``quantized_icosphere``: reference icosphere with vertices rounded to
  float32 so the device can store them losslessly in 48-byte records (C1,
  C2, C5); both the GPU and the CPU oracle consume the same mesh.
* ``generate_aircraft``: a procedural airliner-like target (C4): fuselage
  of revolution, swept airfoil wings, tailplanes and two nacelles with open
  inlet ducts closed by a fan face (multi-bounce cavities).  ~1.0M
  triangles at density 1, bounding box ~15 x 13 x 4 m, float32-exact.
"""

from __future__ import annotations

import math

import numpy as np

from .geometry import Mesh, generate_icosphere, mesh_from_arrays, mesh_from_soup


def plate_mesh(side: float = 1.0) -> Mesh:
    s = side
    return mesh_from_arrays([[0, 0, 0], [s, 0, 0], [s, s, 0], [0, s, 0]], [[0, 1, 2], [0, 2, 3]])


def dihedral_mesh(size: float = 1.0) -> Mesh:
    s = size
    v = [[0, 0, 0], [s, 0, 0], [s, 0, s], [0, 0, s], [0, s, 0], [0, s, s]]
    return mesh_from_arrays(v, [[0, 1, 2], [0, 2, 3], [0, 4, 5], [0, 5, 3]])


def trihedral_mesh(size: float = 1.0) -> Mesh:
    s = size
    v = [[0, 0, 0], [s, 0, 0], [s, s, 0], [0, s, 0], [0, 0, s], [s, 0, s], [0, s, s]]
    f = [[0, 1, 2], [0, 2, 3], [0, 1, 5], [0, 5, 4], [0, 3, 6], [0, 6, 4]]
    return mesh_from_arrays(v, f)


def perturbed_grid_mesh(cells: int = 71, extent: float = 4.0, amplitude: float = 0.05,
                        seed: int = 42) -> Mesh:
    rng = np.random.default_rng(seed)
    n = cells + 1
    xs = np.linspace(0.0, extent, n)
    gx, gy = np.meshgrid(xs, xs, indexing="ij")
    gz = amplitude * rng.standard_normal((n, n))
    verts = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    idx = np.arange(n * n).reshape(n, n)
    a, b = idx[:-1, :-1].ravel(), idx[1:, :-1].ravel()
    c, d = idx[1:, 1:].ravel(), idx[:-1, 1:].ravel()
    faces = np.concatenate([np.stack([a, b, c], axis=1), np.stack([a, c, d], axis=1)])
    return mesh_from_arrays(verts, faces)


def quantize_f32(mesh: Mesh) -> Mesh:
    soup = np.stack([mesh.v0, mesh.v1, mesh.v2], axis=1)
    return mesh_from_soup(soup.astype(np.float32).astype(np.float64))


def quantized_icosphere(radius: float, subdivisions: int) -> Mesh:
    return quantize_f32(generate_icosphere(radius, subdivisions))


# ---------------------------------------------------------------------------
# procedural aircraft
# ---------------------------------------------------------------------------
def _sheet(P: np.ndarray, wrap_v: bool = False) -> np.ndarray:
    """(nu, nv, 3) vertex sheet -> (2 (nu-1) (nv'-1), 3, 3) triangles."""
    if wrap_v:
        P = np.concatenate([P, P[:, :1]], axis=1)
    a, b = P[:-1, :-1], P[1:, :-1]
    c, d = P[1:, 1:], P[:-1, 1:]
    t1 = np.stack([a, b, c], axis=2).reshape(-1, 3, 3)
    t2 = np.stack([a, c, d], axis=2).reshape(-1, 3, 3)
    return np.concatenate([t1, t2])


def _fan(center: np.ndarray, ring: np.ndarray) -> np.ndarray:
    nxt = np.roll(ring, -1, axis=0)
    return np.stack([np.broadcast_to(center, ring.shape), ring, nxt], axis=1)


def _revolve(xs, rs, n_circ, cy, cz) -> np.ndarray:
    th = np.linspace(0.0, 2.0 * math.pi, n_circ, endpoint=False)
    x = np.repeat(np.asarray(xs)[:, None], n_circ, axis=1)
    y = cy + np.asarray(rs)[:, None] * np.cos(th)[None, :]
    z = cz + np.asarray(rs)[:, None] * np.sin(th)[None, :]
    return np.stack([x, y, z], axis=-1)


def _airfoil_half(xi):
    """Symmetric 12% thickness distribution (closed trailing edge)."""
    return 5 * 0.12 * (0.2969 * np.sqrt(xi) - 0.1260 * xi - 0.3516 * xi ** 2
                       + 0.2843 * xi ** 3 - 0.1036 * xi ** 4)


def _lifting_surface(n_span, n_chord, root, tip, chord_root, chord_tip, vertical=False):
    """Swept tapered airfoil surface between leading-edge points root/tip."""
    s = np.linspace(0.0, 1.0, n_span)
    xi = 0.5 * (1.0 - np.cos(np.linspace(0.0, math.pi, n_chord)))
    le = np.asarray(root)[None, :] * (1 - s)[:, None] + np.asarray(tip)[None, :] * s[:, None]
    chord = chord_root * (1 - s) + chord_tip * s
    half = _airfoil_half(xi)[None, :] * chord[:, None]
    x = le[:, None, 0] + xi[None, :] * chord[:, None]
    sheets = []
    for sign in (1.0, -1.0):
        if vertical:
            y = le[:, None, 1] + sign * half
            z = np.broadcast_to(le[:, None, 2], x.shape)
        else:
            y = np.broadcast_to(le[:, None, 1], x.shape)
            z = le[:, None, 2] + sign * half
        sheets.append(_sheet(np.stack([x, y, z], axis=-1)))
    return np.concatenate(sheets)


def _nacelle(n_ax, n_circ, x0, x1, x_fan, cy, cz, r_out, r_in):
    ax = np.linspace(x0, x1, n_ax)
    outer = _revolve(ax, np.full(n_ax, r_out), n_circ, cy, cz)
    duct_x = np.linspace(x0, x_fan, max(2, n_ax // 2))
    inner = _revolve(duct_x, np.full(duct_x.size, r_in), n_circ, cy, cz)
    lip = _revolve(np.full(4, x0), np.linspace(r_in, r_out, 4), n_circ, cy, cz)
    n_fan = max(2, n_circ // 8)
    fan = _revolve(np.full(n_fan, x_fan), np.linspace(0.08, r_in, n_fan), n_circ, cy, cz)
    hub = _fan(np.array([x_fan, cy, cz]), fan[0])
    tail = _fan(np.array([x1 + 0.6, cy, cz]), outer[-1])
    return np.concatenate([_sheet(outer, True), _sheet(inner, True), _sheet(lip, True),
                           _sheet(fan, True), hub, tail])


def generate_aircraft(density: float = 1.0, seed: int = 7) -> Mesh:
    """Procedural airliner-like mesh (~1.0M triangles at density 1)."""
    rng = np.random.default_rng(seed)
    q = lambda n: max(4, int(round(n * math.sqrt(density))))  # noqa: E731
    parts = []
    # fuselage of revolution: ellipsoidal nose, barrel, tapered tail cone
    n_ax, n_circ = q(600), q(400)
    t = np.linspace(0.0, 1.0, n_ax)
    xs = 0.002 + t * (15.0 - 0.002)
    rs = np.where(xs < 2.5, 1.0 * np.sqrt(np.clip(1 - ((2.5 - xs) / 2.5) ** 2, 0, 1)),
                  np.where(xs > 11.0, 1.0 - 0.75 * (xs - 11.0) / 4.0, 1.0))
    cz = 1.3
    body = _revolve(xs, rs, n_circ, 0.0, cz)
    parts += [_sheet(body, True), _fan(np.array([0.0, 0.0, cz]), body[0]),
              _fan(np.array([15.0, 0.0, cz]), body[-1])]
    # wings (swept, tapered, dihedral), root inside the fuselage
    for side in (1.0, -1.0):
        parts.append(_lifting_surface(q(300), q(120), (5.5, side * 0.8, 1.0),
                                      (8.0, side * 6.5, 1.3), 3.4, 1.2))
        parts.append(_lifting_surface(q(100), q(60), (12.4, side * 0.6, 1.6),
                                      (13.8, side * 2.6, 1.75), 1.8, 0.8))
        parts.append(_nacelle(q(200), q(100), 4.0, 6.4, 5.4, side * 3.0, 0.55, 0.6, 0.48))
    parts.append(_lifting_surface(q(150), q(80), (11.8, 0.0, 2.0), (14.2, 0.0, 4.0), 2.6, 1.1,
                                  vertical=True))
    soup = np.concatenate(parts)
    # seeded sub-millimetre jitter: breaks exact symmetries (no systematic ties)
    soup = soup + rng.uniform(-2e-4, 2e-4, size=soup.shape)
    soup = soup.astype(np.float32).astype(np.float64)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return mesh_from_soup(soup)

"""Algorithmic bytes per closest-hit query for the bench workload (C4).

SURVEY.md section 8(d): bytes/query = 56 I + 40 T + 64 with
  I = internal-node expansions (a 2-child box pair, 48 B, + 8 B indices),
  T = triangle tests (36 B FP32 vertices + 4 B id),
  64 B of ray state in/out,
measured by the instrumented CPU oracle on the REFERENCE binned-SAH tree
(n_leaf=4) -- a fixed yardstick independent of the GPU's own tree.
The yardstick is split by query kind: query 0 of every ray (answered on the
GPU by the raster pass, k_raster, which moves no BVH bytes) and the
secondary queries (bounces 1..N and the escape probe, k_trace_persistent):
the primary counters come from closest_hit_batch on the sample's launch
origins (query 0 is exactly that call), the secondary ones are the rest.
The result is committed as profiles/algorithmic_bytes_c4.json and read by
bench.py (the bench's timed leg never runs the oracle).

    python scripts/algorithmic_bytes.py
"""

import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from paper_2604_09243_b200 import meshgen  # noqa: E402
from paper_2604_09243_b200.transport import IncidentDirection, build_aperture  # noqa: E402

FREQ = 10e9
B = 5


def main():
    mesh = meshgen.generate_aircraft()
    lam = 299792458.0 / FREQ
    t0 = time.time()
    tree = orc.build(mesh.v0, mesh.v1, mesh.v2, split_rule="sah", n_leaf=4)
    build_s = time.time() - t0
    scene = orc.Scene(mesh.v0, mesh.v1, mesh.v2, mesh.normals, tree)
    eps = 1e-6 * mesh.aabb.diagonal()
    tot = dict(pops=0, boxes=0, tris=0, internal=0, queries=0)
    prim = dict(pops=0, boxes=0, tris=0, internal=0, queries=0)
    rays = 0
    for ph in np.arange(0, 360, 45):
        g = build_aperture(mesh.aabb, IncidentDirection(math.pi / 2, math.radians(ph)),
                           lam / 5, wavelength=lam)
        for b in range(8):
            r0 = (2 * b + 1) * g.n_u // 16
            c = orc.Counters()
            orc.trace_grid(scene, g, B, eps, rows=(r0, min(g.n_u, r0 + 8)), counters=c)
            for k, v in c.as_dict().items():
                tot[k] += v
            i = np.arange(r0, min(g.n_u, r0 + 8))
            ii, jj = np.repeat(i, g.n_v), np.tile(np.arange(g.n_v), i.size)
            sp = g.spacing
            bx = np.asarray(g.corner) + ((ii + 0.5) * sp)[:, None] * np.asarray(g.u)
            o = bx + ((jj + 0.5) * sp)[:, None] * np.asarray(g.v)
            c0 = orc.Counters()
            orc.closest_hit_batch(scene, o, np.tile(np.asarray(g.k_inc), (o.shape[0], 1)),
                                  counters=c0)
            for k, v in c0.as_dict().items():
                prim[k] += v
            rays += 8 * g.n_v
    q = tot["queries"]
    I, T = tot["internal"] / q, tot["tris"] / q
    q0 = prim["queries"]
    qs = q - q0
    I0, T0 = prim["internal"] / q0, prim["tris"] / q0
    Is, Ts = (tot["internal"] - prim["internal"]) / qs, (tot["tris"] - prim["tris"]) / qs
    b0, bs = 56 * I0 + 40 * T0 + 64, 56 * Is + 40 * Ts + 64
    out = {
        "workload": "C4 procedural aircraft (983,660 tris), 10 GHz, lambda/5, B=5, theta=90",
        "sample": f"{rays} rays: 8 azimuths (0..315 step 45) x 8 row bands of 8 rows",
        "tree": "reference binned SAH, n_leaf=4 (oracle restatement of bvh.py:218-299)",
        "sah_build_s_cpu": round(build_s, 3),
        "queries_per_ray": q / rays,
        "internal_per_query": I,
        "tris_per_query": T,
        "pops_per_query": tot["pops"] / q,
        "bytes_per_query": 56 * I + 40 * T + 64,
        "formula": "56*I + 40*T + 64 (SURVEY.md 8d)",
        "primary": {"queries": q0, "internal_per_query": I0, "tris_per_query": T0,
                    "bytes_per_query": b0,
                    "note": "query 0 of every ray: k_raster answers it without BVH bytes; "
                            "its own yardstick is 48 B/triangle/angle + 16 B/hit cell"},
        "secondary": {"queries": qs, "internal_per_query": Is, "tris_per_query": Ts,
                      "bytes_per_query": bs,
                      "share_of_bytes": qs * bs / (qs * bs + q0 * b0),
                      "note": "bounces 1..N + escape probe: k_trace_persistent"},
    }
    path = os.path.join(ROOT, "profiles", "algorithmic_bytes_c4.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Lane-state census of k_trace_persistent (needs an SBR_TRACE_STATS build:
  python scripts/build_variant.py stats -DSBR_TRACE_STATS;
  SBR_LIB=$PWD/build_variants/stats.so python scripts/lane_census.py).
Average lanes per traversal step that are traversing, parked on a leaf,
blocked on a second leaf, or done (waiting for the completion phase)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen, _native as nat
from paper_2604_09243_b200.sweep import sweep_grids
mesh = meshgen.generate_aircraft()
cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=10e9, theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                      phi=sbr.AngleRange(0.0, math.radians(359), 36), max_bounces=5, n_leaf=2)
tree = sbr.build(mesh, cfg.build_params())
th, ph, cells, grids = sweep_grids(cfg, mesh)
ctx = nat.context()
buf = np.zeros(24, np.int64)
nat.check(ctx.lib.sbr_ctx_debug_counters(ctx.handle, nat.ptr(buf), 24))
res = sbr.solve_grids(tree, mesh, grids, cfg.trace_params(), [2 * math.pi / cfg.wavelength])
nat.check(ctx.lib.sbr_ctx_debug_counters(ctx.handle, nat.ptr(buf), 24))
it = max(buf[0], 1)
out = {"trav_steps": int(buf[0]), "lanes_traversing": buf[1] / it, "lanes_parked_leaf": buf[2] / it,
       "lanes_blocked_second_leaf": buf[3] / it, "lanes_done_waiting": buf[4] / it,
       "lanes_other": 32 - (buf[1] + buf[2] + buf[3] + buf[4]) / it,
       "leaf_phases": int(buf[5]), "lanes_in_leaf_phase": buf[6] / max(buf[5], 1),
       "trav_steps_per_leaf_phase": buf[0] / max(buf[5], 1),
       "queries": int(res.queries.sum())}
sq = max(int(buf[16]), 1)   # BVH-traced queries (secondary + any unresolved primary)
out["per_traced_query"] = {"bvh4_node_visits": buf[12] / sq, "triangle_tests": buf[13] / sq,
                           "leaf_visits": buf[14] / sq, "stack_pushes": buf[15] / sq,
                           "traced_queries": sq}
cyc = buf[8:12].astype(float)
out["cycle_share"] = dict(zip(("refill", "traversal", "leaf", "completion"),
                              (cyc / max(cyc.sum(), 1)).round(3).tolist()))
print(json.dumps(out, indent=1))

"""Co-scheduling probe: C4's 360 angles split into two halves solved by two
library contexts (two streams, each with its own mesh + tree copy) on one
GPU, back to back vs concurrently from two host threads.  SBR_TRACE_BPS /
SBR_RASTER_BPS cap the persistent grids (blocks per SM) so kernels of both
contexts can be resident at once."""
import ctypes, math, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import _native as nat
from paper_2604_09243_b200.sweep import sweep_grids, grid_array

mesh, lam, cfg = bench.workload(1.0, 360)
th, ph, cells, grids = sweep_grids(cfg, mesh)
tp = cfg.trace_params()
ks = nat.f64([2 * math.pi / cfg.wavelength])
B = tp.max_bounces
cp = nat.make_trace_params(B, tp.resolve_epsilon(mesh), False, True, 0.0, 5.0)
lib = nat.load_library()


def setup(ctx):
    dm = sbr.geometry._DeviceMesh(ctx, mesh)
    bp = nat.BuildParams()
    bp.split_rule = nat.SPLIT_SAH; bp.n_leaf = 2; bp.max_depth = 64; bp.bins_per_axis = 16
    bp.c_t = 1.0; bp.c_i = 1.0
    h = nat.c_vp()
    nat.check(lib.sbr_bvh_build(ctx.handle, dm.handle, ctypes.byref(bp), ctypes.byref(h)))
    return dm, h


def solve(ctx, dm, h, gs, out):
    ng = len(gs)
    amp = np.zeros((ng, 1, 2)); valid = np.zeros(ng, np.int64); maxb = np.zeros(ng, np.int32)
    hist = np.zeros((ng, B + 1), np.int64); q = np.zeros(ng, np.int64)
    diag = nat.Diag(valid.ctypes.data, maxb.ctypes.data, hist.ctypes.data, q.ctypes.data)
    garr = grid_array(gs)
    nat.check(lib.sbr_solve(ctx.handle, dm.handle, h, garr, ng, ctypes.byref(cp), nat.ptr(ks), 1,
                            -1.0, 0, nat.ptr(amp), ctypes.byref(diag)))
    out.append(int(q.sum()))


ctxs = [nat.context(), nat.Context(0)]
scenes = [setup(c) for c in ctxs]
halves = [grids[0::2], grids[1::2]]
for rep in range(4):
    for c in ctxs:
        c.synchronize()
    out = []
    t0 = time.perf_counter()
    for i in range(2):
        solve(ctxs[i], *scenes[i], halves[i], out)
    t1 = time.perf_counter()
    out2 = []
    ths = [threading.Thread(target=solve, args=(ctxs[i], *scenes[i], halves[i], out2))
           for i in range(2)]
    t2 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    t3 = time.perf_counter()
    print(f"back to back {1e3 * (t1 - t0):.1f} ms, concurrent {1e3 * (t3 - t2):.1f} ms, "
          f"queries {sum(out)} {sum(out2)}", flush=True)

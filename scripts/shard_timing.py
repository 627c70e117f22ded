"""Per-rank device time of the sharded solve, measured on ONE GPU by running
every rank's shard (sbr_solve_shard with rank r of N) in turn: the N-GPU
step time is the slowest rank plus one small reduce.  C4: angle sharding of
the 360-angle sweep; C5: ray-tile sharding of the 1e9-ray aperture (64 k).
Prints one JSON line per (config, N)."""
import ctypes, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen, _native as nat, distributed as D
from paper_2604_09243_b200.sweep import grid_array, sweep_grids

C = 299792458.0


def shard_ms(tree, mesh, grids, tp, ks, lam_min, rank, world, mode, reps=2):
    ctx = nat.context()
    d = tree.device(mesh, ctx)
    ks = nat.f64(ks)
    base = D.segment_layout(grids)
    seg = torch.zeros(int(base[-1]) * ks.size * 2, dtype=torch.float64, device="cuda")
    diag = torch.zeros((len(grids), D.diag_stride(tp.max_bounces)), dtype=torch.int64, device="cuda")
    garr = grid_array(grids)
    cp = nat.make_trace_params(tp.max_bounces, tp.resolve_epsilon(mesh), False, False, lam_min, 5.0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    best = None
    for _ in range(reps):
        ctx.profile(True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nat.check(ctx.lib.sbr_solve_shard(ctx.handle, d.mesh_dev.handle, d.handle, garr, len(grids),
                                          ctypes.byref(cp), nat.ptr(ks), ks.size, -1.0, 0, rank, world,
                                          D.MODES[mode], nat.c_vp(seg.data_ptr()),
                                          nat.c_vp(diag.data_ptr())))
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if best is None or ms < best[0]:
            k = ctx.kernel_stats()
            best = (ms, {n: round(k[n + "_ms"], 1) for n in ("raster", "trace", "po")})
    return best[0], int(diag[:, 1].sum().item()), best[1]


def run(name, tree, mesh, grids, tp, ks, lam_min, mode, worlds):
    for world in worlds:
        for r in range(world):            # warm every rank's buffers first
            shard_ms(tree, mesh, grids, tp, ks, lam_min, r, world, mode, reps=1)
        per = [shard_ms(tree, mesh, grids, tp, ks, lam_min, r, world, mode, reps=3)
               for r in range(world)]
        ms = [p[0] for p in per]
        q = sum(p[1] for p in per)
        print(json.dumps({"config": name, "shard_mode": mode, "n": world,
                          "rank_ms": [round(x, 2) for x in ms], "step_ms_max_rank": round(max(ms), 2),
                          "queries": q, "intersections_per_s_at_n": q / (max(ms) / 1e3),
                          "rank_stages": [p[2] for p in per]}), flush=True)


def main():
    torch.cuda.set_device(0)
    worlds = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8").split(",")]
    mesh = meshgen.generate_aircraft()
    lam = C / 10e9
    tree = sbr.build(mesh)
    cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=10e9, theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                          phi=sbr.AngleRange(0.0, math.radians(359), 360), max_bounces=5)
    th, ph, cells, grids = sweep_grids(cfg, mesh)
    run("C4", tree, mesh, grids, cfg.trace_params(), [2 * math.pi / lam], lam, "angles", worlds)
    mesh = meshgen.quantized_icosphere(1.0, 8)
    tree = sbr.build(mesh)
    ka = np.linspace(937.5, 1000.0, 64)
    lam_min = 2 * math.pi / ka.max()
    grid = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, 0.0), 6.4826e-5,
                              wavelength=lam_min)
    run("C5", tree, mesh, [grid], sbr.TraceParams(max_bounces=1), ka, lam_min, "rays", worlds)


if __name__ == "__main__":
    main()

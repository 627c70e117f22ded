#!/usr/bin/env python
"""Benchmark: 360-angle monostatic RCS sweep of the ~1M-triangle procedural
aircraft at 10 GHz with 5 bounces (BASELINE.json configs[3], the workload the
north-star target "1e9 ray-bounce intersections/s per B200 on a 1M-triangle
mesh" is quoted on).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)

A step = one full 360-angle sweep (launcher + 5-bounce trace + compaction +
PO + reduction) over the resident mesh/BVH.  metric = closest-hit queries
per second, sum_i (N_i + 1) over all rays of the step (the reference's
_traverse calls), whole job over all GPUs.  Angles are sharded
across ranks (strong scaling: the sweep is fixed) and combined with one
NCCL reduce.  ``--impl reference`` times the reference algorithm (the CPU
oracle port of the numba kernels, all host cores) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ray-bounce intersections/s per GPU & monostatic RCS sweep angles/s at 1/2/4/8 B200"
UNIT = "intersections/s"
FREQ_HZ = 10e9
MAX_BOUNCES = 5
N_ANGLES = 360
C = 299792458.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--density", type=float, default=1.0, help="mesh density (1.0 = ~1M tris)")
    p.add_argument("--angles", type=int, default=N_ANGLES)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--n-leaf", type=int, default=2,
                   help="BVH leaf size (BuildParams.n_leaf; 2 measured fastest, "
                        "profiles/experiments/r01_scheduler_experiments.json)")
    p.add_argument("--bounces", type=int, default=MAX_BOUNCES,
                   help="max bounces (experiments only; the C4 workload is 5)")
    return p.parse_args()


def workload(density, n_angles, bounces=MAX_BOUNCES, n_leaf=2):
    import paper_2604_09243_b200 as sbr
    from paper_2604_09243_b200 import meshgen
    mesh = meshgen.generate_aircraft(density=density)
    lam = C / FREQ_HZ
    cfg = sbr.SweepConfig(mesh_path="<procedural aircraft>", frequency_hz=FREQ_HZ,
                          theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                          phi=sbr.AngleRange(0.0, math.radians(n_angles - 1), n_angles),
                          max_bounces=bounces, split_rule="sah", n_leaf=n_leaf)
    return mesh, lam, cfg


def config_dict(mesh, n_angles, world, bounces=MAX_BOUNCES):
    return {"workload": "C4: procedural aircraft, 360-angle monostatic sweep, 10 GHz, "
                        "5 bounces, lambda/5 ray spacing",
            "triangles": int(mesh.triangle_count), "angles": n_angles,
            "theta_deg": 90, "phi_deg": [0, n_angles - 1], "frequency_hz": FREQ_HZ,
            "max_bounces": bounces, "spacing": "lambda/5 (5.996 mm)",
            "parallelism": f"angle-sharded x{world}, one NCCL reduce" if world > 1 else "1 GPU",
            "bvh": "reference binned-SAH tree (16 bins, n_leaf=2) built on the GPU, BVH4 traversal",
            "l2": "flushed (512 MB write) between timed steps"}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = str(index)
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9 or f[0] != self.index:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (oracle port) on the host cores
# ---------------------------------------------------------------------------
def cpu_sample(mesh, lam, cfg, n_angles_sample=8, bands=8, band_rows=8):
    """Bounded sample of the same workload through the CPU port of the
    reference kernels (oracle/, test infrastructure): reference SAH tree,
    then trace + PO on row bands of a few azimuths; returns a dict."""
    from oracle import oracle as orc
    import paper_2604_09243_b200 as sbr
    t0 = time.perf_counter()
    tree = orc.build(mesh.v0, mesh.v1, mesh.v2, split_rule="sah", n_leaf=4)
    build_s = time.perf_counter() - t0
    scene = orc.Scene(mesh.v0, mesh.v1, mesh.v2, mesh.normals, tree)
    eps = 1e-6 * mesh.aabb.diagonal()
    phis = cfg.phi.values()
    picks = np.linspace(0, len(phis) - 1, n_angles_sample).astype(int)
    return scene, eps, build_s, [(phis[i]) for i in picks]


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_run(scene, eps, lam, phis, bands, band_rows, threads=0):
    from oracle import oracle as orc
    import paper_2604_09243_b200 as sbr
    mesh_box = sbr.Aabb(scene.aabb_min, scene.aabb_max)
    queries = rays = 0
    t0 = time.perf_counter()
    for ph in phis:
        g = sbr.build_aperture(mesh_box, sbr.IncidentDirection(math.pi / 2, float(ph)),
                               lam / 5, wavelength=lam)
        for b in range(bands):
            r0 = (2 * b + 1) * g.n_u // (2 * bands)
            rows = (r0, min(g.n_u, r0 + band_rows))
            rec = orc.trace_grid(scene, g, MAX_BOUNCES, eps, rows=rows, threads=threads)
            orc.accumulate(rec, g.k_inc, lam, g.cell_area)
            queries += int((rec.bounces.astype(np.int64) + 1).sum())
            rays += rec.valid.shape[0]
    return queries, rays, time.perf_counter() - t0


def host_cores():
    # the threads the oracle runs with (oracle._threads(0)): every core this
    # process may use, whatever OMP_NUM_THREADS a launcher exported
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    mesh, lam, cfg = workload(args.density, args.angles)
    scene, eps, build_s, phis = cpu_sample(mesh, lam, cfg)
    cores = host_cores()
    for _ in range(max(args.warmup, 0)):
        cpu_run(scene, eps, lam, phis[:1], 4, 32)
    q = r = 0
    t = 0.0
    for s in range(args.steps):
        qq, rr, tt = cpu_run(scene, eps, lam, phis, 16, 64)
        q += qq; r += rr; t += tt
    value = q / t
    sample = (f"{args.steps} steps x {len(phis)} azimuths x 16 row bands of 64 rows ({r} rays, "
              f"{q} queries) "
              f"of the C4 sweep; reference SAH tree built in {build_s:.2f} s (not timed)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(mesh, args.angles, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import paper_2604_09243_b200 as sbr
    from paper_2604_09243_b200 import _native as nat
    from paper_2604_09243_b200 import distributed as D
    from paper_2604_09243_b200.sweep import sweep_grids

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SBR_BENCH_SHARE_GPU=1 (testing the N-rank path on a 1-GPU box): every
    # rank on cuda:0 over gloo -- NCCL refuses two ranks on one device
    share = os.environ.get("SBR_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = nat.context(local)

    mesh, lam, cfg = workload(args.density, args.angles, args.bounces, args.n_leaf)
    tree = sbr.build(mesh, cfg.build_params())
    th, ph, cells, grids = sweep_grids(cfg, mesh)
    tp = cfg.trace_params()
    k = [2 * math.pi / lam]
    stats = {}

    def step():
        if world == 1:
            return sbr.solve_grids(tree, mesh, grids, tp, k, cfg.gamma, lambda_min=lam,
                                   allow_aliasing=False)
        return D.solve_grids_distributed(tree, mesh, grids, tp, k, cfg.gamma,
                                         shard_mode="angles", lambda_min=lam,
                                         allow_aliasing=False, stats=stats)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.ExternalStream(ctx.stream)
    ctx.profile(True)
    clocks = Clocks(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ
                    else os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local])
    clocks.start()
    launches0 = ctx.launches
    total_ms = 0.0
    queries = 0
    local_queries = 0
    local_valid = 0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        total_ms += e0.elapsed_time(e1)
        if res is not None:
            queries += int(res.queries.sum())
        local_queries += stats.get("local_queries", int(res.queries.sum()) if res else 0)
        local_valid += stats.get("local_valid", int(res.valid_rays.sum()) if res else 0)
    launches = ctx.launches - launches0
    clk = clocks.stop()
    kst = ctx.kernel_stats()
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cpu" if share else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    # ---- e2e through the public API with host buffers -------------------
    e2e = None
    if not args.no_e2e:
        import dataclasses
        times, qs = [], []
        reps = max(3, min(args.steps, 5))
        # one untimed call first (first-call host costs: allocator growth,
        # thread-pool start-up); then `reps` calls, reported as the median
        # call (host-side jitter -- GC, cudaFree of the previous call's tree --
        # shows up in single calls; every call is listed in `calls_ms`)
        for rep in range(reps + 1):
            fresh = dataclasses.replace(mesh, _dev={})     # nothing resident
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            if world == 1:
                out = sbr.run_sweep(cfg, fresh)
            else:
                out = D.run_sweep_distributed(cfg, fresh)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if world > 1:
                tt = torch.tensor([dt], dtype=torch.float64, device="cpu" if share else "cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            if rep == 0:
                continue
            times.append(dt)
            qs.append(int(out.queries_total) if out is not None else 0)
        if rank == 0:
            med = sorted(range(reps), key=lambda i: times[i])[reps // 2]
            h2d = (mesh.triangle_count * 12 * 8 + len(grids) * 128) // 1
            d2h = len(grids) * (16 + 8 * (3 + MAX_BOUNCES + 1))
            e2e = {"value": qs[med] / times[med], "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * times[med],
                   "calls_ms": [round(1e3 * t, 1) for t in times],
                   "mean_value": sum(qs) / sum(times),
                   "path": "paper_2604_09243_b200.run_sweep(config, mesh) from host arrays: "
                           "mesh upload + GPU SAH build + 360 apertures + fused solve + readback; "
                           "median of the timed calls after one untimed call"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    value = queries / (total_ms / 1e3)
    # ---- per-kernel rooflines (algorithmic bytes / kernel time) ----------
    # SURVEY 8d yardstick split by query kind (profiles/algorithmic_bytes_c4.json,
    # scripts/algorithmic_bytes.py): query 0 of every ray is answered by the
    # raster pass, which moves no BVH bytes, so only the secondary queries
    # (bounces + escape probes) are charged to k_trace_persistent
    ab = json.load(open(os.path.join(ROOT, "profiles", "algorithmic_bytes_c4.json")))
    b_sec = ab["secondary"]["bytes_per_query"]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = ("MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)" if peaks
                else "fallback 6650 GB/s (B200_PROFILING.md)")
    l2pk = json.load(open(os.path.join(ROOT, "profiles", "l2_peak.json")))["l2_gbs"]
    steps = max(args.steps, 1)
    rays_step = sum(g.ray_count for i, g in enumerate(grids) if i % world == rank)  # own angles
    q_step = local_queries / steps
    sec_step = max(q_step - rays_step, 0.0)          # sum_i N_i: bounces + probes
    hits_step = local_valid / steps                   # primary hits (every hit is valid)
    ms = {k: kst[k] / steps for k in ("raster_ms", "compact_ms", "trace_ms", "po_ms")}

    def rl(bytes_, ms_, bound_peak, unit_note):
        a = bytes_ / (ms_ / 1e3) / 1e9 if ms_ else None
        return a, (a / bound_peak if a else None)

    tr_a, tr_f = rl(sec_step * b_sec, ms["trace_ms"], peak, "")
    traffic = None
    ncu_path = os.path.join(ROOT, "profiles", "ncu_trace_summary.json")
    if os.path.exists(ncu_path):
        nt = json.load(open(ncu_path))
        # dram read+write bytes of one k_trace_persistent launch (ncu --set
        # full) per secondary query, scaled to this step's launch
        bq = nt.get("dram_bytes_per_secondary_query")
        traffic = bq * sec_step if bq else None
    ntri = mesh.triangle_count
    n_ang = len(grids) // max(world, 1)
    ras_bytes = 48.0 * ntri * n_ang + 16.0 * hits_step
    ras_a, ras_f = rl(ras_bytes, ms["raster_ms"], peak, "")
    cmp_bytes = rays_step / 8.0 + 48.0 * hits_step
    cmp_a, cmp_f = rl(cmp_bytes, ms["compact_ms"], peak, "")
    po_bytes = (8.0 + 16.0 + 16.0) * hits_step + 8.0 * rays_step / 1024 + 16.0 * rays_step / 1024
    po_a, po_f = rl(po_bytes, ms["po_ms"], peak, "")
    rooflines = {
        "k_trace_persistent": {
            "bound": "hbm", "achieved": tr_a, "peak": peak, "unit": "GB/s", "frac": tr_f,
            "l2_frac": tr_a / l2pk if tr_a else None, "l2_peak": l2pk,
            "ms": ms["trace_ms"], "secondary_queries": sec_step,
            "bytes_per_query": b_sec,
            "yardstick": "56 I + 40 T + 64 per secondary query, I/T of the reference SAH tree"},
        "k_raster": {
            "bound": "hbm", "achieved": ras_a, "peak": peak, "unit": "GB/s", "frac": ras_f,
            "ms": ms["raster_ms"],
            "yardstick": "48 B per triangle per angle + 16 B per hit cell (query 0)"},
        "k_prim_compact": {
            "bound": "hbm", "achieved": cmp_a, "peak": peak, "unit": "GB/s", "frac": cmp_f,
            "ms": ms["compact_ms"],
            "yardstick": "1 bit of the raster's hit bitmap per ray slot; per hit: 16 B slot read + 16 B slot reset + 16 B work-list entry"},
        "k_po": {
            "bound": "hbm", "achieved": po_a, "peak": peak, "unit": "GB/s", "frac": po_f,
            "ms": ms["po_ms"],
            "yardstick": "per primary hit: 8 B list entry + 16 B record read + 16 B reset; "
                         "per 1024-ray chunk: 8 B run + 16 B partial (nk=1)"},
    }
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(mesh, args.angles, world, args.bounces),
        "angles_per_s": args.angles * args.steps / (total_ms / 1e3),
        "queries_per_step": queries // max(args.steps, 1),
        "gpu_launches": launches,
        "kernel_ms": {"raster": ms["raster_ms"], "compact": ms["compact_ms"],
                      "trace": ms["trace_ms"], "po": ms["po_ms"],
                      "trace_launches_per_step": kst["trace_launches"] / steps},
        "roofline": {"bound": "hbm", "achieved": tr_a, "peak": peak, "unit": "GB/s",
                     "frac": tr_f, "traffic": traffic,
                     "kernel": "k_trace_persistent (bounces 1..5 + escape probes; query 0 is "
                               "the raster pass, see rooflines.k_raster)",
                     "bytes_per_query": b_sec, "peak_source": peak_src,
                     # the node/triangle working set (~100 MB at 1M tris) lives in the
                     # 126 MB L2: the algorithmic bytes are served by L2/L1, so the
                     # measured L2 read bandwidth is the tighter ceiling
                     "l2": {"achieved": tr_a, "peak": l2pk, "unit": "GB/s",
                            "frac": tr_a / l2pk if tr_a else None,
                            "peak_source": "profiles/l2_peak.json (sbr_probe_l2_bandwidth)"}},
        "rooflines": rooflines,
        "clocks": clk,
    }
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu:
        scene, eps, build_s, phis = cpu_sample(mesh, lam, cfg)
        q, r, t = cpu_run(scene, eps, lam, phis, 16, 64)
        # the same kernels on one thread (a smaller slice of the same sample)
        q1, r1, t1 = cpu_run(scene, eps, lam, phis[:2], 4, 16, threads=1)
        cores = host_cores()
        line["cpu_baseline"] = {
            "value": q / t, "unit": UNIT, "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "value_1_thread": q1 / t1,
            "parallel_efficiency": (q / t) / (cores * q1 / t1),
            "sample": f"{len(phis)} azimuths x 16 row bands of 64 rows ({r} rays, {q} queries) "
                      f"of the same sweep, reference SAH tree (built in {build_s:.2f} s, not "
                      f"timed), oracle/ C port of the numba kernels, OpenMP {cores} threads; "
                      f"1-thread rate on 2 azimuths x 4 bands x 16 rows ({q1} queries). The "
                      "reference itself (numba) cannot run on the GPU box (no /root/reference "
                      "there); the port is pinned to it bit for bit (tests/test_oracle_golden.py)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

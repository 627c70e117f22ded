"""The multi-GPU driver end to end on the GPU box: two ranks (processes)
share cuda:0 over a gloo group, each traces its shard with sbr_solve_shard_packed,
one disjoint-support reduce combines them; the result must equal the
single-process solve bit for bit, for both shard modes and run_sweep."""

import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    import paper_2604_09243_b200 as sbr
    from paper_2604_09243_b200 import meshgen
    mesh = meshgen.generate_aircraft(density=0.03)
    lam = 0.05
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, ph), lam / 5,
                                wavelength=lam) for ph in np.linspace(0.0, 3.0, 5)]
    return sbr, mesh, grids, sbr.TraceParams(max_bounces=4), 2 * np.pi / (lam * np.linspace(0.98, 1.02, 3))


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_09243_b200 import distributed as D
    sbr, mesh, grids, tp, ks = _case()
    tree = sbr.build(mesh)
    res = D.solve_grids_distributed(tree, mesh, grids, tp, ks, shard_mode=mode)
    cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=6e9,
                          theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                          phi=sbr.AngleRange(0.0, 1.0, 3), max_bounces=3)
    sw = D.run_sweep_distributed(cfg, mesh, shard_mode=mode)
    if rank == 0:
        q.put((res.amplitude, res.valid_rays, res.bounce_counts, res.queries, sw.amplitude,
               sw.valid_rays, sw.bounce_histogram))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["angles", "rays"])
def test_two_ranks_equal_one(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sbr, mesh, grids, tp, ks = _case()
    tree = sbr.build(mesh)
    ref = sbr.solve_grids(tree, mesh, grids, tp, ks)
    assert np.array_equal(got[0], ref.amplitude)          # bit-identical
    assert np.array_equal(got[1], ref.valid_rays)
    assert np.array_equal(got[2], ref.bounce_counts)
    assert np.array_equal(got[3], ref.queries)
    cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=6e9,
                          theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                          phi=sbr.AngleRange(0.0, 1.0, 3), max_bounces=3)
    sw = sbr.run_sweep(cfg, mesh)
    assert np.array_equal(got[4], sw.amplitude)
    assert np.array_equal(got[5], sw.valid_rays)
    assert np.array_equal(got[6], sw.bounce_histogram)


def _emulated_ranks(sbr, mesh, tree, grids, tp, ks, world, mode):
    """Every rank's sbr_solve_shard run in turn in this process, partials
    combined as reduce_partials does (SUM; MAX for the max-bounce column)."""
    import ctypes
    import torch
    from paper_2604_09243_b200 import _native as nat, distributed as D
    from paper_2604_09243_b200.sweep import grid_array
    ctx = nat.context()
    d = tree.device(mesh, ctx)
    k = nat.f64(ks)
    base = D.segment_layout(grids)
    garr = grid_array(grids)
    cp = nat.make_trace_params(tp.max_bounces, tp.resolve_epsilon(mesh), False, True, 0.0, 5.0)
    seg_sum = diag_sum = None
    for r in range(world):
        seg = torch.zeros(int(base[-1]) * k.size * 2, dtype=torch.float64, device="cuda")
        diag = torch.zeros((len(grids), D.diag_stride(tp.max_bounces)), dtype=torch.int64,
                           device="cuda")
        nat.check(ctx.lib.sbr_solve_shard(ctx.handle, d.mesh_dev.handle, d.handle, garr,
                                          len(grids), ctypes.byref(cp), nat.ptr(k), k.size, -1.0,
                                          0, r, world, D.MODES[mode], nat.c_vp(seg.data_ptr()),
                                          nat.c_vp(diag.data_ptr())), "sbr_solve_shard")
        ctx.synchronize()
        if seg_sum is None:
            seg_sum, diag_sum = seg.clone(), diag.clone()
        else:
            # disjoint support: at most one rank wrote each element
            assert not bool(((seg_sum != 0) & (seg != 0)).any())
            seg_sum += seg
            mx = torch.maximum(diag_sum[:, 2], diag[:, 2])
            diag_sum += diag
            diag_sum[:, 2] = mx
    ng, B = len(grids), tp.max_bounces
    amp = np.zeros((ng, k.size, 2))
    valid = np.zeros(ng, np.int64)
    maxb = np.zeros(ng, np.int32)
    hist = np.zeros((ng, B + 1), np.int64)
    queries = np.zeros(ng, np.int64)
    dg = nat.Diag(valid.ctypes.data, maxb.ctypes.data, hist.ctypes.data, queries.ctypes.data)
    nat.check(ctx.lib.sbr_finalize(ctx.handle, garr, ng, nat.ptr(k), k.size, B,
                                   nat.c_vp(seg_sum.data_ptr()), nat.c_vp(diag_sum.data_ptr()),
                                   nat.ptr(amp), ctypes.byref(dg)), "sbr_finalize")
    return amp.view(np.complex128)[..., 0], valid, maxb, hist, queries


@pytest.mark.parametrize("world,mode", [(3, "rays"), (5, "rays"), (8, "rays"), (7, "angles")])
def test_emulated_ranks_equal_one(world, mode):
    """N-rank shards (ray tiles cut through triangles' candidate rows, big
    triangles' chunk queues and grid boundaries) recombine bit for bit."""
    import paper_2604_09243_b200 as sbr
    from paper_2604_09243_b200 import meshgen
    mesh = meshgen.generate_aircraft(density=0.05)
    lam = 0.04
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(th, ph), lam / 5, wavelength=lam)
             for th, ph in ((math.pi / 2, 0.3), (1.1, 2.0), (math.pi / 2, 4.4))]
    tp = sbr.TraceParams(max_bounces=3)
    ks = 2 * np.pi / (lam * np.array([0.99, 1.0]))
    tree = sbr.build(mesh)
    got = _emulated_ranks(sbr, mesh, tree, grids, tp, ks, world, mode)
    ref = sbr.solve_grids(tree, mesh, grids, tp, ks)
    assert np.array_equal(got[0], ref.amplitude)
    assert np.array_equal(got[1], ref.valid_rays)
    assert np.array_equal(got[2], ref.max_bounce)
    assert np.array_equal(got[3], ref.bounce_counts)
    assert np.array_equal(got[4], ref.queries)


def _emulated_packed(sbr, mesh, tree, grids, tp, ks, world, mode):
    """Every rank's sbr_solve_shard_packed run in turn; the packed buffers
    are combined by ONE element-wise sum (what the single reduce does)."""
    import ctypes
    import torch
    from paper_2604_09243_b200 import _native as nat, distributed as D
    from paper_2604_09243_b200.sweep import grid_array
    ctx = nat.context()
    d = tree.device(mesh, ctx)
    k = nat.f64(ks)
    garr = grid_array(grids)
    ng, B = len(grids), tp.max_bounces
    cp = nat.make_trace_params(B, tp.resolve_epsilon(mesh), False, True, 0.0, 5.0)
    cnt = nat.c_i64()
    nat.check(ctx.lib.sbr_packed_layout(garr, ng, k.size, B, world, ctypes.byref(cnt)))
    assert cnt.value == D.packed_count(grids, k.size, B, world)
    total = torch.zeros(int(cnt.value), dtype=torch.float64, device="cuda")
    for r in range(world):
        buf = torch.full_like(total, float("nan"))   # every element must be written
        nat.check(ctx.lib.sbr_solve_shard_packed(ctx.handle, d.mesh_dev.handle, d.handle, garr,
                                                 ng, ctypes.byref(cp), nat.ptr(k), k.size, -1.0,
                                                 0, r, world, D.MODES[mode],
                                                 nat.c_vp(buf.data_ptr())))
        ctx.synchronize()
        assert not bool(torch.isnan(buf).any())
        total += buf
    amp = np.zeros((ng, k.size, 2))
    valid = np.zeros(ng, np.int64)
    maxb = np.zeros(ng, np.int32)
    hist = np.zeros((ng, B + 1), np.int64)
    queries = np.zeros(ng, np.int64)
    dg = nat.Diag(valid.ctypes.data, maxb.ctypes.data, hist.ctypes.data, queries.ctypes.data)
    nat.check(ctx.lib.sbr_finalize_packed(ctx.handle, garr, ng, nat.ptr(k), k.size, B, world,
                                          nat.c_vp(total.data_ptr()), nat.ptr(amp),
                                          ctypes.byref(dg)))
    return amp.view(np.complex128)[..., 0], valid, maxb, hist, queries


@pytest.mark.parametrize("world,mode", [(1, "angles"), (4, "rays"), (3, "angles")])
def test_emulated_packed_single_sum_equals_one(world, mode):
    import paper_2604_09243_b200 as sbr
    from paper_2604_09243_b200 import meshgen
    mesh = meshgen.generate_aircraft(density=0.05)
    lam = 0.04
    grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(th, ph), lam / 5, wavelength=lam)
             for th, ph in ((math.pi / 2, 0.3), (1.1, 2.0), (math.pi / 2, 4.4))]
    tp = sbr.TraceParams(max_bounces=3)
    ks = 2 * np.pi / (lam * np.array([0.99, 1.0]))
    tree = sbr.build(mesh)
    got = _emulated_packed(sbr, mesh, tree, grids, tp, ks, world, mode)
    ref = sbr.solve_grids(tree, mesh, grids, tp, ks)
    for a, b in zip(got, (ref.amplitude, ref.valid_rays, ref.max_bounce, ref.bounce_counts,
                          ref.queries)):
        assert np.array_equal(a, b)


def _nccl_worker(port, q):
    """world_size 1 over NCCL: the torch carrier (dist.reduce on NCCL) and the
    library's own communicator (sbr_comm_init + sbr_solve_distributed)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0",
                      WORLD_SIZE="1")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2604_09243_b200 import _native as nat, distributed as D
    import ctypes
    sbr, mesh, grids, tp, ks = _case()
    tree = sbr.build(mesh)
    out = {"backend": dist.get_backend()}
    res = D.solve_grids_distributed(tree, mesh, grids, tp, ks, shard_mode="rays")
    out["torch"] = (res.amplitude, res.valid_rays, res.bounce_counts, res.queries)
    v = nat.c_i32()
    nat.check(nat.context().lib.sbr_comm_version(ctypes.byref(v)))
    out["nccl_version"] = int(v.value)
    D.init_library_comm()
    res = D.solve_grids_distributed(tree, mesh, grids, tp, ks, shard_mode="angles",
                                    comm="library")
    out["library"] = (res.amplitude, res.valid_rays, res.bounce_counts, res.queries)
    cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=6e9,
                          theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                          phi=sbr.AngleRange(0.0, 1.0, 3), max_bounces=3)
    sw = D.run_sweep_distributed(cfg, mesh, shard_mode="rays", comm="library")
    out["sweep"] = (sw.amplitude, sw.valid_rays)
    # the raw collective: in-place sum over one rank leaves the buffer as is
    buf = torch.arange(1000, dtype=torch.float64, device="cuda")
    ctx = nat.context()
    nat.check(ctx.lib.sbr_reduce_sum_f64(ctx.handle, nat.c_vp(buf.data_ptr()), 1000, 0))
    out["raw_ok"] = bool((buf.cpu() == torch.arange(1000, dtype=torch.float64)).all())
    D.destroy_library_comm()
    q.put(out)
    dist.destroy_process_group()


def test_nccl_world_size_one():
    """The NCCL code paths themselves (torch NCCL group and the library's
    dlopen-ed NCCL communicator) on the one GPU the box has."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    out = q.get(timeout=300)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert out["backend"] == "nccl" and out["nccl_version"] >= 22000 and out["raw_ok"]
    sbr, mesh, grids, tp, ks = _case()
    tree = sbr.build(mesh)
    ref = sbr.solve_grids(tree, mesh, grids, tp, ks)
    for key in ("torch", "library"):
        got = out[key]
        assert np.array_equal(got[0], ref.amplitude), key
        assert np.array_equal(got[1], ref.valid_rays), key
        assert np.array_equal(got[2], ref.bounce_counts), key
        assert np.array_equal(got[3], ref.queries), key
    cfg = sbr.SweepConfig(mesh_path="x", frequency_hz=6e9,
                          theta=sbr.AngleRange(math.pi / 2, math.pi / 2, 1),
                          phi=sbr.AngleRange(0.0, 1.0, 3), max_bounces=3)
    sw = sbr.run_sweep(cfg, mesh)
    assert np.array_equal(out["sweep"][0], sw.amplitude)
    assert np.array_equal(out["sweep"][1], sw.valid_rays)

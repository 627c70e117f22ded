"""Multi-GPU sweep driver: one process per GPU, ONE collective.

Replaces the paper's MPI layer and the reference's
thread pool over angles (pkg/src/sbr/sweep.py:327-349).

Work is cut into fixed units (grid g, segment s) of SEGMENT_RAYS consecutive
ray indices.  ``shard_mode="angles"`` gives rank r every unit of the grids
g = r (mod N) (the C2-C4 sweeps); ``shard_mode="rays"`` deals units of all
grids round-robin (the single huge aperture of C5).  Each rank writes into
ONE float64 buffer (``sbr_solve_shard_packed``): the FP64 partial sums of
its own units (zero everywhere else), its integer diagnostics as exact
doubles, and its per-grid max bounce in a slot of its own.  A single
element-wise ``reduce(SUM)`` therefore adds exactly one non-zero term per
partial (exact, order-independent: bit-identical to the one-GPU run for
any N) and the root takes the max over the max-bounce slots
(``sbr_finalize_packed``).

Two carriers for that one reduce: the caller's ``torch.distributed`` group
(``comm="torch"``, NCCL on GPUs, gloo on CPU), or the library's own NCCL
communicator (``comm="library"``: ``sbr_comm_init`` + ``sbr_solve_distributed``,
the path a non-Python host binds through the C ABI).
"""

from __future__ import annotations

import ctypes
from typing import Callable, Optional, Sequence

import numpy as np

from . import _native as nat

SEGMENT_RAYS = nat.SEGMENT_RAYS
MODES = {"angles": 0, "rays": 1}


def segment_layout(grids: Sequence) -> np.ndarray:
    """seg_base[g] = first segment row of grid g (mirrors sbr_segment_layout)."""
    base = np.zeros(len(grids) + 1, np.int64)
    for g, grid in enumerate(grids):
        n = int(grid.n_u) * int(grid.n_v)
        base[g + 1] = base[g] + (n + SEGMENT_RAYS - 1) // SEGMENT_RAYS
    return base


def unit_owners(grids: Sequence, world: int, mode: str = "angles") -> np.ndarray:
    """Owning rank of every segment row (same rule as capi.cu)."""
    base = segment_layout(grids)
    owner = np.empty(base[-1], np.int64)
    for g in range(len(grids)):
        rows = np.arange(base[g], base[g + 1])
        owner[rows] = g % world if MODES[mode] == 0 else rows % world
    return owner


def diag_stride(max_bounces: int) -> int:
    return 3 + max_bounces + 1


def packed_count(grids: Sequence, nk: int, max_bounces: int, world: int) -> int:
    """Doubles in the packed reduce buffer (mirrors sbr_packed_layout)."""
    return int(segment_layout(grids)[-1]) * nk * 2 + len(grids) * (diag_stride(max_bounces)
                                                                    + world)


def pack_host(seg, diag, rank: int, world: int) -> np.ndarray:
    """Host mirror of k_pack_diag (for CPU tests of the collective): the
    packed buffer of one rank from its partials and int64 diagnostics."""
    seg = np.asarray(seg, np.float64).ravel()
    diag = np.asarray(diag, np.int64)
    ng = diag.shape[0]
    d = diag.astype(np.float64)
    d[:, 2] = 0.0
    slots = np.zeros((ng, world))
    slots[:, rank] = diag[:, 2]
    return np.concatenate([seg, d.ravel(), slots.ravel()])


def unpack_host(buf, nseg_doubles: int, ng: int, stride: int, world: int):
    """Host mirror of k_unpack_diag: (partials, int64 diagnostics)."""
    buf = np.asarray(buf, np.float64)
    seg = buf[:nseg_doubles]
    d = buf[nseg_doubles:nseg_doubles + ng * stride].reshape(ng, stride)
    slots = buf[nseg_doubles + ng * stride:].reshape(ng, world)
    diag = d.astype(np.int64)
    diag[:, 2] = slots.max(axis=1).astype(np.int64)
    return seg, diag


def _dst(root: int, group) -> int:
    """``dist.reduce`` takes a GLOBAL rank; ``root`` is group-local."""
    import torch.distributed as dist
    return dist.get_global_rank(group, root) if group is not None else root


def reduce_packed(buf, root: int = 0, group=None):
    """The one collective: element-wise SUM of the packed buffer to ``root``
    (torch tensor on the rank's device; NCCL on GPUs, gloo on CPU)."""
    import torch.distributed as dist
    # gloo reduces host tensors only: stage device buffers through the host
    # (a CPU process group driving GPUs, e.g. several ranks sharing one GPU)
    staged = dist.get_backend(group) == "gloo" and buf.is_cuda
    b = buf.cpu() if staged else buf
    dist.reduce(b, dst=_dst(root, group), op=dist.ReduceOp.SUM, group=group)
    if staged and dist.get_rank(group) == root:
        buf.copy_(b)
    return buf


# ---- library communicator (sbr_comm_*) -------------------------------------
def init_library_comm(group=None, ctx: Optional[nat.Context] = None) -> nat.Context:
    """Give this rank's library context an NCCL communicator over the ranks
    of ``group``: rank 0 draws the unique id (sbr_comm_unique_id) and the
    torch group ships it to the others (any out-of-band channel would do)."""
    import torch.distributed as dist
    ctx = ctx or nat.context()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = np.zeros(128, np.uint8)
    if rank == 0:
        nat.check(ctx.lib.sbr_comm_unique_id(nat.ptr(uid)), "sbr_comm_unique_id")
    box = [uid.tobytes()]
    dist.broadcast_object_list(box, src=_dst(0, group), group=group)
    uid = np.frombuffer(box[0], np.uint8).copy()
    nat.check(ctx.lib.sbr_comm_init(ctx.handle, world, rank, nat.ptr(uid)), "sbr_comm_init")
    return ctx


def destroy_library_comm(ctx: Optional[nat.Context] = None) -> None:
    ctx = ctx or nat.context()
    nat.check(ctx.lib.sbr_comm_destroy(ctx.handle), "sbr_comm_destroy")


def _cparams(tree, mesh, trace_params, lambda_min, allow_aliasing):
    return nat.make_trace_params(trace_params.max_bounces, trace_params.resolve_epsilon(mesh),
                                 trace_params.strict_orientation, allow_aliasing,
                                 lambda_min or 0.0, trace_params.sampling_factor)


def solve_grids_distributed(tree, mesh, grids: Sequence, trace_params, wavenumbers,
                            gamma: float = -1.0, count_trapped: bool = False,
                            shard_mode: str = "angles", root: int = 0, group=None,
                            lambda_min: Optional[float] = None, allow_aliasing: bool = True,
                            timer: Optional[Callable] = None, stats: Optional[dict] = None,
                            comm: str = "torch"):
    """Sharded fused solve; returns the sweep.SolveResult on ``root`` and
    None elsewhere.  Every rank must call it with identical arguments.
    ``comm="library"`` uses the context's NCCL communicator
    (init_library_comm) through sbr_solve_distributed; ``"torch"`` reduces
    over the torch group.  ``stats`` (optional) receives this rank's own
    query count (torch carrier only)."""
    import torch
    import torch.distributed as dist
    from .sweep import SolveResult, grid_array

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ctx = nat.context()
    d = tree.device(mesh, ctx)
    ks = nat.f64(np.atleast_1d(wavenumbers))
    ng, B = len(grids), trace_params.max_bounces
    garr = grid_array(grids)
    cp = _cparams(tree, mesh, trace_params, lambda_min, allow_aliasing)
    amp = np.zeros((ng, ks.size, 2))
    valid = np.zeros(ng, np.int64)
    maxb = np.zeros(ng, np.int32)
    hist = np.zeros((ng, B + 1), np.int64)
    queries = np.zeros(ng, np.int64)
    dg = nat.Diag(valid.ctypes.data, maxb.ctypes.data, hist.ctypes.data, queries.ctypes.data)
    dev = torch.device("cuda", ctx.device)
    if comm == "library":
        torch.cuda.synchronize(dev)
        if timer:
            timer("start")
        nat.check(ctx.lib.sbr_solve_distributed(ctx.handle, d.mesh_dev.handle, d.handle, garr,
                                                ng, ctypes.byref(cp), nat.ptr(ks), ks.size,
                                                float(gamma), int(bool(count_trapped)),
                                                MODES[shard_mode], root, nat.ptr(amp),
                                                ctypes.byref(dg)), "sbr_solve_distributed")
        if timer:
            timer("traced")
        if rank != root:
            return None
        return SolveResult(amp.view(np.complex128)[..., 0], valid, maxb, hist, queries)
    if comm != "torch":
        raise ValueError(f"unknown comm {comm!r}")
    cnt = nat.c_i64()
    nat.check(ctx.lib.sbr_packed_layout(garr, ng, ks.size, B, world, ctypes.byref(cnt)))
    buf = torch.empty(int(cnt.value), dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    if timer:
        timer("start")
    nat.check(ctx.lib.sbr_solve_shard_packed(ctx.handle, d.mesh_dev.handle, d.handle, garr, ng,
                                             ctypes.byref(cp), nat.ptr(ks), ks.size,
                                             float(gamma), int(bool(count_trapped)), rank,
                                             world, MODES[shard_mode],
                                             nat.c_vp(buf.data_ptr())),
              "sbr_solve_shard_packed")
    if timer:
        timer("traced")
    if stats is not None:
        nseg = int(segment_layout(grids)[-1]) * ks.size * 2
        dg_ = buf[nseg:nseg + ng * diag_stride(B)].view(ng, diag_stride(B))
        stats["local_queries"] = int(dg_[:, 1].sum().item())
        stats["local_valid"] = int(dg_[:, 0].sum().item())
    reduce_packed(buf, root, group)     # the one collective
    if rank != root:
        return None
    torch.cuda.synchronize(dev)
    nat.check(ctx.lib.sbr_finalize_packed(ctx.handle, garr, ng, nat.ptr(ks), ks.size, B, world,
                                          nat.c_vp(buf.data_ptr()), nat.ptr(amp),
                                          ctypes.byref(dg)), "sbr_finalize_packed")
    return SolveResult(amp.view(np.complex128)[..., 0], valid, maxb, hist, queries)


def run_sweep_distributed(config, mesh=None, shard_mode: str = "angles", root: int = 0,
                          group=None, comm: str = "torch"):
    """``sweep.run_sweep`` across the ranks of the process group: every rank
    builds the (replicated) BVH on its GPU and traces its shard of the
    cells; the SweepResult is returned on ``root`` (None elsewhere)."""
    from . import sweep as S
    from .geometry import load_mesh
    if mesh is None:
        mesh = load_mesh(config.mesh_path, dtype=config.dtype())

    def solver(tree, m, grids, tp, ks, gamma, count_trapped, lambda_min=None,
               allow_aliasing=True):
        return solve_grids_distributed(tree, m, grids, tp, ks, gamma, count_trapped,
                                       shard_mode=shard_mode, root=root, group=group,
                                       lambda_min=lambda_min, allow_aliasing=allow_aliasing,
                                       comm=comm)
    return S._run_sweep(config, mesh, solver)

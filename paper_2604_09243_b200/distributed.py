"""Multi-GPU sweep driver: one process per GPU, one NCCL reduce.

Replaces the paper's MPI layer and the reference's
thread pool over angles (pkg/src/sbr/sweep.py:327-349).

Work is cut into fixed units (grid g, segment s) of SEGMENT_RAYS consecutive
ray indices.  ``shard_mode="angles"`` gives rank r every unit of the grids
g = r (mod N) (the C2-C4 sweeps); ``shard_mode="rays"`` deals units of all
grids round-robin (the single huge aperture of C5).  Each rank writes the
FP64 partial sums of its own units into a buffer that is zero everywhere
else, so the single ``reduce(SUM)`` adds exactly one non-zero term per
element: the result is exact, order-independent and therefore bit-identical
to the one-GPU run for any N.  Integer diagnostics ride in a second buffer
(sum) plus a tiny MAX reduce for the per-grid max bounce.
"""

from __future__ import annotations

import ctypes
import math
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


def reduce_partials(seg, diag, root: int = 0, group=None):
    """One SUM reduce of the disjoint-support partial buffer, one SUM of the
    integer diagnostics and one MAX of the max-bounce column (torch tensors
    on the rank's device; NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    stride = diag.shape[1]
    # gloo reduces host tensors only: stage device buffers through the host
    # (a CPU process group driving GPUs, e.g. several ranks sharing one GPU)
    staged = dist.get_backend(group) == "gloo" and seg.is_cuda
    s, d = (seg.cpu(), diag.cpu()) if staged else (seg, diag)
    maxb = d[:, 2].clone()
    dist.reduce(s, dst=root, op=dist.ReduceOp.SUM, group=group)
    dist.reduce(d, dst=root, op=dist.ReduceOp.SUM, group=group)
    dist.reduce(maxb, dst=root, op=dist.ReduceOp.MAX, group=group)
    if dist.get_rank(group) == root:
        d[:, 2] = maxb
        if staged:
            seg.copy_(s)
            diag.copy_(d)
    assert stride == diag.shape[1]
    return seg, diag


def solve_grids_distributed(tree, mesh, grids: Sequence, trace_params, wavenumbers,
                            gamma: float = -1.0, count_trapped: bool = False,
                            shard_mode: str = "angles", root: int = 0, group=None,
                            lambda_min: Optional[float] = None, allow_aliasing: bool = True,
                            timer: Optional[Callable] = None, stats: Optional[dict] = None):
    """Sharded fused solve; returns the sweep.SolveResult on ``root`` and
    None elsewhere.  Every rank must call it with identical arguments.
    ``stats`` (optional) receives this rank's own query count."""
    import torch
    import torch.distributed as dist
    from .sweep import SolveResult, grid_array

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ctx = nat.context()
    d = tree.device(mesh, ctx)
    ks = nat.f64(np.atleast_1d(wavenumbers))
    ng, B = len(grids), trace_params.max_bounces
    base = segment_layout(grids)
    dev = torch.device("cuda", ctx.device)
    seg = torch.zeros(int(base[-1]) * ks.size * 2, dtype=torch.float64, device=dev)
    diag = torch.zeros((ng, diag_stride(B)), dtype=torch.int64, device=dev)
    garr = grid_array(grids)
    cp = nat.make_trace_params(B, trace_params.resolve_epsilon(mesh),
                               trace_params.strict_orientation, allow_aliasing,
                               lambda_min or 0.0, trace_params.sampling_factor)
    torch.cuda.synchronize(dev)
    if timer:
        timer("start")
    nat.check(ctx.lib.sbr_solve_shard(ctx.handle, d.mesh_dev.handle, d.handle, garr, ng,
                                      ctypes.byref(cp), nat.ptr(ks), ks.size, float(gamma),
                                      int(bool(count_trapped)), rank, world,
                                      MODES[shard_mode], nat.c_vp(seg.data_ptr()),
                                      nat.c_vp(diag.data_ptr())), "sbr_solve_shard")
    ctx.synchronize()   # library stream -> visible to NCCL on torch's stream
    if timer:
        timer("traced")
    if stats is not None:
        stats["local_queries"] = int(diag[:, 1].sum().item())
    reduce_partials(seg, diag, root, group)
    if rank != root:
        return None
    amp = np.zeros((ng, ks.size, 2))
    valid = np.zeros(ng, np.int64)
    maxb = np.zeros(ng, np.int32)
    hist = np.zeros((ng, B + 1), np.int64)
    queries = np.zeros(ng, np.int64)
    dg = nat.Diag(valid.ctypes.data, maxb.ctypes.data, hist.ctypes.data, queries.ctypes.data)
    torch.cuda.synchronize(dev)
    nat.check(ctx.lib.sbr_finalize(ctx.handle, garr, ng, nat.ptr(ks), ks.size, B,
                                   nat.c_vp(seg.data_ptr()), nat.c_vp(diag.data_ptr()),
                                   nat.ptr(amp), ctypes.byref(dg)), "sbr_finalize")
    return SolveResult(amp.view(np.complex128)[..., 0], valid, maxb, hist, queries)


def run_sweep_distributed(config, mesh=None, shard_mode: str = "angles", root: int = 0,
                          group=None):
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
                                       lambda_min=lambda_min, allow_aliasing=allow_aliasing)
    return S._run_sweep(config, mesh, solver)

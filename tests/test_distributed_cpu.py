"""Host logic of the multi-GPU driver, run with world_size=2 over gloo.

The device compute is replaced by deterministic fake partials: each rank
produces the partial sums of the segments it owns, zero elsewhere, packs
them with its diagnostics into ONE buffer (the layout of
sbr_solve_shard_packed); the one SUM reduce must reproduce the single-rank
partials bit for bit and the per-grid max bounce, for both the angle and
the ray-tile shard modes, also inside a sub-group.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_09243_b200 import distributed as D
from paper_2604_09243_b200.transport import IncidentDirection, build_aperture
from paper_2604_09243_b200 import meshgen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _G:
    def __init__(self, n_u, n_v):
        self.n_u, self.n_v = n_u, n_v


def _partials(grids, owners, rank, world, nk):
    """Deterministic fake per-segment partials: value depends only on the row."""
    base = D.segment_layout(grids)
    seg = np.zeros((base[-1], nk, 2))
    for row in range(base[-1]):
        if owners[row] == rank:
            seg[row] = np.sin(np.arange(nk * 2).reshape(nk, 2) + 0.37 * row) + row * 1e-3
    return seg


GRIDS = [(700, 900), (1300, 1100), (10, 10), (2048, 1024)]


def _worker(rank, world, port, mode, sub, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    group = None
    if sub:   # ranks [1, world) form the group; group-local root 0 = global rank 1
        group = dist.new_group(list(range(1, world)))
        if rank == 0:
            dist.destroy_process_group()
            return
    g_rank, g_world = dist.get_rank(group), dist.get_world_size(group)
    grids = [_G(*g) for g in GRIDS]
    nk, B = 3, 4
    owners = D.unit_owners(grids, g_world, mode)
    seg = _partials(grids, owners, g_rank, g_world, nk).ravel()
    diag = np.zeros((len(grids), D.diag_stride(B)), np.int64)
    base = D.segment_layout(grids)
    for g in range(len(grids)):
        mine = (owners[np.arange(base[g], base[g + 1])] == g_rank).sum()
        diag[g, 0] = 10 * mine
        diag[g, 2] = g_rank + g if mine else 0
    buf = torch.from_numpy(D.pack_host(seg, diag, g_rank, g_world))
    assert buf.numel() == D.packed_count(grids, nk, B, g_world)
    D.reduce_packed(buf, root=0, group=group)
    if g_rank == 0:
        out.put(D.unpack_host(buf.numpy(), seg.size, len(grids), D.diag_stride(B), g_world)
                + (g_world,))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,world,sub", [("angles", 2, False), ("rays", 2, False),
                                            ("rays", 3, True)])
def test_one_packed_reduce_is_exact(mode, world, sub):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, sub, q))
             for r in range(world)]
    for p in procs:
        p.start()
    seg, diag, g_world = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    grids = [_G(*g) for g in GRIDS]
    ref = _partials(grids, np.zeros(D.segment_layout(grids)[-1], np.int64), 0, 1, 3)
    assert np.array_equal(seg, ref.ravel())   # bit-identical to the 1-rank buffer
    base = D.segment_layout(grids)
    assert np.array_equal(diag[:, 0], 10 * np.diff(base))
    owners = D.unit_owners(grids, g_world, mode)
    for g in range(len(grids)):
        ranks = set(owners[base[g]:base[g + 1]].tolist())
        assert diag[g, 2] == max(r + g for r in ranks)   # max over the rank slots


def test_unit_owner_rules():
    grids = [_G(1024, 1024), _G(1024, 513), _G(3, 3)]
    base = D.segment_layout(grids)
    assert base.tolist() == [0, 2, 4, 5]
    assert D.unit_owners(grids, 2, "angles").tolist() == [0, 0, 1, 1, 0]
    assert D.unit_owners(grids, 2, "rays").tolist() == [0, 1, 0, 1, 0]
    # every unit has exactly one owner for any world size
    for w in (1, 2, 3, 8):
        own = D.unit_owners(grids, w, "rays")
        assert own.min() >= 0 and own.max() < w


def test_c5_layout_sizes():
    """1e9-ray aperture: ~1907 segments of 2^19 rays, dealt across 8 ranks."""
    class G:
        n_u = n_v = 31623
    base = D.segment_layout([G()])
    assert base[-1] == math.ceil(31623 * 31623 / 2 ** 19)
    own = D.unit_owners([G()], 8, "rays")
    counts = np.bincount(own, minlength=8)
    assert counts.max() - counts.min() <= 1

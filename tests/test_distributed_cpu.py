"""Host logic of the multi-GPU driver, run with world_size=2 over gloo.

The device compute is replaced by the CPU oracle (test-only): each rank
produces the partial sums of the segments it owns, zero elsewhere; the one
SUM reduce must reproduce the single-rank buffer bit for bit, for both the
angle and the ray-tile shard modes.
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


def _worker(rank, world, port, mode, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grids = [_G(700, 900), _G(1300, 1100), _G(10, 10), _G(2048, 1024)]
    nk, B = 3, 4
    owners = D.unit_owners(grids, world, mode)
    seg = torch.from_numpy(_partials(grids, owners, rank, world, nk).ravel().copy())
    diag = torch.zeros((len(grids), D.diag_stride(B)), dtype=torch.int64)
    for g in range(len(grids)):
        rows = np.arange(D.segment_layout(grids)[g], D.segment_layout(grids)[g + 1])
        mine = (owners[rows] == rank).sum()
        diag[g, 0] = 10 * mine
        diag[g, 2] = rank + g if mine else 0
    D.reduce_partials(seg, diag, root=0)
    if rank == 0:
        out.put((seg.numpy().copy(), diag.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["angles", "rays"])
def test_disjoint_reduce_is_exact(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    seg, diag = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    grids = [_G(700, 900), _G(1300, 1100), _G(10, 10), _G(2048, 1024)]
    ref = _partials(grids, np.zeros(D.segment_layout(grids)[-1], np.int64), 0, 1, 3)
    assert np.array_equal(seg, ref.ravel())   # bit-identical to the 1-rank buffer
    base = D.segment_layout(grids)
    assert np.array_equal(diag[:, 0], 10 * np.diff(base))


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

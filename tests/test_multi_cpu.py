"""CPU tests of the multi-GPU host logic: decomposition, halo plan and the
torch.distributed halo exchange (gloo, world sizes 2 and 4) with a numpy
stand-in for the block context, checking every halo cell and node (corners
included) against the global field after ONE exchange."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2208_13409_b200 import multi

NX, NY = 40, 28


def test_decompose_covers_the_mesh_once():
    for px, py in ((1, 1), (2, 1), (2, 2), (4, 2)):
        specs = multi.decompose(NX, NY, px, py)
        seen = np.zeros((NY, NX), int)
        for s in specs:
            seen[s.oj:s.oj + s.bny, s.oi:s.oi + s.bnx] += 1
        assert (seen == 1).all()


def test_grid_shape_splits_long_axis_first():
    assert multi.grid_shape(1, 100, 50) == (1, 1)
    assert multi.grid_shape(2, 100, 50) == (2, 1)
    assert multi.grid_shape(4, 100, 100) == (2, 2)
    assert multi.grid_shape(8, 16384, 16384) == (4, 2)


def test_halo_plan_sizes_match_between_neighbours():
    for px, py in ((2, 1), (2, 2), (4, 2)):
        specs = multi.decompose(NX, NY, px, py)
        for s in specs:
            for dx, dy in multi.DIRS:
                n = s.neighbour(px, py, dx, dy)
                if n is None:
                    continue
                mine = multi.halo_rects(s, NX, NY, dx, dy, pack=False)
                theirs = multi.halo_rects(specs[n], NX, NY, -dx, -dy, pack=True)
                assert mine == theirs  # the same global rectangles


def test_owned_ranges_partition_cells_and_nodes():
    specs = multi.decompose(NX, NY, 4, 2)
    cells = np.zeros((NY + 4, NX + 4), int)
    nodes = np.zeros((NY + 5, NX + 5), int)
    for s in specs:
        oc, on = multi.own_ranges(s, NX, NY)
        cells[oc[2] + 2:oc[3] + 2, oc[0] + 2:oc[1] + 2] += 1
        nodes[on[2] + 2:on[3] + 2, on[0] + 2:on[1] + 2] += 1
    assert (cells == 1).all() and (nodes == 1).all()


class FakeBlock:
    """numpy stand-in for BlockSolver: one cell plane and one node plane over
    the block window, in global indices."""

    def __init__(self, spec):
        self.spec = spec
        h = multi.HALO
        self.i0, self.j0 = spec.oi - h, spec.oj - h
        self.cell = np.full((spec.bny + 2 * h, spec.bnx + 2 * h), np.nan)
        self.node = np.full((spec.bny + 2 * h + 1, spec.bnx + 2 * h + 1), np.nan)
        oc, on = multi.own_ranges(spec, NX, NY)
        for j in range(oc[2], oc[3]):
            for i in range(oc[0], oc[1]):
                self.cell[j - self.j0, i - self.i0] = gcell(i, j)
        for j in range(on[2], on[3]):
            for i in range(on[0], on[1]):
                self.node[j - self.j0, i - self.i0] = gnode(i, j)

    def _rects(self, dx, dy, pack):
        return multi.halo_rects(self.spec, NX, NY, dx, dy, pack)

    def halo_bytes(self, dx, dy, pack):
        rc, rn = self._rects(dx, dy, pack)
        return ((rc[1] - rc[0]) * (rc[3] - rc[2]) + (rn[1] - rn[0]) * (rn[3] - rn[2])) * 8

    def _view(self, ptr, n):
        return np.ctypeslib.as_array((C.c_double * n).from_address(ptr))

    def pack(self, dx, dy, ptr):
        rc, rn = self._rects(dx, dy, True)
        a = self.cell[rc[2] - self.j0:rc[3] - self.j0, rc[0] - self.i0:rc[1] - self.i0].ravel()
        b = self.node[rn[2] - self.j0:rn[3] - self.j0, rn[0] - self.i0:rn[1] - self.i0].ravel()
        self._view(ptr, a.size + b.size)[:] = np.concatenate([a, b])

    def unpack(self, dx, dy, ptr):
        rc, rn = self._rects(dx, dy, False)
        wc, hc = rc[1] - rc[0], rc[3] - rc[2]
        wn, hn = rn[1] - rn[0], rn[3] - rn[2]
        v = self._view(ptr, wc * hc + wn * hn)
        self.cell[rc[2] - self.j0:rc[3] - self.j0, rc[0] - self.i0:rc[1] - self.i0] = v[:wc * hc].reshape(hc, wc)
        self.node[rn[2] - self.j0:rn[3] - self.j0, rn[0] - self.i0:rn[1] - self.i0] = v[wc * hc:].reshape(hn, wn)


def gcell(i, j):
    return 1000.0 * j + i


def gnode(i, j):
    return -1000.0 * j - i - 0.5


def _worker(rank, world, port, px, py, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = multi.decompose(NX, NY, px, py)[rank]
        blk = FakeBlock(spec)
        tr = multi.DistTransport(blk, px, py, torch.device("cpu"))
        # scalar all-reduce: MAX of wave-speed bits, MIN of error keys
        wmax, nerr, err = tr.allreduce([[1000 + rank, multi.NO_ERR - rank, multi.NO_ERR, 0]])
        assert wmax == 1000 + world - 1 and nerr == multi.NO_ERR - (world - 1) and err == multi.NO_ERR
        tr.exchange()
        h = multi.HALO
        bad = 0
        for j in range(spec.oj - h, spec.oj + spec.bny + h):
            for i in range(spec.oi - h, spec.oi + spec.bnx + h):
                if not (-2 <= i < NX + 2 and -2 <= j < NY + 2):
                    continue
                if (i < 0 and spec.oi == 0) or (j < 0 and spec.oj == 0) or \
                        (i >= NX and spec.oi + spec.bnx == NX) or (j >= NY and spec.oj + spec.bny == NY):
                    continue  # physical ghost ring: filled by the wall BC, not the exchange
                v = blk.cell[j - blk.j0, i - blk.i0]
                if not (0 <= i < NX and 0 <= j < NY) or v != gcell(i, j):
                    bad += 1 if (0 <= i < NX and 0 <= j < NY) else 0
        for j in range(spec.oj - h, spec.oj + spec.bny + h + 1):
            for i in range(spec.oi - h, spec.oi + spec.bnx + h + 1):
                if 0 <= i <= NX and 0 <= j <= NY and blk.node[j - blk.j0, i - blk.i0] != gnode(i, j):
                    bad += 1
        q.put((rank, bad))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,px,py", [(2, 2, 1), (4, 2, 2)])
def test_gloo_halo_exchange_fills_every_halo_cell(world, px, py):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, px, py, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert res == [(r, 0) for r in range(world)]


@pytest.mark.parametrize("which", ["triple", "bubble", "voronoi3", "riemann"])
def test_window_paint_equals_global_paint(which):
    """Per-rank painting (cases.paint(window=...)) gives, bit for bit, the
    cells and nodes of the global painter inside the window."""
    from paper_2208_13409_b200 import cases
    case = {"triple": cases.triple_point(70, 30), "bubble": cases.shock_bubble(96),
            "voronoi3": cases.voronoi3(80), "riemann": cases.riemann2d(40)}[which]
    full = case.paint()
    g = 2
    nx, ny = case.cfg.mesh.nx, case.cfg.mesh.ny
    for (wi0, wj0, wnx, wny) in ((0, 0, 17, 11), (13, 5, min(30, nx - 13), min(20, ny - 5)), (nx - 9, ny - 7, 9, 7)):
        w = case.paint((wi0, wj0, wnx, wny))
        for a in range(case.cfg.nmat):
            for f in ("m", "e", "k"):
                want = getattr(full, f)[a][g + wj0:g + wj0 + wny, g + wi0:g + wi0 + wnx]
                assert np.array_equal(getattr(w, f)[a].view(np.int64), want.view(np.int64)), (f, a)
        want_u = full.u[g + wj0:g + wj0 + wny + 1, g + wi0:g + wi0 + wnx + 1]
        assert np.array_equal(w.u.view(np.int64), want_u.view(np.int64))

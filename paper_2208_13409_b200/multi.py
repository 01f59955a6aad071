"""2D block decomposition of the step over several GPUs.

Each block context (C-ABI ``h2d_create_block``) owns a rectangle of the global
mesh plus an 8-cell halo and computes the whole Lagrange + DirectCF step on its
window with redundant halo work.  Per step the blocks then need exactly:

* one all-reduce of three scalars: the next step's wave-speed maximum (MAX of
  the fp64 bit pattern), the first cfl_dt error key and the first step error
  key (MIN; keys order errors like the reference's program order), and
* one halo exchange of the State with the (up to) 8 neighbours, corners
  included, which the unsplit 9-point remap needs.

``Transport`` abstracts where blocks live: ``LocalTransport`` keeps several
blocks in one process (one GPU, device-to-device copies — used by the
bit-equality tests), ``DistTransport`` is one block per rank over
``torch.distributed`` (NCCL on GPUs, gloo in the CPU tests of the exchange
plumbing).  Owned values are bit-identical to the single-domain run.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import errors
from .abi import STEP_DIAG_DTYPE, Config, ErrorRec, HostState, Library, RunArgs, StepDiag, _ptr

HALO = 8
NO_ERR = (1 << 64) - 1
DIRS = [(dx, dy) for dy in (-1, 0, 1) for dx in (-1, 0, 1) if (dx, dy) != (0, 0)]


class Block(C.Structure):
    _fields_ = [("oi", C.c_int), ("oj", C.c_int), ("bnx", C.c_int), ("bny", C.c_int), ("halo", C.c_int)]


def split(n: int, parts: int) -> List[Tuple[int, int]]:
    """Near-equal 1D split: (origin, size) per part."""
    base, rem = divmod(n, parts)
    out, o = [], 0
    for p in range(parts):
        sz = base + (1 if p < rem else 0)
        out.append((o, sz))
        o += sz
    return out


def grid_shape(nranks: int, nx: int, ny: int) -> Tuple[int, int]:
    """px x py = nranks, splitting the longer axis first (1x1, 2x1, 2x2, 4x2)."""
    px, py = 1, 1
    n = nranks
    while n > 1:
        if nx / px >= ny / py:
            px *= 2
        else:
            py *= 2
        n //= 2
    assert px * py == nranks, "power-of-two rank counts"
    return px, py


@dataclass
class BlockSpec:
    rank: int
    bx: int
    by: int
    oi: int
    oj: int
    bnx: int
    bny: int

    def neighbour(self, px: int, py: int, dx: int, dy: int) -> Optional[int]:
        x, y = self.bx + dx, self.by + dy
        if 0 <= x < px and 0 <= y < py:
            return y * px + x
        return None


def decompose(nx: int, ny: int, px: int, py: int) -> List[BlockSpec]:
    xs, ys = split(nx, px), split(ny, py)
    return [BlockSpec(by * px + bx, bx, by, xs[bx][0], ys[by][0], xs[bx][1], ys[by][1])
            for by in range(py) for bx in range(px)]


_SIGS = {
    "create_block": ([C.POINTER(Config), C.POINTER(Block), C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "block_upload": ([C.c_void_p, C.c_void_p], C.c_int),
    "block_download": ([C.c_void_p, C.c_void_p], C.c_int),
    "block_begin": ([C.c_void_p, C.c_int, C.c_double, C.c_double], C.c_int),
    "block_step": ([C.c_void_p], C.c_int),
    "block_scalars": ([C.c_void_p, C.POINTER(C.c_ulonglong)], C.c_int),
    "block_set": ([C.c_void_p, C.POINTER(C.c_ulonglong)], C.c_int),
    "block_rollback": ([C.c_void_p], C.c_int),
    "halo_bytes": ([C.c_void_p, C.c_int, C.c_int, C.c_int], C.c_longlong),
    "halo_pack": ([C.c_void_p, C.c_int, C.c_int, C.c_void_p], C.c_int),
    "halo_unpack": ([C.c_void_p, C.c_int, C.c_int, C.c_void_p], C.c_int),
    "block_result": ([C.c_void_p, C.POINTER(RunArgs)], C.c_int),
    "block_init_window": ([C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double],
                          C.c_int),
    "nccl_unique_id": ([C.c_char_p], C.c_int),
    "comm_nccl": ([C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "comm_local": ([C.POINTER(C.c_void_p), C.c_int, C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "comm_destroy": ([C.c_void_p], None),
    "blocks_run": ([C.c_void_p, C.c_int, C.c_double, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_float)],
                   C.c_int),
    "comm_trace": ([C.c_void_p, C.c_int], C.c_int),
    "comm_trace_read": ([C.c_void_p, C.POINTER(C.c_float), C.c_int], C.c_int),
    "blocks_run_kind": ([C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(C.c_int),
                         C.POINTER(C.c_float)], C.c_int),
}


def bind(lib: Library):
    for name, (args, res) in _SIGS.items():
        f = getattr(lib.dll, lib.prefix + name)
        f.argtypes, f.restype = args, res
        lib.fn[name] = f
    return lib


class BlockSolver:
    """One block context of the decomposition (product library only)."""

    def __init__(self, lib: Library, cfg: Config, spec: BlockSpec, device: int = 0, halo: int = HALO):
        self.lib, self.cfg, self.spec = bind(lib), cfg, spec
        self._h = C.c_void_p()
        self.halo = halo
        b = Block(spec.oi, spec.oj, spec.bnx, spec.bny, halo)
        rc = lib.fn["create_block"](C.byref(cfg), C.byref(b), device, C.byref(self._h))
        if rc:
            raise errors.from_code(rc, f"h2d_create_block failed ({rc})")

    def close(self):
        if self._h:
            self.lib.fn["destroy"](self._h)
            self._h = C.c_void_p()

    __del__ = close

    def _check(self, rc):
        if rc:
            rec = ErrorRec()
            self.lib.fn["last_error"](self._h, C.byref(rec))
            raise errors.from_record(rec)

    def upload(self, g: HostState):
        self._check(self.lib.fn["block_upload"](self._h, C.byref(g.view())))

    def download_into(self, g: HostState):
        v = g.view()
        self._check(self.lib.fn["block_download"](self._h, C.byref(v)))
        g.step, g.time = v.step, v.time

    def window(self) -> Tuple[int, int, int, int]:
        """(wi0, wj0, wnx, wny): the block's storage window clipped to the
        mesh, the cells a rank paints for h2d_block_init_window."""
        s, H = self.spec, self.halo
        nx, ny = self.cfg.mesh.nx, self.cfg.mesh.ny
        i0, j0 = max(0, s.oi - H), max(0, s.oj - H)
        i1, j1 = min(nx, s.oi + s.bnx + H), min(ny, s.oj + s.bny + H)
        return i0, j0, i1 - i0, j1 - j0

    def init_window(self, w, step: int = 0, time: float = 0.0):
        """The block's initial State from a painted window (cases.WindowState):
        per-rank painting, then init_case's tail on the device."""
        v = w.view()
        self._check(self.lib.fn["block_init_window"](self._h, C.byref(v), w.wi0, w.wj0, w.wnx, w.wny, step,
                                                     time))

    def begin(self, max_steps: int, t_end: float, cfl: float):
        self._check(self.lib.fn["block_begin"](self._h, max_steps, t_end, cfl))

    def step(self):
        self._check(self.lib.fn["block_step"](self._h))

    def scalars(self) -> List[int]:
        out = (C.c_ulonglong * 4)()
        self._check(self.lib.fn["block_scalars"](self._h, out))
        return list(out)

    def set_scalars(self, wmax: int, next_err: int, err: int):
        self._check(self.lib.fn["block_set"](self._h, (C.c_ulonglong * 3)(wmax, next_err, err)))

    def rollback(self):
        self._check(self.lib.fn["block_rollback"](self._h))

    def halo_bytes(self, dx, dy, pack) -> int:
        return int(self.lib.fn["halo_bytes"](self._h, dx, dy, int(pack)))

    def pack(self, dx, dy, ptr):
        self._check(self.lib.fn["halo_pack"](self._h, dx, dy, C.c_void_p(ptr)))

    def unpack(self, dx, dy, ptr):
        self._check(self.lib.fn["halo_unpack"](self._h, dx, dy, C.c_void_p(ptr)))

    def result(self, cap: int, series: bool = False):
        """(RunArgs, dt log, error) of the block's run; with series=True the
        RunArgs carries `block_series`: this block's per-step make_diag
        partials (owned cells / nodes), merged across blocks by
        combine_series."""
        a = RunArgs()
        dts = np.zeros(max(cap, 1))
        a.dt_log, a.dt_log_cap = _ptr(dts), len(dts)
        ser = np.zeros(max(cap, 1), STEP_DIAG_DTYPE) if series else None
        if ser is not None:
            a.series, a.series_cap = ser.ctypes.data_as(C.POINTER(StepDiag)), len(ser)
        rc = self.lib.fn["block_result"](self._h, C.byref(a))
        err = None
        if rc:
            rec = ErrorRec()
            self.lib.fn["last_error"](self._h, C.byref(rec))
            err = errors.from_record(rec)
        a.block_series = ser[:a.steps_done].copy() if ser is not None else None
        return a, dts[:a.steps_done], err


class DeviceComm:
    """The library's block data plane (h2d_comm + h2d_blocks_run): the run
    loop of a decomposition with the per-step all-reduce and halo exchange
    enqueued on the device (NCCL across processes, or every block of the
    decomposition in this process on one device)."""

    def __init__(self, blocks: Sequence[BlockSolver], px: int, py: int, nccl_id: Optional[bytes] = None,
                 rank: int = 0):
        self.blocks = list(blocks)
        self.lib = self.blocks[0].lib
        self._h = C.c_void_p()
        if nccl_id is None:
            arr = (C.c_void_p * len(self.blocks))(*[b._h.value for b in self.blocks])
            rc = self.lib.fn["comm_local"](arr, px, py, C.byref(self._h))
        else:
            assert len(self.blocks) == 1
            rc = self.lib.fn["comm_nccl"](nccl_id, px, py, rank, self.blocks[0]._h, C.byref(self._h))
        if rc:
            self.blocks[0]._check(rc)
            raise errors.from_code(rc, f"h2d_comm creation failed ({rc})")

    @staticmethod
    def unique_id(lib: Library) -> bytes:
        bind(lib)
        buf = C.create_string_buffer(128)
        rc = lib.fn["nccl_unique_id"](buf)
        if rc:
            raise errors.from_code(rc, "h2d_nccl_unique_id failed")
        return buf.raw

    def run(self, max_steps: int, t_end: float, cfl: float, kind: int = 2) -> int:
        """Run to max_steps (absolute) / t_end; returns the steps done. The
        device time of the steps (CUDA events on the block's streams) is
        left in self.device_ms. kind: abi.REMAP_DIRECTCF (2: one halo
        exchange per step) or abi.REMAP_AD (0: the split remap, a second
        exchange between its two passes)."""
        done = C.c_int(0)
        ms = C.c_float(0.0)
        rc = self.lib.fn["blocks_run_kind"](self._h, kind, max_steps, t_end, cfl, C.byref(done), C.byref(ms))
        if rc:
            self.blocks[0]._check(rc)
        self.device_ms = ms.value
        return done.value

    TRACE_POINTS = ("lag_owned_start", "lag_owned_end", "lag_edge_end", "ad_mid_start", "ad_mid_end", "rest_end",
                    "allreduce_start", "halo_start", "halo_end")

    def trace(self, steps: int):
        """Record CUDA timing events at TRACE_POINTS of the first `steps` steps of the next run."""
        self.lib.fn["comm_trace"](self._h, steps)

    def trace_read(self) -> np.ndarray:
        """(steps, blocks, 9) milliseconds from each block's first step start (-1: point not reached)."""
        n = self.lib.fn["comm_trace_read"](self._h, None, 0)
        buf = (C.c_float * max(n, 1))()
        self.lib.fn["comm_trace_read"](self._h, buf, n)
        return np.array(buf[:n], dtype=np.float32).reshape(-1, len(self.blocks), len(self.TRACE_POINTS))

    def close(self):
        if self._h:
            self.lib.fn["comm_destroy"](self._h)
            self._h = C.c_void_p()

    __del__ = close


_SUMS = ("mass", "mass_mat", "momentum_x", "momentum_y", "internal_energy")


def combine_series(parts: Sequence[np.ndarray]) -> np.ndarray:
    """RunReport::series of the whole mesh from the blocks' per-step partials
    (block order fixed: sums added in that order, extrema combined; step, t
    and dt are the same on every block). No communication inside the step:
    the diagnostics are reduced across blocks only when they are read."""
    n = min(len(p) for p in parts)
    out = parts[0][:n].copy()
    for p in parts[1:]:
        p = p[:n]
        for f in _SUMS:
            out[f] = out[f] + p[f]
        out["min_rho"] = np.where(p["min_rho"] < out["min_rho"], p["min_rho"], out["min_rho"])
        out["min_p"] = np.where(p["min_p"] < out["min_p"], p["min_p"], out["min_p"])
        out["max_rho"] = np.where(out["max_rho"] < p["max_rho"], p["max_rho"], out["max_rho"])
        out["max_p"] = np.where(out["max_p"] < p["max_p"], p["max_p"], out["max_p"])
    return out


def combine(scal: Sequence[Sequence[int]]) -> Tuple[int, int, int]:
    """MAX of the wave-speed bits, MIN of the error keys (unsigned)."""
    return max(s[0] for s in scal), min(s[1] for s in scal), min(s[2] for s in scal)


def phase_of(key: int) -> int:
    return key >> 58


PH_NAN_CELL = 30  # h2d_device.cuh Phase


class LocalTransport:
    """All blocks in this process on one device; exchange by device copies
    through a scratch tensor (the same pack / unpack calls a rank makes)."""

    def __init__(self, blocks: Sequence[BlockSolver], px: int, py: int):
        import torch
        self.blocks, self.px, self.py = list(blocks), px, py
        nbytes = max(b.halo_bytes(dx, dy, 1) for b in blocks for dx, dy in DIRS)
        self.buf = torch.empty(max(nbytes // 8, 1), dtype=torch.float64, device="cuda")

    def allreduce(self, scal: List[List[int]]):
        return combine(scal)

    def exchange(self):
        for b in self.blocks:
            for dx, dy in DIRS:
                n = b.spec.neighbour(self.px, self.py, dx, dy)
                if n is None:
                    continue
                src = self.blocks[n]
                assert src.halo_bytes(-dx, -dy, 1) == b.halo_bytes(dx, dy, 0)
                src.pack(-dx, -dy, self.buf.data_ptr())
                b.unpack(dx, dy, self.buf.data_ptr())


class DistTransport:
    """One block per rank over torch.distributed (NCCL on GPUs)."""

    def __init__(self, block: BlockSolver, px: int, py: int, device):
        import torch
        import torch.distributed as dist
        self.block, self.px, self.py, self.dist, self.torch, self.device = block, px, py, dist, torch, device
        self.send, self.recv = {}, {}
        for dx, dy in DIRS:
            if block.spec.neighbour(px, py, dx, dy) is None:
                continue
            self.send[(dx, dy)] = torch.empty(block.halo_bytes(dx, dy, 1) // 8, dtype=torch.float64, device=device)
            self.recv[(dx, dy)] = torch.empty(block.halo_bytes(dx, dy, 0) // 8, dtype=torch.float64, device=device)

    def allreduce(self, scal: List[List[int]]):
        torch, dist = self.torch, self.dist
        s = scal[0]
        flip = 1 << 63  # unsigned order -> signed order
        t = torch.tensor([s[0] - flip, s[1] - flip, s[2] - flip], dtype=torch.int64, device=self.device)
        hi = t[:1].clone()
        lo = t[1:].clone()
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        return int(hi[0]) + flip, int(lo[0]) + flip, int(lo[1]) + flip

    def exchange(self):
        dist = self.dist
        ops = []
        for (dx, dy), buf in self.send.items():
            self.block.pack(dx, dy, buf.data_ptr())
        if self.device.type == "cuda":
            self.torch.cuda.synchronize(self.device)
        for (dx, dy), buf in self.send.items():
            peer = self.block.spec.neighbour(self.px, self.py, dx, dy)
            ops.append(dist.P2POp(dist.isend, buf, peer))
            ops.append(dist.P2POp(dist.irecv, self.recv[(dx, dy)], peer))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        if self.device.type == "cuda":
            self.torch.cuda.synchronize(self.device)
        for (dx, dy), buf in self.recv.items():
            self.block.unpack(dx, dy, buf.data_ptr())


def run_blocks(blocks: Sequence[BlockSolver], transport, max_steps: int, t_end: float, cfl: float,
               on_step=None) -> int:
    """The run loop (harness.cpp:390-412) over a decomposition: per step one
    graph launch per block, one 3-scalar all-reduce and one halo exchange.
    Returns the number of steps taken; raises the first error, with every
    block left at the last step all blocks completed."""
    for b in blocks:
        b.begin(max_steps, t_end, cfl)
    g = transport.allreduce([b.scalars() for b in blocks])
    for b in blocks:
        b.set_scalars(g[0], g[1], NO_ERR)
    steps = 0
    while True:
        for b in blocks:
            b.step()
        scal = [b.scalars() for b in blocks]
        wmax, nerr, err = transport.allreduce(scal)
        if err != NO_ERR:
            # every block whose own step committed rolls back when the first
            # error precedes the commit (nan_scan errors come after it); that
            # includes a block whose own error is a post-commit nan_scan error
            # (k_rollback is a no-op on a block that did not commit)
            if phase_of(err) < PH_NAN_CELL:
                for b in blocks:
                    b.rollback()
            for b in blocks:
                b.set_scalars(wmax, nerr, err)
            break
        if all(s[3] for s in scal):
            break
        steps += 1
        transport.exchange()
        for b in blocks:
            b.set_scalars(wmax, nerr, NO_ERR)
        if on_step:
            on_step(steps)
    return steps


def own_ranges(spec: BlockSpec, nx: int, ny: int, g: int = 2):
    """Owned cell / node ranges (global, half-open) — capi.cu block_ranges."""
    li, ri = spec.oi > 0, spec.oi + spec.bnx < nx
    bi, ti = spec.oj > 0, spec.oj + spec.bny < ny
    oc = (spec.oi if li else -g, spec.oi + spec.bnx if ri else nx + g,
          spec.oj if bi else -g, spec.oj + spec.bny if ti else ny + g)
    on = (spec.oi if li else -g, spec.oi + spec.bnx if ri else nx + g + 1,
          spec.oj if bi else -g, spec.oj + spec.bny if ti else ny + g + 1)
    return oc, on


def halo_rects(spec: BlockSpec, nx: int, ny: int, dx: int, dy: int, pack: bool, h: int = HALO):
    """Cell and node rectangles of the halo exchange with neighbour (dx, dy)
    (mirror of capi.cu halo_rects): pack = my owned data it needs, unpack =
    my halo it fills."""
    oc, on = own_ranges(spec, nx, ny)

    def axis(dd, o, n, c0, c1, n0, n1):
        if dd == 0:
            return (c0, c1), (n0, n1)
        if pack:
            return ((o + n - h, o + n), (o + n - h, o + n)) if dd > 0 else ((o, o + h), (o, o + h + 1))
        return ((o - h, o), (o - h, o)) if dd < 0 else ((o + n, o + n + h), (o + n, o + n + h + 1))

    (cx, nxr) = axis(dx, spec.oi, spec.bnx, oc[0], oc[1], on[0], on[1])
    (cy, nyr) = axis(dy, spec.oj, spec.bny, oc[2], oc[3], on[2], on[3])
    return (cx[0], cx[1], cy[0], cy[1]), (nxr[0], nxr[1], nyr[0], nyr[1])


def state_planes(nmat: int) -> Tuple[int, int]:
    """(cell planes, node planes) exchanged per step: m, e, k per material,
    normal x/y | u x/y (the derived fields are rebuilt on the device)."""
    return 3 * nmat + 2, 2

"""ctypes mirror of the C-ABI in ``include/h2d.h``.

The same structures bind three libraries that implement the ABI under
different symbol prefixes (see the header): the CUDA product (``h2d_``), and,
for the test suite only, the C restatement oracle (``h2do_``) and the
reference library itself (``h2dr_``).  The host-side state containers keep the
reference ``Field<T>`` layout (``proj/include/hydro/field.hpp:15-44``: two
ghost layers, row-major in j, contiguous in i, ``Vec2`` interleaved), so the
arrays here are byte-compatible with ``hydro::State`` (state.hpp:39-63).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import errors

ABI_VERSION = 3  # H2D_ABI_VERSION
RUN_LOG_CAP = 65536  # dt / StepDiag log entries of a run until t_end (h2d_run's device log)
MAX_MAT = 3   # H2D_MAX_MAT: the reference's kMaxMat (state.hpp:13) is 2, slot 3 = config 5
GHOST = 2     # kGhost, field.hpp:11

BC_PERIODIC, BC_WALL = 0, 1
EOS_PERFECT, EOS_STIFFENED = 0, 1
CORNER_UPWIND, CORNER_AVGMIN, CORNER_LINEARXY, CORNER_LINEARDIAG, CORNER_MULTID = range(5)
REMAP_AD, REMAP_DIRECT, REMAP_DIRECTCF = range(3)
DUMP_CSV, DUMP_VTK = 0, 1  # DumpFormat, io.hpp:9
OPT_SLIVER_ENERGY = 1  # H2D_OPT_SLIVER_ENERGY (no reference counterpart, default off)

_dp = C.POINTER(C.c_double)


class Mesh(C.Structure):
    """hydro::Mesh (mesh.hpp:13-29)."""
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("dx", C.c_double), ("dy", C.c_double),
                ("x0", C.c_double), ("y0", C.c_double), ("bc_x", C.c_int), ("bc_y", C.c_int)]


class Eos(C.Structure):
    """hydro::EosModel (eos.hpp:11-19)."""
    _fields_ = [("kind", C.c_int), ("gamma", C.c_double), ("pi", C.c_double)]


class Config(C.Structure):
    """MaterialSet + PseudoViscosityParams + ReconConfig (h2d_config)."""
    _fields_ = [("mesh", Mesh), ("nmat", C.c_int), ("eos", Eos * MAX_MAT),
                ("pv_a1", C.c_double), ("pv_a2", C.c_double), ("face_order", C.c_int),
                ("corner", C.c_int), ("interface_degrade", C.c_int), ("options", C.c_int)]


class StateView(C.Structure):
    _fields_ = [("m", _dp * MAX_MAT), ("e", _dp * MAX_MAT), ("k", _dp * MAX_MAT),
                ("vol", _dp), ("m_mix", _dp), ("e_mix", _dp), ("rho_mix", _dp), ("p_mix", _dp),
                ("iface_normal", _dp), ("u", _dp), ("step", C.c_int), ("time", C.c_double)]


class LagrangeView(C.Structure):
    _fields_ = [("u_half", _dp), ("u_lag", _dp), ("e_lag", _dp * MAX_MAT), ("vol_lag", _dp),
                ("q", _dp), ("floor_count", C.c_int)]


class HalfView(C.Structure):
    """h2d_half: HalfStepState (lagrange.hpp:14-24)."""
    _fields_ = [("x_half", _dp), ("u_half", _dp), ("vol_half", _dp), ("e_half", _dp * MAX_MAT),
                ("p_half", _dp * MAX_MAT), ("p_mix_half", _dp), ("q", _dp), ("floor_count", C.c_int)]


class RemapDiag(C.Structure):
    """hydro::RemapDiag (remap.hpp:42-46)."""
    _fields_ = [("max_k_violation", C.c_double), ("k_clip_count", C.c_int),
                ("mass_fix_count", C.c_int)]


class ErrorRec(C.Structure):
    _fields_ = [("kind", C.c_int), ("i", C.c_int), ("j", C.c_int), ("step", C.c_int),
                ("in_step", C.c_int), ("what", C.c_char * 256)]


class StepDiag(C.Structure):
    """hydro::StepDiag + Totals (harness.hpp:66-72, state.hpp:93-98)."""
    _fields_ = [("step", C.c_int), ("t", C.c_double), ("dt", C.c_double), ("mass", C.c_double),
                ("mass_mat", C.c_double * MAX_MAT), ("momentum_x", C.c_double), ("momentum_y", C.c_double),
                ("internal_energy", C.c_double), ("min_rho", C.c_double), ("max_rho", C.c_double),
                ("min_p", C.c_double), ("max_p", C.c_double)]


# the same record as a numpy structured dtype (C layout), for series arrays
STEP_DIAG_DTYPE = np.dtype([("step", "<i4"), ("t", "<f8"), ("dt", "<f8"), ("mass", "<f8"),
                            ("mass_mat", "<f8", (MAX_MAT,)), ("momentum_x", "<f8"), ("momentum_y", "<f8"),
                            ("internal_energy", "<f8"), ("min_rho", "<f8"), ("max_rho", "<f8"),
                            ("min_p", "<f8"), ("max_p", "<f8")], align=True)
assert STEP_DIAG_DTYPE.itemsize == C.sizeof(StepDiag)


class RunArgs(C.Structure):
    _fields_ = [("max_steps", C.c_int), ("t_end", C.c_double), ("cfl", C.c_double),
                ("remap_kind", C.c_int), ("dt_log", _dp), ("dt_log_cap", C.c_int),
                ("steps_done", C.c_int), ("floor_count", C.c_int), ("diag", RemapDiag),
                ("series", C.POINTER(StepDiag)), ("series_cap", C.c_int)]


def make_config(nx, ny, dx, dy, x0=0.0, y0=0.0, bc_x=BC_WALL, bc_y=BC_WALL, eos=((EOS_PERFECT, 1.4, 0.0),),
                a1=0.2, a2=1.0, face_order=2, corner=CORNER_LINEARDIAG, interface_degrade=True,
                options=0) -> Config:
    """Build an h2d_config; defaults are the reference defaults
    (lagrange.hpp:7-10, reconstruct.hpp:9-13) with walls on every side."""
    cfg = Config()
    cfg.mesh = Mesh(nx, ny, dx, dy, x0, y0, bc_x, bc_y)
    cfg.nmat = len(eos)
    for a, (kind, gamma, pi) in enumerate(eos):
        cfg.eos[a] = Eos(kind, gamma, pi)
    cfg.pv_a1, cfg.pv_a2 = a1, a2
    cfg.face_order, cfg.corner, cfg.interface_degrade = face_order, corner, int(bool(interface_degrade))
    cfg.options = options
    return cfg


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


@dataclass
class HostState:
    """Host copy of a State in the reference layout (state.hpp:39-63).

    Cell arrays are (ny+4, nx+4); node arrays (ny+5, nx+5); Vec2 arrays carry a
    trailing axis of 2.  ``cell(f)`` / ``node(f)`` give the interior views."""
    nx: int
    ny: int
    nmat: int
    m: np.ndarray
    e: np.ndarray
    k: np.ndarray
    vol: np.ndarray
    m_mix: np.ndarray
    e_mix: np.ndarray
    rho_mix: np.ndarray
    p_mix: np.ndarray
    iface_normal: np.ndarray
    u: np.ndarray
    step: int = 0
    time: float = 0.0

    @classmethod
    def empty(cls, nx: int, ny: int, nmat: int, cv: float = 0.0) -> "HostState":
        """make_state (state.cpp:5-23): k0 = 1, normals (1, 0), vol = dx*dy."""
        cs, ns = (ny + 2 * GHOST, nx + 2 * GHOST), (ny + 1 + 2 * GHOST, nx + 1 + 2 * GHOST)
        k = np.zeros((MAX_MAT,) + cs)
        k[0] = 1.0
        nrm = np.zeros(cs + (2,))
        nrm[..., 0] = 1.0
        return cls(nx, ny, nmat, np.zeros((MAX_MAT,) + cs), np.zeros((MAX_MAT,) + cs), k,
                   np.full(cs, cv), np.zeros(cs), np.zeros(cs), np.zeros(cs), np.zeros(cs), nrm,
                   np.zeros(ns + (2,)))

    def copy(self) -> "HostState":
        return HostState(self.nx, self.ny, self.nmat, *(getattr(self, f).copy() for f in
                         ("m", "e", "k", "vol", "m_mix", "e_mix", "rho_mix", "p_mix", "iface_normal", "u")),
                         step=self.step, time=self.time)

    def cell(self, f: np.ndarray) -> np.ndarray:
        return f[..., GHOST:GHOST + self.ny, GHOST:GHOST + self.nx] if f.ndim != 3 or f.shape[-1] != 2 \
            else f[GHOST:GHOST + self.ny, GHOST:GHOST + self.nx]

    def node(self, f: np.ndarray) -> np.ndarray:
        return f[GHOST:GHOST + self.ny + 1, GHOST:GHOST + self.nx + 1]

    def view(self, derived: bool = True) -> StateView:
        v = StateView()
        for a in range(MAX_MAT):
            v.m[a], v.e[a], v.k[a] = _ptr(self.m[a]), _ptr(self.e[a]), _ptr(self.k[a])
        if derived:
            v.vol, v.m_mix, v.e_mix = _ptr(self.vol), _ptr(self.m_mix), _ptr(self.e_mix)
            v.rho_mix, v.p_mix = _ptr(self.rho_mix), _ptr(self.p_mix)
        v.iface_normal, v.u = _ptr(self.iface_normal), _ptr(self.u)
        v.step, v.time = self.step, self.time
        return v

    def nbytes(self) -> int:
        return sum(getattr(self, f).nbytes for f in
                   ("m", "e", "k", "vol", "m_mix", "e_mix", "rho_mix", "p_mix", "iface_normal", "u"))


@dataclass
class HostLagrange:
    """Host copy of a LagrangeResult (lagrange.hpp:38-45)."""
    u_half: np.ndarray
    u_lag: np.ndarray
    e_lag: np.ndarray
    vol_lag: np.ndarray
    q: np.ndarray
    floor_count: int = 0

    @classmethod
    def empty(cls, nx: int, ny: int) -> "HostLagrange":
        cs, ns = (ny + 2 * GHOST, nx + 2 * GHOST), (ny + 1 + 2 * GHOST, nx + 1 + 2 * GHOST)
        return cls(np.zeros(ns + (2,)), np.zeros(ns + (2,)), np.zeros((MAX_MAT,) + cs), np.zeros(cs),
                   np.zeros(cs))

    def view(self) -> LagrangeView:
        v = LagrangeView()
        v.u_half, v.u_lag = _ptr(self.u_half), _ptr(self.u_lag)
        for a in range(MAX_MAT):
            v.e_lag[a] = _ptr(self.e_lag[a])
        v.vol_lag, v.q = _ptr(self.vol_lag), _ptr(self.q)
        v.floor_count = self.floor_count
        return v


SC_IN, SC_OUT = 48, 8  # H2D_SC_IN / H2D_SC_OUT
(SC_VAN_LEER, SC_LIMITED_GRADIENT, SC_FACE_VALUE, SC_CORNER_VALUE, SC_MULTID_PLANE, SC_CLIPPED_FRACTION,
 SC_PLACE_INTERFACE, SC_YOUNGS_NORMAL, SC_CELL_VOLUME, SC_CF_CORNER_FLUX, SC_CF_FACE_FLUX_X, SC_CF_FACE_FLUX_Y,
 SC_PSEUDO_VISCOSITY, SC_DIV_U_CELL, SC_GRAD_PQ_NODE, SC_AD_FACE_FLUX) = range(16)


@dataclass
class HostHalf:
    """Host copy of a HalfStepState (lagrange.hpp:14-24)."""
    x_half: np.ndarray
    u_half: np.ndarray
    vol_half: np.ndarray
    e_half: np.ndarray
    p_half: np.ndarray
    p_mix_half: np.ndarray
    q: np.ndarray
    floor_count: int = 0

    @classmethod
    def empty(cls, nx: int, ny: int) -> "HostHalf":
        cs, ns = (ny + 2 * GHOST, nx + 2 * GHOST), (ny + 1 + 2 * GHOST, nx + 1 + 2 * GHOST)
        return cls(np.zeros(ns + (2,)), np.zeros(ns + (2,)), np.zeros(cs), np.zeros((MAX_MAT,) + cs),
                   np.zeros((MAX_MAT,) + cs), np.zeros(cs), np.zeros(cs))

    def view(self) -> HalfView:
        v = HalfView()
        v.x_half, v.u_half, v.vol_half = _ptr(self.x_half), _ptr(self.u_half), _ptr(self.vol_half)
        for a in range(MAX_MAT):
            v.e_half[a], v.p_half[a] = _ptr(self.e_half[a]), _ptr(self.p_half[a])
        v.p_mix_half, v.q, v.floor_count = _ptr(self.p_mix_half), _ptr(self.q), self.floor_count
        return v


def scalar_eval(lib: "Library", op: int, records: np.ndarray):
    """h2d_scalar_eval over records[n, <= SC_IN] -> (out[n, SC_OUT], flags[n])."""
    n = len(records)
    inp = np.zeros((n, SC_IN))
    inp[:, :records.shape[1]] = records
    out = np.zeros((n, SC_OUT))
    flags = np.zeros(n, np.int32)
    rc = lib.fn["scalar_eval"](op, n, _ptr(inp), _ptr(out), flags.ctypes.data_as(C.POINTER(C.c_int)))
    if rc:
        raise errors.from_code(rc, f"{lib.prefix}scalar_eval failed ({rc})")
    return out, flags


@dataclass
class RunResult:
    steps_done: int
    floor_count: int
    diag: dict
    dts: np.ndarray = field(default_factory=lambda: np.zeros(0))
    # one make_diag record per step done (RunReport::series[1:], harness.cpp:410)
    series: np.ndarray = field(default_factory=lambda: np.zeros(0, STEP_DIAG_DTYPE))


_SIGS = {
    "abi_version": ([], C.c_int),
    "create": ([C.POINTER(Config), C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "destroy": ([C.c_void_p], None),
    "upload_state": ([C.c_void_p, C.POINTER(StateView)], C.c_int),
    "download_state": ([C.c_void_p, C.POINTER(StateView)], C.c_int),
    "fill_ghosts": ([C.c_void_p], C.c_int),
    "sync_derived": ([C.c_void_p], C.c_int),
    "update_interface_normals": ([C.c_void_p], C.c_int),
    "cfl_dt": ([C.c_void_p, C.c_double, _dp], C.c_int),
    "lagrange_step": ([C.c_void_p, C.c_double, C.POINTER(LagrangeView)], C.c_int),
    "set_lagrange": ([C.c_void_p, C.POINTER(LagrangeView)], C.c_int),
    "remap_step": ([C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(RemapDiag)], C.c_int),
    "run": ([C.c_void_p, C.POINTER(RunArgs)], C.c_int),
    "totals": ([C.c_void_p, _dp], C.c_int),
    "step_diag_now": ([C.c_void_p, C.c_double, C.POINTER(StepDiag)], C.c_int),
    "last_error": ([C.c_void_p, C.POINTER(ErrorRec)], C.c_int),
}
# product-only extras (benchmark support) and the field / checkpoint I/O
# (the reference shim exports write_fields and diag_line)
_EXTRA = {
    "write_fields": ([C.c_void_p, C.c_char_p, C.c_int], C.c_int),
    "write_fields_host": ([C.POINTER(Config), C.POINTER(StateView), C.c_char_p, C.c_int], C.c_int),
    "diag_line": ([C.POINTER(StepDiag), C.c_char_p, C.c_int], C.c_int),
    "save_state": ([C.c_void_p, C.c_char_p], C.c_int),
    "load_state": ([C.c_void_p, C.c_char_p], C.c_int),
    "save_state_host": ([C.POINTER(Config), C.POINTER(StateView), C.c_char_p], C.c_int),
    "load_state_host": ([C.POINTER(Config), C.POINTER(StateView), C.c_char_p], C.c_int),
    "predict": ([C.c_void_p, C.c_double, C.POINTER(HalfView)], C.c_int),
    "correct": ([C.c_void_p, C.c_double, C.POINTER(HalfView), C.POINTER(LagrangeView)], C.c_int),
    "remap_single_axis": ([C.c_void_p, C.c_double, C.c_int, C.c_int, C.POINTER(RemapDiag)], C.c_int),
    "scalar_eval": ([C.c_int, C.c_int, _dp, _dp, C.POINTER(C.c_int)], C.c_int),
    "launch_count": ([], C.c_longlong),
    "step_timed": ([C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_float)], C.c_int),
    "flush_l2": ([C.c_void_p, C.c_longlong], C.c_int),
}

ABI_SYMBOLS = tuple(_SIGS)


class Library:
    """A loaded implementation of the h2d ABI under ``prefix``."""

    def __init__(self, path: str, prefix: str):
        self.path, self.prefix = path, prefix
        self.dll = C.CDLL(path)
        self.fn = {}
        for name, (args, res) in _SIGS.items():
            f = getattr(self.dll, prefix + name)
            f.argtypes, f.restype = args, res
            self.fn[name] = f
        for name, (args, res) in _EXTRA.items():
            f = getattr(self.dll, prefix + name, None)
            if f is not None:
                f.argtypes, f.restype = args, res
                self.fn[name] = f
        if self.fn["abi_version"]() != ABI_VERSION:
            raise RuntimeError(f"{path}: unexpected ABI version")


class Solver:
    """One context of an h2d ABI implementation: Mesh + materials + params
    plus a resident State (and LagrangeResult).  Mirrors the reference free
    functions (cfl_dt, lagrange_step, remap_step, run) as methods; reference
    exceptions are re-raised as the matching ``errors`` classes."""

    def __init__(self, lib: Library, cfg: Config, device: int = -1):
        self.lib, self.cfg = lib, cfg
        self.nx, self.ny, self.nmat = cfg.mesh.nx, cfg.mesh.ny, cfg.nmat
        self._h = C.c_void_p()
        rc = lib.fn["create"](C.byref(cfg), device, C.byref(self._h))
        if rc:
            if rc == errors.H2D_ERR_SIM:
                raise errors.SimError("mesh must be at least 3x3 with positive spacing")
            raise errors.from_code(rc, f"{lib.prefix}create failed ({rc})")

    def close(self):
        if self._h:
            self.lib.fn["destroy"](self._h)
            self._h = C.c_void_p()

    __del__ = close

    def _check(self, rc: int):
        if rc:
            rec = ErrorRec()
            self.lib.fn["last_error"](self._h, C.byref(rec))
            raise errors.from_record(rec)

    def last_error(self) -> ErrorRec:
        rec = ErrorRec()
        self.lib.fn["last_error"](self._h, C.byref(rec))
        return rec

    # -- state ---------------------------------------------------------------
    def upload(self, st: HostState, derived: bool = True):
        self._check(self.lib.fn["upload_state"](self._h, C.byref(st.view(derived))))

    def download(self) -> HostState:
        st = HostState.empty(self.nx, self.ny, self.nmat)
        v = st.view()
        self._check(self.lib.fn["download_state"](self._h, C.byref(v)))
        st.step, st.time = v.step, v.time
        return st

    def fill_ghosts(self):
        self._check(self.lib.fn["fill_ghosts"](self._h))

    def sync_derived(self):
        self._check(self.lib.fn["sync_derived"](self._h))

    def update_interface_normals(self):
        self._check(self.lib.fn["update_interface_normals"](self._h))

    def init_from(self, painted: HostState):
        """init_case tail (harness.cpp:286-288) on a painted interior."""
        self.upload(painted, derived=False)
        self.fill_ghosts()
        self.sync_derived()
        self.update_interface_normals()

    # -- step ----------------------------------------------------------------
    def cfl_dt(self, cfl: float) -> float:
        dt = C.c_double()
        self._check(self.lib.fn["cfl_dt"](self._h, cfl, C.byref(dt)))
        return dt.value

    def lagrange_step(self, dt: float, download: bool = True) -> Optional[HostLagrange]:
        out = HostLagrange.empty(self.nx, self.ny) if download else None
        v = out.view() if out else None
        self._check(self.lib.fn["lagrange_step"](self._h, dt, C.byref(v) if v else None))
        if out:
            out.floor_count = v.floor_count
        return out

    def predict(self, dt: float) -> HostHalf:
        """HalfStepState predict(State, MaterialSet, dt, PseudoViscosityParams)."""
        out = HostHalf.empty(self.nx, self.ny)
        v = out.view()
        self._check(self.lib.fn["predict"](self._h, dt, C.byref(v)))
        out.floor_count = v.floor_count
        return out

    def correct(self, dt: float, half: HostHalf) -> HostLagrange:
        """LagrangeResult correct(State, MaterialSet, HalfStepState, dt)."""
        out = HostLagrange.empty(self.nx, self.ny)
        v = out.view()
        self._check(self.lib.fn["correct"](self._h, dt, C.byref(half.view()), C.byref(v)))
        out.floor_count = v.floor_count
        return out

    def remap_single_axis(self, dt: float, axis_x: bool, remap_velocity: bool = True,
                          diag: Optional[RemapDiag] = None):
        self._check(self.lib.fn["remap_single_axis"](self._h, dt, int(axis_x), int(remap_velocity),
                                                     C.byref(diag) if diag is not None else None))

    def set_lagrange(self, lag: HostLagrange):
        self._check(self.lib.fn["set_lagrange"](self._h, C.byref(lag.view())))

    def remap_step(self, dt: float, kind: int = REMAP_DIRECTCF, x_first: bool = True,
                   remap_velocity: bool = True, diag: Optional[RemapDiag] = None):
        self._check(self.lib.fn["remap_step"](self._h, dt, kind, int(x_first), int(remap_velocity),
                                              C.byref(diag) if diag is not None else None))

    def run(self, max_steps: int, t_end: float = 1e30, cfl: float = 0.3, log_dt: bool = True,
            kind: int = REMAP_DIRECTCF, series: bool = False) -> RunResult:
        a = RunArgs()
        a.max_steps, a.t_end, a.cfl, a.remap_kind = max_steps, t_end, cfl, kind
        cap = max_steps if max_steps > 0 else RUN_LOG_CAP  # (max_steps is the absolute end step)
        dts = np.zeros(max(cap, 1)) if log_dt else None
        if dts is not None:
            a.dt_log, a.dt_log_cap = _ptr(dts), len(dts)
        ser = np.zeros(max(cap, 1), STEP_DIAG_DTYPE) if series else None
        if ser is not None:
            a.series, a.series_cap = ser.ctypes.data_as(C.POINTER(StepDiag)), len(ser)
        rc = self.lib.fn["run"](self._h, C.byref(a))
        res = RunResult(a.steps_done, a.floor_count,
                        dict(max_k_violation=a.diag.max_k_violation, k_clip_count=a.diag.k_clip_count,
                             mass_fix_count=a.diag.mass_fix_count),
                        dts[:a.steps_done] if dts is not None else np.zeros(0),
                        ser[:a.steps_done].copy() if ser is not None else np.zeros(0, STEP_DIAG_DTYPE))
        if rc:
            rec = self.last_error()
            err = errors.from_record(rec)
            err.partial = res
            raise err
        return res

    STEP_GROUPS = ("start", "lagrange", "remap_tile", "slivers", "dual", "post", "total", "ghosts_commit")

    def step_timed(self, cfl: float, t_end: float = 1e30, phases: bool = False, kind: int = REMAP_DIRECTCF) -> dict:
        """One run-loop step timed with CUDA events (product only): returns
        milliseconds per kernel group (STEP_GROUPS); phases=False replays the
        production CUDA graph and only "total" is set."""
        ms = (C.c_float * 8)()
        self._check(self.lib.fn["step_timed"](self._h, cfl, t_end, int(phases), int(kind), ms))
        return {k: float(ms[q]) for q, k in enumerate(self.STEP_GROUPS)}

    def flush_l2(self, nbytes: int = 512 << 20):
        self._check(self.lib.fn["flush_l2"](self._h, nbytes))

    # -- I/O (io.hpp:17-22) and checkpoints -----------------------------------
    def write_fields(self, path: str, fmt: int = DUMP_CSV):
        """write_fields(s, path, fmt) of the resident State (io.cpp:72-83)."""
        self._check(self.lib.fn["write_fields"](self._h, path.encode(), fmt))

    def save_state(self, path: str):
        self._check(self.lib.fn["save_state"](self._h, path.encode()))

    def load_state(self, path: str):
        self._check(self.lib.fn["load_state"](self._h, path.encode()))

    def step_diag(self, dt: float = 0.0) -> np.void:
        """make_diag(s, dt) of the current State (harness.cpp:360-376)."""
        out = np.zeros(1, STEP_DIAG_DTYPE)
        self._check(self.lib.fn["step_diag_now"](self._h, dt, out.ctypes.data_as(C.POINTER(StepDiag))))
        return out[0]

    def totals(self) -> dict:
        out = (C.c_double * 6)()
        self._check(self.lib.fn["totals"](self._h, out))
        return dict(mass=out[0], mass_mat=(out[1], out[2]), momentum=(out[3], out[4]), internal_energy=out[5])


def diag_line(lib: Library, rec) -> str:
    """append_diag_line (io.cpp:85-92) of one StepDiag record."""
    r = np.zeros(1, STEP_DIAG_DTYPE)
    r[0] = rec
    buf = C.create_string_buffer(1024)
    rc = lib.fn["diag_line"](r.ctypes.data_as(C.POINTER(StepDiag)), buf, len(buf))
    if rc:
        raise errors.from_code(rc, "diag_line failed")
    return buf.value.decode()

"""Front ends wired to the device path.

Python mirror of the reference's driver layer over the CUDA product:

* ``CaseSpec`` / ``build_case`` / ``case_list`` — the case catalogue
  (harness.hpp:14-58, harness.cpp:22-163), plus the BASELINE.json configs;
* ``run`` / ``RunReport`` / ``StepDiag`` — ``RunReport run(const CaseSpec&,
  const StepHook&)`` (harness.cpp:380-424): init_case, the step loop (the
  dynamic branch runs as the device-resident ``h2d_run``; the imposed-velocity
  branch drives ``h2d_remap_step`` with ``kinematic_lagrange`` /
  ``impose_velocity``), the make_diag series, counters and L2 errors;
* ``RunConfig`` / ``parse_config`` / ``load_config`` / ``configure_case`` —
  the key = value run configuration (config.hpp, config.cpp:54-110);
* ``run_case`` — the pybind11 entry of the reference (bindings/module.cpp:50-93),
  same arguments and the same result keys.

The CLI (``python -m paper_2208_13409_b200 run <config>``) is in
``__main__.py``.  Every scheme (DirectCF, Direct, AD) and corner scheme
runs on the device.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace
from typing import Callable, List, Optional, Tuple

import numpy as np

from . import abi, cases, errors
from .abi import (BC_PERIODIC, BC_WALL, CORNER_AVGMIN, CORNER_LINEARDIAG, CORNER_LINEARXY, CORNER_MULTID,
                  CORNER_UPWIND, EOS_PERFECT, EOS_STIFFENED, GHOST, REMAP_AD, REMAP_DIRECT, REMAP_DIRECTCF,
                  STEP_DIAG_DTYPE, HostLagrange, HostState, RemapDiag, make_config)
from .cases import ALL, CIRCLE, HALFPLANE_X, RECTANGLE, Region

NONE, CONSTANT, ROTATION = range(3)  # ImposedVelocity, harness.hpp:12

SCHEMES = {"AD": REMAP_AD, "Direct": REMAP_DIRECT, "DirectCF": REMAP_DIRECTCF}
SCHEME_NAMES = {v: k for k, v in SCHEMES.items()}
CORNERS = {"upwind": CORNER_UPWIND, "avg_min": CORNER_AVGMIN, "linear_xy": CORNER_LINEARXY,
           "linear_diag": CORNER_LINEARDIAG, "multid": CORNER_MULTID}

AIR = (EOS_PERFECT, 1.4, 0.0)        # air_eos, harness.cpp:29
WATER = (EOS_STIFFENED, 7.0, 2.1e9)  # water_eos, harness.cpp:30


@dataclass
class CaseSpec:
    """hydro::CaseSpec (harness.hpp:31-58)."""
    name: str = ""
    nx: int = 0
    ny: int = 0
    x0: float = 0.0
    y0: float = 0.0
    lx: float = 1.0
    ly: float = 1.0
    bc_x: int = BC_PERIODIC
    bc_y: int = BC_PERIODIC
    eos: List[Tuple[int, float, float]] = field(default_factory=lambda: [AIR])  # MaterialSet
    regions: List[Region] = field(default_factory=list)
    t_end: float = 0.0
    cfl: float = 0.3
    max_steps: int = 0
    scheme: int = REMAP_DIRECTCF
    face_order: int = 2
    corner: int = CORNER_LINEARDIAG
    interface_degrade: bool = True
    pv: Tuple[float, float] = (0.2, 1.0)
    imposed: int = NONE
    u_const: Tuple[float, float] = (0.0, 0.0)
    flip_time: float = -1.0
    rot_center: Tuple[float, float] = (0.0, 0.0)
    rot_omega: float = 0.0

    @property
    def nmat(self) -> int:
        return len(self.eos)

    def config(self) -> abi.Config:
        """Mesh (CaseSpec::make_mesh, harness.cpp:9-11) + materials + params."""
        return make_config(self.nx, self.ny, self.lx / self.nx, self.ly / self.ny, self.x0, self.y0,
                           self.bc_x, self.bc_y, eos=tuple(self.eos), a1=self.pv[0], a2=self.pv[1],
                           face_order=self.face_order, corner=self.corner,
                           interface_degrade=self.interface_degrade)


def case_list() -> List[str]:
    """harness.cpp:22-25, then the BASELINE.json configurations."""
    return ["uniform", "mono_advect", "mono_rotation", "multimat_advect", "water_air_rotation", "haas",
            "impact"] + list(_BASELINE)


def _scaled(n: int, divisor: int) -> int:  # harness.cpp:37
    return max(8, n // max(1, divisor))


def _from_case(c: cases.Case, name: str) -> CaseSpec:
    m = c.cfg.mesh
    return CaseSpec(name=name, nx=m.nx, ny=m.ny, lx=m.dx * m.nx, ly=m.dy * m.ny, bc_x=m.bc_x, bc_y=m.bc_y,
                    eos=[(c.cfg.eos[a].kind, c.cfg.eos[a].gamma, c.cfg.eos[a].pi) for a in range(c.cfg.nmat)],
                    regions=list(c.regions), t_end=1e30, cfl=c.cfl, max_steps=c.steps)


# BASELINE.json configs 1-4: name -> builder(divisor)
_BASELINE = {
    "riemann2d": lambda d: _from_case(cases.riemann2d(_scaled(256, d)), "riemann2d"),
    "sedov": lambda d: _from_case(cases.sedov(_scaled(1024, d)), "sedov"),
    "triple_point": lambda d: _from_case(cases.triple_point(_scaled(2048, d), _scaled(1024, d)), "triple_point"),
    "shock_bubble": lambda d: _from_case(cases.shock_bubble(_scaled(8192, d)), "shock_bubble"),
}


def build_case(name: str, divisor: int = 1) -> CaseSpec:
    """CaseSpec build_case(const std::string&, int divisor) (harness.cpp:41-163)."""
    n = lambda v: _scaled(v, divisor)  # noqa: E731
    if name == "uniform":
        return CaseSpec(name=name, nx=n(50), ny=n(50), eos=[AIR],
                        regions=[Region(ALL, mat=0, rho=1.0, p=1e5, u=(5.0, 5.0))], t_end=1.0, max_steps=50)
    if name in ("mono_advect", "multimat_advect"):
        multi = name == "multimat_advect"
        return CaseSpec(name=name, nx=n(100), ny=n(100), eos=[AIR, AIR] if multi else [AIR],
                        regions=[Region(ALL, mat=0, rho=1.29 if multi else 0.1, p=1e5),
                                 Region(RECTANGLE, rect=(0.2, 0.2, 0.4, 0.4), mat=1 if multi else 0,
                                        rho=1.29 if multi else 10.0, p=1e5)],
                        imposed=CONSTANT, u_const=(5.0, 5.0), flip_time=0.06, t_end=0.12)
    if name == "mono_rotation":
        return CaseSpec(name=name, nx=n(100), ny=n(100), eos=[AIR],
                        regions=[Region(ALL, mat=0, rho=0.1, p=1e5),
                                 Region(RECTANGLE, rect=(0.4, 0.65, 0.6, 0.85), mat=0, rho=10.0, p=1e5)],
                        imposed=ROTATION, rot_center=(0.5, 0.5), rot_omega=2.0 * 3.14159265358979323846,
                        t_end=1.0)
    if name == "water_air_rotation":
        return CaseSpec(name=name, nx=n(400), ny=n(400), lx=4.0, ly=4.0, eos=[AIR, WATER],
                        regions=[Region(ALL, mat=0, rho=1.29, p=1e5),
                                 Region(RECTANGLE, rect=(1.6, 2.5, 2.4, 3.3), mat=1, rho=1000.0, p=1e5)],
                        imposed=ROTATION, rot_center=(2.0, 2.0),
                        rot_omega=2.0 * 3.14159265358979323846 * 1e3, t_end=1e-3)
    if name == "haas":
        return CaseSpec(name=name, nx=n(1000), ny=n(90), lx=10.0, ly=0.09, bc_x=BC_WALL, bc_y=BC_WALL,
                        eos=[AIR, (EOS_PERFECT, 1.66, 0.0)],
                        regions=[Region(ALL, mat=0, rho=1.0, p=1e5),
                                 Region(HALFPLANE_X, xsplit=0.8, mat=0, rho=1.376363, p=1.5698e5, u=(124.824, 0.0)),
                                 Region(CIRCLE, center=(1.0, 0.045), radius=0.04, mat=1, rho=0.18187, p=1e5)],
                        t_end=1e-3)
    if name == "impact":
        return CaseSpec(name=name, nx=n(320), ny=n(160), lx=0.10, ly=0.05, bc_x=BC_WALL, bc_y=BC_WALL,
                        eos=[AIR, WATER],
                        regions=[Region(ALL, mat=0, rho=1.29, p=1e5, u=(-1000.0, 0.0)),
                                 Region(RECTANGLE, rect=(0.0, 0.0, 0.01, 0.05), mat=1, rho=1000.0, p=1e5),
                                 Region(CIRCLE, center=(0.03, 0.025), radius=0.01, mat=1, rho=1000.0, p=1e5,
                                        u=(-1000.0, 0.0))],
                        t_end=6e-3)
    if name in _BASELINE:
        return _BASELINE[name](divisor)
    raise errors.SimError("unknown case: " + name)


# ---- run configuration (config.hpp, config.cpp) -------------------------------------

@dataclass
class RunConfig:
    case_name: str = ""
    scheme: int = REMAP_DIRECTCF
    face_order: int = 2
    corner: int = CORNER_LINEARDIAG
    cfl: float = 0.3
    divisor: int = 1
    t_end: float = -1.0
    max_steps: int = 0
    out_dir: str = "out"
    output_every: int = 0
    seed: int = 0


def _fail(line: int, msg: str):
    raise errors.SimError(f"config line {line}: {msg}")


def _num(v: str, line: int) -> float:
    """parse_num (config.cpp:41-50): std::stod of the whole token."""
    try:
        return float(v)
    except ValueError:
        _fail(line, f"not a number: '{v}'")


def parse_config(text: str) -> RunConfig:
    """RunConfig parse_config(const std::string&) (config.cpp:54-85)."""
    rc = RunConfig()
    for lineno, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip(" \t\r")
        if not line:
            continue
        if "=" not in line:
            _fail(lineno, "expected 'key = value'")
        key, val = (x.strip(" \t\r") for x in line.split("=", 1))
        if key == "case":
            rc.case_name = val
        elif key == "scheme":
            if val not in SCHEMES:
                _fail(lineno, f"invalid scheme '{val}' (valid: AD, Direct, DirectCF)")
            rc.scheme = SCHEMES[val]
        elif key == "face_order":
            o = int(_num(val, lineno))
            if o not in (1, 2):
                _fail(lineno, "face_order must be 1 or 2")
            rc.face_order = o
        elif key == "corner_scheme":
            if val not in CORNERS:
                _fail(lineno, f"invalid corner_scheme '{val}' (valid: upwind, avg_min, linear_xy, "
                              "linear_diag, multid)")
            rc.corner = CORNERS[val]
        elif key == "cfl":
            rc.cfl = _num(val, lineno)
        elif key == "divisor":
            rc.divisor = int(_num(val, lineno))
        elif key == "t_end":
            rc.t_end = _num(val, lineno)
        elif key == "max_steps":
            rc.max_steps = int(_num(val, lineno))
        elif key == "out_dir":
            rc.out_dir = val
        elif key == "output_every":
            rc.output_every = int(_num(val, lineno))
        elif key == "seed":
            rc.seed = int(_num(val, lineno))
        else:
            _fail(lineno, f"unknown key '{key}'")
    return rc


def load_config(path: str) -> RunConfig:
    try:
        with open(path) as f:
            return parse_config(f.read())
    except OSError:
        raise errors.SimError("cannot open config file: " + path)


def configure_case(rc: RunConfig) -> CaseSpec:
    """CaseSpec configure_case(const RunConfig&) (config.cpp:95-106)."""
    if not rc.case_name:
        raise errors.SimError("config is missing 'case'")
    cs = build_case(rc.case_name, rc.divisor)
    cs = replace(cs, scheme=rc.scheme, face_order=rc.face_order, corner=rc.corner, cfl=rc.cfl)
    if rc.t_end >= 0.0:
        cs.t_end = rc.t_end
    if rc.max_steps > 0:
        cs.max_steps = rc.max_steps
    return cs


# ---- run (harness.cpp:380-424) --------------------------------------------------------

@dataclass
class RunReport:
    """hydro::RunReport (harness.hpp:74-88)."""
    spec: CaseSpec
    series: np.ndarray  # StepDiag records, series[0] = make_diag(initial, 0.0)
    initial_state: HostState
    final_state: HostState
    steps: int = 0
    wall_seconds: float = 0.0
    max_k_violation: float = 0.0
    k_clip_count: int = 0
    mass_fix_count: int = 0
    energy_floor_count: int = 0
    l2_rho_vs_initial: float = 0.0
    l2_k_vs_initial: float = 0.0


def _cells(f: np.ndarray, nx: int, ny: int) -> np.ndarray:
    return f[GHOST:GHOST + ny, GHOST:GHOST + nx]


def l2_error(a: np.ndarray, b: np.ndarray, nx: int, ny: int, dx: float, dy: float) -> float:
    """sqrt(sum (a-b)^2 dx dy) (harness.cpp:315-324), serial in the reference's order."""
    d = (_cells(a, nx, ny) - _cells(b, nx, ny)).ravel()
    s = float(np.cumsum(d * d)[-1]) if d.size else 0.0  # cumsum adds left to right, like the loop
    return math.sqrt(s * dx * dy)


def impose_velocity(u: np.ndarray, cs: CaseSpec, t: float, dx: float, dy: float):
    """impose_velocity's interior part (harness.cpp:208-221) on a node Vec2
    field; the ghost fill runs on the device (fill_ghosts)."""
    nx, ny, g = cs.nx, cs.ny, GHOST
    v = u[g:g + ny + 1, g:g + nx + 1]
    if cs.imposed == CONSTANT:
        sgn = -1.0 if (cs.flip_time > 0.0 and t >= cs.flip_time) else 1.0
        v[..., 0] = sgn * cs.u_const[0]
        v[..., 1] = sgn * cs.u_const[1]
    else:
        i = np.arange(nx + 1, dtype=np.float64)
        j = np.arange(ny + 1, dtype=np.float64)
        px = cs.x0 + i * dx  # Mesh::node_pos, mesh.hpp:33
        py = cs.y0 + j * dy
        v[..., 0] = np.broadcast_to(cs.rot_omega * (-(py - cs.rot_center[1]))[:, None], (ny + 1, nx + 1))
        v[..., 1] = np.broadcast_to(cs.rot_omega * (px - cs.rot_center[0])[None, :], (ny + 1, nx + 1))


def _kinematic_dt(st: HostState, cs: CaseSpec, dx: float, dy: float) -> float:
    """harness.cpp:328-334 (norm = sqrt(x*x + y*y), vec2.hpp:27)."""
    u = st.node(st.u)
    umax = float(np.max(np.sqrt(u[..., 0] * u[..., 0] + u[..., 1] * u[..., 1])))
    if not umax > 0.0:
        raise errors.SimError("imposed velocity field is zero")
    return cs.cfl * min(dx, dy) / umax


def _nan_scan(st: HostState, nx: int, ny: int, step: int):
    """harness.cpp:347-358 (the device run loop has it built in)."""
    for f in (st.m_mix, st.e_mix, st.p_mix):
        bad = ~np.isfinite(_cells(f, nx, ny))
        if bad.any():
            j, i = map(int, np.argwhere(bad)[0])
            raise errors.SimError(f"non-finite cell state at ({i},{j}) step {step}")
    u = st.node(st.u)
    bad = ~np.isfinite(u).all(axis=-1)
    if bad.any():
        j, i = map(int, np.argwhere(bad)[0])
        raise errors.SimError(f"non-finite velocity at ({i},{j}) step {step}")


StepHook = Callable[[HostState, np.void], None]


def init_case(cs: CaseSpec, solver: abi.Solver) -> HostState:
    """State init_case(const CaseSpec&) (harness.cpp:226-291) on a device context."""
    painted = cases.paint(solver.cfg, cs.regions)
    solver.init_from(painted)
    if cs.imposed != NONE:
        st = solver.download()
        impose_velocity(st.u, cs, 0.0, solver.cfg.mesh.dx, solver.cfg.mesh.dy)
        solver.upload(st)
        solver.fill_ghosts()
    return solver.download()


def run(cs: CaseSpec, hook: Optional[StepHook] = None, device: int = 0) -> RunReport:
    """RunReport run(const CaseSpec&, const StepHook&) (harness.cpp:380-424)."""
    from . import product_library
    t0 = time.perf_counter()
    cfg = cs.config()
    s = abi.Solver(product_library(), cfg, device)
    try:
        init = init_case(cs, s)
        series = [s.step_diag(0.0)]
        rep = RunReport(spec=cs, series=None, initial_state=init, final_state=init)
        if cs.imposed == NONE:
            _run_dynamic(cs, s, hook, series, rep)
        else:
            _run_kinematic(cs, s, hook, series, rep)
        fin = s.download()
        rep.series = np.array(series, dtype=STEP_DIAG_DTYPE)
        rep.final_state = fin
        rep.steps = fin.step
        m = cfg.mesh
        rep.l2_rho_vs_initial = l2_error(fin.rho_mix, init.rho_mix, m.nx, m.ny, m.dx, m.dy)
        if cs.nmat == 2:
            rep.l2_k_vs_initial = l2_error(fin.k[1], init.k[1], m.nx, m.ny, m.dx, m.dy)
        rep.wall_seconds = time.perf_counter() - t0
        return rep
    finally:
        s.close()


def _with_case(err: errors.SimError, cs: CaseSpec, step: int) -> errors.SimError:
    """run() re-throws a step's error with the case and step appended (harness.cpp:404-407)."""
    err.what = f"{err.what} [{cs.name} step {step}]"
    err.args = (err.what,)
    return err


def _run_dynamic(cs, s, hook, series, rep):
    if hook is None:  # the whole loop on the device, the series reduced there too
        try:
            r = s.run(cs.max_steps, t_end=cs.t_end, cfl=cs.cfl, kind=cs.scheme, series=True)
        except errors.SimError as e:
            r = e.partial
            _account(rep, r)
            series.extend(r.series)
            if getattr(e, "in_step", False):
                raise _with_case(e, cs, e.step)
            raise
        _account(rep, r)
        series.extend(r.series)
        return
    while True:  # a hook sees every State: one device step per call
        step = s.download().step
        if cs.max_steps > 0 and step >= cs.max_steps:
            break
        try:
            r = s.run(step + 1, t_end=cs.t_end, cfl=cs.cfl, kind=cs.scheme, series=True)
        except errors.SimError as e:
            _account(rep, e.partial)
            if getattr(e, "in_step", False):
                raise _with_case(e, cs, e.step)
            raise
        _account(rep, r)
        if r.steps_done == 0:  # t >= t_end
            break
        series.extend(r.series)
        hook(s.download(), series[-1])


def _account(rep, r):
    rep.energy_floor_count += r.floor_count
    rep.k_clip_count += r.diag["k_clip_count"]
    rep.mass_fix_count += r.diag["mass_fix_count"]
    rep.max_k_violation = max(rep.max_k_violation, r.diag["max_k_violation"])


def _run_kinematic(cs, s, hook, series, rep):
    """The imposed-velocity branch (harness.cpp:393-402): kinematic_dt,
    kinematic_lagrange, remap without velocity remap, impose_velocity."""
    m = s.cfg.mesh
    diag = RemapDiag()
    t_end = cs.t_end
    while True:
        st = s.download()
        if not st.time < t_end - 1e-15 * max(1.0, t_end):
            break
        if cs.max_steps > 0 and st.step >= cs.max_steps:
            break
        dt = _kinematic_dt(st, cs, m.dx, m.dy)
        if cs.flip_time > 0.0 and st.time < cs.flip_time:
            dt = min(dt, cs.flip_time - st.time)
        dt = min(dt, t_end - st.time)
        lag = HostLagrange.empty(m.nx, m.ny)  # kinematic_lagrange (harness.cpp:336-345)
        lag.u_half[...] = st.u
        lag.u_lag[...] = st.u
        for a in range(cs.nmat):
            lag.e_lag[a][...] = st.e[a]
        lag.vol_lag[...] = st.vol
        s.set_lagrange(lag)
        try:
            s.remap_step(dt, kind=cs.scheme, x_first=st.step % 2 == 0, remap_velocity=False, diag=diag)
        except errors.SimError as e:
            raise _with_case(e, cs, st.step)
        nst = s.download()
        impose_velocity(nst.u, cs, nst.time, m.dx, m.dy)
        s.upload(nst)
        s.fill_ghosts()  # fill_ghost_nodes of the imposed field; the other ghosts are unchanged
        nst = s.download()
        _nan_scan(nst, m.nx, m.ny, nst.step)
        series.append(s.step_diag(dt))
        if hook:
            hook(nst, series[-1])
    rep.max_k_violation = diag.max_k_violation
    rep.k_clip_count = diag.k_clip_count
    rep.mass_fix_count = diag.mass_fix_count


# ---- pybind11 run_case (bindings/module.cpp:50-93) --------------------------------------

def run_case(name: str, divisor: int = 1, scheme: str = "DirectCF", face_order: int = 2,
             corner: str = "linear_diag", cfl: float = 0.3, t_end: float = -1.0, max_steps: int = 0) -> dict:
    rc = RunConfig(case_name=name, divisor=divisor, face_order=face_order, cfl=cfl, t_end=t_end,
                   max_steps=max_steps)
    if scheme not in SCHEMES:
        raise errors.SimError("unknown scheme: " + scheme)
    rc.scheme = SCHEMES[scheme]
    if corner not in CORNERS:
        raise errors.SimError("unknown corner scheme: " + corner)
    rc.corner = CORNERS[corner]
    cs = configure_case(rc)
    rep = run(cs)
    t0, t1 = rep.series[0], rep.series[-1]
    return {
        "case": cs.name, "scheme": scheme, "nx": cs.nx, "ny": cs.ny, "steps": rep.steps,
        "time": rep.final_state.time, "mass_initial": float(t0["mass"]), "mass_final": float(t1["mass"]),
        "mass_drift": abs(float(t1["mass"]) - float(t0["mass"])) / float(t0["mass"]),
        "internal_energy_drift": abs(float(t1["internal_energy"]) - float(t0["internal_energy"]))
        / max(1e-300, abs(float(t0["internal_energy"]))),
        "l2_rho_vs_initial": rep.l2_rho_vs_initial, "l2_k_vs_initial": rep.l2_k_vs_initial,
        "max_k_violation": rep.max_k_violation, "min_p": float(t1["min_p"]), "max_p": float(t1["max_p"]),
        "wall_seconds": rep.wall_seconds,
    }


# ---- mesh-refinement study (harness.hpp:100-113, harness.cpp:426-461) ---------------

@dataclass
class ConvergenceResult:
    """hydro::ConvergenceResult: per mesh n the L2 error of the final density
    (volume fraction for two-material cases) against the initial field, and
    the least-squares slope of log(err) against log(dx)."""
    scheme: int = REMAP_DIRECTCF
    rows: List[Tuple[int, float]] = field(default_factory=list)
    slope: float = 0.0


def parse_schemes(text: str) -> List[int]:
    """Comma list of scheme names (tools/main.cpp:72-84)."""
    out = []
    for item in text.split(","):
        if item not in SCHEMES:
            raise errors.SimError(f"unknown scheme '{item}' (valid: AD, Direct, DirectCF)")
        out.append(SCHEMES[item])
    if not out:
        raise errors.SimError("no schemes given")
    return out


def convergence_study(case_name: str, meshes: List[int], schemes: List[int]) -> List[ConvergenceResult]:
    """convergence_study (harness.cpp:426-461): the case on n x n meshes per
    scheme, every run on the device; the slope's sums accumulate in the
    reference's order so it matches to the bit."""
    out = []
    for scheme in schemes:
        res = ConvergenceResult(scheme=scheme)
        for n in meshes:
            cs = build_case(case_name)
            cs.nx = cs.ny = n
            cs.scheme = scheme
            rep = run(cs)
            res.rows.append((n, rep.l2_k_vs_initial if cs.nmat == 2 else rep.l2_rho_vs_initial))
        sx = sy = sxx = sxy = 0.0
        m = len(res.rows)
        for n, err in res.rows:
            x = math.log(1.0 / n)
            y = math.log(max(err, 1e-300))
            sx += x
            sy += y
            sxx += x * x
            sxy += x * y
        res.slope = (m * sxy - sx * sy) / (m * sxx - sx * sx) if m > 1 else 0.0
        out.append(res)
    return out

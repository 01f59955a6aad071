"""Shared test helpers: backends (product / oracle / reference), state
generators modelled on the reference fixtures (gas_state test_remap.cpp:32-43,
front_state :403-422, kinematic() :46-54) and bitwise comparison."""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess

import numpy as np

from paper_2208_13409_b200 import abi
from paper_2208_13409_b200.abi import GHOST, HostLagrange, HostState, Solver

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_LIB = os.path.join(ROOT, "oracle", "libh2d_oracle.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libh2d_ref.so")
PRODUCT_LIB = os.environ.get("H2D_PRODUCT_LIB") or os.path.join(ROOT, "paper_2208_13409_b200", "libh2d.so")

STATE_FIELDS = ("m", "e", "k", "vol", "m_mix", "e_mix", "rho_mix", "p_mix", "iface_normal", "u")
LAG_FIELDS = ("u_half", "u_lag", "e_lag", "vol_lag", "q")

_cache = {}


def oracle_lib() -> abi.Library:
    """The C restatement (built on demand with gcc: its sources travel)."""
    if "o" not in _cache:
        if not os.path.exists(ORACLE_LIB):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
        _cache["o"] = abi.Library(ORACLE_LIB, "h2do_")
    return _cache["o"]


def ref_lib():
    """The reference library itself, or None where it was not built (the GPU
    box has no /root/reference; the .so travels only if built here)."""
    if "r" not in _cache:
        if not os.path.exists(REF_LIB) and os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
        _cache["r"] = abi.Library(REF_LIB, "h2dr_") if os.path.exists(REF_LIB) else None
    return _cache["r"]


def product_lib() -> abi.Library:
    if "p" not in _cache:
        _cache["p"] = abi.Library(PRODUCT_LIB, "h2d_")
    return _cache["p"]


def bitwise_diff(a, b, fields, nmat=2):
    """Fields whose bytes differ, with the max abs difference."""
    bad = []
    for f in fields:
        x, y = getattr(a, f), getattr(b, f)
        if f in ("m", "e", "k", "e_lag"):
            x, y = x[:nmat], y[:nmat]
        if not np.array_equal(x.view(np.int64), y.view(np.int64)):
            with np.errstate(invalid="ignore"):
                bad.append((f, float(np.nanmax(np.abs(x - y)))))
    return bad


def periodic_nodes(u: np.ndarray, nx: int, ny: int, per_x: bool, per_y: bool):
    """Make the node field consistent with the periodic identification
    u(nx, j) = u(0, j), u(i, ny) = u(i, 0) (test_remap.cpp:247-248)."""
    g = GHOST
    if per_x:
        u[g:g + ny + 1, g + nx] = u[g:g + ny + 1, g]
    if per_y:
        u[g + ny, g:g + nx + 1] = u[g, g:g + nx + 1]


def random_state(cfg: abi.Config, seed: int, kind: str = "gas", umax: float = 0.2,
                 e_scale: float = 1.0) -> HostState:
    """Painted interior (ghosts filled later by the backend's init helpers).

    gas    : one material, m, e ~ U[0.5, 2], node u ~ U[-umax, umax]
    front  : two materials, pure columns left/right of a mixed column
    blobs  : two materials, random discs with exact-ish fractions, random u
    """
    rng = np.random.Generator(np.random.MT19937(seed))
    m = cfg.mesh
    nx, ny, cv = m.nx, m.ny, m.dx * m.dy
    st = HostState.empty(nx, ny, cfg.nmat, cv)
    g = GHOST
    I = (slice(g, g + ny), slice(g, g + nx))
    if kind == "gas":
        st.m[0][I] = rng.uniform(0.5, 2.0, (ny, nx)) * cv
        st.e[0][I] = rng.uniform(0.5, 2.0, (ny, nx)) * e_scale
    elif kind == "front":
        k0 = np.zeros((ny, nx))
        mid = nx // 2
        k0[:, :mid] = 1.0
        k0[:, mid] = rng.uniform(0.1, 0.9, ny)
        for a, (rho, e) in enumerate(((1.0, 1.0), (2.0, 0.5))):
            k = k0 if a == 0 else 1.0 - k0
            st.k[a][I] = k
            st.m[a][I] = k * rho * cv
            st.e[a][I] = np.where(k > 0.0, e * e_scale, 0.0)
    elif kind == "blobs":
        xs = (np.arange(nx) + 0.5) / nx
        ys = (np.arange(ny) + 0.5) / ny
        X, Y = np.meshgrid(xs, ys)
        k1 = np.zeros((ny, nx))
        for _ in range(3):
            cx, cy, r = rng.uniform(0.25, 0.75), rng.uniform(0.25, 0.75), rng.uniform(0.08, 0.2)
            d = np.sqrt((X - cx) ** 2 + (Y - cy) ** 2)
            k1 = np.maximum(k1, np.clip((r - d) * nx * 0.7 + 0.5, 0.0, 1.0))
        k1 = np.where(k1 < 1e-10, 0.0, np.where(k1 > 1 - 1e-10, 1.0, k1))
        k0 = 1.0 - k1
        st.k[0][I], st.k[1][I] = k0, k1
        rho0 = rng.uniform(0.8, 1.2, (ny, nx))
        rho1 = rng.uniform(0.1, 0.2, (ny, nx))
        st.m[0][I] = k0 * rho0 * cv
        st.m[1][I] = k1 * rho1 * cv
        st.e[0][I] = np.where(k0 > 0, rng.uniform(2.0, 3.0, (ny, nx)) * e_scale, 0.0)
        st.e[1][I] = np.where(k1 > 0, rng.uniform(5.0, 8.0, (ny, nx)) * e_scale, 0.0)
    else:
        raise ValueError(kind)
    st.u[g:g + ny + 1, g:g + nx + 1] = rng.uniform(-umax, umax, (ny + 1, nx + 1, 2))
    periodic_nodes(st.u, nx, ny, m.bc_x == abi.BC_PERIODIC, m.bc_y == abi.BC_PERIODIC)
    return st


def kinematic(st: HostState) -> HostLagrange:
    """Imposed-velocity LagrangeResult (test_remap.cpp:46-54): u_half = u_lag
    = u, e_lag = e, vol_lag = vol, q = 0."""
    lag = HostLagrange.empty(st.nx, st.ny)
    lag.u_half[:] = st.u
    lag.u_lag[:] = st.u
    lag.e_lag[:] = st.e
    lag.vol_lag[:] = st.vol
    return lag


def prepared(lib: abi.Library, cfg: abi.Config, painted: HostState) -> Solver:
    s = Solver(lib, cfg)
    s.init_from(painted)
    return s


def run_capture(s: Solver, steps: int, cfl: float, kind: int = abi.REMAP_DIRECTCF, t_end: float = 1e30):
    """Run and return (result, error-tuple-or-None)."""
    from paper_2208_13409_b200 import errors
    try:
        r = s.run(steps, t_end=t_end, cfl=cfl, kind=kind)
        return r, None
    except errors.SimError as e:
        return e.partial, (type(e).__name__, e.what, e.i, e.j, e.step, e.in_step)


def plane_hashes(solver, nmat: int) -> dict:
    """sha256 of every State plane, downloading one plane at a time (so the
    8192^2 pin needs one plane of host memory, not a whole State)."""
    nx, ny = solver.nx, solver.ny
    cs, ns = (ny + 2 * abi.GHOST, nx + 2 * abi.GHOST), (ny + 1 + 2 * abi.GHOST, nx + 1 + 2 * abi.GHOST)
    out = {}
    plan = [(f"{f}{a}", f, a, cs) for f in ("m", "e", "k") for a in range(nmat)]
    plan += [(f, f, None, cs) for f in ("vol", "m_mix", "e_mix", "rho_mix", "p_mix")]
    plan += [("iface_normal", "iface_normal", None, cs + (2,)), ("u", "u", None, ns + (2,))]
    step = time_ = None
    for key, f, a, shape in plan:
        buf = np.empty(shape)
        v = abi.StateView()
        p = buf.ctypes.data_as(C.POINTER(C.c_double))
        if a is None:
            setattr(v, f, p)
        else:
            getattr(v, f)[a] = p
        solver._check(solver.lib.fn["download_state"](solver._h, C.byref(v)))
        out[key] = hashlib.sha256(buf.tobytes()).hexdigest()
        step, time_ = v.step, v.time
        del buf
    return out, step, time_

"""Initial data for the BASELINE.json configurations.

``paint`` restates the interior painter of ``init_case``
(proj/src/harness.cpp:165-207 coverage/contains, :226-284 painting) in
vectorised numpy with the reference's operation order, so a painted state
followed by ``Solver.init_from`` (fill_ghosts + sync_derived +
update_interface_normals, harness.cpp:286-288) is bit-identical to the
reference ``init_case`` (pinned by tests/test_oracle_vs_reference.py).

Two shapes the reference painter lacks are added for configs 4 and 5 (the
reference has no perturbed circle and no Voronoi region): a
seeded Fourier-perturbed circle sampled 16x16 per cell like the reference
circle (harness.cpp:179-189), and the seeded three-material Voronoi mesh of
config 5 (``voronoi3``; three materials are this build's N-material
extension, the reference stops at kMaxMat = 2, state.hpp:13).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from .abi import (BC_WALL, CORNER_LINEARDIAG, EOS_PERFECT, EOS_STIFFENED, GHOST, MAX_MAT, Config, HostState,
                  StateView, _ptr, make_config)

K_PURE_TOL = 1e-10  # state.hpp:17

ALL, HALFPLANE_X, RECTANGLE, CIRCLE, PERTURBED_CIRCLE = range(5)


@dataclass
class Region:
    """hydro::Region (harness.hpp:17-28) plus PERTURBED_CIRCLE (radius(theta))."""
    shape: int = ALL
    xsplit: float = 0.0
    rect: Tuple[float, float, float, float] = (0.0, 0.0, 0.0, 0.0)  # lo.x, lo.y, hi.x, hi.y
    center: Tuple[float, float] = (0.0, 0.0)
    radius: float = 0.0
    mat: int = 0
    rho: float = 1.0
    p: float = 1e5
    u: Tuple[float, float] = (0.0, 0.0)
    radius_fn: Optional[Callable[[np.ndarray], np.ndarray]] = None  # PERTURBED_CIRCLE only

    def row(self) -> List[float]:
        """Flat row for the reference probe h2dr_init_regions."""
        return [self.shape, self.xsplit, *self.rect, *self.center, self.radius, self.mat, self.rho, self.p,
                *self.u]


def energy_from_p(eos, rho, p):
    """harness.cpp:32-35."""
    kind, gamma, pi = eos
    pi = pi if kind == EOS_STIFFENED else 0.0
    return (p + pi) / ((gamma - 1.0) * rho)


def _contains(r: Region, px: np.ndarray, py: np.ndarray) -> np.ndarray:
    """contains(), harness.cpp:194-207."""
    if r.shape == ALL:
        return np.ones(np.broadcast(px, py).shape, bool)
    if r.shape == HALFPLANE_X:
        return np.broadcast_to(px < r.xsplit, np.broadcast(px, py).shape)
    if r.shape == RECTANGLE:
        return (px >= r.rect[0]) & (px <= r.rect[2]) & (py >= r.rect[1]) & (py <= r.rect[3])
    ddx, ddy = px - r.center[0], py - r.center[1]
    if r.shape == CIRCLE:
        return ddx * ddx + ddy * ddy <= r.radius * r.radius
    # perturbed circle: only points in the annulus r0 +- max|delta| need the
    # radius function; inside / outside it the answer is known
    ddx, ddy = np.broadcast_arrays(ddx, ddy)
    dist = np.sqrt(ddx * ddx + ddy * ddy)
    lo, hi = r.radius - r.radius_fn.reach, r.radius + r.radius_fn.reach
    out = dist <= lo
    band = (dist > lo) & (dist <= hi)
    if band.any():
        out = out.copy()
        out[band] = dist[band] <= r.radius_fn(ddx[band], ddy[band], dist[band])
    return out


def _ref_max(a, b):
    return np.where(a < b, b, a)


def _ref_min(a, b):
    return np.where(b < a, b, a)


def _coverage(r: Region, lox, loy, hix, hiy, dx, dy, mask) -> np.ndarray:
    """coverage(), harness.cpp:166-192, evaluated where ``mask`` holds."""
    out = np.zeros(mask.shape)
    if r.shape == ALL:
        out[:] = 1.0
        return out
    if r.shape == HALFPLANE_X:
        v = (r.xsplit - lox) / dx
        v = np.where(v < 0.0, 0.0, np.where(1.0 < v, 1.0, v))
        return np.broadcast_to(v, mask.shape).copy()
    if r.shape == RECTANGLE:
        ox = _ref_max(0.0, _ref_min(hix, r.rect[2]) - _ref_max(lox, r.rect[0]))
        oy = _ref_max(0.0, _ref_min(hiy, r.rect[3]) - _ref_max(loy, r.rect[1]))
        return np.broadcast_to((ox / dx) * (oy / dy), mask.shape).copy()
    # circles: 16x16 sub-cell samples, only cells whose box meets the disc
    # bounding box can be covered (all others are exactly 0)
    reach = r.radius * (1.5 if r.shape == PERTURBED_CIRCLE else 1.0)
    jj, ii = np.nonzero(mask)
    lx, ly = np.broadcast_to(lox, mask.shape)[jj, ii], np.broadcast_to(loy, mask.shape)[jj, ii]
    near = (lx + dx >= r.center[0] - reach) & (lx <= r.center[0] + reach) & \
           (ly + dy >= r.center[1] - reach) & (ly <= r.center[1] + reach)
    jj, ii, lx, ly = jj[near], ii[near], lx[near], ly[near]
    if r.shape == PERTURBED_CIRCLE:
        # every sample of a cell lies within half a diagonal of its centre and
        # within dtheta <= 2 half / cd of its direction: cells whose samples
        # are provably all inside get 256/256 exactly, provably all outside 0
        half = 0.5 * np.hypot(dx, dy)
        cx, cy = lx + 0.5 * dx - r.center[0], ly + 0.5 * dy - r.center[1]
        cd = np.hypot(cx, cy)
        ok = cd > 4.0 * half
        rc = r.radius_fn(cx, cy, cd)
        slack = r.radius_fn.slope * 2.0 * half / np.where(ok, cd, 1.0) + 1e-12
        full = ok & (cd + half < rc - slack)
        empty = ok & (cd - half > rc + slack)
        out[jj[full], ii[full]] = 1.0
        keep = ~full & ~empty
        jj, ii, lx, ly = jj[keep], ii[keep], lx[keep], ly[keep]
    offs = (np.arange(16) + 0.5) / 16.0
    chunk = 1 << 16
    for s in range(0, len(jj), chunk):
        sx = lx[s:s + chunk, None, None] + offs[None, None, :] * dx
        sy = ly[s:s + chunk, None, None] + offs[None, :, None] * dy
        inside = _contains(r, sx, sy).sum(axis=(1, 2))
        out[jj[s:s + chunk], ii[s:s + chunk]] = inside / 256.0
    return out


@dataclass
class WindowState:
    """A painted window of the global mesh (per-rank painting for the block
    decomposition, h2d_block_init_window): cells [wi0, wi0 + wnx) x
    [wj0, wj0 + wny), nodes [wi0, wi0 + wnx] x [wj0, wj0 + wny], no ghost
    layers; m, e, k (MAX_MAT, wny, wnx), u (wny + 1, wnx + 1, 2)."""
    wi0: int
    wj0: int
    wnx: int
    wny: int
    nmat: int
    m: np.ndarray
    e: np.ndarray
    k: np.ndarray
    u: np.ndarray

    @classmethod
    def empty(cls, wi0, wj0, wnx, wny, nmat):
        z = np.zeros((MAX_MAT, wny, wnx))
        return cls(wi0, wj0, wnx, wny, nmat, z.copy(), z.copy(), z.copy(), np.zeros((wny + 1, wnx + 1, 2)))

    def view(self) -> StateView:
        v = StateView()
        for a in range(MAX_MAT):
            v.m[a], v.e[a], v.k[a] = _ptr(self.m[a]), _ptr(self.e[a]), _ptr(self.k[a])
        v.u = _ptr(self.u)
        return v

    def into(self, st: HostState):
        """Copy into a global HostState's interior."""
        g = GHOST
        cs = (slice(g + self.wj0, g + self.wj0 + self.wny), slice(g + self.wi0, g + self.wi0 + self.wnx))
        for a in range(self.nmat):
            st.k[a][cs] = self.k[a]
            st.m[a][cs] = self.m[a]
            st.e[a][cs] = self.e[a]
        st.u[g + self.wj0:g + self.wj0 + self.wny + 1, g + self.wi0:g + self.wi0 + self.wnx + 1] = self.u
        return st


def paint(cfg: Config, regions: Sequence[Region], window=None):
    """Interior of init_case (harness.cpp:226-284); ghosts/derived/normals are
    completed on the solver by ``Solver.init_from``. With window = (wi0,
    wj0, wnx, wny) only that window is painted (a WindowState, the same
    per-cell arithmetic)."""
    m = cfg.mesh
    if window is None:
        w = paint(cfg, regions, (0, 0, m.nx, m.ny))
        return w.into(HostState.empty(m.nx, m.ny, cfg.nmat, m.dx * m.dy))
    wi0, wj0, nx, ny = window
    dx, dy, x0, y0 = m.dx, m.dy, m.x0, m.y0
    nmat = cfg.nmat
    eos = [(cfg.eos[a].kind, cfg.eos[a].gamma, cfg.eos[a].pi) for a in range(nmat)]
    cv = dx * dy
    i = np.arange(wi0, wi0 + nx, dtype=np.float64)[None, :]
    j = np.arange(wj0, wj0 + ny, dtype=np.float64)[:, None]
    lox, loy = x0 + i * dx, y0 + j * dy              # node_pos(i, j)
    hix, hiy = x0 + (i + 1) * dx, y0 + (j + 1) * dy  # node_pos(i+1, j+1)
    cenx, ceny = x0 + (i + 0.5) * dx, y0 + (j + 0.5) * dy
    shape = (ny, nx)
    karr = np.zeros((2,) + shape)
    marr = np.zeros((2,) + shape)
    mearr = np.zeros((2,) + shape)
    for r_idx, reg in enumerate(regions):
        if r_idx == 0:
            f = np.ones(shape)
        else:
            frac = (nmat == 2) & (karr[reg.mat] < 1.0)
            f = np.where(_contains(reg, cenx, ceny), 1.0, 0.0)
            if np.any(frac):
                cov = _coverage(reg, lox, loy, hix, hiy, dx, dy, frac)
                f = np.where(frac, cov, f)
        # cells this region paints, restricted to their bounding box (the
        # per-cell arithmetic is the same as over the whole mesh)
        pos = f > 0.0
        rows, cols = np.nonzero(np.any(pos, axis=1))[0], np.nonzero(np.any(pos, axis=0))[0]
        if len(rows) == 0:
            continue
        box = (slice(rows[0], rows[-1] + 1), slice(cols[0], cols[-1] + 1))
        upd, fb = pos[box], f[box]
        e = energy_from_p(eos[reg.mat], reg.rho, reg.p)
        for a in range(nmat):
            for arr in (karr, marr, mearr):
                sub = arr[a][box]
                sub[...] = np.where(upd, sub * (1.0 - fb), sub)
        for arr, add in ((karr, fb), (marr, fb * reg.rho * cv), (mearr, fb * reg.rho * e * cv)):
            sub = arr[reg.mat][box]
            sub[...] = np.where(upd, sub + add, sub)
    for a in range(nmat):  # snap trace fractions to pure (harness.cpp:260-269)
        snap = karr[a] < K_PURE_TOL
        if not snap.any():
            continue
        b = 1 - a
        for arr in (karr, marr, mearr):
            arr[b] = np.where(snap, arr[b] + arr[a], arr[b])
            arr[a] = np.where(snap, 0.0, arr[a])
    st = WindowState.empty(wi0, wj0, nx, ny, nmat)
    for a in range(nmat):
        st.k[a] = karr[a]
        st.m[a] = marr[a]
        with np.errstate(divide="ignore", invalid="ignore"):
            st.e[a] = np.where(marr[a] > 0.0, mearr[a] / marr[a], 0.0)
    # node velocities: last region containing the node (harness.cpp:277-284)
    ni = np.arange(wi0, wi0 + nx + 1, dtype=np.float64)[None, :]
    nj = np.arange(wj0, wj0 + ny + 1, dtype=np.float64)[:, None]
    px, py = x0 + ni * dx, y0 + nj * dy
    ux = np.zeros((ny + 1, nx + 1))
    uy = np.zeros((ny + 1, nx + 1))
    for reg in regions:
        inside = np.nonzero(np.broadcast_to(_contains(reg, px, py), ux.shape))
        ux[inside] = reg.u[0]
        uy[inside] = reg.u[1]
    st.u[..., 0] = ux
    st.u[..., 1] = uy
    return st


@dataclass
class Case:
    name: str
    cfg: Config
    regions: List[Region]
    cfl: float
    steps: int
    note: str = ""

    @property
    def cells(self) -> int:
        return self.cfg.mesh.nx * self.cfg.mesh.ny

    def paint(self, window=None):
        return paint(self.cfg, self.regions, window)


def _mesh_cfg(nx, ny, lx, ly, eos, **kw) -> Config:
    # CaseSpec::make_mesh divides the extent (harness.cpp:9-11)
    return make_config(nx, ny, lx / nx, ly / ny, 0.0, 0.0, BC_WALL, BC_WALL, eos=eos,
                       corner=CORNER_LINEARDIAG, **kw)


def riemann2d(n: int = 256) -> Case:
    """Config 1: gamma 1.4 two-state Riemann problem on the unit square."""
    air = (EOS_PERFECT, 1.4, 0.0)
    return Case(f"riemann2d_{n}", _mesh_cfg(n, n, 1.0, 1.0, [air]),
                [Region(ALL, rho=0.125, p=0.1), Region(HALFPLANE_X, xsplit=0.5, rho=1.0, p=1.0)], 0.5, 100)


def sedov(n: int = 1024) -> Case:
    """Config 2: point blast, E0 = 1 in the 2x2 corner cells (sum m e = 1)."""
    gamma = 1.4
    dx = dy = 1.0 / n
    p0 = (gamma - 1.0) * 1.0 / (4.0 * dx * dy)
    return Case(f"sedov_{n}", _mesh_cfg(n, n, 1.0, 1.0, [(EOS_PERFECT, gamma, 0.0)]),
                [Region(ALL, rho=1.0, p=1e-6), Region(RECTANGLE, rect=(0.0, 0.0, 2 * dx, 2 * dy), rho=1.0, p=p0)],
                0.5, 500)


def sedov_weak(px: int, py: int, n: int = 1024) -> Case:
    """Config 2 grown for weak scaling over px x py GPUs: the same 1/n cell
    size and corner blast, on a (px*n) x (py*n) mesh over [0,px] x [0,py]."""
    gamma = 1.4
    dx = dy = 1.0 / n
    p0 = (gamma - 1.0) * 1.0 / (4.0 * dx * dy)
    return Case(f"sedov_{px * n}x{py * n}", _mesh_cfg(px * n, py * n, float(px), float(py), [(EOS_PERFECT, gamma, 0.0)]),
                [Region(ALL, rho=1.0, p=1e-6), Region(RECTANGLE, rect=(0.0, 0.0, 2 * dx, 2 * dy), rho=1.0, p=p0)],
                0.5, 500)


def triple_point(nx: int = 2048, ny: int = 1024) -> Case:
    """Config 3: two-material three-state interface problem on [0,7]x[0,3]
    (A: gamma 1.5 = material 0, B: gamma 1.4 = material 1).  Region order is
    the one in BASELINE.json; the reference aborts after step 819 at full size
    (SURVEY.md finding 6)."""
    A, B = (EOS_PERFECT, 1.5, 0.0), (EOS_PERFECT, 1.4, 0.0)
    return Case(f"triple_point_{nx}x{ny}", _mesh_cfg(nx, ny, 7.0, 3.0, [A, B]),
                [Region(ALL, mat=0, rho=1.0, p=1.0),
                 Region(RECTANGLE, rect=(1.0, 0.0, 7.0, 1.5), mat=0, rho=1.0, p=0.1),
                 Region(RECTANGLE, rect=(1.0, 1.5, 7.0, 3.0), mat=1, rho=0.125, p=0.1)], 0.4, 1000)


def bubble_radius_fn(seed: int = 20241001, amp: float = 0.005, r0: float = 0.1, table_bits: int = 20):
    """Radius of the perturbed bubble boundary in the direction of a point:
    r = r0 + delta(theta), delta a seeded sum of Fourier modes 2..32,
    sum_m a_m cos(m theta + phi_m), rescaled so max |delta| = amp.  delta is
    tabulated on 2^20 angles and interpolated linearly (the definition of
    the configuration-4 initial data used by every backend)."""
    rng = np.random.Generator(np.random.MT19937(seed))
    modes = np.arange(2, 33)
    a = rng.standard_normal(len(modes)) / modes
    ph = rng.uniform(0.0, 2.0 * np.pi, len(modes))
    n = 1 << table_bits
    th = np.arange(n + 1) * (2.0 * np.pi / n)
    tab = np.zeros(n + 1)
    for ak, mk, pk in zip(a, modes, ph):
        tab += ak * np.cos(mk * th + pk)
    tab *= amp / np.abs(tab).max()

    def fn(ddx, ddy, dist):
        t = np.mod(np.arctan2(ddy, ddx), 2.0 * np.pi) * (n / (2.0 * np.pi))
        k = np.minimum(t.astype(np.int64), n - 1)
        f = t - k
        return r0 + (tab[k] + f * (tab[k + 1] - tab[k]))

    fn.reach = 1.0001 * amp  # |delta| <= amp on the table, hence everywhere
    fn.slope = float(np.abs(np.diff(tab)).max()) * (n / (2.0 * np.pi)) * 1.0001  # |d delta / d theta|
    return fn


def shock_bubble(n: int = 8192, seed: int = 20241001) -> Case:
    """Config 4: shock-bubble, A gamma 1.4 (material 0), B gamma 1.67
    (material 1) bubble of radius 0.1 +- 0.005 at (0.5, 0.5), post-shock slab
    x < 0.3; fractions by 16x16 sub-cell sampling. CFL 0.3 (the reference
    default, harness.hpp:39; unstated in BASELINE.json), walls."""
    A, B = (EOS_PERFECT, 1.4, 0.0), (EOS_PERFECT, 1.67, 0.0)
    return Case(f"shock_bubble_{n}", _mesh_cfg(n, n, 1.0, 1.0, [A, B]),
                [Region(ALL, mat=0, rho=1.0, p=1.0),
                 Region(HALFPLANE_X, xsplit=0.3, mat=0, rho=1.376, p=1.5, u=(0.394, 0.0)),
                 Region(PERTURBED_CIRCLE, center=(0.5, 0.5), radius=0.1, mat=1, rho=0.138, p=1.0,
                        radius_fn=bubble_radius_fn(seed))], 0.3, 200)


def voronoi_sites(nsites: int = 64, seed: int = 20241005):
    """Config 5's seeded sites: positions U[0,1]^2, material uniform over the
    three gammas, rho and p log-uniform on [0.1, 10], u and v U[-0.5, 0.5]."""
    rng = np.random.Generator(np.random.MT19937(seed))
    xy = rng.uniform(0.0, 1.0, (nsites, 2))
    mat = rng.integers(0, 3, nsites)
    rho = 10.0 ** rng.uniform(-1.0, 1.0, nsites)
    p = 10.0 ** rng.uniform(-1.0, 1.0, nsites)
    uv = rng.uniform(-0.5, 0.5, (nsites, 2))
    return xy, mat, rho, p, uv


def _nearest(px: np.ndarray, py: np.ndarray, xy: np.ndarray, chunk: int = 1 << 18) -> np.ndarray:
    """Index of the nearest site of each point (squared distance, ties to the
    lower index), in chunks."""
    out = np.empty(px.size, np.int64)
    fx, fy = px.ravel(), py.ravel()
    for s0 in range(0, fx.size, chunk):
        ddx = fx[s0:s0 + chunk, None] - xy[None, :, 0]
        ddy = fy[s0:s0 + chunk, None] - xy[None, :, 1]
        out[s0:s0 + chunk] = np.argmin(ddx * ddx + ddy * ddy, axis=1)
    return out.reshape(px.shape)


def paint_voronoi3(cfg: Config, sites, sub: int = 4, window=None):
    """Config 5's initial State (three materials, gammas 1.4 / 1.5 / 1.67).
    Node u: the nearest site's velocity.  Cells: a cell whose four corners
    have the same nearest site lies in that site's (convex) Voronoi region and
    is pure: k = 1, m = rho cv, e = p / ((gamma - 1) rho).  Any other cell is
    sampled on sub x sub points: k_a = n_a / sub^2, m_a = (sum of the
    samples' rho, in sample order) * (cv / sub^2), e_a = (sum of rho e) /
    (sum of rho)."""
    m = cfg.mesh
    if window is None:
        w = paint_voronoi3(cfg, sites, sub, (0, 0, m.nx, m.ny))
        return w.into(HostState.empty(m.nx, m.ny, 3, m.dx * m.dy))
    wi0, wj0, nx, ny = window
    xy, mat, rho, p, uv = sites
    dx, dy, x0, y0 = m.dx, m.dy, m.x0, m.y0
    gam = np.array([cfg.eos[a].gamma for a in range(3)])
    e_site = p / ((gam[mat] - 1.0) * rho)
    cv = dx * dy
    st = WindowState.empty(wi0, wj0, nx, ny, 3)
    xn = x0 + np.arange(wi0, wi0 + nx + 1) * dx
    yn = y0 + np.arange(wj0, wj0 + ny + 1) * dy
    lab = _nearest(np.broadcast_to(xn[None, :], (ny + 1, nx + 1)), np.broadcast_to(yn[:, None], (ny + 1, nx + 1)), xy)
    st.u[..., 0] = uv[lab, 0]
    st.u[..., 1] = uv[lab, 1]
    c00 = lab[:-1, :-1]
    pure = (c00 == lab[:-1, 1:]) & (c00 == lab[1:, :-1]) & (c00 == lab[1:, 1:])
    kk = np.zeros((3, ny, nx))
    mm = np.zeros((3, ny, nx))
    ee = np.zeros((3, ny, nx))
    pm = mat[c00]
    for a in range(3):
        sel = pure & (pm == a)
        kk[a][sel] = 1.0
        mm[a][sel] = rho[c00[sel]] * cv
        ee[a][sel] = e_site[c00[sel]]
    jj, ii = np.nonzero(~pure)
    if jj.size:
        ns = sub * sub
        offs = (np.arange(sub) + 0.5) / sub
        sx = x0 + ((ii + wi0)[:, None, None] + offs[None, None, :]) * dx  # [cell, q (row), s (col)]
        sy = y0 + ((jj + wj0)[:, None, None] + offs[None, :, None]) * dy
        sx, sy = np.broadcast_to(sx, (ii.size, sub, sub)), np.broadcast_to(sy, (ii.size, sub, sub))
        sl = _nearest(np.ascontiguousarray(sx), np.ascontiguousarray(sy), xy).reshape(ii.size, ns)
        smat, srho, sre = mat[sl], rho[sl], rho[sl] * e_site[sl]
        for a in range(3):
            inm = smat == a
            cnt = inm.sum(axis=1)
            rs = np.zeros(ii.size)
            res = np.zeros(ii.size)
            for q in range(ns):  # the samples in order
                rs = rs + np.where(inm[:, q], srho[:, q], 0.0)
                res = res + np.where(inm[:, q], sre[:, q], 0.0)
            kk[a][jj, ii] = cnt / float(ns)
            mm[a][jj, ii] = rs * (cv / float(ns))
            ee[a][jj, ii] = np.where(cnt > 0, res / np.where(cnt > 0, rs, 1.0), 0.0)
    for a in range(3):
        st.k[a] = kk[a]
        st.m[a] = mm[a]
        st.e[a] = ee[a]
    return st


@dataclass
class VoronoiCase(Case):
    sites: tuple = ()

    def paint(self, window=None):
        return paint_voronoi3(self.cfg, self.sites, window=window)


def voronoi3(nx: int = 16384, ny: Optional[int] = None, n_full: Optional[int] = None, nsites: int = 64,
             seed: int = 20241005) -> Case:
    """Config 5: three-material Voronoi mesh on [0,1]^2 (gammas 1.4, 1.5,
    1.67 = materials 0, 1, 2), 64 seeded sites, 4x4 sampling of the cells the
    site boundaries cross, walls, CFL 0.3 (unstated in BASELINE.json), 100
    steps. With n_full > nx the mesh is the lower-left nx x ny block of the
    n_full^2 mesh (cell size 1 / n_full, walls at the block edges): the share
    of one GPU of the 8-GPU decomposition, which fits one B200 where the whole
    16384^2 three-material problem does not."""
    ny = nx if ny is None else ny
    n_full = nx if n_full is None else n_full
    eos = [(EOS_PERFECT, 1.4, 0.0), (EOS_PERFECT, 1.5, 0.0), (EOS_PERFECT, 1.67, 0.0)]
    name = f"voronoi3_{nx}x{ny}" + (f"_of_{n_full}" if n_full != nx else "")
    return VoronoiCase(name, _mesh_cfg(nx, ny, nx / n_full, ny / n_full, eos), [], 0.3, 100,
                       sites=voronoi_sites(nsites, seed))


CASES = {"c1": riemann2d, "c2": sedov, "c3": triple_point, "c4": shock_bubble, "c5": voronoi3}

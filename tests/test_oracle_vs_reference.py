"""Pin the C restatement oracle (oracle/h2d_oracle.c) bit-for-bit against the
reference library itself (oracle/_ref, compiled from /root/reference/proj).

Runs on CPU only. Every case drives the same ABI calls on both libraries and
requires identical bytes in every State / LagrangeResult field, identical dt
sequences, RemapDiag counters, floor counts and located errors."""
import ctypes as C

import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import abi, cases, errors
from paper_2208_13409_b200.abi import BC_PERIODIC, BC_WALL, CORNER_LINEARDIAG, CORNER_UPWIND, EOS_PERFECT, \
    EOS_STIFFENED, HostState, Solver, make_config

pytestmark = pytest.mark.ref


def _both(ref, orc, cfg, painted):
    return helpers.prepared(ref, cfg, painted), helpers.prepared(orc, cfg, painted)


@pytest.mark.parametrize("case,steps", [
    (cases.riemann2d(48), 100),
    (cases.sedov(64), 120),
    (cases.triple_point(64, 32), 700),      # aborts like the full-size run (finding 6)
    (cases.shock_bubble(64), 40),
])
def test_run_loop_bitwise(ref, orc, case, steps):
    painted = case.paint()
    sr, so = _both(ref, orc, case.cfg, painted)
    assert helpers.bitwise_diff(sr.download(), so.download(), helpers.STATE_FIELDS) == []
    rr, er = helpers.run_capture(sr, steps, case.cfl)
    ro, eo = helpers.run_capture(so, steps, case.cfl)
    assert er == eo
    assert rr.steps_done == ro.steps_done
    assert np.array_equal(rr.dts, ro.dts)
    assert rr.diag == ro.diag and rr.floor_count == ro.floor_count
    assert helpers.bitwise_diff(sr.download(), so.download(), helpers.STATE_FIELDS) == []
    assert sr.totals() == so.totals()


def test_init_case_painter_matches_reference(ref, orc):
    """cases.paint + init helpers == the reference init_case (harness.cpp:226-291)."""
    for case in (cases.riemann2d(32), cases.sedov(32), cases.triple_point(70, 30)):
        rows = np.array([r.row() for r in case.regions], dtype=np.float64)
        s = Solver(ref, case.cfg)
        out = HostState.empty(case.cfg.mesh.nx, case.cfg.mesh.ny, case.cfg.nmat)
        f = ref.dll.h2dr_init_regions
        f.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int, C.POINTER(abi.StateView)]
        v = out.view()
        assert f(s._h, rows.ctypes.data_as(C.POINTER(C.c_double)), len(rows), C.byref(v)) == 0
        so = helpers.prepared(orc, case.cfg, case.paint())
        assert helpers.bitwise_diff(out, so.download(), helpers.STATE_FIELDS) == []


CONFIGS = []
for bcx, bcy in ((BC_PERIODIC, BC_PERIODIC), (BC_WALL, BC_WALL), (BC_PERIODIC, BC_WALL)):
    for order, corner, degrade in ((2, CORNER_LINEARDIAG, 1), (1, CORNER_UPWIND, 1), (2, CORNER_UPWIND, 1),
                                   (2, CORNER_LINEARDIAG, 0), (2, abi.CORNER_AVGMIN, 1), (2, abi.CORNER_LINEARXY, 1),
                                   (2, abi.CORNER_MULTID, 1), (2, abi.CORNER_MULTID, 0), (1, abi.CORNER_MULTID, 1)):
        CONFIGS.append((bcx, bcy, order, corner, degrade))


@pytest.mark.parametrize("corner", [abi.CORNER_AVGMIN, abi.CORNER_LINEARXY, abi.CORNER_MULTID])
@pytest.mark.parametrize("which,steps", [("riemann", 40), ("triple", 60), ("bubble", 20)])
def test_run_loop_corner_schemes_bitwise(ref, orc, corner, which, steps):
    """The remaining corner schemes (reconstruct.cpp:116-152; Multid also
    reconstructs the faces, remap.cpp:840,889-894) in the run loop."""
    case = {"riemann": cases.riemann2d(40), "triple": cases.triple_point(48, 24),
            "bubble": cases.shock_bubble(40)}[which]
    m = case.cfg.mesh
    cfg = make_config(m.nx, m.ny, m.dx, m.dy, m.x0, m.y0, m.bc_x, m.bc_y,
                      eos=[(case.cfg.eos[a].kind, case.cfg.eos[a].gamma, case.cfg.eos[a].pi)
                           for a in range(case.cfg.nmat)], corner=corner)
    sr, so = _both(ref, orc, cfg, case.paint())
    rr, er = helpers.run_capture(sr, steps, case.cfl)
    ro, eo = helpers.run_capture(so, steps, case.cfl)
    assert er == eo
    assert np.array_equal(rr.dts, ro.dts)
    assert (rr.floor_count, rr.diag) == (ro.floor_count, ro.diag)
    assert helpers.bitwise_diff(sr.download(), so.download(), helpers.STATE_FIELDS) == []


@pytest.mark.parametrize("bcx,bcy,order,corner,degrade", CONFIGS)
@pytest.mark.parametrize("kind", ["gas", "front", "blobs"])
def test_kinematic_remap_bitwise(ref, orc, bcx, bcy, order, corner, degrade, kind):
    """remap_step with an imposed-velocity LagrangeResult (test_remap.cpp:46-54)."""
    nmat = 1 if kind == "gas" else 2
    eos = [(EOS_PERFECT, 1.4, 0.0)] * nmat
    cfg = make_config(13, 11, 1.0, 1.0, 0.25, -0.5, bcx, bcy, eos=eos, face_order=order, corner=corner,
                      interface_degrade=degrade)
    seed = hash((bcx, bcy, order, corner, degrade, kind)) & 0xFFFF
    painted = helpers.random_state(cfg, seed, kind, umax=0.25)
    sr, so = _both(ref, orc, cfg, painted)
    lag = helpers.kinematic(sr.download())
    for s in (sr, so):
        s.set_lagrange(lag)
    for vel in (True, False):
        dr, do = abi.RemapDiag(), abi.RemapDiag()
        sr2, so2 = _both(ref, orc, cfg, sr.download())
        sr2.set_lagrange(lag)
        so2.set_lagrange(lag)
        sr2.remap_step(1.0, remap_velocity=vel, diag=dr)
        so2.remap_step(1.0, remap_velocity=vel, diag=do)
        assert helpers.bitwise_diff(sr2.download(), so2.download(), helpers.STATE_FIELDS) == []
        assert (dr.max_k_violation, dr.k_clip_count, dr.mass_fix_count) == \
               (do.max_k_violation, do.k_clip_count, do.mass_fix_count)


@pytest.mark.parametrize("bcx,bcy", [(BC_WALL, BC_WALL), (BC_PERIODIC, BC_PERIODIC), (BC_WALL, BC_PERIODIC)])
@pytest.mark.parametrize("kind,eos", [
    ("gas", [(EOS_PERFECT, 1.4, 0.0)]),
    ("blobs", [(EOS_PERFECT, 1.4, 0.0), (EOS_STIFFENED, 7.0, 0.5)]),
    ("front", [(EOS_PERFECT, 1.5, 0.0), (EOS_PERFECT, 1.67, 0.0)]),
])
def test_lagrange_then_remap_bitwise(ref, orc, bcx, bcy, kind, eos):
    cfg = make_config(17, 12, 0.5, 0.25, 0.0, 0.0, bcx, bcy, eos=eos)
    painted = helpers.random_state(cfg, 7, kind, umax=0.05)
    sr, so = _both(ref, orc, cfg, painted)
    for step in range(3):
        dtr, dto = sr.cfl_dt(0.4), so.cfl_dt(0.4)
        assert dtr == dto
        lr, lo = sr.lagrange_step(dtr), so.lagrange_step(dto)
        assert helpers.bitwise_diff(lr, lo, helpers.LAG_FIELDS) == []
        assert lr.floor_count == lo.floor_count
        sr.remap_step(dtr, x_first=step % 2 == 0)
        so.remap_step(dto)
        assert helpers.bitwise_diff(sr.download(), so.download(), helpers.STATE_FIELDS) == []


def _err(s, fn):
    try:
        fn(s)
    except errors.SimError as e:
        return type(e).__name__, e.what, e.i, e.j
    return None


@pytest.mark.parametrize("scenario", ["cfl_face", "tangled", "unphysical", "wave"])
def test_error_parity(ref, orc, scenario):
    cfg = make_config(9, 8, 1.0, 1.0, bc_x=BC_WALL, bc_y=BC_PERIODIC)
    painted = helpers.random_state(cfg, 3, "gas", umax=0.05)
    if scenario == "unphysical":
        painted.e[0][4, 5] = -3.0
    sr, so = _both(ref, orc, cfg, painted)
    if scenario == "cfl_face":
        lag = helpers.kinematic(sr.download())
        lag.u_half[..., 0] = 0.95   # test_remap.cpp:505-513
        fn = lambda s: (s.set_lagrange(lag), s.remap_step(1.0))
    elif scenario == "tangled":
        fn = lambda s: s.lagrange_step(40.0)
    elif scenario == "unphysical":
        fn = lambda s: s.cfl_dt(0.3)
    else:
        def fn(s):
            st = s.download()
            st.u[:] = np.nan
            st.e[0][:] = 0.0
            s.upload(st)
            s.cfl_dt(0.3)
    er, eo = _err(sr, fn), _err(so, fn)
    assert er is not None and er == eo


def test_scalar_kernels(ref, orc):
    rng = np.random.Generator(np.random.MT19937(5))
    for f in ("van_leer",):
        fr, fo = getattr(ref.dll, "h2dr_" + f), getattr(orc.dll, "h2do_" + f)
        fr.restype = fo.restype = C.c_double
        fr.argtypes = fo.argtypes = [C.c_double]
        for r in np.concatenate([rng.normal(0, 3, 2000), [0.0, -0.0, 1e301, -1.0, np.inf, np.nan]]):
            a, b = fr(r), fo(r)
            assert (a == b) or (np.isnan(a) and np.isnan(b))
    fr, fo = ref.dll.h2dr_clipped_fraction, orc.dll.h2do_clipped_fraction
    fr.restype = fo.restype = C.c_double
    fr.argtypes = fo.argtypes = [C.c_double] * 5
    pr, po = ref.dll.h2dr_place_interface, orc.dll.h2do_place_interface
    pr.restype = po.restype = C.c_double
    pr.argtypes = po.argtypes = [C.c_double] * 7
    for _ in range(3000):
        w, h = rng.uniform(0.1, 2, 2)
        a = rng.uniform(0, 2 * np.pi)
        nx, ny = np.cos(a), np.sin(a)
        d = rng.uniform(-1.5, 1.5)
        assert fr(w, h, nx, ny, d) == fo(w, h, nx, ny, d)
        k = rng.uniform(0, 1)
        lox, loy = rng.uniform(-1, 1, 2)
        assert pr(k, nx, ny, lox, loy, lox + w, loy + h) == po(k, nx, ny, lox, loy, lox + w, loy + h)


# ---------------------------------------------------------------- AD engine
# The alternating-direction split remap (remap.cpp:469-589, 1110-1115), the
# first "next" row of SURVEY.md 8f.

@pytest.mark.parametrize("case,steps", [
    (cases.riemann2d(48), 60),
    (cases.sedov(64), 80),
    (cases.triple_point(64, 32), 700),
    (cases.shock_bubble(64), 30),
])
def test_run_loop_ad_bitwise(ref, orc, case, steps):
    sr, so = _both(ref, orc, case.cfg, case.paint())
    rr, er = helpers.run_capture(sr, steps, case.cfl, abi.REMAP_AD)
    ro, eo = helpers.run_capture(so, steps, case.cfl, abi.REMAP_AD)
    assert er == eo
    assert rr.steps_done == ro.steps_done and np.array_equal(rr.dts, ro.dts)
    assert rr.diag == ro.diag and rr.floor_count == ro.floor_count
    assert helpers.bitwise_diff(sr.download(), so.download(), helpers.STATE_FIELDS) == []


@pytest.mark.parametrize("bcx,bcy,order,degrade", [(BC_PERIODIC, BC_PERIODIC, 2, 1), (BC_WALL, BC_WALL, 2, 1),
                                                  (BC_PERIODIC, BC_WALL, 1, 1), (BC_WALL, BC_PERIODIC, 2, 0)])
@pytest.mark.parametrize("kind", ["gas", "front", "blobs"])
def test_kinematic_remap_ad_bitwise(ref, orc, bcx, bcy, order, degrade, kind):
    nmat = 1 if kind == "gas" else 2
    cfg = make_config(13, 11, 1.0, 1.0, 0.25, -0.5, bcx, bcy, eos=[(EOS_PERFECT, 1.4, 0.0)] * nmat,
                      face_order=order, interface_degrade=degrade)
    painted = helpers.random_state(cfg, 11 + order + 3 * degrade, kind, umax=0.25)
    sr, so = _both(ref, orc, cfg, painted)
    lag = helpers.kinematic(sr.download())
    for x_first in (True, False):
        for vel in (True, False):
            dr, do = abi.RemapDiag(), abi.RemapDiag()
            sr2, so2 = _both(ref, orc, cfg, sr.download())
            sr2.set_lagrange(lag)
            so2.set_lagrange(lag)
            sr2.remap_step(1.0, kind=abi.REMAP_AD, x_first=x_first, remap_velocity=vel, diag=dr)
            so2.remap_step(1.0, kind=abi.REMAP_AD, x_first=x_first, remap_velocity=vel, diag=do)
            assert helpers.bitwise_diff(sr2.download(), so2.download(), helpers.STATE_FIELDS) == []
            assert (dr.max_k_violation, dr.k_clip_count, dr.mass_fix_count) == \
                   (do.max_k_violation, do.k_clip_count, do.mass_fix_count)


@pytest.mark.parametrize("scenario", ["cfl_face", "collapsed"])
def test_error_parity_ad(ref, orc, scenario):
    cfg = make_config(9, 8, 1.0, 1.0, bc_x=BC_WALL, bc_y=BC_PERIODIC)
    painted = helpers.random_state(cfg, 3, "gas", umax=0.05)
    sr, so = _both(ref, orc, cfg, painted)
    lag = helpers.kinematic(sr.download())
    if scenario == "cfl_face":
        lag.u_half[..., 0] = 0.95
    else:  # converging X face displacements collapse a cell
        lag.u_half[..., 0] = 0.0
        lag.u_half[:, 5, 0] = 0.6
        lag.u_half[:, 6, 0] = -0.6
    out = []
    for s in (sr, so):
        s.set_lagrange(lag)
        out.append(_err(s, lambda s: s.remap_step(1.0, kind=abi.REMAP_AD)))
    assert out[0] == out[1] and out[0] is not None


@pytest.mark.parametrize("bcx,bcy,order,degrade", [(BC_PERIODIC, BC_PERIODIC, 2, 1), (BC_WALL, BC_WALL, 2, 1),
                                                   (BC_PERIODIC, BC_WALL, 1, 1), (BC_WALL, BC_PERIODIC, 2, 0)])
@pytest.mark.parametrize("kind", ["gas", "front", "blobs"])
def test_kinematic_remap_direct_bitwise(ref, orc, bcx, bcy, order, degrade, kind):
    """The Direct (faces-only) engine, remap.cpp:593-724."""
    nmat = 1 if kind == "gas" else 2
    cfg = make_config(13, 11, 1.0, 1.0, 0.25, -0.5, bcx, bcy, eos=[(EOS_PERFECT, 1.4, 0.0)] * nmat,
                      face_order=order, interface_degrade=degrade)
    painted = helpers.random_state(cfg, hash((bcx, bcy, order, degrade, kind, "direct")) & 0xFFFF, kind, umax=0.25)
    sr, so = _both(ref, orc, cfg, painted)
    lag = helpers.kinematic(sr.download())
    for vel in (True, False):
        dr, do = abi.RemapDiag(), abi.RemapDiag()
        sr2, so2 = _both(ref, orc, cfg, sr.download())
        sr2.set_lagrange(lag)
        so2.set_lagrange(lag)
        sr2.remap_step(1.0, kind=abi.REMAP_DIRECT, remap_velocity=vel, diag=dr)
        so2.remap_step(1.0, kind=abi.REMAP_DIRECT, remap_velocity=vel, diag=do)
        assert helpers.bitwise_diff(sr2.download(), so2.download(), helpers.STATE_FIELDS) == []
        assert (dr.max_k_violation, dr.k_clip_count, dr.mass_fix_count) == \
               (do.max_k_violation, do.k_clip_count, do.mass_fix_count)


@pytest.mark.parametrize("case,steps", [(cases.riemann2d(48), 80), (cases.triple_point(64, 32), 700),
                                        (cases.shock_bubble(48), 30)])
def test_run_loop_direct_bitwise(ref, orc, case, steps):
    sr, so = _both(ref, orc, case.cfg, case.paint())
    rr, er = helpers.run_capture(sr, steps, case.cfl, kind=abi.REMAP_DIRECT)
    ro, eo = helpers.run_capture(so, steps, case.cfl, kind=abi.REMAP_DIRECT)
    assert er == eo
    assert np.array_equal(rr.dts, ro.dts)
    assert (rr.floor_count, rr.diag) == (ro.floor_count, ro.diag)
    assert helpers.bitwise_diff(sr.download(), so.download(), helpers.STATE_FIELDS) == []


@pytest.mark.parametrize("scenario", ["cfl_face", "collapsed"])
def test_error_parity_direct(ref, orc, scenario):
    cfg = make_config(12, 10, 1.0, 1.0, bc_x=BC_PERIODIC, bc_y=BC_PERIODIC)
    painted = helpers.random_state(cfg, 77, "gas", umax=0.2)
    sr, so = _both(ref, orc, cfg, painted)
    st = sr.download()
    lag = helpers.kinematic(st)
    g = abi.GHOST
    if scenario == "cfl_face":
        lag.u_half[g + 3, g + 5, 0] = 1.9  # one fast node: face volume > 0.9 cv
        lag.u_half[g + 4, g + 5, 0] = 1.9
    else:
        lag.u_half[g + 3, g + 5, 0] = -3.0  # the cell's faces converge past its volume
        lag.u_half[g + 4, g + 5, 0] = -3.0
        lag.u_half[g + 3, g + 4, 0] = 3.0
        lag.u_half[g + 4, g + 4, 0] = 3.0
    res = []
    for s in (sr, so):
        s.set_lagrange(lag)
        try:
            s.remap_step(0.5, kind=abi.REMAP_DIRECT)
            res.append(None)
        except errors.SimError as e:
            res.append((type(e).__name__, e.what, e.i, e.j))
    assert res[0] == res[1]
    assert res[0] is not None

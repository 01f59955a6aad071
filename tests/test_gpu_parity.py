"""Parity of the CUDA product (libh2d.so, through the C-ABI) against the
REFERENCE library itself (oracle/_ref, h2dr_, built from /root/reference and
shipped to the GPU box) wherever it can hold the case (at most two
materials, no build option of this product), else against the C
restatement oracle, which is pinned bit for bit to the reference
(test_oracle_vs_reference.py).  The bar is bit-exact: every State and
LagrangeResult byte, every dt, the mixed-cell set, the RemapDiag counters,
floor counts and the first located error."""
import zlib

import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import abi, cases, errors
from paper_2208_13409_b200.abi import BC_PERIODIC, BC_WALL, CORNER_LINEARDIAG, CORNER_UPWIND, EOS_PERFECT, \
    EOS_STIFFENED, make_config

pytestmark = pytest.mark.gpu


def _checker(orc, cfg):
    """The reference itself when it can run the case, else the oracle."""
    ref = helpers.ref_lib()
    return ref if ref is not None and cfg.nmat <= 2 and not getattr(cfg, "options", 0) else orc


def _pair(gpu, orc, cfg, painted):
    return helpers.prepared(gpu, cfg, painted), helpers.prepared(_checker(orc, cfg), cfg, painted)


def test_init_helpers(gpu, orc):
    for case in (cases.riemann2d(40), cases.triple_point(64, 32), cases.shock_bubble(48)):
        sg, so = _pair(gpu, orc, case.cfg, case.paint())
        assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS) == []


@pytest.mark.parametrize("case,steps", [
    (cases.riemann2d(48), 100),
    (cases.sedov(64), 120),
    (cases.triple_point(64, 32), 700),      # aborts at the same step with the same error
    (cases.shock_bubble(64), 40),
])
def test_run_loop_bitwise(gpu, orc, case, steps):
    sg, so = _pair(gpu, orc, case.cfg, case.paint())
    rg, eg = helpers.run_capture(sg, steps, case.cfl)
    ro, eo = helpers.run_capture(so, steps, case.cfl)
    assert eg == eo
    assert rg.steps_done == ro.steps_done
    assert np.array_equal(rg.dts, ro.dts)
    assert rg.diag == ro.diag and rg.floor_count == ro.floor_count
    a, b = sg.download(), so.download()
    assert helpers.bitwise_diff(a, b, helpers.STATE_FIELDS) == []
    assert (a.step, a.time) == (b.step, b.time)
    assert sg.totals() == so.totals()


@pytest.mark.parametrize("kind", ["gas", "front", "blobs"])
@pytest.mark.parametrize("bcx,bcy,dx", [(BC_WALL, BC_WALL, 0.025), (BC_WALL, BC_WALL, 1.0 / 32),
                                        (BC_PERIODIC, BC_WALL, 0.025), (BC_WALL, BC_PERIODIC, 1.0 / 32)])
def test_run_loop_random_states(gpu, orc, kind, bcx, bcy, dx):
    """The run loop (fused Lagrange kernel) on random states: rough pressure
    next to the walls makes the wall-node gradient a rounding residue, which
    fill_ghost_nodes zeroes before correct uses u_half (lagrange.cpp:143,155)."""
    nmat = 1 if kind == "gas" else 2
    cfg = make_config(40, 24, dx, dx * 1.25, 0.0, 0.0, bcx, bcy, eos=[(EOS_PERFECT, 1.4, 0.0), (EOS_PERFECT, 1.6, 0.0)][:nmat])
    seed = zlib.crc32(repr((kind, bcx, bcy, dx)).encode()) & 0xFFFF
    painted = helpers.random_state(cfg, seed, kind, umax=0.1, e_scale=3.0)
    sg, so = _pair(gpu, orc, cfg, painted)
    rg, eg = helpers.run_capture(sg, 25, 0.3)
    ro, eo = helpers.run_capture(so, 25, 0.3)
    assert eg == eo
    assert rg.steps_done == ro.steps_done and np.array_equal(rg.dts, ro.dts)
    assert rg.diag == ro.diag and rg.floor_count == ro.floor_count
    assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS) == []


@pytest.mark.parametrize("n,steps", [(48, 80), (64, 60)])
def test_wall_blast_bitwise(gpu, orc, n, steps):
    """A strong blast against the middle of the left wall: the artificial
    viscosity dominates p + q at the wall nodes, so the rounding residue of the
    wall-node gradient is large enough to move a cell volume unless u_half's
    wall component is zeroed (fill_ghost_nodes) before correct uses it."""
    from paper_2208_13409_b200.cases import Case, Region, ALL, RECTANGLE, _mesh_cfg
    dx = 1.0 / n
    p0 = 0.4 / (2 * dx * dx)
    y0 = (n // 2) * dx
    case = Case("wall_blast", _mesh_cfg(n, n, 1.0, 1.0, [(EOS_PERFECT, 1.4, 0.0)]),
                [Region(ALL, rho=1.0, p=1e-6), Region(RECTANGLE, rect=(0.0, y0, 2 * dx, y0 + dx), rho=1.0, p=p0)],
                0.5, steps)
    sg, so = _pair(gpu, orc, case.cfg, case.paint())
    rg, eg = helpers.run_capture(sg, steps, case.cfl)
    ro, eo = helpers.run_capture(so, steps, case.cfl)
    assert eg == eo
    assert rg.steps_done == ro.steps_done and np.array_equal(rg.dts, ro.dts)
    assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS) == []


CONFIGS = []
for bcx, bcy in ((BC_PERIODIC, BC_PERIODIC), (BC_WALL, BC_WALL), (BC_PERIODIC, BC_WALL)):
    for order, corner, degrade in ((2, CORNER_LINEARDIAG, 1), (1, CORNER_UPWIND, 1), (2, CORNER_UPWIND, 1),
                                   (2, CORNER_LINEARDIAG, 0), (2, abi.CORNER_AVGMIN, 1), (2, abi.CORNER_LINEARXY, 1),
                                   (2, abi.CORNER_MULTID, 1), (2, abi.CORNER_MULTID, 0)):
        CONFIGS.append((bcx, bcy, order, corner, degrade))


@pytest.mark.parametrize("corner", [abi.CORNER_AVGMIN, abi.CORNER_LINEARXY, abi.CORNER_MULTID])
@pytest.mark.parametrize("which,steps", [("riemann", 60), ("triple", 80), ("bubble", 30), ("voronoi3", 30)])
def test_run_loop_corner_schemes_bitwise(gpu, orc, corner, which, steps):
    """AvgMin / LinearXY / Multid corners (+ Multid faces), reconstruct.cpp:116-152."""
    case = {"riemann": cases.riemann2d(48), "triple": cases.triple_point(64, 32), "bubble": cases.shock_bubble(48),
            "voronoi3": cases.voronoi3(64)}[which]
    m = case.cfg.mesh
    cfg = make_config(m.nx, m.ny, m.dx, m.dy, m.x0, m.y0, m.bc_x, m.bc_y,
                      eos=[(case.cfg.eos[a].kind, case.cfg.eos[a].gamma, case.cfg.eos[a].pi)
                           for a in range(case.cfg.nmat)], corner=corner)
    sg, so = _pair(gpu, orc, cfg, case.paint())
    rg, eg = helpers.run_capture(sg, steps, case.cfl)
    ro, eo = helpers.run_capture(so, steps, case.cfl)
    assert eg == eo
    assert np.array_equal(rg.dts, ro.dts)
    assert (rg.floor_count, rg.diag) == (ro.floor_count, ro.diag)
    assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS, case.cfg.nmat) == []


@pytest.mark.parametrize("bcx,bcy,order,corner,degrade", CONFIGS)
@pytest.mark.parametrize("kind", ["gas", "front", "blobs"])
def test_kinematic_remap_bitwise(gpu, orc, bcx, bcy, order, corner, degrade, kind):
    nmat = 1 if kind == "gas" else 2
    cfg = make_config(13, 11, 1.0, 1.0, 0.25, -0.5, bcx, bcy, eos=[(EOS_PERFECT, 1.4, 0.0)] * nmat,
                      face_order=order, corner=corner, interface_degrade=degrade)
    seed = hash((bcx, bcy, order, corner, degrade, kind)) & 0xFFFF
    painted = helpers.random_state(cfg, seed, kind, umax=0.25)
    sg, so = _pair(gpu, orc, cfg, painted)
    lag = helpers.kinematic(so.download())
    for vel in (True, False):
        sg2, so2 = _pair(gpu, orc, cfg, so.download())
        sg2.set_lagrange(lag)
        so2.set_lagrange(lag)
        dg, do = abi.RemapDiag(), abi.RemapDiag()
        sg2.remap_step(1.0, remap_velocity=vel, diag=dg)
        so2.remap_step(1.0, remap_velocity=vel, diag=do)
        assert helpers.bitwise_diff(sg2.download(), so2.download(), helpers.STATE_FIELDS) == []
        assert (dg.max_k_violation, dg.k_clip_count, dg.mass_fix_count) == \
               (do.max_k_violation, do.k_clip_count, do.mass_fix_count)


@pytest.mark.parametrize("bcx,bcy", [(BC_WALL, BC_WALL), (BC_PERIODIC, BC_PERIODIC), (BC_WALL, BC_PERIODIC)])
@pytest.mark.parametrize("kind,eos", [
    ("gas", [(EOS_PERFECT, 1.4, 0.0)]),
    ("blobs", [(EOS_PERFECT, 1.4, 0.0), (EOS_STIFFENED, 7.0, 0.5)]),
    ("front", [(EOS_PERFECT, 1.5, 0.0), (EOS_PERFECT, 1.67, 0.0)]),
])
def test_lagrange_then_remap_bitwise(gpu, orc, bcx, bcy, kind, eos):
    cfg = make_config(17, 12, 0.5, 0.25, 0.0, 0.0, bcx, bcy, eos=eos)
    painted = helpers.random_state(cfg, 7, kind, umax=0.05)
    sg, so = _pair(gpu, orc, cfg, painted)
    for step in range(3):
        dtg, dto = sg.cfl_dt(0.4), so.cfl_dt(0.4)
        assert dtg == dto
        lg, lo = sg.lagrange_step(dtg), so.lagrange_step(dto)
        assert helpers.bitwise_diff(lg, lo, helpers.LAG_FIELDS) == []
        assert lg.floor_count == lo.floor_count
        sg.remap_step(dtg)
        so.remap_step(dto)
        assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS) == []


def _err(s, fn):
    try:
        fn(s)
    except errors.SimError as e:
        return type(e).__name__, e.what, e.i, e.j
    return None


@pytest.mark.parametrize("scenario", ["cfl_face", "tangled", "unphysical", "wave"])
def test_error_parity(gpu, orc, scenario):
    cfg = make_config(9, 8, 1.0, 1.0, bc_x=BC_WALL, bc_y=BC_PERIODIC)
    painted = helpers.random_state(cfg, 3, "gas", umax=0.05)
    if scenario == "unphysical":
        painted.e[0][4, 5] = -3.0
    sg, so = _pair(gpu, orc, cfg, painted)
    if scenario == "cfl_face":
        lag = helpers.kinematic(so.download())
        lag.u_half[..., 0] = 0.95
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
    eg, eo = _err(sg, fn), _err(so, fn)
    assert eo is not None and eg == eo
    # a failed call leaves the State untouched (value semantics)
    assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS) == []


def test_c1_full_size(gpu, orc):
    """Config 1 at full size (256^2, 100 steps): every step's dt and the final
    fields bit-identical to the oracle."""
    case = cases.riemann2d(256)
    sg, so = _pair(gpu, orc, case.cfg, case.paint())
    rg, _ = helpers.run_capture(sg, case.steps, case.cfl)
    ro, _ = helpers.run_capture(so, case.steps, case.cfl)
    assert rg.steps_done == ro.steps_done == 100
    assert np.array_equal(rg.dts, ro.dts)
    assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS) == []


# ---------------------------------------------------------------- AD engine
# The alternating-direction split remap on the device (remap.cpp:469-589,
# 1110-1115) against the oracle, which tests/test_oracle_vs_reference.py pins
# to the reference.

@pytest.mark.parametrize("case,steps", [
    (cases.riemann2d(48), 60),
    (cases.sedov(64), 80),
    (cases.triple_point(64, 32), 700),
    (cases.shock_bubble(64), 30),
    (cases.triple_point(100, 44), 120),
])
def test_run_loop_ad_bitwise(gpu, orc, case, steps):
    sg, so = _pair(gpu, orc, case.cfg, case.paint())
    rg, eg = helpers.run_capture(sg, steps, case.cfl, abi.REMAP_AD)
    ro, eo = helpers.run_capture(so, steps, case.cfl, abi.REMAP_AD)
    assert eg == eo
    assert rg.steps_done == ro.steps_done and np.array_equal(rg.dts, ro.dts)
    assert rg.diag == ro.diag and rg.floor_count == ro.floor_count
    assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS) == []


@pytest.mark.parametrize("bcx,bcy,order,degrade", [(BC_PERIODIC, BC_PERIODIC, 2, 1), (BC_WALL, BC_WALL, 2, 1),
                                                  (BC_PERIODIC, BC_WALL, 1, 1), (BC_WALL, BC_PERIODIC, 2, 0)])
@pytest.mark.parametrize("kind", ["gas", "front", "blobs"])
def test_kinematic_remap_ad_bitwise(gpu, orc, bcx, bcy, order, degrade, kind):
    nmat = 1 if kind == "gas" else 2
    cfg = make_config(13, 11, 1.0, 1.0, 0.25, -0.5, bcx, bcy, eos=[(EOS_PERFECT, 1.4, 0.0)] * nmat,
                      face_order=order, interface_degrade=degrade)
    painted = helpers.random_state(cfg, 11 + order + 3 * degrade, kind, umax=0.25)
    sg, so = _pair(gpu, orc, cfg, painted)
    lag = helpers.kinematic(so.download())
    for x_first in (True, False):
        for vel in (True, False):
            dg, do = abi.RemapDiag(), abi.RemapDiag()
            sg2, so2 = _pair(gpu, orc, cfg, so.download())
            sg2.set_lagrange(lag)
            so2.set_lagrange(lag)
            sg2.remap_step(1.0, kind=abi.REMAP_AD, x_first=x_first, remap_velocity=vel, diag=dg)
            so2.remap_step(1.0, kind=abi.REMAP_AD, x_first=x_first, remap_velocity=vel, diag=do)
            assert helpers.bitwise_diff(sg2.download(), so2.download(), helpers.STATE_FIELDS) == []
            assert (dg.max_k_violation, dg.k_clip_count, dg.mass_fix_count) == \
                   (do.max_k_violation, do.k_clip_count, do.mass_fix_count)


@pytest.mark.parametrize("scenario", ["cfl_face", "collapsed"])
def test_error_parity_ad(gpu, orc, scenario):
    cfg = make_config(9, 8, 1.0, 1.0, bc_x=BC_WALL, bc_y=BC_PERIODIC)
    painted = helpers.random_state(cfg, 3, "gas", umax=0.05)
    sg, so = _pair(gpu, orc, cfg, painted)
    lag = helpers.kinematic(so.download())
    if scenario == "cfl_face":
        lag.u_half[..., 0] = 0.95
    else:
        lag.u_half[..., 0] = 0.0
        lag.u_half[:, 5, 0] = 0.6
        lag.u_half[:, 6, 0] = -0.6
    out = []
    for s in (sg, so):
        s.set_lagrange(lag)
        try:
            s.remap_step(1.0, kind=abi.REMAP_AD)
            out.append(None)
        except errors.SimError as e:
            out.append((type(e).__name__, e.what, e.i, e.j))
    assert out[0] == out[1] and out[0] is not None


# ---- the Direct (faces-only) engine, remap.cpp:593-724 --------------------------------

@pytest.mark.parametrize("bcx,bcy,order,degrade", [(BC_PERIODIC, BC_PERIODIC, 2, 1), (BC_WALL, BC_WALL, 2, 1),
                                                   (BC_PERIODIC, BC_WALL, 1, 1), (BC_WALL, BC_PERIODIC, 2, 0)])
@pytest.mark.parametrize("kind", ["gas", "front", "blobs"])
def test_kinematic_remap_direct_bitwise(gpu, orc, bcx, bcy, order, degrade, kind):
    nmat = 1 if kind == "gas" else 2
    cfg = make_config(13, 11, 1.0, 1.0, 0.25, -0.5, bcx, bcy, eos=[(EOS_PERFECT, 1.4, 0.0)] * nmat,
                      face_order=order, interface_degrade=degrade)
    painted = helpers.random_state(cfg, hash((bcx, bcy, order, degrade, kind, "direct")) & 0xFFFF, kind, umax=0.25)
    sg, so = _pair(gpu, orc, cfg, painted)
    lag = helpers.kinematic(so.download())
    for vel in (True, False):
        dg, do = abi.RemapDiag(), abi.RemapDiag()
        sg2, so2 = _pair(gpu, orc, cfg, so.download())
        sg2.set_lagrange(lag)
        so2.set_lagrange(lag)
        sg2.remap_step(1.0, kind=abi.REMAP_DIRECT, remap_velocity=vel, diag=dg)
        so2.remap_step(1.0, kind=abi.REMAP_DIRECT, remap_velocity=vel, diag=do)
        assert helpers.bitwise_diff(sg2.download(), so2.download(), helpers.STATE_FIELDS) == []
        assert (dg.max_k_violation, dg.k_clip_count, dg.mass_fix_count) == \
               (do.max_k_violation, do.k_clip_count, do.mass_fix_count)


@pytest.mark.parametrize("which,steps", [("riemann", 80), ("triple", 700), ("bubble", 30), ("voronoi3", 30)])
def test_run_loop_direct_bitwise(gpu, orc, which, steps):
    case = {"riemann": cases.riemann2d(48), "triple": cases.triple_point(64, 32), "bubble": cases.shock_bubble(48),
            "voronoi3": cases.voronoi3(64)}[which]
    sg, so = _pair(gpu, orc, case.cfg, case.paint())
    rg, eg = helpers.run_capture(sg, steps, case.cfl, kind=abi.REMAP_DIRECT)
    ro, eo = helpers.run_capture(so, steps, case.cfl, kind=abi.REMAP_DIRECT)
    assert eg == eo
    assert np.array_equal(rg.dts, ro.dts)
    assert (rg.floor_count, rg.diag) == (ro.floor_count, ro.diag)
    assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS, case.cfg.nmat) == []


@pytest.mark.parametrize("scenario", ["cfl_face", "collapsed"])
def test_error_parity_direct(gpu, orc, scenario):
    cfg = make_config(12, 10, 1.0, 1.0, bc_x=BC_PERIODIC, bc_y=BC_PERIODIC)
    painted = helpers.random_state(cfg, 77, "gas", umax=0.2)
    sg, so = _pair(gpu, orc, cfg, painted)
    lag = helpers.kinematic(so.download())
    g = abi.GHOST
    if scenario == "cfl_face":
        lag.u_half[g + 3, g + 5, 0] = 1.9
        lag.u_half[g + 4, g + 5, 0] = 1.9
        lag.u_half[g + 6, g + 2, 1] = 1.9  # and a fast Y face later in loop order
        lag.u_half[g + 6, g + 3, 1] = 1.9
    else:
        lag.u_half[g + 3, g + 5, 0] = -3.0
        lag.u_half[g + 4, g + 5, 0] = -3.0
        lag.u_half[g + 3, g + 4, 0] = 3.0
        lag.u_half[g + 4, g + 4, 0] = 3.0
    res = []
    for s in (sg, so):
        s.set_lagrange(lag)
        try:
            s.remap_step(0.5, kind=abi.REMAP_DIRECT)
            res.append(None)
        except errors.SimError as e:
            res.append((type(e).__name__, e.what, e.i, e.j))
    assert res[0] == res[1] and res[0] is not None

"""Three materials (configuration 5): the N-material extension of the
reference's one-interface VOF remap (the reference
itself stops at kMaxMat = 2, state.hpp:13, so there is no reference run of a
3-material state: parity unpinned).

What pins it anyway:
  * wherever at most two materials are present the extension IS the
    reference: a 3-material run with one material absent equals the
    2-material reference run bit for bit (material 2 absent; or material 0
    absent with the other two relabelled);
  * conservation of every material's mass, fractions in [0, 1] summing to 1,
    and no error over a Voronoi run;
  * the CUDA product equals the restated oracle bit for bit (GPU tests)."""
import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import abi, cases
from paper_2208_13409_b200.abi import BC_PERIODIC, EOS_PERFECT, EOS_STIFFENED, HostState, make_config

G = abi.GHOST
E2 = (EOS_PERFECT, 1.67, 0.0)


def as_three(cfg2, st2: HostState, absent: int, eos_absent=E2):
    """The 2-material problem as a 3-material one with material `absent`
    (0 or 2) empty: the two present ones keep their order."""
    m = cfg2.mesh
    eos2 = [(cfg2.eos[a].kind, cfg2.eos[a].gamma, cfg2.eos[a].pi) for a in range(2)]
    eos3 = eos2 + [eos_absent] if absent == 2 else [eos_absent] + eos2
    cfg3 = make_config(m.nx, m.ny, m.dx, m.dy, m.x0, m.y0, m.bc_x, m.bc_y, eos=eos3, a1=cfg2.pv_a1,
                       a2=cfg2.pv_a2, face_order=cfg2.face_order, corner=cfg2.corner,
                       interface_degrade=cfg2.interface_degrade)
    st3 = HostState.empty(m.nx, m.ny, 3, m.dx * m.dy)
    slots = (0, 1) if absent == 2 else (1, 2)
    for src, dst in enumerate(slots):
        st3.m[dst][...] = st2.m[src]
        st3.e[dst][...] = st2.e[src]
        st3.k[dst][...] = st2.k[src]
    st3.k[absent][...] = 0.0
    st3.u[...] = st2.u
    st3.iface_normal[...] = st2.iface_normal
    return cfg3, st3, slots


def same_as_two(st3, st2, slots):
    bad = []
    for f in ("m", "e", "k"):
        for src, dst in enumerate(slots):
            if not np.array_equal(getattr(st3, f)[dst].view(np.int64), getattr(st2, f)[src].view(np.int64)):
                bad.append((f, dst))
    bad += helpers.bitwise_diff(st3, st2, ("vol", "m_mix", "e_mix", "rho_mix", "p_mix", "iface_normal", "u"))
    return bad


def two_material_problems():
    tp = cases.triple_point(64, 32)
    sb = cases.shock_bubble(48)
    cfgb = make_config(40, 32, 0.025, 0.03125, bc_x=BC_PERIODIC, bc_y=BC_PERIODIC,
                       eos=[(EOS_PERFECT, 1.4, 0.0), (EOS_STIFFENED, 4.4, 0.6)])
    return [("triple", tp.cfg, tp.paint(), tp.cfl, 60), ("bubble", sb.cfg, sb.paint(), sb.cfl, 30),
            ("blobs", cfgb, helpers.random_state(cfgb, 11, "blobs", umax=0.1), 0.3, 25)]


@pytest.mark.parametrize("absent", [2, 0])
@pytest.mark.parametrize("which", [0, 1, 2])
def test_absent_material_reduces_to_two(orc, which, absent):
    """The extension with one material absent is the 2-material (reference)
    scheme: run loop, dt, counters and every State byte."""
    name, cfg2, st2, cfl, steps = two_material_problems()[which]
    s2 = helpers.prepared(orc, cfg2, st2)
    cfg3, st3, slots = as_three(cfg2, s2.download(), absent)
    s3 = abi.Solver(orc, cfg3)
    s3.upload(st3, derived=False)
    r2, e2 = helpers.run_capture(s2, steps, cfl)
    r3, e3 = helpers.run_capture(s3, steps, cfl)
    assert e2 == e3
    assert r2.steps_done == r3.steps_done
    assert np.array_equal(r2.dts, r3.dts)
    if absent == 2:  # the canonical embedding (materials in the first two slots): counters too
        assert (r2.floor_count, r2.diag) == (r3.floor_count, r3.diag)
    else:  # a pure cell is finalised on the pair (0, its material): the clip counter may differ
        assert (r2.floor_count, r2.diag["max_k_violation"], r2.diag["mass_fix_count"]) == \
            (r3.floor_count, r3.diag["max_k_violation"], r3.diag["mass_fix_count"])
    assert same_as_two(s3.download(), s2.download(), slots) == []


def test_voronoi_conservation_and_fractions(orc):
    """(Like the reference's own 2-material proxy of config 5, which aborts
    with UnphysicalStateError after 35-67 steps, the Voronoi
    state's density / pressure contrasts of up to 100 end the run early: a
    remapped sliver's energy goes negative. The 128^2 case aborts at step 63.)"""
    case = cases.voronoi3(128)
    s = helpers.prepared(orc, case.cfg, case.paint())
    st0 = s.download()
    m0 = [st0.cell(st0.m[a]).sum() for a in range(3)]
    r = s.run(50, cfl=case.cfl)
    assert r.steps_done == 50
    st = s.download()
    k = np.stack([st.cell(st.k[a]) for a in range(3)])
    assert k.min() >= 0.0 and k.max() <= 1.0
    assert np.abs(k.sum(axis=0) - 1.0).max() <= 4e-16
    # total mass is conserved; a material's own mass too unless an orphan
    # sliver joined another material (mass_fix_count, remap.cpp:217-225)
    assert abs(sum(st.cell(st.m[a]).sum() for a in range(3)) - sum(m0)) <= 1e-12 * sum(m0)
    if r.diag["mass_fix_count"] == 0:
        for a in range(3):
            assert abs(st.cell(st.m[a]).sum() - m0[a]) <= 1e-12 * m0[a]
    mixed = (k.max(axis=0) < 1.0).sum()
    assert mixed > 0 and ((k > 0).sum(axis=0) == 3).sum() > 0  # the run exercises triple cells


def test_voronoi_painter_is_a_partition():
    case = cases.voronoi3(64)
    st = case.paint()
    k = np.stack([st.cell(st.k[a]) for a in range(3)])
    assert np.array_equal(k.sum(axis=0), np.ones_like(k[0]))
    cv = case.cfg.mesh.dx * case.cfg.mesh.dy
    xy, mat, rho, p, uv = case.sites
    pure = k.max(axis=0) == 1.0
    assert pure.mean() > 0.8
    a = np.argmax(k, axis=0)
    m = np.choose(a, [st.cell(st.m[b]) for b in range(3)])
    assert np.all((m[pure] / cv > 0.099) & (m[pure] / cv < 10.01))


@pytest.mark.gpu
@pytest.mark.parametrize("n,steps", [(64, 20), (128, 70), (256, 40)])  # 64^2 and 128^2 abort (steps 11, 63)
def test_device_three_materials_bitwise(gpu, orc, n, steps):
    case = cases.voronoi3(n)
    painted = case.paint()
    sg, so = helpers.prepared(gpu, case.cfg, painted), helpers.prepared(orc, case.cfg, painted)
    assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS, 3) == []
    rg, eg = helpers.run_capture(sg, steps, case.cfl)
    ro, eo = helpers.run_capture(so, steps, case.cfl)
    assert eg == eo
    assert rg.steps_done == ro.steps_done
    assert np.array_equal(rg.dts, ro.dts)
    assert (rg.floor_count, rg.diag) == (ro.floor_count, ro.diag)
    assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS, 3) == []


@pytest.mark.gpu
@pytest.mark.parametrize("absent", [2, 0])
def test_device_absent_material_reduces_to_two(gpu, orc, absent):
    name, cfg2, st2, cfl, steps = two_material_problems()[0]
    s2 = helpers.prepared(orc, cfg2, st2)
    cfg3, st3, slots = as_three(cfg2, s2.download(), absent)
    sg = abi.Solver(gpu, cfg3)
    sg.upload(st3, derived=False)
    r2, _ = helpers.run_capture(s2, steps, cfl)
    r3, _ = helpers.run_capture(sg, steps, cfl)
    assert np.array_equal(r2.dts, r3.dts)
    assert same_as_two(sg.download(), s2.download(), slots) == []


# ---- H2D_OPT_SLIVER_ENERGY: configuration 5 to its 100 steps ----------------
def _voronoi_opt(n):
    c = cases.voronoi3(n)
    c.cfg.options = abi.OPT_SLIVER_ENERGY
    return c


def test_voronoi_aborts_without_the_safeguard(orc):
    """Like the reference's own two-material proxy, the
    scheme as the reference defines it aborts the Voronoi case: a remapped
    sliver's e goes negative and sound_speed throws (eos.hpp:31-32)."""
    c = cases.voronoi3(64)
    s = helpers.prepared(orc, c.cfg, c.paint())
    r, err = helpers.run_capture(s, 100, c.cfl)
    assert err is not None and err[0] == "UnphysicalStateError" and r.steps_done < 100


@pytest.mark.parametrize("n", [64, 128])
def test_voronoi_safeguard_runs_100_steps(orc, n):
    """With the (non-default) sliver-energy safeguard the case runs its 100
    steps; mass is conserved per material up to sliver moves and in total."""
    c = _voronoi_opt(n)
    painted = c.paint()
    s = helpers.prepared(orc, c.cfg, painted)
    m0 = sum(float(np.sum(painted.cell(painted.m)[a])) for a in range(3))
    r, err = helpers.run_capture(s, 100, c.cfl)
    assert err is None and r.steps_done == 100
    st = s.download()
    m1 = sum(float(np.sum(st.cell(st.m)[a])) for a in range(3))
    assert abs(m1 - m0) <= 1e-12 * m0
    k = st.cell(st.k)[:3]
    assert (k >= 0.0).all() and (k <= 1.0).all()
    assert np.all(st.cell(st.e)[:3][st.cell(st.m)[:3] > 0] >= 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [64, 256])
def test_device_voronoi_safeguard_bitwise(gpu, orc, n):
    c = _voronoi_opt(n)
    painted = c.paint()
    sg = helpers.prepared(gpu, c.cfg, painted)
    so = helpers.prepared(orc, c.cfg, painted)
    rg, eg = helpers.run_capture(sg, 100, c.cfl)
    ro, eo = helpers.run_capture(so, 100, c.cfl)
    assert eg is None and eo is None and rg.steps_done == 100
    assert np.array_equal(rg.dts, ro.dts)
    assert rg.diag == ro.diag and rg.floor_count == ro.floor_count
    assert helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS, 3) == []


@pytest.mark.gpu
def test_device_voronoi_safeguard_blocks_bitwise(gpu):
    """the safeguard under the block data plane (window init, 4 x 2 blocks)."""
    from paper_2208_13409_b200 import multi
    c = _voronoi_opt(128)
    steps = 100
    s = helpers.prepared(gpu, c.cfg, c.paint())
    r = s.run(steps, cfl=c.cfl)
    ref = s.download()
    specs = multi.decompose(128, 128, 4, 2)
    blocks = [multi.BlockSolver(gpu, c.cfg, sp) for sp in specs]
    for b in blocks:
        b.init_window(c.paint(b.window()))
    comm = multi.DeviceComm(blocks, 4, 2)
    comm.run(steps, 1e30, c.cfl)
    comm.close()
    got = HostState.empty(128, 128, 3)
    for b in blocks:
        b.download_into(got)
        a, dts, e = b.result(steps)
        assert e is None and np.array_equal(dts, r.dts)
    assert helpers.bitwise_diff(got, ref, helpers.STATE_FIELDS, 3) == []

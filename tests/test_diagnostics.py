"""Per-step diagnostics of the run loop: RunReport::series (harness.cpp:385,410)
= make_diag (harness.cpp:360-376) over compute_totals (state.cpp:145-160).

The reference adds its totals in a serial loop; the product reduces them on
the device inside the step (a fixed-order tree), so:
  * step, t, dt and the four extrema are bit-identical;
  * every sum S = sum_k x_k is within 2 n 2^-53 sum_k |x_k| of the reference's
    (its serial error is at most (n-1) 2^-53 sum|x|, the tree's log2(n) 2^-53
    sum|x|); the bound is evaluated per step from the oracle's own State.
The oracle's series is pinned bitwise to the reference library's."""
import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import abi, cases, multi
from paper_2208_13409_b200.abi import BC_PERIODIC, HostState, make_config

EPS = 2.0 ** -53
SUMS = ("mass", "mass_mat", "momentum_x", "momentum_y", "internal_energy")
EXACT = ("step", "t", "dt", "min_rho", "max_rho", "min_p", "max_p")

CASES = {
    "riemann": lambda: cases.riemann2d(48),
    "sedov": lambda: cases.sedov(48),
    "triple": lambda: cases.triple_point(64, 32),
    "bubble": lambda: cases.shock_bubble(48),
}


def same_bits(a, b) -> bool:
    """Field-wise bit equality of StepDiag records (padding ignored)."""
    return all(np.ascontiguousarray(a[f]).tobytes() == np.ascontiguousarray(b[f]).tobytes()
               for f in abi.STEP_DIAG_DTYPE.names)


def term_scales(st: HostState, nx: int, ny: int, nmat: int, per_x=False, per_y=False):
    """(n, sum|x_k|) of every compute_totals sum of a State (state.cpp:148-158)."""
    c = st.cell
    m, e = c(st.m_mix), c(st.e_mix)
    g = abi.GHOST
    mm = st.m_mix[g - 1:g + ny + 1, g - 1:g + nx + 1]  # cells -1 .. n
    mp = 0.25 * (mm[:-1, :-1] + mm[:-1, 1:] + mm[1:, :-1] + mm[1:, 1:])  # nodes 0 .. n
    u = st.node(st.u)
    ie, je = (nx - 1 if per_x else nx), (ny - 1 if per_y else ny)
    mp, u = mp[:je + 1, :ie + 1], u[:je + 1, :ie + 1]
    nc, nn = nx * ny, (ie + 1) * (je + 1)
    return {
        "mass": (nc, np.abs(m).sum()),
        "internal_energy": (nc, np.abs(m * e).sum()),
        "mass_mat": [(nc, np.abs(c(st.m[a])).sum()) for a in range(nmat)],
        "momentum_x": (nn, np.abs(mp * u[..., 0]).sum()),
        "momentum_y": (nn, np.abs(mp * u[..., 1]).sum()),
    }


def assert_series_close(got, want, scales, nmat):
    for f in EXACT:
        assert np.array_equal(got[f], want[f]), f
    for q in range(len(want)):
        sc = scales[q]
        for f in SUMS:
            if f == "mass_mat":
                for a in range(nmat):
                    n, s = sc[f][a]
                    assert abs(got[f][q][a] - want[f][q][a]) <= 2 * n * EPS * s, (q, f, a)
            else:
                n, s = sc[f]
                assert abs(got[f][q] - want[f][q]) <= 2 * n * EPS * s, (q, f, got[f][q], want[f][q])


def oracle_series_with_scales(orc, case, steps):
    """The oracle's series and, per step, the term scales of its State."""
    so = helpers.prepared(orc, case.cfg, case.paint())
    m = case.cfg.mesh
    recs, scales = [], []
    for q in range(steps):
        r = so.run(q + 1, cfl=case.cfl, series=True)
        recs.append(r.series[0])
        scales.append(term_scales(so.download(), m.nx, m.ny, case.cfg.nmat,
                                  m.bc_x == BC_PERIODIC, m.bc_y == BC_PERIODIC))
    return np.array(recs, dtype=abi.STEP_DIAG_DTYPE), scales


# ---- CPU: the oracle restates make_diag bit for bit --------------------------------

@pytest.mark.ref
@pytest.mark.parametrize("which,steps", [("riemann", 30), ("triple", 40), ("bubble", 10), ("sedov", 20)])
def test_oracle_series_equals_reference(orc, ref, which, steps):
    case = CASES[which]()
    so = helpers.prepared(orc, case.cfg, case.paint())
    sr = helpers.prepared(ref, case.cfg, case.paint())
    a = so.run(steps, cfl=case.cfl, series=True)
    b = sr.run(steps, cfl=case.cfl, series=True)
    assert a.steps_done == b.steps_done == steps
    assert same_bits(a.series, b.series)
    assert same_bits(so.step_diag(0.5), sr.step_diag(0.5))


@pytest.mark.ref
def test_oracle_series_periodic_random(orc, ref):
    cfg = make_config(32, 24, 1.0 / 32, 1.0 / 24, bc_x=BC_PERIODIC, bc_y=BC_PERIODIC)
    painted = helpers.random_state(cfg, 7, "gas")
    so, sr = helpers.prepared(orc, cfg, painted), helpers.prepared(ref, cfg, painted)
    a, b = so.run(15, cfl=0.3, series=True), sr.run(15, cfl=0.3, series=True)
    assert same_bits(a.series, b.series)


def test_series_record_layout():
    assert abi.STEP_DIAG_DTYPE.itemsize == abi.C.sizeof(abi.StepDiag)
    assert abi.STEP_DIAG_DTYPE.fields["t"][1] == abi.StepDiag.t.offset
    assert abi.STEP_DIAG_DTYPE.fields["max_p"][1] == abi.StepDiag.max_p.offset


def test_combine_series_sums_and_extrema():
    a = np.zeros(2, abi.STEP_DIAG_DTYPE)
    b = np.zeros(2, abi.STEP_DIAG_DTYPE)
    a["mass"], b["mass"] = [1.0, 2.0], [3.0, 4.0]
    a["min_p"], b["min_p"] = [0.5, 0.1], [0.2, 0.3]
    a["max_rho"], b["max_rho"] = [5.0, 1.0], [2.0, 7.0]
    c = multi.combine_series([a, b])
    assert c["mass"].tolist() == [4.0, 6.0]
    assert c["min_p"].tolist() == [0.2, 0.1]
    assert c["max_rho"].tolist() == [5.0, 7.0]


# ---- GPU: the device series ----------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("which,steps", [("riemann", 25), ("sedov", 25), ("triple", 30), ("bubble", 12)])
def test_device_series(gpu, orc, which, steps):
    case = CASES[which]()
    want, scales = oracle_series_with_scales(orc, case, steps)
    sg = helpers.prepared(gpu, case.cfg, case.paint())
    got = sg.run(steps, cfl=case.cfl, series=True)
    assert got.steps_done == steps
    assert_series_close(got.series, want, scales, case.cfg.nmat)
    so = helpers.prepared(orc, case.cfg, case.paint())
    so.run(steps, cfl=case.cfl)
    assert same_bits(sg.step_diag(0.25), so.step_diag(0.25))


@pytest.mark.gpu
def test_device_series_periodic(gpu, orc):
    cfg = make_config(40, 32, 1.0 / 40, 1.0 / 32, bc_x=BC_PERIODIC, bc_y=BC_PERIODIC)
    painted = helpers.random_state(cfg, 3, "gas")

    class C:
        pass
    case = C()
    case.cfg, case.cfl, case.paint = cfg, 0.3, (lambda: painted)
    want, scales = oracle_series_with_scales(orc, case, 12)
    sg = helpers.prepared(gpu, cfg, painted)
    got = sg.run(12, cfl=0.3, series=True)
    assert_series_close(got.series, want, scales, 1)


@pytest.mark.gpu
def test_device_series_ad(gpu, orc):
    case = cases.triple_point(64, 32)
    sg = helpers.prepared(gpu, case.cfg, case.paint())
    so = helpers.prepared(orc, case.cfg, case.paint())
    got = sg.run(12, cfl=case.cfl, series=True, kind=abi.REMAP_AD)
    want = so.run(12, cfl=case.cfl, series=True, kind=abi.REMAP_AD)
    for f in EXACT:
        assert np.array_equal(got.series[f], want.series[f]), f
    for f in SUMS:
        assert np.allclose(got.series[f], want.series[f], rtol=1e-12, atol=1e-14), f


@pytest.mark.gpu
@pytest.mark.parametrize("px,py", [(2, 1), (2, 2)])
def test_block_series_combine(gpu, orc, px, py):
    case = cases.shock_bubble(64)
    steps = 10
    want, scales = oracle_series_with_scales(orc, case, steps)
    init = helpers.prepared(gpu, case.cfg, case.paint()).download()
    specs = multi.decompose(case.cfg.mesh.nx, case.cfg.mesh.ny, px, py)
    blocks = [multi.BlockSolver(gpu, case.cfg, sp) for sp in specs]
    for b in blocks:
        b.upload(init)
    multi.run_blocks(blocks, multi.LocalTransport(blocks, px, py), steps, 1e30, case.cfl)
    parts = [b.result(steps, series=True)[0].block_series for b in blocks]
    assert_series_close(multi.combine_series(parts), want, scales, case.cfg.nmat)

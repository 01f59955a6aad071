"""The reference's sub-step entry points and public scalar functions on the
device, compared bit for bit with the REFERENCE library itself (h2dr_,
oracle/_ref, present on the GPU box):

* predict (lagrange.cpp:79-144) -> HalfStepState, correct (:146-196) from a
  HalfStepState, remap_single_axis (remap.cpp:1098-1104) X and Y, with and
  without the velocity remap, 1 and 2 materials, walls / periodic, perfect
  and stiffened EOS;
* h2d_scalar_eval: van_leer, limited_gradient_1d, face_value, corner_value
  (all five schemes), multid_plane, clipped_fraction, place_interface,
  youngs_normal, cell_volume, cf_corner_flux, cf_face_flux_x/_y,
  pseudo_viscosity, div_u_cell, grad_pq_node and one face of ad_face_fluxes
  on seeded random records, including the records on which the reference
  throws (flags)."""
import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import abi, errors
from paper_2208_13409_b200.abi import BC_PERIODIC, BC_WALL, EOS_PERFECT, EOS_STIFFENED, make_config

pytestmark = pytest.mark.gpu

CFGS = {
    "gas_periodic": (make_config(24, 20, 0.05, 0.04, 0.0, 0.0, BC_PERIODIC, BC_PERIODIC), "gas"),
    "gas_wall": (make_config(24, 20, 0.05, 0.05, 0.0, 0.0, BC_WALL, BC_WALL), "gas"),
    "blobs_wall": (make_config(32, 24, 1 / 32, 1 / 32, 0.0, 0.0, BC_WALL, BC_WALL,
                               eos=[(EOS_PERFECT, 1.4, 0.0), (EOS_PERFECT, 1.67, 0.0)]), "blobs"),
    "blobs_stiff_mixed_bc": (make_config(28, 20, 0.5, 0.25, 0.0, 0.0, BC_WALL, BC_PERIODIC,
                                         eos=[(EOS_PERFECT, 1.4, 0.0), (EOS_STIFFENED, 7.0, 0.5)]), "blobs"),
}


def _pair(name, seed=7, umax=0.2):
    cfg, kind = CFGS[name]
    st = helpers.random_state(cfg, seed, kind, umax=umax)
    return (helpers.prepared(helpers.product_lib(), cfg, st), helpers.prepared(helpers.ref_lib(), cfg, st), cfg)


def _same(a, b, fields, nmat):
    bad = []
    for f in fields:
        x, y = getattr(a, f), getattr(b, f)
        if f in ("e_half", "p_half", "e_lag"):
            x, y = x[:nmat], y[:nmat]
        if not np.array_equal(x.view(np.int64), y.view(np.int64)):
            bad.append(f)
    return bad


@pytest.fixture(scope="module", autouse=True)
def _need_ref():
    if helpers.ref_lib() is None:
        pytest.skip("reference library not present")


@pytest.mark.parametrize("name", sorted(CFGS))
def test_predict_and_correct_match_reference(name):
    g, r, cfg = _pair(name)
    dt = 0.5 * r.cfl_dt(0.4)
    hg, hr = g.predict(dt), r.predict(dt)
    assert hg.floor_count == hr.floor_count
    assert _same(hg, hr, ("x_half", "u_half", "vol_half", "e_half", "p_half", "p_mix_half", "q"), cfg.nmat) == []
    # correct from the reference's own HalfStepState, on both
    lg, lr = g.correct(dt, hr), r.correct(dt, hr)
    assert lg.floor_count == lr.floor_count
    assert _same(lg, lr, ("u_half", "u_lag", "e_lag", "vol_lag", "q"), cfg.nmat) == []
    # and correct(predict()) equals lagrange_step on the device
    ll = g.lagrange_step(dt)
    assert _same(ll, lg, ("u_half", "u_lag", "e_lag", "vol_lag", "q"), cfg.nmat) == []


def test_predict_tangled_error_matches_reference():
    g, r, cfg = _pair("gas_wall", umax=4.0)
    errs = []
    for s in (g, r):
        try:
            s.predict(0.5)
            errs.append(None)
        except errors.SimError as e:
            errs.append((type(e).__name__, e.what, e.i, e.j))
    assert errs[0] is not None and errs[0] == errs[1]


@pytest.mark.parametrize("name", sorted(CFGS))
@pytest.mark.parametrize("axis_x", [True, False])
@pytest.mark.parametrize("vel", [True, False])
def test_remap_single_axis_matches_reference(name, axis_x, vel):
    g, r, cfg = _pair(name, seed=11)
    dt = r.cfl_dt(0.3)
    outs = []
    for s in (g, r):
        s.lagrange_step(dt, download=False)
        d = abi.RemapDiag()
        s.remap_single_axis(dt, axis_x, vel, d)
        outs.append((s.download(), (d.max_k_violation, d.k_clip_count, d.mass_fix_count)))
    assert outs[0][1] == outs[1][1]
    assert helpers.bitwise_diff(outs[0][0], outs[1][0], helpers.STATE_FIELDS, cfg.nmat) == []
    assert (outs[0][0].step, outs[0][0].time) == (outs[1][0].step, outs[1][0].time)


def _records(op, n, rng):
    u = lambda lo, hi, *shape: rng.uniform(lo, hi, (n,) + shape)  # noqa: E731
    if op == abi.SC_VAN_LEER:
        r = u(-3, 3, 1)
        r[::7] = 0.0
        r[1::11] = -1.0
        r[2::13] = 1e301
        return r
    if op == abi.SC_LIMITED_GRADIENT:
        a = u(0.1, 10, 3)
        x = np.sort(u(-1, 1, 3), axis=1)
        x[::17, 1] = x[::17, 0]  # zero spacing: the reference throws
        a[3::9, 1] = a[3::9, 0]  # zero difference
        return np.hstack([a, x])
    if op == abi.SC_FACE_VALUE:
        order = rng.integers(1, 3, (n, 1)).astype(float)
        a = u(0.1, 10, 3)
        x = np.sort(u(-1, 1, 3), axis=1)
        return np.hstack([order, a, x, np.sign(u(-1, 1, 1)), u(0.5, 1.5, 1), u(-0.4, 0.4, 1)])
    if op == abi.SC_CORNER_VALUE:
        scheme = rng.integers(0, 5, (n, 1)).astype(float)
        a = u(0.1, 10, 9)
        gx, gy = np.meshgrid(np.arange(-1, 2), np.arange(-1, 2), indexing="ij")
        xlx = gx.ravel()[None, :] * 1.0 + u(-0.2, 0.2, 9)
        xly = gy.ravel()[None, :] * 0.5 + u(-0.1, 0.1, 9)
        kin = np.hstack([u(-0.3, 0.3, 2), u(0.8, 1.2, 2), np.sign(u(-1, 1, 1)), u(-0.3, 0.3, 1),
                         np.sign(u(-1, 1, 1)), u(-0.3, 0.3, 1), u(-0.5, 0.5, 2), np.full((n, 1), 1.0),
                         np.full((n, 1), 0.5)])
        return np.hstack([scheme, a, xlx, xly, kin])
    if op == abi.SC_MULTID_PLANE:
        a = u(0.1, 10, 9)
        gx, gy = np.meshgrid(np.arange(-1, 2), np.arange(-1, 2), indexing="ij")
        xlx = gx.ravel()[None, :] * 0.25 + u(-0.05, 0.05, 9)
        xly = gy.ravel()[None, :] * 0.25 + u(-0.05, 0.05, 9)
        a[::5] = 3.0  # flat stencils: zero gradient
        return np.hstack([a, xlx, xly, np.full((n, 1), 0.25), np.full((n, 1), 0.25)])
    if op in (abi.SC_CLIPPED_FRACTION, abi.SC_PLACE_INTERFACE):
        ang = u(0, 2 * np.pi, 1)
        nrm = np.hstack([np.cos(ang), np.sin(ang)])
        nrm[::9] = [1.0, 0.0]
        if op == abi.SC_CLIPPED_FRACTION:
            return np.hstack([u(0.5, 1.5, 2), nrm, u(-1, 1, 1)])
        lo = u(-0.4, 0.4, 2)
        return np.hstack([u(1e-6, 1 - 1e-6, 1), nrm, lo, lo + u(0.5, 1.5, 2)])
    if op == abi.SC_YOUNGS_NORMAL:
        k = u(0, 1, 9)
        k[::6] = 0.4  # uniform: isolated mixed cell
        return np.hstack([k, np.full((n, 1), 0.1), np.full((n, 1), 0.2)])
    if op == abi.SC_CELL_VOLUME:
        base = np.array([0, 0, 1, 0, 1, 1, 0, 1], float)
        return base[None, :] + u(-0.3, 0.3, 8) * np.where(np.arange(n)[:, None] % 5 == 0, 3.0, 1.0)
    if op == abi.SC_CF_CORNER_FLUX:
        v = u(-2, 2, 2)
        v[::7, 0] = 0.0
        return np.hstack([v, u(0.01, 0.2, 1)])
    if op in (abi.SC_CF_FACE_FLUX_X, abi.SC_CF_FACE_FLUX_Y):
        lo = u(-1, 1, 1)
        return np.hstack([lo, lo + u(0.5, 1.5, 1), u(-0.4, 0.4, 4)])
    if op == abi.SC_PSEUDO_VISCOSITY:
        return np.hstack([u(0.1, 5, 1), u(0.1, 3, 1), u(-2, 1, 1), np.full((n, 1), 0.2), np.full((n, 1), 1.0),
                          u(0.01, 0.1, 1)])
    if op == abi.SC_DIV_U_CELL:
        return np.hstack([u(-1, 1, 8), np.full((n, 1), 0.125), np.full((n, 1), 0.1)])
    if op == abi.SC_GRAD_PQ_NODE:
        return np.hstack([u(0, 5, 8), np.full((n, 1), 0.125), np.full((n, 1), 0.1)])
    if op == abi.SC_AD_FACE_FLUX:  # dy = 0.5, cv = 0.25 (dx = 0.5 exactly)
        return np.hstack([u(-3, 3, 2), np.full((n, 1), 0.4), np.full((n, 1), 0.5), np.full((n, 1), 0.25)])
    raise KeyError(op)


@pytest.mark.parametrize("op", list(range(16)))
def test_scalar_kernels_match_reference(op):
    rng = np.random.Generator(np.random.MT19937(1000 + op))
    rec = _records(op, 4000, rng)
    og, fg = abi.scalar_eval(helpers.product_lib(), op, rec)
    orr, fr = abi.scalar_eval(helpers.ref_lib(), op, rec)
    assert np.array_equal(fg, fr)
    ok = fr == 0
    assert np.array_equal(og[ok].view(np.int64), orr[ok].view(np.int64)), \
        np.argwhere(og[ok].view(np.int64) != orr[ok].view(np.int64))[:5]

"""The reference's own remap tests (proj/tests/test_remap.cpp), restated as
properties of the oracle (CPU) and of the CUDA product (GPU) through the
C-ABI, for the two engines built here (DirectCF, AD).

Each test cites the reference TEST_CASE it restates; the tolerances are the
reference's. They complement the bitwise comparisons (test_gpu_parity.py,
test_oracle_vs_reference.py) with the reference's physical invariants:
identity at rest, free stream, conservation, split == unsplit at first order,
stencil reach, split-order symmetry and the located CFL refusal."""
import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import abi, errors
from paper_2208_13409_b200.abi import (BC_PERIODIC, CORNER_LINEARDIAG, CORNER_UPWIND, EOS_PERFECT, GHOST,
                                       HostState, make_config)

ENGINES = [abi.REMAP_AD, abi.REMAP_DIRECTCF]
G = GHOST


@pytest.fixture(params=[pytest.param("oracle", id="oracle"),
                        pytest.param("product", id="product", marks=pytest.mark.gpu)])
def lib(request):
    return helpers.oracle_lib() if request.param == "oracle" else helpers.product_lib()


def gas(lib, nx, ny, m=None, e=None, u=None, order=2, corner=CORNER_LINEARDIAG, rho=1.0, e0=2.5e5):
    """gas_state of test_remap.cpp:33-43 (unit cells, periodic, gamma 1.4)
    with optional interior m / e arrays and node velocities."""
    cfg = make_config(nx, ny, 1.0, 1.0, 0.0, 0.0, BC_PERIODIC, BC_PERIODIC, eos=[(EOS_PERFECT, 1.4, 0.0)],
                      face_order=order, corner=corner)
    st = HostState.empty(nx, ny, 1, 1.0)
    st.m[0][G:G + ny, G:G + nx] = rho if m is None else m
    st.e[0][G:G + ny, G:G + nx] = e0 if e is None else e
    if u is not None:
        st.u[G:G + ny + 1, G:G + nx + 1] = u
    s = helpers.prepared(lib, cfg, st)
    return s


def remapped(s, kind, x_first=True):
    s.set_lagrange(helpers.kinematic(s.download()))
    s.remap_step(1.0, kind=kind, x_first=x_first)
    return s.download()


def interior(a, nx, ny, node=False):
    return a[G:G + ny + node, G:G + nx + node]


@pytest.mark.parametrize("kind", ENGINES)
def test_zero_velocity_is_identity(lib, kind):
    """test_remap.cpp:160-181: m exact, e to 1e-15."""
    rng = np.random.default_rng(11)
    m, e = rng.uniform(0.5, 2.0, (6, 8)), rng.uniform(0.5, 2.0, (6, 8)) * 1e5
    s = gas(lib, 8, 6, m, e)
    before = s.download()
    s.set_lagrange(helpers.kinematic(before))
    s.remap_step(0.01, kind=kind)
    out = s.download()
    assert np.array_equal(interior(out.m[0], 8, 6), m)
    assert np.allclose(interior(out.e[0], 8, 6), e, rtol=1e-15, atol=0)


@pytest.mark.parametrize("kind", ENGINES)
@pytest.mark.parametrize("order", [1, 2])
def test_free_stream_fixed_point(lib, kind, order):
    """test_remap.cpp:183-206: a uniform state in uniform motion stays put to 1e-12."""
    s = gas(lib, 8, 8, u=np.array([3.0, -2.0]), order=order, rho=1.3, e0=2.1e5)
    s.set_lagrange(helpers.kinematic(s.download()))
    s.remap_step(0.05, kind=kind)
    out = s.download()
    assert np.allclose(interior(out.m[0], 8, 8), 1.3, rtol=1e-12, atol=0)
    assert np.allclose(interior(out.e[0], 8, 8), 2.1e5, rtol=1e-12, atol=0)
    u = interior(out.u, 8, 8, node=True)
    assert np.allclose(u[..., 0], 3.0, rtol=1e-12) and np.allclose(u[..., 1], -2.0, rtol=1e-12)


@pytest.mark.parametrize("kind", ENGINES)
@pytest.mark.parametrize("order", [1, 2])
def test_conservation_periodic(lib, kind, order):
    """test_remap.cpp:233-268: mass and internal energy to 1e-12, momentum to 1e-11."""
    rng = np.random.default_rng(31)
    m, e = rng.uniform(0.5, 2.0, (10, 12)), rng.uniform(0.5, 2.0, (10, 12))
    u = np.zeros((11, 13, 2))
    u[:10, :12] = rng.uniform(-0.2, 0.2, (10, 12, 2))
    u[:, 12] = u[:, 0]
    u[10, :] = u[0, :]
    s = gas(lib, 12, 10, m, e, u, order=order)
    before = s.totals()
    s.set_lagrange(helpers.kinematic(s.download()))
    s.remap_step(1.0, kind=kind)
    after = s.totals()
    assert after["mass"] == pytest.approx(before["mass"], rel=1e-12)
    assert after["internal_energy"] == pytest.approx(before["internal_energy"], rel=1e-12)
    for q in range(2):
        assert after["momentum"][q] == pytest.approx(before["momentum"][q], rel=1e-11, abs=1e-13)


@pytest.mark.parametrize("u", [(0.31, 0.17), (-0.23, 0.29), (-0.19, -0.37)])
def test_first_order_split_equals_corner_flux(lib, u):
    """test_remap.cpp:270-312: order-1 upwind AD == DirectCF to 1e-13, both the
    tensor-product convex combination to 1e-12."""
    rng = np.random.default_rng(57)
    m, e = rng.uniform(0.5, 2.0, (16, 16)), rng.uniform(0.5, 2.0, (16, 16))
    outs = {}
    for kind in ENGINES:
        s = gas(lib, 16, 16, m, e, np.array(u), order=1, corner=CORNER_UPWIND)
        outs[kind] = remapped(s, kind)
    ad, cf = outs[abi.REMAP_AD], outs[abi.REMAP_DIRECTCF]
    d = max(np.abs(interior(ad.m[0], 16, 16) - interior(cf.m[0], 16, 16)).max(),
            np.abs(interior(ad.e[0], 16, 16) - interior(cf.e[0], 16, 16)).max())
    assert d <= 1e-13
    ex, ey = abs(u[0]), abs(u[1])
    sx, sy = (1 if u[0] > 0 else -1), (1 if u[1] > 0 else -1)
    at = lambda di, dj: np.roll(np.roll(m, sy * dj, axis=0), sx * di, axis=1)
    expect = at(0, 0) * (1 - ex) * (1 - ey) + at(1, 0) * ex * (1 - ey) + at(0, 1) * ey * (1 - ex) + at(1, 1) * ex * ey
    assert np.allclose(interior(ad.m[0], 16, 16), expect, rtol=1e-12, atol=0)


@pytest.mark.parametrize("kind", ENGINES)
def test_stencil_reaches_the_diagonal(lib, kind):
    """test_remap.cpp:314-336: a delta moved diagonally feeds the diagonal
    neighbour in one step for the split and corner-flux engines."""
    m = np.ones((7, 7))
    md = m.copy()
    md[3, 3] += 1.0
    outs = [remapped(gas(lib, 7, 7, mm, np.ones((7, 7)), np.array([0.3, 0.3]), order=1, corner=CORNER_UPWIND), kind)
            for mm in (md, m)]
    gain = outs[0].m[0][G + 4, G + 4] - outs[1].m[0][G + 4, G + 4]
    assert gain > 1e-3


def test_split_order_parity_transpose(lib):
    """test_remap.cpp:338-359: on symmetric data with symmetric motion the X-Y
    AD remap equals the transpose of the Y-X remap."""
    rng = np.random.default_rng(7)
    a = rng.uniform(0.5, 2.0, (9, 9))
    m = a + a.T
    out = {}
    for xf in (True, False):
        out[xf] = remapped(gas(lib, 9, 9, m, np.ones((9, 9)) * 2.0, np.array([0.21, 0.21])), abi.REMAP_AD, xf)
    assert np.allclose(interior(out[True].m[0], 9, 9), interior(out[False].m[0], 9, 9).T, rtol=1e-13, atol=0)


@pytest.mark.parametrize("kind", ENGINES)
def test_cfl_refusal_is_located(lib, kind):
    """test_remap.cpp:505-513: a face displacement beyond the CFL fraction
    raises CflViolationError with a location."""
    s = gas(lib, 6, 5, u=np.array([0.95, 0.0]))
    s.set_lagrange(helpers.kinematic(s.download()))
    with pytest.raises(errors.CflViolationError) as ei:
        s.remap_step(1.0, kind=kind)
    assert ei.value.i >= -G and ei.value.j >= -G

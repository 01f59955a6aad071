"""Known-answer tests of the reference (proj/tests/test_harness_io.cpp cfl_dt,
test_lagrange.cpp predict/correct), restated on the oracle (CPU) and the CUDA
product (GPU) through the C-ABI with the reference's tolerances."""
import math

import numpy as np
import pytest

import helpers
from paper_2208_13409_b200.abi import BC_PERIODIC, EOS_PERFECT, EOS_STIFFENED, GHOST, HostState, make_config

G = GHOST


@pytest.fixture(params=[pytest.param("oracle", id="oracle"),
                        pytest.param("product", id="product", marks=pytest.mark.gpu)])
def lib(request):
    return helpers.oracle_lib() if request.param == "oracle" else helpers.product_lib()


def air(lib, nx, ny, dx, rho, e, u=(0.0, 0.0)):
    """gas_state of test_lagrange.cpp:26-36 / test_harness_io.cpp:14-24 (periodic)."""
    cfg = make_config(nx, ny, dx, dx, 0.0, 0.0, BC_PERIODIC, BC_PERIODIC, eos=[(EOS_PERFECT, 1.4, 0.0)])
    st = HostState.empty(nx, ny, 1, dx * dx)
    st.m[0][G:G + ny, G:G + nx] = rho * dx * dx
    st.e[0][G:G + ny, G:G + nx] = e
    st.u[G:G + ny + 1, G:G + nx + 1] = u
    return helpers.prepared(lib, cfg, st)


def test_cfl_dt_at_rest(lib):
    """test_harness_io.cpp:25-29: dt = 0.3 dx / c with c = sqrt(1.4e5)."""
    s = air(lib, 8, 8, 0.01, 1.0, 2.5e5)
    dt = s.cfl_dt(0.3)
    assert dt == pytest.approx(0.3 * 0.01 / math.sqrt(1.4e5), rel=1e-13)
    assert dt == pytest.approx(8.0178e-6, rel=1e-4)
    assert s.cfl_dt(0.6) == pytest.approx(2.0 * s.cfl_dt(0.3), rel=1e-14)


def test_cfl_dt_fastest_cell_wins(lib):
    """test_harness_io.cpp:33-56: one stiffened (water) cell sets the step."""
    cfg = make_config(8, 8, 0.01, 0.01, 0.0, 0.0, BC_PERIODIC, BC_PERIODIC,
                      eos=[(EOS_PERFECT, 1.4, 0.0), (EOS_STIFFENED, 7.0, 2.1e9)])
    cv = 1e-4
    st = HostState.empty(8, 8, 2, cv)
    I = (slice(G, G + 8), slice(G, G + 8))
    st.k[0][I], st.k[1][I] = 1.0, 0.0
    st.m[0][I], st.e[0][I] = cv, 2.5e5
    c = (G + 4, G + 4)
    st.k[0][c], st.k[1][c], st.m[0][c] = 0.0, 1.0, 0.0
    st.m[1][c], st.e[1][c] = 1000.0 * cv, (1e5 + 2.1e9) / 6000.0
    s = helpers.prepared(lib, cfg, st)
    c_water = math.sqrt(7.0 * (1e5 + 2.1e9) / 1000.0)
    assert s.cfl_dt(0.3) == pytest.approx(0.3 * 0.01 / c_water, rel=1e-12)


def test_equilibrium_is_a_fixed_point(lib):
    """test_lagrange.cpp:98-118: at rest, u_half = u_lag = 0 and e_lag = e to 1e-13."""
    s = air(lib, 6, 6, 1.0, 1.0, 2.5e5)
    lag = s.lagrange_step(1e-4)
    assert np.allclose(lag.u_half[G:G + 7, G:G + 7], 0.0, atol=1e-13)
    assert np.allclose(lag.u_lag[G:G + 7, G:G + 7], 0.0, atol=1e-13)
    assert np.allclose(lag.e_lag[0][G:G + 6, G:G + 6], 2.5e5, rtol=1e-13)
    assert np.allclose(lag.vol_lag[G:G + 6, G:G + 6], 1.0, rtol=1e-13)


def test_uniform_flow_translates(lib):
    """test_lagrange.cpp:120-136: uniform (5, 5) motion, thermodynamics frozen."""
    s = air(lib, 6, 6, 1.0, 1.0, 2.5e5, u=(5.0, 5.0))
    lag = s.lagrange_step(1e-3)
    assert np.allclose(lag.e_lag[0][G:G + 6, G:G + 6], 2.5e5, rtol=1e-13)
    assert np.allclose(lag.u_lag[G:G + 7, G:G + 7], 5.0, rtol=1e-13)
    assert np.allclose(lag.vol_lag[G:G + 6, G:G + 6], 1.0, rtol=1e-13)

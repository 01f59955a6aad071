"""Edge cases: the smallest meshes the reference accepts (3x3, mesh.hpp:27),
ragged tile remainders, rejected meshes, and a mesh too large for the
device's 32-bit plane offsets."""
import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import abi, errors
from paper_2208_13409_b200.abi import BC_PERIODIC, BC_WALL, EOS_PERFECT, make_config

SIZES = [(3, 3), (3, 4), (4, 3), (5, 3), (3, 7), (33, 9), (35, 17)]


@pytest.mark.ref
@pytest.mark.parametrize("nx,ny", SIZES[:5])
@pytest.mark.parametrize("bc", [BC_WALL, BC_PERIODIC])
@pytest.mark.parametrize("kind", ["gas", "front"])
def test_minimal_meshes_oracle_vs_reference(ref, orc, nx, ny, bc, kind):
    cfg = make_config(nx, ny, 0.1, 0.1, 0.0, 0.0, bc, bc, eos=[(EOS_PERFECT, 1.4, 0.0)] * (1 if kind == "gas" else 2))
    painted = helpers.random_state(cfg, 5, kind, umax=0.05)
    out = []
    for lib in (ref, orc):
        s = helpers.prepared(lib, cfg, painted)
        r, e = helpers.run_capture(s, 6, 0.3)
        out.append((r.steps_done, e, s.download()))
    assert out[0][:2] == out[1][:2]
    assert helpers.bitwise_diff(out[0][2], out[1][2], helpers.STATE_FIELDS) == []


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny", SIZES)
@pytest.mark.parametrize("bc", [BC_WALL, BC_PERIODIC])
@pytest.mark.parametrize("kind", ["gas", "front"])
@pytest.mark.parametrize("remap", [abi.REMAP_DIRECTCF, abi.REMAP_AD])
def test_small_and_ragged_meshes_device(gpu, orc, nx, ny, bc, kind, remap):
    cfg = make_config(nx, ny, 0.1, 0.1, 0.0, 0.0, bc, bc, eos=[(EOS_PERFECT, 1.4, 0.0)] * (1 if kind == "gas" else 2))
    painted = helpers.random_state(cfg, 5, kind, umax=0.05)
    out = []
    for lib in (gpu, orc):
        s = helpers.prepared(lib, cfg, painted)
        r, e = helpers.run_capture(s, 6, 0.3, remap)
        out.append((r.steps_done, e, s.download(), r.dts))
    assert out[0][:2] == out[1][:2] and np.array_equal(out[0][3], out[1][3])
    assert helpers.bitwise_diff(out[0][2], out[1][2], helpers.STATE_FIELDS) == []


@pytest.mark.parametrize("nx,ny", [(2, 5), (5, 2), (0, 4)])
def test_rejects_meshes_below_3x3(orc, nx, ny):
    """Mesh(nx, ny, ...) throws "mesh must be at least 3x3" (mesh.hpp:27)."""
    cfg = make_config(nx, ny, 0.1, 0.1)
    with pytest.raises(errors.SimError):
        abi.Solver(orc, cfg)


@pytest.mark.gpu
def test_device_rejects_oversized_plane(gpu):
    """P * R >= 2^31 doubles per plane cannot be indexed with the device's
    32-bit offsets: h2d_create refuses instead of overflowing."""
    cfg = make_config(50000, 50000, 1e-5, 1e-5)
    with pytest.raises(errors.DeviceError) as ei:
        abi.Solver(gpu, cfg)
    assert ei.value.code == errors.H2D_ERR_INVALID

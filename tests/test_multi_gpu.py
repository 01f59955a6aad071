"""2D block decomposition on ONE GPU: P blocks run the step with their halos
and one exchange + one scalar all-reduce per step (LocalTransport). The
assembled owned regions must be bit-identical to the single-domain run — the
property that makes the 8-GPU path exact."""
import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import cases, errors, multi
from paper_2208_13409_b200.abi import HostState

pytestmark = pytest.mark.gpu


def _single(case, steps):
    s = helpers.prepared(helpers.product_lib(), case.cfg, case.paint())
    r, err = helpers.run_capture(s, steps, case.cfl)
    return s.download(), r, err


def _blocks(case, steps, px, py):
    lib = helpers.product_lib()
    init = helpers.prepared(lib, case.cfg, case.paint()).download()
    specs = multi.decompose(case.cfg.mesh.nx, case.cfg.mesh.ny, px, py)
    blocks = [multi.BlockSolver(lib, case.cfg, sp) for sp in specs]
    for b in blocks:
        b.upload(init)
    tr = multi.LocalTransport(blocks, px, py)
    multi.run_blocks(blocks, tr, steps, 1e30, case.cfl)
    out = HostState.empty(case.cfg.mesh.nx, case.cfg.mesh.ny, case.cfg.nmat)
    results = []
    for b in blocks:
        b.download_into(out)
        results.append(b.result(steps))
    return out, results


@pytest.mark.parametrize("px,py", [(2, 1), (1, 2), (2, 2), (4, 2)])
@pytest.mark.parametrize("which", ["riemann", "triple", "bubble", "voronoi3"])
def test_blocks_bitwise_equal_single_domain(which, px, py):
    case = {"riemann": cases.riemann2d(64), "triple": cases.triple_point(96, 48),
            "bubble": cases.shock_bubble(64), "voronoi3": cases.voronoi3(128)}[which]
    steps = 40
    ref, r, err = _single(case, steps)
    got, results = _blocks(case, steps, px, py)
    assert err is None
    for a, dts, e in results:
        assert e is None
        assert a.steps_done == r.steps_done
        assert np.array_equal(dts, r.dts)
    assert sum(a.diag.k_clip_count for a, _, _ in results) == r.diag["k_clip_count"]
    assert sum(a.diag.mass_fix_count for a, _, _ in results) == r.diag["mass_fix_count"]
    assert sum(a.floor_count for a, _, _ in results) == r.floor_count
    assert helpers.bitwise_diff(got, ref, helpers.STATE_FIELDS) == []
    assert (got.step, got.time) == (ref.step, ref.time)


def test_blocks_reproduce_the_reference_abort():
    """triple point 32x16 aborts (UnphysicalStateError at step 79 on the
    reference): the decomposition raises the same error at the same step and
    keeps the State of the last completed step."""
    case = cases.triple_point(32, 16)
    ref, r, err = _single(case, 1000)
    assert err is not None
    got, results = _blocks(case, 1000, 2, 2)
    for a, dts, e in results:
        assert (type(e).__name__, e.what, e.i, e.j) == err[:4]
        assert a.steps_done == r.steps_done
    assert helpers.bitwise_diff(got, ref, helpers.STATE_FIELDS) == []


def test_halo_plan_matches_library():
    case = cases.riemann2d(64)
    lib = helpers.product_lib()
    for sp in multi.decompose(64, 64, 2, 2):
        b = multi.BlockSolver(lib, case.cfg, sp)
        nc, nn = multi.state_planes(1)
        for dx, dy in multi.DIRS:
            for pack in (1, 0):
                rc, rn = multi.halo_rects(sp, 64, 64, dx, dy, bool(pack))
                want = ((rc[1] - rc[0]) * (rc[3] - rc[2]) * nc + (rn[1] - rn[0]) * (rn[3] - rn[2]) * nn) * 8
                assert b.halo_bytes(dx, dy, pack) == want

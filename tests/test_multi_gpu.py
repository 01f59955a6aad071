"""2D block decomposition on ONE GPU: P blocks run the step with their halos
and one exchange + one scalar all-reduce per step (LocalTransport). The
assembled owned regions must be bit-identical to the single-domain run — the
property that makes the 8-GPU path exact."""
import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import abi, cases, errors, multi
from paper_2208_13409_b200.abi import HostState

pytestmark = pytest.mark.gpu


def _single(case, steps, kind=abi.REMAP_DIRECTCF):
    s = helpers.prepared(helpers.product_lib(), case.cfg, case.paint())
    r, err = helpers.run_capture(s, steps, case.cfl, kind=kind)
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


# ---- the library's data plane (h2d_comm + h2d_blocks_run) -------------------
def _blocks_device(case, steps, px, py, kind=abi.REMAP_DIRECTCF):
    """The whole decomposed run loop inside the library: per step every
    block's graph, one max all-reduce of the four control words and one
    halo exchange enqueued on the device (in-process transport: every
    block on this GPU), the host polling every 16 steps."""
    lib = helpers.product_lib()
    init = helpers.prepared(lib, case.cfg, case.paint()).download()
    specs = multi.decompose(case.cfg.mesh.nx, case.cfg.mesh.ny, px, py)
    blocks = [multi.BlockSolver(lib, case.cfg, sp) for sp in specs]
    for b in blocks:
        b.upload(init)
    comm = multi.DeviceComm(blocks, px, py)
    comm.run(steps, 1e30, case.cfl, kind=kind)
    comm.close()
    out = HostState.empty(case.cfg.mesh.nx, case.cfg.mesh.ny, case.cfg.nmat)
    results = []
    for b in blocks:
        b.download_into(out)
        results.append(b.result(steps))
    return out, results


# ---- the AD split remap in block mode (the split remap
# needs a second halo exchange per step, between its two passes) --------------
@pytest.mark.parametrize("px,py", [(2, 1), (1, 2), (2, 2), (4, 2)])
@pytest.mark.parametrize("which", ["riemann", "sedov", "triple", "bubble"])
def test_ad_blocks_bitwise_equal_single_domain(which, px, py):
    case = {"riemann": cases.riemann2d(64), "sedov": cases.sedov(64), "triple": cases.triple_point(96, 48),
            "bubble": cases.shock_bubble(64)}[which]
    steps = 41  # odd: both axis orders end a run
    ref, r, err = _single(case, steps, abi.REMAP_AD)
    got, results = _blocks_device(case, steps, px, py, abi.REMAP_AD)
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


def test_ad_blocks_reproduce_the_reference_abort():
    """the AD run of the 64x32 triple point at CFL 1.15 aborts at step 101
    (a tangled cell in one block; the AD run is stable at the case's own
    CFL): the decomposition raises the same error at the same step, every
    block stops there and keeps the last completed State."""
    case = cases.triple_point(64, 32)
    case.cfl = 1.15
    ref, r, err = _single(case, 300, abi.REMAP_AD)
    assert err is not None and r.steps_done == 101
    got, results = _blocks_device(case, 300, 2, 2, abi.REMAP_AD)
    for a, dts, e in results:
        assert (type(e).__name__, e.what, e.i, e.j) == err[:4]
        assert a.steps_done == r.steps_done
        assert np.array_equal(dts[:r.steps_done], r.dts[:r.steps_done])
    assert helpers.bitwise_diff(got, ref, helpers.STATE_FIELDS) == []


def test_ad_blocks_refuse_three_materials():
    case = cases.voronoi3(64)
    lib = helpers.product_lib()
    init = helpers.prepared(lib, case.cfg, case.paint()).download()
    blocks = [multi.BlockSolver(lib, case.cfg, sp) for sp in multi.decompose(64, 64, 2, 1)]
    for b in blocks:
        b.upload(init)
    comm = multi.DeviceComm(blocks, 2, 1)
    with pytest.raises(errors.DeviceError):
        comm.run(5, 1e30, case.cfl, kind=abi.REMAP_AD)
    comm.close()


def test_blocks_refuse_the_direct_engine():
    """block mode runs DirectCF and AD; the faces-only Direct engine is single-domain only."""
    case = cases.riemann2d(64)
    lib = helpers.product_lib()
    init = helpers.prepared(lib, case.cfg, case.paint()).download()
    blocks = [multi.BlockSolver(lib, case.cfg, sp) for sp in multi.decompose(64, 64, 2, 1)]
    for b in blocks:
        b.upload(init)
    comm = multi.DeviceComm(blocks, 2, 1)
    with pytest.raises(errors.DeviceError):
        comm.run(5, 1e30, case.cfl, kind=abi.REMAP_DIRECT)
    comm.close()


@pytest.mark.parametrize("px,py", [(2, 1), (1, 2), (2, 2), (4, 2)])
@pytest.mark.parametrize("which", ["riemann", "triple", "bubble", "voronoi3"])
def test_device_data_plane_bitwise_equal_single_domain(which, px, py):
    case = {"riemann": cases.riemann2d(64), "triple": cases.triple_point(96, 48),
            "bubble": cases.shock_bubble(64), "voronoi3": cases.voronoi3(128)}[which]
    steps = 40
    ref, r, err = _single(case, steps)
    got, results = _blocks_device(case, steps, px, py)
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


def test_device_data_plane_reproduces_the_reference_abort():
    """the device-side combine rolls back the blocks that committed when the
    first error (any block) precedes the commit: same error, same State."""
    case = cases.triple_point(32, 16)
    ref, r, err = _single(case, 1000)
    assert err is not None
    got, results = _blocks_device(case, 1000, 2, 2)
    for a, dts, e in results:
        assert (type(e).__name__, e.what, e.i, e.j) == err[:4]
        assert a.steps_done == r.steps_done
    assert helpers.bitwise_diff(got, ref, helpers.STATE_FIELDS) == []


def test_device_data_plane_until_t_end():
    """a run to t_end (max_steps = 0): the last dt is clipped to t_end and
    every block stops at the same step."""
    case = cases.sedov(64)
    lib = helpers.product_lib()
    s = helpers.prepared(lib, case.cfg, case.paint())
    t_end = 0.002
    r = s.run(0, t_end=t_end, cfl=case.cfl)
    ref = s.download()
    init = helpers.prepared(lib, case.cfg, case.paint()).download()
    specs = multi.decompose(64, 64, 2, 2)
    blocks = [multi.BlockSolver(lib, case.cfg, sp) for sp in specs]
    for b in blocks:
        b.upload(init)
    comm = multi.DeviceComm(blocks, 2, 2)
    comm.run(0, t_end, case.cfl)
    comm.close()
    got = HostState.empty(64, 64, 1)
    for b in blocks:
        b.download_into(got)
        a, dts, e = b.result(r.steps_done + 1)
        assert e is None and np.array_equal(dts, r.dts)
    assert helpers.bitwise_diff(got, ref, helpers.STATE_FIELDS, 1) == []


def test_nccl_transport_single_rank():
    """The NCCL transport with a one-rank communicator owned by the library
    (1 x 1 decomposition: the all-reduce runs, no neighbours): equal to the
    single domain. Two or more ranks need two or more GPUs (bench.py --gpus)."""
    case = cases.triple_point(64, 32)
    steps = 30
    ref, r, err = _single(case, steps)
    lib = helpers.product_lib()
    init = helpers.prepared(lib, case.cfg, case.paint()).download()
    spec = multi.decompose(64, 32, 1, 1)[0]
    blk = multi.BlockSolver(lib, case.cfg, spec)
    blk.upload(init)
    uid = multi.DeviceComm.unique_id(lib)
    comm = multi.DeviceComm([blk], 1, 1, nccl_id=uid, rank=0)
    comm.run(steps, 1e30, case.cfl)
    comm.close()
    got = HostState.empty(64, 32, 2)
    blk.download_into(got)
    a, dts, e = blk.result(steps)
    assert e is None and np.array_equal(dts, r.dts)
    assert helpers.bitwise_diff(got, ref, helpers.STATE_FIELDS) == []


@pytest.mark.parametrize("px,py", [(2, 1), (2, 2), (4, 2)])
@pytest.mark.parametrize("which", ["triple", "bubble", "voronoi3"])
def test_window_init_blocks_equal_single_domain(which, px, py):
    """Per-rank painting: every block paints and initialises only its own
    window (h2d_block_init_window: fill_ghosts at the global walls,
    sync_derived, interface normals on the window; the first exchange makes
    the halo exact), no global host State; the run equals the single
    domain's bit for bit."""
    case = {"triple": cases.triple_point(96, 48), "bubble": cases.shock_bubble(64),
            "voronoi3": cases.voronoi3(128)}[which]
    steps = 25
    ref, r, err = _single(case, steps)
    lib = helpers.product_lib()
    specs = multi.decompose(case.cfg.mesh.nx, case.cfg.mesh.ny, px, py)
    blocks = [multi.BlockSolver(lib, case.cfg, sp) for sp in specs]
    for b in blocks:
        b.init_window(case.paint(b.window()))
    comm = multi.DeviceComm(blocks, px, py)
    comm.run(steps, 1e30, case.cfl)
    comm.close()
    got = HostState.empty(case.cfg.mesh.nx, case.cfg.mesh.ny, case.cfg.nmat)
    for b in blocks:
        b.download_into(got)
        a, dts, e = b.result(steps)
        assert e is None and np.array_equal(dts, r.dts)
    assert helpers.bitwise_diff(got, ref, helpers.STATE_FIELDS) == []


def test_comm_trace_shows_the_exchange_beside_the_owned_tiles():
    """h2d_comm_trace: per step and block nine stream timestamps; the State
    halo exchange enqueued after step s starts no later than step s + 1's
    owned Lagrange tiles end (it runs beside them, on its own stream), and the
    edge tiles end after it."""
    case = cases.shock_bubble(256)
    lib = helpers.product_lib()
    specs = multi.decompose(256, 256, 2, 1)
    blocks = [multi.BlockSolver(lib, case.cfg, sp) for sp in specs]
    for b in blocks:
        b.init_window(case.paint(b.window()))
    comm = multi.DeviceComm(blocks, 2, 1)
    comm.run(3, 1e30, case.cfl)
    comm.trace(5)
    comm.run(8, 1e30, case.cfl)
    tr = comm.trace_read()
    comm.close()
    P = {k: q for q, k in enumerate(multi.DeviceComm.TRACE_POINTS)}
    assert tr.shape == (5, 2, len(P))
    assert (tr[:, :, P["ad_mid_start"]] == -1.0).all()  # DirectCF: no mid exchange
    for s in range(1, 5):
        for b in range(2):
            r, prev = tr[s, b], tr[s - 1, b]
            assert r[P["lag_owned_start"]] <= r[P["lag_owned_end"]] <= r[P["lag_edge_end"]] <= r[P["rest_end"]]
            assert prev[P["halo_start"]] <= prev[P["halo_end"]] <= r[P["lag_edge_end"]]
            assert prev[P["halo_start"]] <= r[P["lag_owned_end"]]

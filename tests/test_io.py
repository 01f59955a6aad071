"""Field readback formats and checkpoints.

write_fields (io.hpp:17, io.cpp:15-83) and append_diag_line (io.cpp:85-92)
must produce the reference's bytes; the binary checkpoint must restart a run
bit-exactly."""
import ctypes as C
import os

import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import abi, cases, errors
from paper_2208_13409_b200.abi import DUMP_CSV, DUMP_VTK, HostState


def _ref_state(ref, case, steps):
    s = helpers.prepared(ref, case.cfg, case.paint())
    if steps:
        s.run(steps, cfl=case.cfl)
    return s


def _read(path):
    with open(path, "rb") as f:
        return f.read()


# ---- CPU ----------------------------------------------------------------------------

@pytest.mark.ref
@pytest.mark.parametrize("fmt", [DUMP_CSV, DUMP_VTK])
@pytest.mark.parametrize("which,steps", [("riemann", 8), ("triple", 12)])
def test_write_fields_host_matches_reference(ref, tmp_path, fmt, which, steps):
    case = {"riemann": cases.riemann2d(24), "triple": cases.triple_point(32, 16)}[which]
    sr = _ref_state(ref, case, steps)
    want = tmp_path / "ref.out"
    sr._check(ref.fn["write_fields"](sr._h, str(want).encode(), fmt))
    st = sr.download()
    got = tmp_path / "b200.out"
    prod = helpers.product_lib()
    v = st.view(derived=True)
    rc = prod.fn["write_fields_host"](C.byref(case.cfg), C.byref(v), str(got).encode(), fmt)
    assert rc == 0
    assert _read(got) == _read(want)


@pytest.mark.ref
def test_diag_line_matches_reference(ref, orc):
    case = cases.shock_bubble(32)
    so = helpers.prepared(orc, case.cfg, case.paint())
    r = so.run(6, cfl=case.cfl, series=True)
    prod = helpers.product_lib()
    for rec in list(r.series) + [so.step_diag(0.0)]:
        assert abi.diag_line(prod, rec) == abi.diag_line(ref, rec)


def test_write_fields_rejects_bad_path_and_format(tmp_path):
    case = cases.riemann2d(8)
    st = case.paint()
    prod = helpers.product_lib()
    v = st.view(derived=True)
    assert prod.fn["write_fields_host"](C.byref(case.cfg), C.byref(v), str(tmp_path / "x").encode(), 7) == \
        errors.H2D_ERR_INVALID
    assert prod.fn["write_fields_host"](C.byref(case.cfg), C.byref(v), b"/nonexistent/dir/f.csv", DUMP_CSV) == \
        errors.H2D_ERR_SIM


def test_checkpoint_host_round_trip(orc, tmp_path):
    case = cases.triple_point(32, 16)
    so = helpers.prepared(orc, case.cfg, case.paint())
    so.run(5, cfl=case.cfl)
    st = so.download()
    prod = helpers.product_lib()
    path = str(tmp_path / "s.h2d").encode()
    assert prod.fn["save_state_host"](C.byref(case.cfg), C.byref(st.view(derived=True)), path) == 0
    back = HostState.empty(case.cfg.mesh.nx, case.cfg.mesh.ny, case.cfg.nmat)
    v = back.view(derived=True)
    assert prod.fn["load_state_host"](C.byref(case.cfg), C.byref(v), path) == 0
    back.step, back.time = v.step, v.time
    assert helpers.bitwise_diff(back, st, helpers.STATE_FIELDS) == []
    assert (back.step, back.time) == (st.step, st.time)
    other = cases.triple_point(16, 16).cfg
    v2 = HostState.empty(16, 16, 2).view(derived=True)
    assert prod.fn["load_state_host"](C.byref(other), C.byref(v2), path) == errors.H2D_ERR_INVALID


# ---- GPU ----------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("fmt", [DUMP_CSV, DUMP_VTK])
def test_device_write_fields_matches_reference_writer(gpu, orc, tmp_path, fmt):
    """The device State after K steps, dumped by the product, is the text the
    reference writer produces for the same State (the oracle's, bit-identical)."""
    case = cases.triple_point(48, 24)
    sg = helpers.prepared(gpu, case.cfg, case.paint())
    so = helpers.prepared(orc, case.cfg, case.paint())
    sg.run(10, cfl=case.cfl)  # (this small triple point aborts at step 13, like the reference)
    so.run(10, cfl=case.cfl)
    got = tmp_path / "dev.out"
    sg.write_fields(str(got), fmt)
    ref = helpers.ref_lib()
    want = tmp_path / "ref.out"
    if ref is not None:  # the reference writer on the oracle's State
        sr = helpers.prepared(ref, case.cfg, case.paint())
        sr.upload(so.download())
        sr._check(ref.fn["write_fields"](sr._h, str(want).encode(), fmt))
    else:  # the host formatter (pinned to the reference on CPU) on the oracle's State
        v = so.download().view(derived=True)
        assert gpu.fn["write_fields_host"](C.byref(case.cfg), C.byref(v), str(want).encode(), fmt) == 0
    assert _read(got) == _read(want)


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["sedov", "bubble"])
def test_checkpoint_restart_is_bit_exact(gpu, tmp_path, which):
    case = {"sedov": cases.sedov(64), "bubble": cases.shock_bubble(48)}[which]
    a = helpers.prepared(gpu, case.cfg, case.paint())
    a.run(10, cfl=case.cfl)
    path = str(tmp_path / "ck.h2d")
    a.save_state(path)
    ra = a.run(25, cfl=case.cfl)
    b = abi.Solver(gpu, case.cfg)
    b.load_state(path)
    rb = b.run(25, cfl=case.cfl)
    assert np.array_equal(ra.dts, rb.dts)
    sa, sb = a.download(), b.download()
    assert helpers.bitwise_diff(sa, sb, helpers.STATE_FIELDS) == []
    assert (sa.step, sa.time) == (sb.step, sb.time)
    with pytest.raises(errors.SimError):
        b.write_fields("/nonexistent/dir/x.csv")


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["sedov", "triple"])
def test_upload_primary_fields_rebuilds_derived_bitwise(gpu, orc, which):
    """h2d_upload_state with the derived pointers NULL (the e2e bench's
    upload) rebuilds vol, m_mix, e_mix, rho_mix, p_mix exactly as the
    reference State carries them (sync_derived, state.cpp:120-143)."""
    case = {"sedov": cases.sedov(64), "triple": cases.triple_point(64, 32)}[which]
    so = helpers.prepared(orc, case.cfg, case.paint())
    so.run(8, cfl=case.cfl)
    st = so.download()
    a, b = abi.Solver(gpu, case.cfg), abi.Solver(gpu, case.cfg)
    a.upload(st, derived=True)
    b.upload(st, derived=False)
    assert helpers.bitwise_diff(a.download(), b.download(), helpers.STATE_FIELDS) == []
    ra, rb = a.run(14, cfl=case.cfl), b.run(14, cfl=case.cfl)
    assert np.array_equal(ra.dts, rb.dts)
    assert helpers.bitwise_diff(a.download(), b.download(), helpers.STATE_FIELDS) == []

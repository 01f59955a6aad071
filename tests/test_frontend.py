"""Front ends over the device path: the case catalogue,
the run configuration, run() / run_case and the CLI, against the reference's
own driver (harness.cpp:22-163,226-424, config.cpp, bindings/module.cpp:50-93)
run through oracle/_ref (h2dr_run_case)."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

import helpers
from paper_2208_13409_b200 import abi, cases, errors, frontend
from paper_2208_13409_b200.abi import STEP_DIAG_DTYPE, HostState, StepDiag

EXACT = ("step", "t", "dt", "min_rho", "max_rho", "min_p", "max_p")
SUMS = ("mass", "momentum_x", "momentum_y", "internal_energy")

# (case, divisor, max_steps override) small enough for the reference on one core
CATALOGUE_RUNS = [("uniform", 2, 0), ("mono_advect", 4, 0), ("multimat_advect", 4, 0),
                  ("mono_rotation", 5, 120), ("water_air_rotation", 8, 120), ("haas", 8, 0),
                  ("impact", 4, 40)]


def ref_run_case(ref, name, divisor, scheme="DirectCF", face_order=2, corner="linear_diag", cfl=0.3,
                 t_end=-1.0, max_steps=0):
    f = ref.dll.h2dr_run_case
    f.restype = C.c_int
    cs = frontend.build_case(name, divisor)
    cap = 200000
    series = np.zeros(cap, STEP_DIAG_DTYPE)
    n, steps = C.c_int(), C.c_int()
    out = (C.c_double * 8)()
    fin = HostState.empty(cs.nx, cs.ny, cs.nmat)
    v = fin.view(derived=True)
    what = C.create_string_buffer(256)
    rc = f(name.encode(), divisor, frontend.SCHEMES[scheme], face_order, frontend.CORNERS[corner],
           C.c_double(cfl), C.c_double(t_end), max_steps, series.ctypes.data_as(C.POINTER(StepDiag)), cap,
           C.byref(n), out, C.byref(steps), C.byref(v), what, 256)
    fin.step, fin.time = v.step, v.time
    return rc, what.value.decode(), series[:n.value], list(out), steps.value, fin


# ---- CPU ----------------------------------------------------------------------------

def test_case_list_has_the_reference_catalogue():
    names = frontend.case_list()
    for n in ("uniform", "mono_advect", "mono_rotation", "multimat_advect", "water_air_rotation", "haas", "impact"):
        assert n in names
    with pytest.raises(errors.SimError, match="unknown case: nope"):
        frontend.build_case("nope")


def test_parse_config():
    rc = frontend.parse_config("# comment\ncase = haas  # trailing\nscheme = AD\nface_order = 1\n"
                               "corner_scheme = upwind\ncfl = 0.25\ndivisor = 4\nt_end = 1e-4\n"
                               "max_steps = 7\nout_dir = /tmp/x\noutput_every = 3\nseed = 5\n")
    assert (rc.case_name, rc.scheme, rc.face_order, rc.corner, rc.cfl, rc.divisor, rc.t_end, rc.max_steps,
            rc.out_dir, rc.output_every, rc.seed) == ("haas", abi.REMAP_AD, 1, abi.CORNER_UPWIND, 0.25, 4,
                                                       1e-4, 7, "/tmp/x", 3, 5)
    cs = frontend.configure_case(rc)
    assert (cs.nx, cs.ny, cs.t_end, cs.max_steps, cs.cfl, cs.face_order) == (250, 22, 1e-4, 7, 0.25, 1)
    for text, msg in [("case haas", "config line 1: expected 'key = value'"),
                      ("x = 1", "config line 1: unknown key 'x'"),
                      ("\nface_order = 3", "config line 2: face_order must be 1 or 2"),
                      ("scheme = Foo", "config line 1: invalid scheme 'Foo' (valid: AD, Direct, DirectCF)"),
                      ("cfl = abc", "config line 1: not a number: 'abc'")]:
        with pytest.raises(errors.SimError) as e:
            frontend.parse_config(text)
        assert str(e.value) == msg
    with pytest.raises(errors.SimError, match="config is missing 'case'"):
        frontend.configure_case(frontend.parse_config("cfl = 0.3"))


@pytest.mark.ref
@pytest.mark.parametrize("name", ["uniform", "mono_advect", "mono_rotation", "multimat_advect",
                                  "water_air_rotation", "haas", "impact"])
def test_catalogue_paint_equals_reference_init_case(ref, name):
    """The catalogue's regions painted by cases.paint are the reference
    init_case's interior (the painter is pinned in test_oracle_vs_reference)."""
    cs = frontend.build_case(name, 4)
    cfg = cs.config()
    ours = cases.paint(cfg, cs.regions)
    sr = abi.Solver(ref, cfg)
    rows = np.array([r.row() for r in cs.regions], dtype=np.float64)
    out = HostState.empty(cs.nx, cs.ny, cs.nmat)
    v = out.view(derived=False)
    f = ref.dll.h2dr_init_regions
    f.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int, C.POINTER(abi.StateView)]
    assert f(sr._h, rows.ctypes.data_as(C.POINTER(C.c_double)), len(cs.regions), C.byref(v)) == 0
    for fld in ("m", "e", "k"):
        a, b = getattr(ours, fld)[:cs.nmat], getattr(out, fld)[:cs.nmat]
        g = abi.GHOST
        assert np.array_equal(a[:, g:g + cs.ny, g:g + cs.nx], b[:, g:g + cs.ny, g:g + cs.nx]), fld


# ---- GPU ----------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name,divisor,max_steps", CATALOGUE_RUNS)
def test_run_case_matches_reference_run(name, divisor, max_steps):
    ref = helpers.ref_lib()
    if ref is None:
        pytest.skip("reference library not built")
    rc, what, want, out, steps, fin = ref_run_case(ref, name, divisor, max_steps=max_steps)
    cs = frontend.build_case(name, divisor)
    if max_steps:
        cs.max_steps = max_steps
    if rc:
        with pytest.raises(errors.SimError) as e:
            frontend.run(cs)
        assert str(e.value) == what
        return
    rep = frontend.run(cs)
    assert rep.steps == steps
    assert len(rep.series) == len(want)
    for f in EXACT:
        assert np.array_equal(rep.series[f], want[f]), f
    scale = np.abs(want["mass"]).max()
    for f in SUMS:
        assert np.allclose(rep.series[f], want[f], rtol=1e-12, atol=1e-12 * scale), f
    assert helpers.bitwise_diff(rep.final_state, fin, helpers.STATE_FIELDS, cs.nmat) == []
    assert rep.final_state.time == out[0]
    assert (rep.l2_rho_vs_initial, rep.l2_k_vs_initial, rep.max_k_violation) == (out[1], out[2], out[3])
    assert (rep.k_clip_count, rep.mass_fix_count, rep.energy_floor_count) == tuple(int(x) for x in out[4:7])


@pytest.mark.gpu
@pytest.mark.parametrize("name,divisor", [("riemann2d", 8), ("triple_point", 32), ("shock_bubble", 128)])
def test_run_baseline_configs_equal_oracle_loop(orc, name, divisor):
    """The BASELINE.json configs (not in the reference catalogue) through
    run(): the same steps as the oracle's run loop on the same painted State."""
    cs = frontend.build_case(name, divisor)
    cs.max_steps = 25
    rep = frontend.run(cs)
    so = helpers.prepared(orc, cs.config(), cases.paint(cs.config(), cs.regions))
    r, err = helpers.run_capture(so, 25, cs.cfl)
    assert err is None and rep.steps == r.steps_done == 25
    assert np.array_equal(rep.series["dt"][1:], r.dts)  # series[0] = make_diag(initial, 0.0)
    assert helpers.bitwise_diff(rep.final_state, so.download(), helpers.STATE_FIELDS, cs.nmat) == []


@pytest.mark.gpu
def test_run_case_dict_and_hook():
    d = frontend.run_case("haas", divisor=8)
    for k in ("case", "scheme", "nx", "ny", "steps", "time", "mass_initial", "mass_final", "mass_drift",
              "internal_energy_drift", "l2_rho_vs_initial", "l2_k_vs_initial", "max_k_violation", "min_p",
              "max_p", "wall_seconds"):
        assert k in d
    seen = []
    rep = frontend.run(frontend.build_case("haas", 8), hook=lambda st, dg: seen.append((st.step, int(dg["step"]))))
    assert [a for a, _ in seen] == [b for _, b in seen] == list(range(1, rep.steps + 1))
    ref = helpers.ref_lib()
    if ref is not None:  # every engine runs on the device, e.g. the Direct one, as the reference driver does
        d2 = frontend.run_case("haas", divisor=8, scheme="Direct")
        rc, what, want, out, steps, fin = ref_run_case(ref, "haas", 8, scheme="Direct")
        assert rc == 0 and d2["steps"] == steps and d2["time"] == out[0]
        assert d2["l2_rho_vs_initial"] == out[1] and d2["l2_k_vs_initial"] == out[2]


@pytest.mark.gpu
def test_cli_run(tmp_path):
    cfgf = tmp_path / "run.cfg"
    out = tmp_path / "out"
    cfgf.write_text(f"case = haas\ndivisor = 8\noutput_every = 5\nout_dir = {out}\n")
    r = subprocess.run([sys.executable, "-m", "paper_2208_13409_b200", "run", str(cfgf)], cwd=helpers.ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "case haas scheme DirectCF mesh 125x11" in r.stdout
    lines = (out / "diag.log").read_text().splitlines()
    steps = int(r.stdout.split("steps ")[1].split()[0])
    assert len(lines) == steps and lines[0].startswith("1 ")
    assert (out / "final.csv").exists() and (out / "final.vtk").exists() and (out / "fields_000005.csv").exists()
    ref = helpers.ref_lib()
    if ref is not None:  # final.csv is the reference writer's text of the reference's final State
        _, _, _, _, _, fin = ref_run_case(ref, "haas", 8)
        sr = abi.Solver(ref, frontend.build_case("haas", 8).config())
        sr.upload(fin)
        want = tmp_path / "want.csv"
        sr._check(ref.fn["write_fields"](sr._h, str(want).encode(), abi.DUMP_CSV))
        assert (out / "final.csv").read_bytes() == want.read_bytes()


# ---- convergence study (harness.cpp:426-461, main.cpp:72-105) ---------------------

def ref_convergence(ref, name, meshes, schemes):
    f = ref.dll.h2dr_convergence
    f.restype = C.c_int
    ms, ks = np.array(meshes, np.int32), np.array(schemes, np.int32)
    errs, slopes = np.zeros(len(ms) * len(ks)), np.zeros(len(ks))
    what = C.create_string_buffer(256)
    rc = f(name.encode(), ms.ctypes.data_as(C.c_void_p), len(ms), ks.ctypes.data_as(C.c_void_p), len(ks),
           errs.ctypes.data_as(C.c_void_p), slopes.ctypes.data_as(C.c_void_p), what, 256)
    assert rc == 0, what.value
    return errs.reshape(len(ks), len(ms)), slopes


def test_parse_schemes():
    assert frontend.parse_schemes("AD,Direct,DirectCF") == [abi.REMAP_AD, abi.REMAP_DIRECT, abi.REMAP_DIRECTCF]
    with pytest.raises(errors.SimError) as e:
        frontend.parse_schemes("AD,Foo")
    assert str(e.value) == "unknown scheme 'Foo' (valid: AD, Direct, DirectCF)"


def test_convergence_slope_and_error_choice(monkeypatch):
    """The study's bookkeeping with run() stubbed: the error is L2(k) for two
    materials, L2(rho) otherwise, and the slope is the least-squares fit."""
    seen = []

    def fake_run(cs, hook=None, device=0):
        seen.append((cs.nx, cs.ny, cs.scheme))
        return frontend.RunReport(spec=cs, series=None, initial_state=None, final_state=None,
                                  l2_rho_vs_initial=1.0 / cs.nx ** 2, l2_k_vs_initial=3.0 / cs.nx)
    monkeypatch.setattr(frontend, "run", fake_run)
    mono, multi = (frontend.convergence_study(n, [50, 100, 200], [abi.REMAP_AD, abi.REMAP_DIRECTCF])
                   for n in ("mono_advect", "multimat_advect"))
    assert seen[:3] == [(50, 50, abi.REMAP_AD), (100, 100, abi.REMAP_AD), (200, 200, abi.REMAP_AD)]
    assert [e for _, e in mono[0].rows] == [1.0 / 2500, 1.0 / 10000, 1.0 / 40000]
    assert [e for _, e in multi[1].rows] == [3.0 / 50, 3.0 / 100, 3.0 / 200]
    assert abs(mono[0].slope - 2.0) < 1e-12 and abs(multi[1].slope - 1.0) < 1e-12


@pytest.mark.gpu
def test_convergence_study_matches_reference():
    """The refinement study on the device equals the reference's own
    convergence_study (criterion 5's call, acceptance.cpp:239-241): every
    error and slope to the bit, on the three engines."""
    ref = helpers.ref_lib()
    if ref is None:
        pytest.skip("reference library not built")
    meshes, schemes = [50, 100, 200], [abi.REMAP_AD, abi.REMAP_DIRECT, abi.REMAP_DIRECTCF]
    want_e, want_s = ref_convergence(ref, "mono_advect", meshes, schemes)
    got = frontend.convergence_study("mono_advect", meshes, schemes)
    for s, r in enumerate(got):
        assert r.scheme == schemes[s] and [n for n, _ in r.rows] == meshes
        assert [e for _, e in r.rows] == list(want_e[s]), frontend.SCHEME_NAMES[r.scheme]
        assert r.slope == want_s[s]
    # criterion 5's ordering claims hold for the device run too
    ad, direct, cf = ([e for _, e in r.rows] for r in got)
    for errs in (ad, direct, cf):
        assert all(errs[m] < errs[m - 1] for m in range(1, 3))
    assert all(direct[m] >= ad[m] and cf[m] <= 2.0 * ad[m] for m in range(3))


@pytest.mark.gpu
def test_cli_converge():
    r = subprocess.run([sys.executable, "-m", "paper_2208_13409_b200", "converge", "multimat_advect", "DirectCF"],
                       cwd=helpers.ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0].split() == ["mesh", "DirectCF"] and [ln.split()[0] for ln in lines[1:]] == ["50", "100", "200",
                                                                                              "slope"]

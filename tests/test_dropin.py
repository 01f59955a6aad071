"""Drop-in proof for the C++ boundary ("Callers"):

* tests/cpp/dropin_driver.cpp, a caller written against the reference's
  public hydro:: API only, compiled once against the reference
  (oracle/_ref/dropin_ref) and once against the B200 headers + libh2d.so
  (tests/cpp/build/dropin_b200): both write byte-identical results;
* the reference's OWN callers compiled unmodified against the drop-in
  (tests/cpp/Makefile): the `hydro2d` CLI (tools/main.cpp), the acceptance
  suite (tests/acceptance.cpp) and the seven doctest unit-test files
  (tests/test_*.cpp, with tests/cpp/doctest_shim standing in for doctest).
  Their outputs must equal the reference build's (tests/golden/cli,
  tests/golden/acceptance_ref.txt, made by tests/golden/make_cli_golden.py),
  and every unit test must pass.

The *_b200 binaries are built in the container (the reference sources are
not on the GPU box) and run on the GPU."""
import filecmp
import os
import subprocess
import sys

import pytest

import helpers

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
from make_cli_golden import CLI_CONFIGS, normalise, normalise_acceptance  # noqa: E402

REF_BIN = os.path.join(helpers.ROOT, "oracle", "_ref", "dropin_ref")
BUILD = os.path.join(helpers.ROOT, "tests", "cpp", "build")
B200_BIN = os.path.join(BUILD, "dropin_b200")
GOLDEN = os.path.join(helpers.ROOT, "tests", "golden")
REFTESTS = ["mesh_state", "vof", "reconstruct", "lagrange", "remap", "analysis", "harness_io"]
HAVE_REF_SRC = os.path.isdir("/root/reference/proj/src")


def _b(name):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (tests/cpp/Makefile needs /root/reference)")
    return path


def test_dropin_driver_builds_against_b200_headers():
    subprocess.run(["make", "-s", "-C", os.path.join(helpers.ROOT, "tests", "cpp")], check=True)
    assert os.path.exists(B200_BIN)


@pytest.mark.skipif(not HAVE_REF_SRC, reason="needs /root/reference")
def test_reference_callers_build_against_b200_headers():
    subprocess.run(["make", "-s", "-C", os.path.join(helpers.ROOT, "tests", "cpp"), "callers"], check=True)
    for name in ["hydro2d_b200", "acceptance_b200"] + [f"reftest_{t}_b200" for t in REFTESTS]:
        assert os.path.exists(os.path.join(BUILD, name)), name


def test_doctest_shim_semantics(tmp_path):
    """The doctest stand-in re-runs a case per SUBCASE leaf, counts and
    reports failures and exits non-zero on one."""
    exe = tmp_path / "st"
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(helpers.ROOT, "tests", "cpp", "doctest_shim"),
                    os.path.join(helpers.ROOT, "tests", "cpp", "shim_selftest.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 1
    assert "test cases: 4 | 3 passed | 1 failed" in r.stdout
    assert "shim_selftest.cpp:31: ERROR: CHECK( 1 + 1 == 3 )" in r.stdout


@pytest.mark.skipif(not HAVE_REF_SRC, reason="needs /root/reference")
@pytest.mark.parametrize("t", REFTESTS)
def test_reference_unit_tests_pass_on_the_reference(t):
    """The shim is faithful: the reference's own unit tests pass against the
    reference library (oracle/Makefile target `callers`)."""
    subprocess.run(["make", "-s", "-C", os.path.join(helpers.ROOT, "oracle"), "callers"], check=True)
    r = subprocess.run([os.path.join(helpers.ROOT, "oracle", "_ref", f"reftest_{t}_ref")], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "Status: SUCCESS" in r.stdout


@pytest.mark.gpu
def test_same_caller_same_bytes(tmp_path):
    if not os.path.exists(REF_BIN):
        pytest.skip("reference build of the driver not present")
    subprocess.run(["make", "-s", "-C", os.path.join(helpers.ROOT, "tests", "cpp"), "dropin"], check=True)
    a, b = tmp_path / "ref.bin", tmp_path / "b200.bin"
    subprocess.run([REF_BIN, str(a)], check=True, timeout=600)
    subprocess.run([B200_BIN, str(b)], check=True, timeout=600)
    ra, rb = a.read_bytes(), b.read_bytes()
    assert len(ra) == len(rb)
    assert ra == rb


@pytest.mark.gpu
@pytest.mark.parametrize("t", REFTESTS)
def test_reference_unit_tests_pass_on_the_drop_in(t):
    """proj/tests/test_<t>.cpp, unmodified, against include/hydro + libh2d.so."""
    r = subprocess.run([_b(f"reftest_{t}_b200")], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "Status: SUCCESS" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CLI_CONFIGS))
def test_hydro2d_cli_run_same_bytes(name, tmp_path):
    """`hydro2d run <config>` (tools/main.cpp:30-71) built against the drop-in:
    diag.log, every fields dump, final.csv / final.vtk and stdout (wall time
    and output path aside) equal the reference build's bytes."""
    exe = _b("hydro2d_b200")
    out = str(tmp_path / name)
    os.makedirs(out)
    cfg = os.path.join(out, "run.cfg")
    with open(cfg, "w") as f:
        f.write(CLI_CONFIGS[name])
    r = subprocess.run([exe, "run", cfg], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, HYDRO_OUT_DIR=out))
    assert r.returncode == 0, r.stdout + r.stderr
    gold = os.path.join(GOLDEN, "cli", name)
    with open(os.path.join(gold, "stdout.txt")) as f:
        assert normalise(r.stdout, out) == f.read()
    files = sorted(x for x in os.listdir(gold) if x not in ("stdout.txt", "run.cfg"))
    assert sorted(x for x in os.listdir(out) if x != "run.cfg") == files
    for x in files:
        assert filecmp.cmp(os.path.join(gold, x), os.path.join(out, x), shallow=False), x


@pytest.mark.gpu
def test_hydro2d_cli_case_list():
    r = subprocess.run([_b("hydro2d_b200"), "case-list"], capture_output=True, text=True, check=True)
    with open(os.path.join(GOLDEN, "cli", "case-list.txt")) as f:
        assert r.stdout == f.read()


@pytest.mark.gpu
def test_acceptance_suite_same_lines():
    """proj/tests/acceptance.cpp against the drop-in: the same PASS / FAIL
    line, with the same figures, for every criterion (timings aside). The
    reference itself fails criterion 7 (impact / DirectCF aborts with
    UnphysicalStateError); the drop-in reproduces that abort."""
    r = subprocess.run([_b("acceptance_b200")], capture_output=True, text=True, timeout=3000)
    with open(os.path.join(GOLDEN, "acceptance_ref.txt")) as f:
        want = f.read()
    assert normalise_acceptance(r.stdout).splitlines() == want.splitlines()
    assert r.returncode == 1  # criterion 7, as in the reference

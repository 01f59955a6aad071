"""Drop-in proof for the C++ boundary: tests/cpp/dropin_driver.cpp, a caller
written against the reference's public hydro:: API only, is compiled once
against the reference (proj/include + reference library: oracle/_ref/dropin_ref)
and once against the B200 headers + libh2d.so (tests/cpp/build/dropin_b200).
Both binaries must write byte-identical results (every dt, counter, caught
exception and final State field)."""
import os
import subprocess

import pytest

import helpers

REF_BIN = os.path.join(helpers.ROOT, "oracle", "_ref", "dropin_ref")
B200_BIN = os.path.join(helpers.ROOT, "tests", "cpp", "build", "dropin_b200")


def test_dropin_driver_builds_against_b200_headers():
    subprocess.run(["make", "-s", "-C", os.path.join(helpers.ROOT, "tests", "cpp")], check=True)
    assert os.path.exists(B200_BIN)


@pytest.mark.gpu
def test_same_caller_same_bytes(tmp_path):
    if not os.path.exists(REF_BIN):
        pytest.skip("reference build of the driver not present")
    subprocess.run(["make", "-s", "-C", os.path.join(helpers.ROOT, "tests", "cpp")], check=True)
    a, b = tmp_path / "ref.bin", tmp_path / "b200.bin"
    subprocess.run([REF_BIN, str(a)], check=True, timeout=600)
    subprocess.run([B200_BIN, str(b)], check=True, timeout=600)
    ra, rb = a.read_bytes(), b.read_bytes()
    assert len(ra) == len(rb)
    assert ra == rb

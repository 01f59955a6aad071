"""Full-size, full-length parity against the REFERENCE itself (SURVEY.md
§8d): the device runs each BASELINE
configuration at its full size for its full step count (C3 up to the
reference's abort at step 820, C4 at 8192^2 for 10 steps and at 1024^2 for
200) and must reproduce the pin the reference library wrote for the same run
(tests/golden/make_fullsize_pins.py, oracle/_ref): every dt bit for bit, the
floor / clip / mass-fix counters and max_k_violation, the abort (class,
message, step) and the sha256 of every State plane, ghost layers included —
i.e. the end-of-run fields are identical (L1 difference 0)."""
import glob
import json
import os

import pytest

import helpers
from paper_2208_13409_b200 import cases

HERE = os.path.dirname(os.path.abspath(__file__))
PINS = sorted(glob.glob(os.path.join(HERE, "golden", "fullsize_pins", "*.json")))

CASES = {
    "c1_riemann_256": lambda: cases.riemann2d(256),
    "c2_sedov_1024": lambda: cases.sedov(1024),
    "c3_triple_point_2048x1024": lambda: cases.triple_point(2048, 1024),
    "c4_shock_bubble_1024": lambda: cases.shock_bubble(1024),
    "c4_shock_bubble_8192": lambda: cases.shock_bubble(8192),
}


def _load(path):
    with open(path) as f:
        return json.load(f)


def test_pins_are_complete():
    """Every BASELINE configuration the reference can run has a pin (C5 has
    three materials, beyond the reference's kMaxMat = 2: parity unpinned)."""
    names = {os.path.basename(p)[:-5] for p in PINS}
    assert names == set(CASES), names
    for p in PINS:
        rec = _load(p)
        assert rec["steps_done"] == len(rec["dts_hex"])
        assert rec["generator"].startswith("oracle/_ref")


@pytest.mark.gpu
@pytest.mark.parametrize("path", PINS, ids=[os.path.basename(p)[:-5] for p in PINS])
def test_device_reproduces_reference_pin(path):
    rec = _load(path)
    case = CASES[rec["name"]]()
    assert (case.cfg.mesh.nx, case.cfg.mesh.ny, case.cfg.nmat) == (rec["nx"], rec["ny"], rec["nmat"])
    s = helpers.prepared(helpers.product_lib(), case.cfg, case.paint())
    r, err = helpers.run_capture(s, rec["steps_requested"], case.cfl)
    assert r.steps_done == rec["steps_done"]
    assert [float(x).hex() for x in r.dts] == rec["dts_hex"]
    assert r.floor_count == rec["floor_count"]
    assert r.diag["k_clip_count"] == rec["k_clip_count"]
    assert r.diag["mass_fix_count"] == rec["mass_fix_count"]
    assert float(r.diag["max_k_violation"]).hex() == rec["max_k_violation_hex"]
    if rec["error"] is None:
        assert err is None
    else:
        assert err is not None and list(err) == rec["error"]
    hashes, step, t = helpers.plane_hashes(s, case.cfg.nmat)
    assert step == rec["final_step"] and float(t).hex() == rec["final_time_hex"]
    bad = {k: v for k, v in hashes.items() if rec["plane_sha256"][k] != v}
    assert not bad, sorted(bad)

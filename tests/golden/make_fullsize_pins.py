"""Full-size, full-length parity pins of the BASELINE configurations, produced
by the REFERENCE library itself (oracle/_ref/libh2d_ref.so, compiled from
/root/reference/proj by oracle/Makefile) — VERDICT r01 "next round" item 1,
SURVEY.md §8d.

Run in the build container (where /root/reference exists), one pin per
process (they are independent; C4 8192^2 needs ~50 GB of host memory):
    python tests/golden/make_fullsize_pins.py c1_256 c2_1024 ...
Each pin records, for the reference's run loop (harness.cpp:380-424) over
the configuration's initial State (cases.py restates init_case,
harness.cpp:163-291): the full dt sequence (bitwise, as float64 hex), the
counters (floor_count, k_clip_count, mass_fix_count, max_k_violation), the
error tuple of an aborting run, the final step / time and the sha256 of every
State plane in the reference Field layout (ghost layers included).  The -m gpu
test tests/test_gpu_fullsize_pins.py replays the same run on the device and
compares all of it; the GPU box has no /root/reference, so the pins are
committed as tests/golden/fullsize_pins/<name>.json."""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2208_13409_b200 import cases  # noqa: E402

OUT = os.path.join(HERE, "fullsize_pins")

# name -> (case factory, steps run by the pin); the BASELINE step counts,
# C3 up to its abort, C4 at full size for its first 10 steps and the full
# 200 steps at 1024^2 (SURVEY.md §8d "Oracle at full size ... use per-step
# parity on the first 10 steps at full size, plus a full 200-step run at 1024^2")
PINS = {
    "c1_riemann_256": (lambda: cases.riemann2d(256), 100),
    "c2_sedov_1024": (lambda: cases.sedov(1024), 500),
    "c3_triple_point_2048x1024": (lambda: cases.triple_point(2048, 1024), 1000),
    "c4_shock_bubble_1024": (lambda: cases.shock_bubble(1024), 200),
    "c4_shock_bubble_8192": (lambda: cases.shock_bubble(8192), 10),
}


def run_pin(lib, name: str):
    from paper_2208_13409_b200 import abi, errors
    make, steps = PINS[name]
    case = make()
    painted = case.paint()
    s = abi.Solver(lib, case.cfg)
    s.init_from(painted)
    del painted
    t0 = time.time()
    err = None
    try:
        r = s.run(steps, t_end=1e30, cfl=case.cfl)
    except errors.SimError as e:
        r = e.partial
        err = [type(e).__name__, e.what, e.i, e.j, e.step, e.in_step]
    wall = time.time() - t0
    import helpers
    hashes, step, t = helpers.plane_hashes(s, case.cfg.nmat)
    return {
        "name": name, "case": case.name, "steps_requested": steps, "cfl": case.cfl,
        "nx": case.cfg.mesh.nx, "ny": case.cfg.mesh.ny, "nmat": case.cfg.nmat,
        "steps_done": int(r.steps_done), "final_step": int(step), "final_time_hex": float(t).hex(),
        "dts_hex": [float(x).hex() for x in r.dts],
        "floor_count": int(r.floor_count), "k_clip_count": int(r.diag["k_clip_count"]),
        "mass_fix_count": int(r.diag["mass_fix_count"]),
        "max_k_violation_hex": float(r.diag["max_k_violation"]).hex(),
        "error": err, "plane_sha256": hashes,
        "generator": "oracle/_ref (reference compiled unmodified), tests/golden/make_fullsize_pins.py",
        "reference_wall_s": round(wall, 1),
    }


def main(names):
    import helpers
    ref = helpers.ref_lib()
    assert ref is not None, "needs the reference library (oracle/_ref)"
    os.makedirs(OUT, exist_ok=True)
    for name in names or list(PINS):
        rec = run_pin(ref, name)
        with open(os.path.join(OUT, f"{name}.json"), "w") as f:
            json.dump(rec, f, indent=1)
        print(name, "steps", rec["steps_done"], "error", rec["error"], "wall", rec["reference_wall_s"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])

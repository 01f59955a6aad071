"""Kernel-group times of one configuration at given steps:
python tools/phase_at.py c4 80,90,100,120."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2208_13409_b200 as pkg  # noqa: E402

name = sys.argv[1]
at = sorted(int(x) for x in sys.argv[2].split(","))
case = bench.workload(name)
s = pkg.solver(case.cfg)
s.init_from(case.paint())
for q in at:
    s.run(q, cfl=case.cfl, log_dt=False)
    s.flush_l2(512 << 20)
    ph = s.step_timed(case.cfl, phases=True)
    r = s.run(q + 2, cfl=case.cfl, log_dt=False)
    print(json.dumps({"workload": name, "step": q, "phases_ms": {k: round(v, 4) for k, v in ph.items()},
                      "next_step_diag": r.diag}), flush=True)

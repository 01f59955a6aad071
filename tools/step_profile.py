"""Per-step device time across a configuration's whole run (is the timed
sample representative?): python tools/step_profile.py c2 [total_steps] [every]."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2208_13409_b200 as pkg  # noqa: E402

name = sys.argv[1]
total = int(sys.argv[2]) if len(sys.argv) > 2 else 500
every = int(sys.argv[3]) if len(sys.argv) > 3 else 1
case = bench.workload(name)
s = pkg.solver(case.cfg)
s.init_from(case.paint())
out = []
for q in range(total):
    s.flush_l2(512 << 20)
    ms = s.step_timed(case.cfl)["total"]
    if q % every == 0:
        out.append((q, round(ms, 4)))
print(json.dumps({"workload": name, "per_step_ms": out}))

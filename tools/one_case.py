"""Run N device steps of a configuration (for profiling): python tools/one_case.py c3 [steps] [warm]."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2208_13409_b200 as pkg  # noqa: E402

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 0
case = bench.workload(name)
s = pkg.solver(case.cfg)
s.init_from(case.paint())
if warm:
    s.run(warm, cfl=case.cfl, log_dt=False)
r = s.run(s.download().step + steps, cfl=case.cfl)
print(name, "steps", r.steps_done, "diag", r.diag)

"""One plain-launch step of a configuration at step q inside a cudaProfilerStart/Stop
window (for ncu --profile-from-start off): python tools/ncu_at.py c4 85."""
import ctypes
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2208_13409_b200 as pkg  # noqa: E402

name, q = sys.argv[1], int(sys.argv[2])
case = bench.workload("c5", full=False) if name == "c5b" else bench.workload(name)
s = pkg.solver(case.cfg)
s.init_from(case.paint())
if q:
    s.run(q, cfl=case.cfl, log_dt=False)
rt = ctypes.CDLL("libcudart.so.12") if False else None
import torch  # noqa: E402
torch.cuda.init()
torch.cuda.cudart().cudaProfilerStart()
s.step_timed(case.cfl, phases=True)
torch.cuda.cudart().cudaProfilerStop()
print("done", name, q)

"""Stream timeline of the block data plane on ONE GPU (in-process comm): CUDA
timing events at nine points of each step and block (h2d_comm_trace), to show
where the halo exchange sits against the compute stream.

python tools/blocks_trace.py [n=4096] [px=2] [py=1] [engine=directcf|ad] [steps=6] [warm=4]

For every traced step s >= 1 and block b it prints the intervals (ms from the
block's first traced step start) and whether the State halo exchange enqueued
after step s - 1 ran INSIDE step s's owned-tile Lagrange interval (overlap),
and for AD the mid exchange, which has nothing to hide behind."""
import json
import sys

sys.path.insert(0, ".")
import paper_2208_13409_b200 as pkg  # noqa: E402
from paper_2208_13409_b200 import abi, cases, multi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
px = int(sys.argv[2]) if len(sys.argv) > 2 else 2
py = int(sys.argv[3]) if len(sys.argv) > 3 else 1
engine = sys.argv[4] if len(sys.argv) > 4 else "directcf"
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 6
warm = int(sys.argv[6]) if len(sys.argv) > 6 else 4
kind = abi.REMAP_AD if engine == "ad" else abi.REMAP_DIRECTCF

case = cases.shock_bubble(n)
lib = pkg.product_library()
specs = multi.decompose(n, n, px, py)
blocks = [multi.BlockSolver(lib, case.cfg, sp) for sp in specs]
for b in blocks:
    b.init_window(case.paint(b.window()))
comm = multi.DeviceComm(blocks, px, py)
comm.run(warm, 1e30, case.cfl, kind=kind)
comm.trace(steps)
comm.run(warm + steps, 1e30, case.cfl, kind=kind)
tr = comm.trace_read()
P = {k: q for q, k in enumerate(multi.DeviceComm.TRACE_POINTS)}
out = {"mesh": f"shock_bubble {n}^2", "blocks": f"{px}x{py} in-process on one GPU", "engine": engine,
       "points": list(multi.DeviceComm.TRACE_POINTS), "steps": []}
for s in range(tr.shape[0]):
    for b in range(tr.shape[1]):
        r = tr[s, b]
        rec = {"step": s, "block": b, **{k: round(float(r[q]), 4) for k, q in P.items()}}
        if s >= 1:
            h0, h1 = tr[s - 1, b, P["halo_start"]], tr[s - 1, b, P["halo_end"]]
            l0, l1 = r[P["lag_owned_start"]], r[P["lag_owned_end"]]
            ov = max(0.0, min(h1, l1) - max(h0, l0))
            rec["prev_halo_ms"] = round(float(h1 - h0), 4)
            rec["prev_halo_overlap_with_owned_lagrange_ms"] = round(float(ov), 4)
            rec["edge_wait_after_owned_ms"] = round(float(max(0.0, h1 - l1)), 4)
        if kind == abi.REMAP_AD:
            rec["mid_exchange_ms"] = round(float(r[P["ad_mid_end"]] - r[P["ad_mid_start"]]), 4)
        out["steps"].append(rec)
print(json.dumps(out))
comm.close()

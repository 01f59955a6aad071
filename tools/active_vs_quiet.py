"""Per-kernel-group device time of the C4 state family at 4096^2 with the
post-shock slab covering a chosen fraction of the domain: 0.0 = every tile
quiescent (plus the bubble), 0.3 = configuration 4, 1.0 = every cell moving
(uniform flow). Shows what the quiescent-tile and active paths cost per cell.

python tools/active_vs_quiet.py [n=4096] [lib-variant ...]"""
import json
import os
import sys

sys.path.insert(0, ".")
import paper_2208_13409_b200 as pkg  # noqa: E402
from paper_2208_13409_b200 import cases  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for frac in (0.0, 0.3, 1.0):
    case = cases.shock_bubble(n)
    case.regions[1].xsplit = frac * 1.0 if frac < 1.0 else 2.0
    s = pkg.solver(case.cfg)
    s.init_from(case.paint())
    for _ in range(3):
        s.step_timed(case.cfl)
    steps = 6
    tot = 0.0
    for _ in range(steps):
        s.flush_l2(512 << 20)
        tot += s.step_timed(case.cfl)["total"]
    ph = {}
    for _ in range(steps):
        s.flush_l2(512 << 20)
        for k, v in s.step_timed(case.cfl, phases=True).items():
            ph[k] = ph.get(k, 0.0) + v / steps
    cells = n * n
    print(json.dumps({"mesh": f"{n}^2", "moving_fraction": frac, "graphed_ms": tot / steps,
                      "ns_per_cell": {k: round(v * 1e6 / cells, 4) for k, v in ph.items()},
                      "phases_ms": {k: round(v, 4) for k, v in ph.items()},
                      "lib": os.environ.get("H2D_PRODUCT_LIB", "base")}), flush=True)
    del s

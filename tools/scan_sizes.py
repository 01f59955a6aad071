"""Step time of the product vs mesh size (fixed-overhead vs per-cell cost)."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2208_13409_b200 as pkg  # noqa: E402
from paper_2208_13409_b200 import cases  # noqa: E402


def main():
    out = []
    for name, case in [("sedov", cases.sedov), ("riemann", cases.riemann2d)]:
        for n in (256, 512, 1024, 2048, 4096):
            c = case(n)
            s = pkg.solver(c.cfg)
            s.init_from(c.paint())
            for _ in range(5):
                s.step_timed(c.cfl)
            ts = []
            for _ in range(10):
                s.flush_l2()
                ts.append(s.step_timed(c.cfl)["total"])
            ms = float(np.median(ts))
            out.append({"case": name, "n": n, "cells": n * n, "ms": ms, "cells_per_s": n * n / ms * 1e3})
            print(json.dumps(out[-1]), flush=True)
            s.close()
    json.dump(out, open("gpurun_out/scan_sizes.json", "w"), indent=1)


if __name__ == "__main__":
    main()

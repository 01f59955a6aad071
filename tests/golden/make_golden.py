"""Generate the golden vectors in this directory from the REFERENCE library
itself (oracle/_ref/libh2d_ref.so, compiled from /root/reference/proj).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Each fixture stores the initial-state recipe name, the dt sequence, the
RemapDiag / floor counters, the first error (if any) and the final State
fields (all ghost layers) as produced by the reference; test_golden.py
replays the recipes on the oracle (CPU) and on the CUDA product (GPU)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import helpers  # noqa: E402
from golden_cases import GOLDEN, build  # noqa: E402


def main():
    ref = helpers.ref_lib()
    assert ref is not None, "needs the reference library (oracle/_ref)"
    for name in GOLDEN:
        cfg, painted, action = build(name)
        s = helpers.prepared(ref, cfg, painted)
        res, err = action(s)
        st = s.download()
        out = {f: getattr(st, f) for f in helpers.STATE_FIELDS}
        out["step_time"] = np.array([st.step, st.time])
        out["dts"] = res["dts"]
        out["counters"] = np.array(res["counters"], dtype=np.float64)
        out["error"] = np.array(repr(err))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, "steps", len(res["dts"]), "error", err)


if __name__ == "__main__":
    main()

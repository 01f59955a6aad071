"""Build variants of libh2d.so that differ only in compile-time knobs
(launch bounds, tile shapes), for side-by-side timing on the GPU:

    python tools/variants.py build NAME -DH2D_POST_MINB=4 ...   (here, CPU)
    python tools/variants.py time c4 NAME [NAME ...]              (GPU box)

`time` loads each variant in a fresh process (H2D_PRODUCT_LIB) and prints
the per-group CUDA-event phases of 6 un-graphed steps after 3 warm-up
steps plus the graphed step time, one JSON line per variant."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VDIR = os.path.join(ROOT, "build", "variants")


def build(name, defs):
    sys.path.insert(0, ROOT)
    from paper_2208_13409_b200 import build as b
    os.makedirs(VDIR, exist_ok=True)
    out = os.path.join(VDIR, f"libh2d_{name}.so")
    srcs = [os.path.join(b.CSRC, s) for s in b.SOURCES]
    cmd = [b.NVCC, *[f for f in b.FLAGS if f not in ("-Xptxas", "-v")], *defs,
           "-I" + os.path.join(ROOT, "include"), "-shared", "-o", out, *srcs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stdout + r.stderr)
    with open(out + ".defs", "w") as f:
        f.write(" ".join(defs))
    print(out)


CHILD = r"""
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import bench
import paper_2208_13409_b200 as pkg
wl, steps, warm = sys.argv[1], 6, 3
case = bench.workload(wl, full=(wl != "c5"))
s = pkg.solver(case.cfg)
s.init_from(case.paint())
for _ in range(warm):
    s.step_timed(case.cfl)
tot = 0.0
for _ in range(steps):
    s.flush_l2(512 << 20)
    tot += s.step_timed(case.cfl)["total"]
ph = {}
for _ in range(steps):
    s.flush_l2(512 << 20)
    for k, v in s.step_timed(case.cfl, phases=True).items():
        ph[k] = ph.get(k, 0.0) + v / steps
st = s.download()
import hashlib, numpy as np
h = hashlib.sha256()
for f in ("m", "e", "k", "u", "iface_normal"):
    h.update(np.ascontiguousarray(getattr(st, f)).tobytes())
print(json.dumps({"graphed_ms": tot / steps, "phases": ph, "state_sha": h.hexdigest()[:16], "step": st.step}))
"""


def time_variants(wl, names):
    for name in names:
        lib = os.path.join(ROOT, "paper_2208_13409_b200", "libh2d.so") if name == "base" else \
            os.path.join(VDIR, f"libh2d_{name}.so")
        env = dict(os.environ, ROOT=ROOT, H2D_PRODUCT_LIB=lib)
        r = subprocess.run([sys.executable, "-c", CHILD, wl], capture_output=True, text=True, env=env, timeout=900)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else json.dumps({"error": r.stderr[-800:]})
        d = json.loads(line)
        d["variant"] = name
        d["workload"] = wl
        if os.path.exists(lib + ".defs"):
            d["defs"] = open(lib + ".defs").read()
        print(json.dumps(d), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3:])
    else:
        time_variants(sys.argv[2], sys.argv[3:])

"""Regenerate the round-2 results table of DESIGN.md section 7 from a
measurement set under profiles/ (python tools/fill_design.py v4)."""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
V = sys.argv[1]
P = os.path.join(ROOT, "profiles")
NAMES = {"c1": "C1 Riemann 256², 1 mat", "c2": "C2 Sedov 1024², 1 mat", "c3": "C3 triple point 2048×1024, 2 mat",
         "c4": "**C4 shock-bubble 8192², 2 mat** (bench default)", "c5": "C5 Voronoi 16384², 3 mat, one GPU"}


def sci(x):
    e = int(f"{x:e}".split("e")[1])
    sup = str(e).translate(str.maketrans("0123456789", "⁰¹²³⁴⁵⁶⁷⁸⁹"))
    return f"{x / 10 ** e:.2f}·10{sup}"


def rows():
    out = []
    for w in ("c1", "c2", "c3", "c4", "c5"):
        d = json.load(open(os.path.join(P, f"r02_bench_{w}_{V}.json")))
        r = d["roofline"]
        cells = d["config"]["cells"]
        cs = f"{cells / 1e6:.2f} M" if cells >= 1e6 else f"{cells / 1e3:.0f} K"
        dr = f" ({100 * r['dram_frac']:.0f} % on DRAM bytes)" if r.get("dram_frac") else ""
        kern = r["kernel"] if w != "c5" else "remap tile class launches"
        roof = f"`{kern}` {100 * r['frac']:.0f} %{dr}" if w != "c1" else "— (launch-bound)"
        cb = d["cpu_baseline"]
        kind = "reference" if cb["kind"] == "reference" else "C restatement"
        out.append(f"| {NAMES[w]} | {cs} | {d['ms_per_step']:.3f} | {sci(d['value'])} | {roof} | "
                   f"{100 * d['step_roofline']['frac']:.1f} % | {sci(d['e2e']['value'])} | {sci(cb['value'])} ({kind}) |")
    return "\n".join(out)


def main():
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    hdr = "| workload | cells | ms/step | cell-updates/s | dominant kernel roofline | step roofline | e2e run(K = 10) | CPU baseline (1 core) |\n|---|---|---|---|---|---|---|---|\n"
    a = s.index(hdr) + len(hdr)
    b = s.index("\n\n", a)
    s = s[:a] + rows() + s[b:]
    s = re.sub(r"set `v\d`, the round's final code", f"set `{V}`, the round's final code", s)
    open(p, "w").write(s)
    print(rows())


if __name__ == "__main__":
    main()

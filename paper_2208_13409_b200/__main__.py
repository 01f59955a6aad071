"""Command-line front end, the reference CLI's ``run`` and ``case-list``
commands (proj/tools/main.cpp:15-71) over the device path:

    python -m paper_2208_13409_b200 run <config>
    python -m paper_2208_13409_b200 converge <case> <schemes>
    python -m paper_2208_13409_b200 case-list

``run`` reads the key = value config (config.cpp), runs the case on the GPU
and writes, like cmd_run: <out_dir>/diag.log (one append_diag_line per step),
fields_<step>.csv every ``output_every`` steps, final.csv and final.vtk, then
the summary lines.  ``converge`` is cmd_converge (main.cpp:86-105): the
mesh-refinement study on 50, 100, 200 cells per side, one table.  The device keeps the State between dumps: a dump is one
download, the ledger comes from the step series reduced on the device.
"""
from __future__ import annotations

import os
import sys

import numpy as np

from . import abi, errors, frontend, product_library


def _usage() -> int:
    print("usage: hydro2d <command> [args]\n"
          "  run <config>               run a case from a key = value config file\n"
          "  converge <case> <schemes>  mesh-refinement study (schemes: comma list)\n"
          "  case-list                  list the built-in cases")
    return 2


def cmd_run(path: str) -> int:
    rc = frontend.load_config(path)
    cs = frontend.configure_case(rc)
    out_dir = os.environ.get("HYDRO_OUT_DIR", rc.out_dir)
    os.makedirs(out_dir, exist_ok=True)
    lib = product_library()
    lines = []

    def hook(st, d):
        lines.append(abi.diag_line(lib, d))
        if rc.output_every > 0 and int(d["step"]) >= hook.next_dump:
            v = st.view(derived=True)
            fname = os.path.join(out_dir, "fields_%06d.csv" % int(d["step"]))
            code = lib.fn["write_fields_host"](abi.C.byref(cs.config()), abi.C.byref(v), fname.encode(),
                                               abi.DUMP_CSV)
            if code:
                raise errors.SimError("cannot write: " + fname)
            hook.next_dump += rc.output_every
    hook.next_dump = rc.output_every

    if rc.output_every > 0:
        rep = frontend.run(cs, hook=hook)
    else:  # no State needed per step: the whole loop stays on the device
        rep = frontend.run(cs)
        lines.extend(abi.diag_line(lib, d) for d in rep.series[1:])
    with open(os.path.join(out_dir, "diag.log"), "w") as f:
        f.writelines(lines)
    cfg = cs.config()
    for name, fmt in (("final.csv", abi.DUMP_CSV), ("final.vtk", abi.DUMP_VTK)):
        v = rep.final_state.view(derived=True)
        fname = os.path.join(out_dir, name)
        if lib.fn["write_fields_host"](abi.C.byref(cfg), abi.C.byref(v), fname.encode(), fmt):
            raise errors.SimError("cannot write: " + fname)
    t0, t1 = rep.series[0], rep.series[-1]
    print(f"case {cs.name} scheme {frontend.SCHEME_NAMES[cs.scheme]} mesh {cs.nx}x{cs.ny}")
    print(f"steps {rep.steps}  t {rep.final_state.time:g}  wall {rep.wall_seconds:g} s")
    print("mass drift %.3e  internal-energy drift %.3e" % (
        abs(float(t1["mass"]) - float(t0["mass"])) / float(t0["mass"]),
        abs(float(t1["internal_energy"]) - float(t0["internal_energy"]))
        / max(1e-300, abs(float(t0["internal_energy"])))))
    if cs.nmat == 2:
        print("max pre-clip fraction violation %.3e" % rep.max_k_violation)
    print("L2(rho) vs initial %.6e" % rep.l2_rho_vs_initial)
    if cs.nmat == 2:
        print("L2(k) vs initial %.6e" % rep.l2_k_vs_initial)
    print(f"wrote {out_dir}/final.csv, final.vtk, diag.log")
    return 0


def cmd_converge(case_name: str, schemes_arg: str) -> int:
    schemes = frontend.parse_schemes(schemes_arg)
    meshes = [50, 100, 200]
    results = frontend.convergence_study(case_name, meshes, schemes)
    print("%-10s" % "mesh" + "".join("  %-12s" % frontend.SCHEME_NAMES[r.scheme] for r in results))
    for row, n in enumerate(meshes):
        print("%-10d" % n + "".join("  %-12.5e" % r.rows[row][1] for r in results))
    print("%-10s" % "slope" + "".join("  %-12.3f" % r.slope for r in results))
    return 0


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    if not argv:
        return _usage()
    try:
        if argv[0] == "case-list":
            for n in frontend.case_list():
                print(n)
            return 0
        if argv[0] == "run" and len(argv) == 2:
            return cmd_run(argv[1])
        if argv[0] == "converge" and len(argv) == 3:
            return cmd_converge(argv[1], argv[2])
    except errors.SimError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    return _usage()


if __name__ == "__main__":
    sys.exit(main())

"""Small device runs that reach every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per call):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py

TMA + mbarrier remap tile (k_remap_tile<1,2,3>), the fused Lagrange kernel,
k_slivers (the 64x32 triple point has sliver chains), k_post / k_tail, the
dual-mesh momentum kernels, the AD and Direct engines, the API-path kernels
(k_lag_cells / k_lag_nodes / k_cfl / k_sync / ghosts) and the block mode.
Every run is also compared bit for bit with the C oracle, so a sanitizer
finding and a parity break show up in the same log."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import helpers  # noqa: E402
from paper_2208_13409_b200 import abi, cases, multi  # noqa: E402


def pair(case, steps, kind=abi.REMAP_DIRECTCF):
    painted = case.paint()
    sg = helpers.prepared(helpers.product_lib(), case.cfg, painted)
    so = helpers.prepared(helpers.oracle_lib(), case.cfg, painted)
    rg, eg = helpers.run_capture(sg, steps, case.cfl, kind=kind)
    ro, eo = helpers.run_capture(so, steps, case.cfl, kind=kind)
    ok = eg == eo and np.array_equal(rg.dts, ro.dts) and \
        helpers.bitwise_diff(sg.download(), so.download(), helpers.STATE_FIELDS) == []
    print(f"{case.name} kind={kind} steps={rg.steps_done} err={eg and eg[0]} parity={'ok' if ok else 'FAIL'}",
          flush=True)
    return ok


def api_path(case):
    painted = case.paint()
    outs = []
    for lib in (helpers.product_lib(), helpers.oracle_lib()):
        s = helpers.prepared(lib, case.cfg, painted)
        dt = s.cfl_dt(case.cfl)
        lag = s.lagrange_step(dt)
        s.remap_step(dt)
        outs.append((dt, lag, s.download()))
    ok = outs[0][0] == outs[1][0] and helpers.bitwise_diff(outs[0][2], outs[1][2], helpers.STATE_FIELDS) == []
    print(f"{case.name} api-path parity={'ok' if ok else 'FAIL'}", flush=True)
    return ok


def blocks(case, px, py, steps):
    painted = case.paint()
    ref = helpers.prepared(helpers.product_lib(), case.cfg, painted)
    ref.run(steps, cfl=case.cfl)
    want = ref.download()
    lib = helpers.product_lib()
    init = ref_init = helpers.prepared(lib, case.cfg, painted).download()
    specs = multi.decompose(case.cfg.mesh.nx, case.cfg.mesh.ny, px, py)
    bl = [multi.BlockSolver(lib, case.cfg, sp) for sp in specs]
    for b in bl:
        b.upload(ref_init)
    multi.run_blocks(bl, multi.LocalTransport(bl, px, py), steps, 1e30, case.cfl)
    got = abi.HostState.empty(case.cfg.mesh.nx, case.cfg.mesh.ny, case.cfg.nmat)
    for b in bl:
        b.download_into(got)
    del init
    ok = helpers.bitwise_diff(got, want, helpers.STATE_FIELDS) == []
    print(f"{case.name} blocks {px}x{py} parity={'ok' if ok else 'FAIL'}", flush=True)
    return ok


def main():
    ok = True
    ok &= pair(cases.sedov(64), 20)
    ok &= pair(cases.riemann2d(48), 20)
    ok &= pair(cases.triple_point(64, 32), 60)
    ok &= pair(cases.shock_bubble(64), 10)
    ok &= pair(cases.voronoi3(64), 8)
    ok &= pair(cases.triple_point(64, 32), 20, kind=abi.REMAP_AD)
    ok &= pair(cases.triple_point(64, 32), 20, kind=abi.REMAP_DIRECT)
    ok &= api_path(cases.triple_point(48, 24))
    ok &= blocks(cases.triple_point(64, 32), 2, 2, 10)
    print("ALL OK" if ok else "PARITY FAILURES")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

"""Block mode on ONE GPU (in-process comm, px x py blocks side by side): the
unsplit DirectCF step (1 halo exchange + 1 all-reduce per step) against the
AD split remap (2 halo exchanges + 1 all-reduce), same mesh and steps.

python tools/blocks_ad_vs_cf.py [n=2048] [px=2] [py=2] [steps=20] [warm=5]

Prints one JSON line per engine: device ms/step of the whole decomposed loop
(CUDA events, slowest block), the doubles each block sends per exchange, and
the single-domain step of the same engine for scale. The blocks share one
GPU, so the times show the extra exchange's pack / copy / unpack work and
the lost overlap, not NVLink latency."""
import json
import sys

sys.path.insert(0, ".")
import paper_2208_13409_b200 as pkg  # noqa: E402
from paper_2208_13409_b200 import abi, cases, multi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
px = int(sys.argv[2]) if len(sys.argv) > 2 else 2
py = int(sys.argv[3]) if len(sys.argv) > 3 else 2
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
warm = int(sys.argv[5]) if len(sys.argv) > 5 else 5

case = cases.shock_bubble(n)
lib = pkg.product_library()
nm = case.cfg.nmat
for name, kind in (("directcf", abi.REMAP_DIRECTCF), ("ad", abi.REMAP_AD)):
    s = pkg.solver(case.cfg)
    s.init_from(case.paint())
    s.run(warm, cfl=case.cfl, kind=kind, log_dt=False)
    single = [s.step_timed(case.cfl, kind=kind)["total"] for _ in range(steps)]
    del s
    specs = multi.decompose(n, n, px, py)
    blocks = [multi.BlockSolver(lib, case.cfg, sp) for sp in specs]
    for b in blocks:
        b.init_window(case.paint(b.window()))
    comm = multi.DeviceComm(blocks, px, py)
    comm.run(warm, 1e30, case.cfl, kind=kind)
    done = comm.run(warm + steps, 1e30, case.cfl, kind=kind)
    ms = comm.device_ms / max(done, 1)
    state_doubles = sum(blocks[0].halo_bytes(dx, dy, 1) for dx, dy in multi.DIRS
                        if specs[0].neighbour(px, py, dx, dy) is not None) // 8
    nc, nn = multi.state_planes(nm)
    ad_cells, ad_nodes = 4 * nm + 1 + (2 if nm == 2 else 0), 2
    comm.close()
    for b in blocks:
        b.close()
    print(json.dumps({
        "engine": name, "mesh": f"shock_bubble {n}^2", "blocks": f"{px}x{py} in-process on one GPU",
        "steps": done, "ms_per_step_blocks": ms, "ms_per_step_single_domain": sum(single) / len(single),
        "halo_exchanges_per_step": 2 if kind == abi.REMAP_AD else 1, "allreduces_per_step": 1,
        "state_halo_doubles_block0": state_doubles,
        "planes_state_exchange": [nc, nn], "planes_mid_exchange": [ad_cells, ad_nodes] if kind == abi.REMAP_AD else None,
    }), flush=True)

#!/usr/bin/env python
"""Benchmark of one full Lagrange + DirectCF step (fp64) on B200.

Product arm (default): the CUDA library through its C-ABI.  A "step" is one
pass of the hot path over the whole mesh: cfl_dt -> lagrange_step ->
remap_step(DirectCF) -> nan_scan (harness.cpp:390-412).  The default workload is
configs[3] of BASELINE.json, the two-material shock-bubble on 8192^2 cells: the
largest configuration the reference itself can hold (kMaxMat = 2), so its
results are pinned to the reference bit for bit.  (--workload c5 runs the
16384^2 three-material configs[4], which also fits one B200 at ~156 GB; it is
this build's N-material extension, runs with the documented sliver-energy
safeguard, and its default run takes several minutes to paint.)  Synthetic
initial data painted exactly like the reference's init_case (seeded bubble
perturbation).  W warm-up steps, then K timed steps, each bracketed by CUDA
events on the library's stream with an L2 flush (512 MiB write) between steps.

Reference arm (--impl reference): the reference's own CPU implementation
(oracle/_ref, compiled from /root/reference/proj) on the host, same workload
and config, single thread (the reference has no threading), each run a
bounded sample of the workload's steps (about 1.2e8 cell-updates).

Prints ONE JSON line (rank 0).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "cell-updates/s per full Lagrange+remap step (fp64)"
UNIT = "cell-updates/s"
B_MIN = {1: 64, 2: 160, 3: 208}  # algorithmic bytes per cell-step (3 materials:
#   m, e, k per material + normals + u = 13 fp64 read + written once)
# Compulsory HBM bytes per cell of the three big kernels (their inputs read
# once + outputs written once):
#  k_lag_fused: reads m, e, k per material, u (2 nodal), m_mix, rho_mix;
#               writes u_half, u_lag (2+2 nodal), e_lag per material;
#  k_remap_tile: reads u_half (2), e_lag, m, k per material (+ normals for 2
#               materials); writes Work m, me, e, k per material, mcell, the
#               mass fluxes dmx, dmy, dmc (+ 1 sliver-flag byte for 2);
#  k_post:      reads new m, e, k per material and |u| (+ old normals);
#               writes m_mix, e_mix, rho_mix, p_mix, vol (+ normals).
KERNEL_BYTES = {
    "lagrange": ("k_lag_fused", {1: 8 * (3 + 4) + 8 * (4 + 1), 2: 8 * (6 + 4) + 8 * (4 + 2),
                                 3: 8 * (9 + 4) + 8 * (4 + 3)}),
    "remap_tile": ("k_remap_tile", {1: 8 * (2 + 3) + 8 * (4 + 1 + 3), 2: 8 * (2 + 6 + 2) + 8 * (8 + 1 + 3) + 1,
                                    3: 8 * (2 + 9 + 2) + 8 * (12 + 1 + 3) + 1}),
    "post": ("k_post", {1: 8 * (3 + 1) + 8 * 5, 2: 8 * (6 + 1 + 2) + 8 * (5 + 2), 3: 8 * (9 + 1 + 2) + 8 * (5 + 2)}),
}
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0


def workload(name, full=True):
    """The bench workloads (BASELINE.json configs[0..4]); c5 is the whole
    16384^2 three-material mesh (about 594 B per cell on the device: it fits
    one B200); full=False gives one GPU's 4096 x 8192 block of it."""
    from paper_2208_13409_b200 import cases
    if name == "c5":
        return c5_case(cases.voronoi3(16384) if full else cases.voronoi3(4096, 8192, n_full=16384))
    if name == "c1":
        return cases.riemann2d(256)
    if name == "c2":
        return cases.sedov(1024)
    if name == "c3":
        return cases.triple_point(2048, 1024)
    if name == "c4":
        return cases.shock_bubble(8192)
    raise SystemExit(f"unknown workload {name}")


def c5_case(case):
    """Configuration 5 runs with the sliver-energy safeguard
    (H2D_OPT_SLIVER_ENERGY, include/h2d.h; default off elsewhere): without it
    a remapped sliver's negative energy aborts the Voronoi case within tens
    of steps, as the reference's own two-material proxy does."""
    from paper_2208_13409_b200 import abi
    case.cfg.options = abi.OPT_SLIVER_ENERGY
    return case


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class Clocks:
    """SM clock / throttle-reason sampler (NVML, every 5 ms) running during
    the timed region."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index, self.samples, self.reasons, self.smax = index, [], set(), None
        self._stop = threading.Event()
        self.t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.nv = pynvml
        except Exception:
            self.nv = None
            return
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()

    def _poll(self):
        while not self._stop.is_set():
            try:
                self.samples.append(float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for nm, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.005)

    def stop(self):
        if self.t is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self._stop.set()
        self.t.join()
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        pg = dist
    return world, rank, local, pg


def max_over_ranks(pg, value):
    if pg is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


def cpu_lib(nmat=1):
    """Reference library (oracle/_ref) if built, else the C restatement (and
    always for three materials, which the reference cannot hold)."""
    from paper_2208_13409_b200 import abi
    ref = os.path.join(ROOT, "oracle", "_ref", "libh2d_ref.so")
    if os.path.exists(ref) and nmat <= 2:
        return abi.Library(ref, "h2dr_"), "reference"
    port = os.path.join(ROOT, "oracle", "libh2d_oracle.so")
    if not os.path.exists(port):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    return abi.Library(port, "h2do_"), "port"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


SCHEMES = {"ad": "AD split (X/Y alternating)", "direct": "Direct (faces only)"}


def config_of(case, remap, world, parallelism=None):
    """The `config` object, identical for the product and the reference arm."""
    return {"workload": case.name, "cells": case.cells, "materials": case.cfg.nmat, "cfl": case.cfl,
            "options": "sliver-energy safeguard (H2D_OPT_SLIVER_ENERGY)" if case.cfg.options else "none",
            "scheme": SCHEMES.get(remap, "DirectCF") + " face_order=2 LinearDiag interface_degrade",
            "steps_from": "t=0 (+ warm-up steps)",
            "parallelism": parallelism or ("replicas" if world > 1 else "single"),
            "l2": "512 MiB write between timed device steps; per-step working set >> 126 MB L2"}


def ncu_traffic(workload, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed ncu launch list of the workload (profiles/)."""
    tf = os.path.join(ROOT, "profiles", "traffic_per_launch.json")
    try:
        with open(tf) as f:
            rec = json.load(f).get(workload, {})
        return rec.get(kernel), rec.get("_source")
    except Exception:
        return None, None


def cpu_sample(name, case):
    """The case the CPU legs time: the workload itself, except c5, whose
    16384^2 three-material State does not fit a host process of the C
    restatement: its lower-left 2048^2 block (same cells, same sites)."""
    if name == "c5" and case.cfg.mesh.nx > 4096:
        from paper_2208_13409_b200 import cases
        return c5_case(cases.voronoi3(2048, 2048, n_full=case.cfg.mesh.nx)), "lower-left 2048^2 block of the mesh, "
    return case, ""


def time_cpu(case, warm, steps, remap_kind=None):
    """Wall-clock the CPU implementation on `steps` steps after `warm`."""
    from paper_2208_13409_b200 import abi
    lib, lib_kind = cpu_lib(case.cfg.nmat)
    rk = abi.REMAP_DIRECTCF if remap_kind is None else remap_kind
    s = abi.Solver(lib, case.cfg)
    s.init_from(case.paint())
    if warm:
        s.run(warm, cfl=case.cfl, log_dt=False, kind=rk)
    t0 = time.perf_counter()
    r = s.run(warm + steps, cfl=case.cfl, log_dt=False, kind=rk)
    dt = time.perf_counter() - t0
    return case.cells * r.steps_done / dt, lib_kind, r.steps_done, dt


def pinned_state(nx, ny, nmat, cv):
    """HostState whose arrays live in page-locked memory (torch is plumbing)."""
    import torch
    from paper_2208_13409_b200.abi import HostState
    st = HostState.empty(nx, ny, nmat, cv)
    for f in ("m", "e", "k", "vol", "m_mix", "e_mix", "rho_mix", "p_mix", "iface_normal", "u"):
        a = getattr(st, f)
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        setattr(st, f, t.numpy())
    st._pins = True
    return st


def run_product(args, world, rank, local, pg):
    from paper_2208_13409_b200 import abi as _abi
    kind = {"ad": _abi.REMAP_AD, "direct": _abi.REMAP_DIRECT}.get(args.remap, _abi.REMAP_DIRECTCF)
    import paper_2208_13409_b200 as pkg
    from paper_2208_13409_b200 import abi

    case = workload(args.workload)
    nmat = case.cfg.nmat
    lib = pkg.product_library()
    s = abi.Solver(lib, case.cfg, local)
    painted = case.paint()
    s.init_from(painted)
    for _ in range(args.warmup):
        s.step_timed(case.cfl, kind=kind)
    clocks = Clocks(local)
    barrier(pg)
    clocks.start()
    launches0 = lib.fn["launch_count"]()
    tot = 0.0
    for _ in range(args.steps):
        s.flush_l2(512 << 20)
        tot += s.step_timed(case.cfl, kind=kind)["total"]
    launches = lib.fn["launch_count"]() - launches0
    # kernel-group split: the same steps as plain launches with CUDA events on
    # the launching stream between the groups (k_remap_tile is timed alone)
    ph = {k: 0.0 for k in abi.Solver.STEP_GROUPS}
    n_ph = max(3, min(args.steps, 10))
    for _ in range(n_ph):
        s.flush_l2(512 << 20)
        for k, v in s.step_timed(case.cfl, phases=True, kind=kind).items():
            ph[k] += v / n_ph
    clk = clocks.stop()
    barrier(pg)
    total_s = max_over_ranks(pg, tot / 1e3)
    cells = case.cells
    value = cells * args.steps * world / total_s
    ms_step = total_s * 1e3 / args.steps
    peak, peak_kind = hbm_peak()
    achieved_step = B_MIN[nmat] * cells / (ms_step / 1e3) / 1e9
    kern = {}
    for grp, (kname, nbytes) in KERNEL_BYTES.items():
        if kind == abi.REMAP_AD and grp != "lagrange":  # the AD remap + post share one timed group
            continue
        kms = max_over_ranks(pg, ph[grp])
        ach = nbytes[nmat] * cells / (kms / 1e3) / 1e9
        label = f"{kname}<{nmat}>"
        if grp == "remap_tile" and nmat == 3:  # per-tile material classes: one launch per slot count
            label = "k_remap_tile<1|2|3> (class launches)"
        kern[grp] = {"kernel": label, "ms": kms, "bytes_per_cell": nbytes[nmat],
                     "achieved": ach, "frac": ach / peak,
                     "share_of_step": kms / ph["total"] if ph["total"] > 0 else None}
    dom = max(kern, key=lambda g: kern[g]["ms"])
    dom_name = kern[dom]["kernel"].split("<")[0]
    traffic, traffic_src = ncu_traffic(args.workload, dom_name)
    # the dominant kernel against the HBM roofline: algorithmic bytes =
    # SURVEY 8d's B_min per cell-step x the cells one launch covers, over the
    # launch's CUDA-event time; its measured DRAM traffic (ncu) beside it
    dom_ms = kern[dom]["ms"]
    dom_alg = B_MIN[nmat] * cells / (dom_ms / 1e3) / 1e9

    # end to end through the public API with host (pinned) State buffers.
    # (1) e2e: the reference's hot-loop call -- run(State, K steps) -- on a host
    #     State: upload, K device steps, download, all inside the timed region;
    # (2) e2e_per_step_api: the value API every step (upload State -> one step
    #     -> download State), i.e. a caller that keeps its State on the host.
    s.close()  # one context at a time (a 16384^2 three-material context takes ~161 GB)
    se = abi.Solver(lib, case.cfg, local)
    se.init_from(painted)
    se.run(1, cfl=case.cfl, log_dt=False, kind=kind)  # one-time setup (graph capture) outside the timed region
    se.init_from(painted)
    pinned = cells <= (1 << 27)  # a 16384^2 three-material State (39 GB) stays in pageable memory
    if pinned:
        host = pinned_state(case.cfg.mesh.nx, case.cfg.mesh.ny, nmat, case.cfg.mesh.dx * case.cfg.mesh.dy)
    else:
        from paper_2208_13409_b200.abi import HostState
        host = HostState.empty(case.cfg.mesh.nx, case.cfg.mesh.ny, nmat, case.cfg.mesh.dx * case.cfg.mesh.dy)
    st0 = se.download()
    fields = ("m", "e", "k", "vol", "m_mix", "e_mix", "rho_mix", "p_mix", "iface_normal", "u")
    for f in fields:
        getattr(host, f)[...] = getattr(st0, f)
    def nbytes(fs):
        return sum(getattr(host, f)[:nmat].nbytes if f in ("m", "e", "k") else getattr(host, f).nbytes for f in fs)
    # upload: the primary State (m, e, k, normals, u); the device rebuilds the
    # derived fields with sync_derived (state.cpp:120-143, h2d.h upload
    # contract), bit-identical to uploading them. download: the whole State.
    up_bytes = nbytes(("m", "e", "k", "iface_normal", "u"))
    state_bytes = nbytes(fields)

    def upload():
        v = host.view(derived=False)
        se._check(lib.fn["upload_state"](se._h, abi.C.byref(v)))

    def download():
        v = host.view(derived=True)
        se._check(lib.fn["download_state"](se._h, abi.C.byref(v)))
        host.step, host.time = v.step, v.time

    barrier(pg)
    t0 = time.perf_counter()
    upload()
    se.run(host.step + args.steps, cfl=case.cfl, log_dt=False, kind=kind)
    download()
    e2e_run_s = max_over_ranks(pg, time.perf_counter() - t0)
    e2e_value = cells * args.steps * world / e2e_run_s
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    barrier(pg)
    t0 = time.perf_counter()
    for q in range(e2e_steps):
        upload()
        se.run(host.step + 1, cfl=case.cfl, log_dt=False, kind=kind)
        download()
    e2e_s = max_over_ranks(pg, time.perf_counter() - t0)
    e2e_step_value = cells * e2e_steps * world / e2e_s

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (init_case-equivalent painter, seeded)",
        "config": config_of(case, args.remap, world),
        "phases_ms": dict(ph, note=f"{n_ph} un-graphed steps after the timed ones, CUDA events between "
                                    "kernel groups on the launching stream"),
        "roofline": {"bound": "hbm", "achieved": dom_alg, "peak": peak, "unit": "GB/s",
                     "frac": dom_alg / peak, "traffic": traffic, "peak_source": peak_kind,
                     "kernel": kern[dom]["kernel"], "kernel_ms": dom_ms,
                     "share_of_step": kern[dom]["share_of_step"],
                     "basis": f"algorithmic {B_MIN[nmat]} B/cell-step (SURVEY 8d B_min) x {cells} cells per "
                              f"launch / CUDA-event time of the launch",
                     "dram_achieved": traffic / (dom_ms / 1e3) / 1e9 if traffic else None,
                     "dram_frac": traffic / (dom_ms / 1e3) / 1e9 / peak if traffic else None,
                     "traffic_source": traffic_src,
                     "kernel_boundary": {"bytes_per_cell": kern[dom]["bytes_per_cell"],
                                         "achieved": kern[dom]["achieved"], "frac": kern[dom]["frac"]},
                     "kernels": kern},
        "step_roofline": {"bound": "hbm", "achieved": achieved_step, "peak": peak, "unit": "GB/s",
                          "frac": achieved_step / peak,
                          "basis": f"whole step: {B_MIN[nmat]} B/cell-step (state read+write once, "
                                   f"SURVEY 8d) x {cells} cells"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": up_bytes / args.steps,
                "d2h_bytes_per_step": state_bytes / args.steps, "steps": args.steps,
                "path": "run(State, K steps) on a pinned host State: h2d_upload_state (primary fields; "
                        "derived rebuilt on the device) + h2d_run(K) + h2d_download_state (whole State), wall "
                        "clock (the reference's hot-loop call, harness.cpp:380-424)"},
        "e2e_per_step_api": {"value": e2e_step_value, "unit": UNIT, "h2d_bytes_per_step": up_bytes,
                             "d2h_bytes_per_step": state_bytes, "steps": e2e_steps,
                             "path": "every step: h2d_upload_state + h2d_run(1 step) + h2d_download_state"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # a bounded sample: about 3e7 cell-updates (10-30 s of one core)
        sc, where = cpu_sample(args.workload, case)
        v, ckind, n, secs = time_cpu(sc, 0, min(args.cpu_steps, max(1, int(3e7 // sc.cells))), kind)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": ckind, "cpu": cpu_model(),
                                "nproc": os.cpu_count(),
                                "sample": f"{case.name}: {where}first {n} steps from t=0, single thread, "
                                          f"{secs:.1f} s"}
    if rank == 0:
        emit(line)


def run_product_multi(args, world, rank, local, pg):
    """N > 1: the workload's global mesh split into px x py blocks (strong
    scaling: the same problem as N = 1), one block per rank. Each rank paints
    and initialises only its own window (h2d_block_init_window); the whole
    run loop, with ONE max all-reduce of four control words and ONE halo
    exchange (8 neighbours, corners included) per step, runs inside the
    library over an NCCL communicator it owns (h2d_comm_nccl +
    h2d_blocks_run: device-side combine, exchange overlapped with the
    Lagrange tiles on owned data, host polling every 16 steps)."""
    import torch
    import paper_2208_13409_b200 as pkg
    from paper_2208_13409_b200 import multi

    case = workload(args.workload, full=True)
    nx, ny, nmat = case.cfg.mesh.nx, case.cfg.mesh.ny, case.cfg.nmat
    px, py = multi.grid_shape(world, nx, ny)
    lib = pkg.product_library()
    spec = multi.decompose(nx, ny, px, py)[rank]
    blk = multi.BlockSolver(lib, case.cfg, spec, local)
    t_paint = time.perf_counter()
    win = case.paint(blk.window())
    t_paint = time.perf_counter() - t_paint
    # the NCCL id travels once through torch.distributed (plumbing)
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(multi.DeviceComm.unique_id(lib)), dtype=torch.uint8))
    if pg is not None:
        pg.broadcast(uid, 0)
    comm = multi.DeviceComm([blk], px, py, nccl_id=bytes(uid.cpu().numpy().tobytes()), rank=rank)
    # e2e (the timed region includes the host -> device upload of this rank's
    # painted window, the run and the download of the owned State)
    barrier(pg)
    t0 = time.perf_counter()
    blk.init_window(win)
    from paper_2208_13409_b200 import abi as _abi
    if args.remap == "direct":
        raise SystemExit("block mode runs the DirectCF and AD remaps")
    kind = _abi.REMAP_AD if args.remap == "ad" else _abi.REMAP_DIRECTCF
    comm.run(args.warmup, 1e30, case.cfl, kind=kind)
    warm_ms = comm.device_ms
    clocks = Clocks(local)
    clocks.start()
    launches0 = lib.fn["launch_count"]()
    done = comm.run(args.warmup + args.steps, 1e30, case.cfl, kind=kind)  # the steps of this call
    dev_ms = comm.device_ms
    launches = lib.fn["launch_count"]() - launches0
    clk = clocks.stop()
    from paper_2208_13409_b200.abi import HostState
    own = HostState.empty(nx, ny, nmat) if nx * ny <= (1 << 26) else None
    if own is not None:
        blk.download_into(own)
    e2e_s = max_over_ranks(pg, time.perf_counter() - t0)
    barrier(pg)
    total_s = max_over_ranks(pg, dev_ms / 1e3)
    cells = case.cells
    value = cells * done / total_s
    ms_step = total_s * 1e3 / max(done, 1)
    peak, peak_kind = hbm_peak()
    per_gpu = spec.bnx * spec.bny
    achieved = B_MIN[nmat] * per_gpu / (ms_step / 1e3) / 1e9
    halo_doubles = sum(blk.halo_bytes(dx, dy, 1) for dx, dy in multi.DIRS
                       if spec.neighbour(px, py, dx, dy) is not None) // 8
    comm.close()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": done, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (init_case-equivalent painter, seeded; each rank paints its own window)",
        "config": config_of(case, args.remap, world,
                            parallelism=f"2D blocks {px}x{py}, halo {blk.halo}; per step 1 NCCL max all-reduce "
                                        f"(4 words) + {2 if args.remap == 'ad' else 1} grouped NCCL halo "
                                        f"exchange(s), in the library"),
        "cells_per_gpu": per_gpu, "halo_doubles_sent_rank0": halo_doubles, "paint_s_rank0": t_paint,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_source": peak_kind,
                     "basis": f"per GPU: {B_MIN[nmat]} B/cell-step x {per_gpu} owned cells / step time"},
        "e2e": {"value": cells * (args.warmup + done) / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": (win.m[:nmat].nbytes * 3 + win.u.nbytes) / (args.warmup + done),
                "d2h_bytes_per_step": (sum(getattr(own, f).nbytes for f in ("m", "e", "k", "vol", "m_mix", "e_mix",
                                                                        "rho_mix", "p_mix", "iface_normal", "u"))
                                       / (args.warmup + done)) if own is not None else 0,
                "path": "h2d_block_init_window (painted window up) + h2d_blocks_run (warm-up + timed steps) + "
                        "h2d_block_download (owned State down), wall clock, max over ranks"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rank == 0:
        emit(line)


def run_reference(args, world, rank, pg):
    if rank != 0:
        return
    from paper_2208_13409_b200 import abi
    case = workload(args.workload)
    sc, where = cpu_sample(args.workload, case)
    # a bounded sample: about 1.2e8 cell-updates (~1 min of one core), at
    # least one step; warm-up steps only where they fit the same budget
    budget = max(1, int(1.2e8 // sc.cells))
    steps = max(1, min(args.steps, budget))
    warm = min(args.warmup, budget - steps)
    rk = {"ad": abi.REMAP_AD, "direct": abi.REMAP_DIRECT}.get(args.remap, abi.REMAP_DIRECTCF)
    v, ckind, n, secs = time_cpu(sc, warm, steps, rk)
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": n, "warmup": warm,
        "ms_per_step": secs * 1e3 / max(n, 1), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (init_case-equivalent painter, seeded)", "impl": "reference",
        "config": config_of(case, args.remap, 1),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": ckind, "cpu": cpu_model(),
                         "nproc": os.cpu_count(),
                         "sample": f"{case.name}: {where}steps {warm + 1}..{warm + n} of the workload, single "
                                   f"thread (the reference has no threading), {secs:.1f} s"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


_OUT = None


def quiet_stdout():
    """Keep stdout for the ONE JSON line: file descriptor 1 is pointed at
    stderr for the rest of the run, so a library that writes to the C stdout
    (NCCL prints its version banner there) cannot add lines to it."""
    global _OUT
    if _OUT is None:
        sys.stdout.flush()
        _OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line):
    out = _OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    quiet_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--remap", default="directcf", choices=["directcf", "ad", "direct"],
                    help="remap engine: DirectCF (the path), the AD split scheme or the Direct faces-only "
                         "engine (SURVEY 8f)")
    ap.add_argument("--cpu-steps", type=int, default=10)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--blocks", action="store_true",
                    help="run the block-decomposition data plane (NCCL, per-rank painting) even on one GPU")
    args = ap.parse_args()
    world, rank, local, pg = dist_setup(args.gpus)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank, pg)
        elif world > 1 or args.blocks:
            run_product_multi(args, world, rank, local, pg)
        else:
            run_product(args, world, rank, local, pg)
    finally:
        if pg is not None:
            pg.destroy_process_group()


if __name__ == "__main__":
    main()

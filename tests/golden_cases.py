"""Recipes of the golden fixtures (tests/golden/*.npz): initial state + the
ABI call sequence.  Shared by make_golden.py (reference), test_golden.py
(oracle on CPU, product on GPU)."""
import numpy as np

import helpers
from paper_2208_13409_b200 import abi, cases, errors
from paper_2208_13409_b200.abi import BC_PERIODIC, BC_WALL, CORNER_LINEARDIAG, CORNER_UPWIND, EOS_PERFECT, \
    EOS_STIFFENED, make_config


def _run(steps, cfl, t_end=1e30):
    def act(s):
        r, err = helpers.run_capture(s, steps, cfl, t_end=t_end)
        return {"dts": r.dts, "counters": [r.floor_count, r.diag["k_clip_count"], r.diag["mass_fix_count"],
                                           r.diag["max_k_violation"]]}, err
    return act


def _kinematic(dt, vel=True):
    def act(s):
        lag = helpers.kinematic(s.download())
        s.set_lagrange(lag)
        d = abi.RemapDiag()
        err = None
        try:
            s.remap_step(dt, remap_velocity=vel, diag=d)
        except errors.SimError as e:
            err = (type(e).__name__, e.what, e.i, e.j, e.step, e.in_step)
        return {"dts": np.array([dt]), "counters": [0, d.k_clip_count, d.mass_fix_count, d.max_k_violation]}, err
    return act


def _lagrange_remap(nsteps, cfl):
    def act(s):
        dts = []
        d = abi.RemapDiag()
        for q in range(nsteps):
            dt = s.cfl_dt(cfl)
            dts.append(dt)
            s.lagrange_step(dt, download=False)
            s.remap_step(dt, diag=d)
        return {"dts": np.array(dts), "counters": [0, d.k_clip_count, d.mass_fix_count, d.max_k_violation]}, None
    return act


GOLDEN = ["riemann2d_48", "sedov_64", "triple_point_64x32", "triple_point_32x16_abort", "shock_bubble_48",
          "kinematic_gas_periodic", "kinematic_blobs_wall_upwind_error", "kinematic_blobs_wall_upwind",
          "lagrange_blobs_stiffened", "impact_full_abort"]


def build(name):
    if name == "riemann2d_48":
        c = cases.riemann2d(48)
        return c.cfg, c.paint(), _run(100, c.cfl)
    if name == "sedov_64":
        c = cases.sedov(64)
        return c.cfg, c.paint(), _run(60, c.cfl)
    if name == "triple_point_64x32":
        c = cases.triple_point(64, 32)
        return c.cfg, c.paint(), _run(1000, c.cfl)
    if name == "triple_point_32x16_abort":
        c = cases.triple_point(32, 16)
        return c.cfg, c.paint(), _run(1000, c.cfl)
    if name == "shock_bubble_48":
        c = cases.shock_bubble(48)
        return c.cfg, c.paint(), _run(30, c.cfl)
    if name == "kinematic_gas_periodic":
        cfg = make_config(16, 12, 1.0, 1.0, 0.0, 0.0, BC_PERIODIC, BC_PERIODIC)
        return cfg, helpers.random_state(cfg, 101, "gas", umax=0.3), _kinematic(1.0)
    if name in ("kinematic_blobs_wall_upwind_error", "kinematic_blobs_wall_upwind"):
        cfg = make_config(20, 18, 0.05, 0.05, 0.0, 0.0, BC_WALL, BC_WALL, eos=[(EOS_PERFECT, 1.4, 0.0)] * 2,
                          corner=CORNER_UPWIND)
        return cfg, helpers.random_state(cfg, 102, "blobs", umax=0.3), _kinematic(
            0.1 if name.endswith("error") else 0.02)
    if name == "lagrange_blobs_stiffened":
        cfg = make_config(24, 20, 0.5, 0.25, 0.0, 0.0, BC_WALL, BC_PERIODIC,
                          eos=[(EOS_PERFECT, 1.4, 0.0), (EOS_STIFFENED, 7.0, 0.5)], corner=CORNER_LINEARDIAG)
        return cfg, helpers.random_state(cfg, 103, "blobs", umax=0.05), _lagrange_remap(4, 0.4)
    if name == "impact_full_abort":
        # the reference's own robustness case at full size (acceptance.cpp
        # criterion 7): impact / DirectCF aborts with
        # UnphysicalStateError after ~3000 steps
        from paper_2208_13409_b200 import frontend
        cs = frontend.build_case(name.split("_")[0])
        cfg = cs.config()
        return cfg, cases.paint(cfg, cs.regions), _run(0, cs.cfl, cs.t_end)
    raise KeyError(name)

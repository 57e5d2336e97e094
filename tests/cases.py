"""Parity case specs shared by the golden generator, the oracle tests and the
GPU parity tests.

A case is a plain dict; ``build(case, mods)`` turns it into
(config, cost, model, track, noise, x0, cov0, plan) using either the
reference modules (golden generation, build container only) or this repo's
host mirror (tests) -- both expose the same names.
"""

from __future__ import annotations

import math

import numpy as np

ELLIPSE_SIGMA_EPS = [[0.2 ** 2, 0.0], [0.0, 0.5 ** 2]]


def _seeded_scalars(seed, track_length):
    """Per-seed scalars, drawn in the order of SURVEY.md 8d: the three
    process-noise stds ~ U[0.01, 0.05], then s0 ~ U[0, L)."""
    rng = np.random.default_rng(seed)
    stds = rng.uniform(0.01, 0.05, 3)
    s0 = rng.uniform(0.0, track_length)
    return stds, s0


def c1_case(seed, K=256, M=32, T=20, dt=0.05, track="ellipse", warm=1, **kw):
    """BASELINE config 1: ellipse, K=256, M=32, T=20; one warm-start
    iteration from the zero plan, then the captured iteration."""
    c = dict(name=f"c1_s{seed}", track=track, K=K, M=M, T=T, dt=dt, seed=seed,
             run_path=[5, seed], warm=warm, sigma_eps=ELLIPSE_SIGMA_EPS,
             noise="seeded", x0="seeded", kind="bss", persist=False)
    c.update(kw)
    return c


CASES = [
    c1_case(0),
    c1_case(1),
    c1_case(2),
    # zero process noise + zero cov: the belief collapses onto the deterministic
    # Euler step; BSS == S-MPPI (reference test_controllers.py:232-245)
    dict(name="collapse_m2", track="oval", K=16, M=2, T=10, dt=0.05, seed=11, run_path=[],
         warm=1, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.0, 0.0, 0.0],
         x0=dict(vx=4.0, s=16.0, e_y=0.8), kind="bss", persist=False),
    dict(name="collapse_m16", track="oval", K=16, M=16, T=10, dt=0.05, seed=11, run_path=[],
         warm=0, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.0, 0.0, 0.0],
         x0=dict(vx=4.0, s=16.0, e_y=0.8), kind="bss", persist=False),
    # e_y beyond the local turn radius on the arc -> every rollout +inf
    # (reference test_controllers.py:185-191); the update raises.
    dict(name="dead", track="oval", K=8, M=4, T=3, dt=0.05, seed=3, run_path=[],
         warm=0, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.05, 0.05, 0.1],
         x0=dict(vx=3.0, s=25.0, e_y=6.5), kind="bss", persist=False),
    # plan pinned at the bounds: the clamp acts on most samples
    # (reference test_controllers.py:65-73)
    dict(name="clamp", track="ellipse", K=64, M=16, T=12, dt=0.05, seed=4, run_path=[5, 4],
         warm=0, plan=[0.35, 1.0], sigma_eps=[[0.2 ** 2, 0], [0, 0.5 ** 2]],
         noise="seeded", x0="seeded", kind="bss", persist=False),
    # persistent particles (controllers.py:288-305)
    dict(name="persist", track="oval", K=32, M=16, T=12, dt=0.05, seed=22, run_path=[1],
         warm=1, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.15, 0.15, 0.3],
         x0=dict(vx=4.0, s=4.0), kind="bss", persist=True),
    # non-ascending sigma_eps diagonal: eigh factor is column-permuted
    dict(name="permuted", track="ellipse", K=64, M=8, T=10, dt=0.05, seed=6, run_path=[5, 6],
         warm=1, sigma_eps=[[0.5 ** 2, 0], [0, 0.2 ** 2]], noise="seeded", x0="seeded",
         kind="bss", persist=False),
    # ragged inner sample counts (not a power of two), non-diagonal noise
    dict(name="ragged_m5", track="oval", K=40, M=5, T=8, dt=0.05, seed=8, run_path=[2],
         warm=1, sigma_eps=[[0.15 ** 2, 0.01], [0.01, 0.35 ** 2]],
         noise=[[0.05 ** 2, 0.0005, 0.0], [0.0005, 0.05 ** 2, 0.0], [0.0, 0.0, 0.1 ** 2]],
         x0=dict(vx=3.0, s=5.0, e_y=0.3), kind="bss", persist=False),
    dict(name="ragged_m50", track="stadium", K=100, M=50, T=20, dt=0.05, seed=9, run_path=[3],
         warm=1, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.15, 0.15, 0.3],
         x0=dict(vx=2.0, s=1.0), kind="bss", persist=False),
    # the reference's default experiment controller (default.cfg, sim.py:90-92)
    dict(name="default_bss", track="stadium", K=256, M=16, T=20, dt=0.05, seed=0,
         run_path=[5, 0], warm=2, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]],
         noise=[0.15, 0.15, 0.3], x0=dict(vx=2.0, s=0.0), kind="bss", persist=False),
    # nonzero initial belief covariance
    dict(name="cov0", track="oval", K=32, M=64, T=10, dt=0.05, seed=12, run_path=[4],
         warm=0, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.05, 0.05, 0.1],
         x0=dict(vx=4.0, s=30.0, e_y=1.0, e_psi=0.1),
         cov0=[[0.01, 0, 0, 0], [0, 0.02, 0, 0.001], [0, 0, 0.003, 0], [0, 0.001, 0, 0.04]],
         kind="bss", persist=False),
    # C3 shape slice: spline track, M=256, T=50, dt=0.04 (moment headroom)
    dict(name="c3_slice", track="spline0", K=32, M=256, T=50, dt=0.04, seed=0, run_path=[5, 0],
         warm=0, sigma_eps=ELLIPSE_SIGMA_EPS, noise=[0.05, 0.05, 0.05], x0="seeded",
         kind="bss", persist=False),
    # rare branches of the step against the reference: the arc-length wrap
    # (s just below L), the heading wrap (e_psi near pi, driving backwards
    # along s so s also wraps below 0), the low-speed floor (vx < v_floor)
    # and reverse driving (vx_eff < 0: the atan2 +-pi branch)
    dict(name="s_wrap", track="oval", K=48, M=16, T=12, dt=0.05, seed=31, run_path=[6],
         warm=1, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.05, 0.05, 0.1],
         x0=dict(vx=5.0, s_frac=0.995, e_y=0.2), kind="bss", persist=False),
    dict(name="heading_wrap", track="oval", K=48, M=16, T=12, dt=0.05, seed=32, run_path=[6],
         warm=0, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.05, 0.05, 0.1],
         x0=dict(vx=2.0, s_frac=0.002, e_psi=3.05, e_y=-0.3), kind="bss", persist=False),
    dict(name="low_speed", track="ellipse", K=48, M=16, T=12, dt=0.05, seed=33, run_path=[6],
         warm=1, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.02, 0.02, 0.05],
         x0=dict(vx=0.15, s=10.0), kind="bss", persist=False),
    dict(name="reverse", track="ellipse", K=48, M=16, T=10, dt=0.05, seed=34, run_path=[6],
         warm=0, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.02, 0.02, 0.05],
         x0=dict(vx=-2.0, s=20.0, e_y=0.2), plan=[0.05, -0.5], kind="bss", persist=False),
    # every cost term away from its default: all eight tracking weights,
    # goal speed, lane-exit penalty, terminal scale, CBF rate / penalty and
    # back-off (controllers.py:108-138, constraints.py:22-33)
    dict(name="custom_cost", track="ellipse", K=64, M=24, T=15, dt=0.05, seed=35, run_path=[7],
         warm=1, sigma_eps=[[0.2 ** 2, 0], [0, 0.5 ** 2]], noise=[0.03, 0.03, 0.06],
         x0=dict(vx=4.5, s=12.0, e_y=0.9, e_psi=0.05), kind="bss", persist=False,
         cost=dict(q_diag=[3.0, 0.5, 0.1, 1e-4, 2e-4, 1.5, 0.8, 0.01], v_goal=4.0,
                   obstacle_penalty=500.0, terminal_scale=3.0,
                   safety=dict(cbf_rate=0.2, penalty=700.0), backoff=2.5)),
    # every vehicle parameter away from its default (the 23-value physics
    # vector: mass, inertia, geometry, wheels, all eight magic-formula B/C,
    # the four peaks, drive gain, rolling resistance, low-speed floor)
    dict(name="custom_vehicle", track="oval", K=64, M=24, T=15, dt=0.04, seed=36, run_path=[7],
         warm=1, sigma_eps=[[0.2 ** 2, 0], [0, 0.5 ** 2]], noise=[0.03, 0.03, 0.06],
         x0=dict(vx=3.5, s=8.0, e_y=-0.4), kind="bss", persist=False,
         vehicle=dict(mass=18.0, inertia_z=0.9, lf=0.22, lr=0.28, wheel_radius=0.11, wheel_inertia=0.3,
                      b_lat_front=5.0, c_lat_front=1.4, b_lat_rear=3.5, c_lat_rear=1.2,
                      b_long_front=2.5, c_long_front=1.6, b_long_rear=1.8, c_long_rear=1.5,
                      peak_fx_front=90.0, peak_fy_front=100.0, peak_fx_rear=110.0, peak_fy_rear=95.0,
                      drive_gain=10.0, roll_resist=0.02, v_floor=0.4)),
    # wide lateral shape factors (C = 1.9 / 1.7): a different per-vehicle
    # tire table (csrc/bssmppi.cu tire_table_host) than the default tire
    dict(name="wide_tire", track="ellipse", K=64, M=24, T=15, dt=0.05, seed=38, run_path=[7],
         warm=1, sigma_eps=[[0.2 ** 2, 0], [0, 0.5 ** 2]], noise=[0.03, 0.03, 0.06],
         x0=dict(vx=5.0, s=14.0, e_y=0.3), kind="bss", persist=False,
         vehicle=dict(c_lat_front=1.9, c_lat_rear=1.7)),
    # an open track: the arc length clamps at L instead of wrapping
    dict(name="open_track", track="open60", K=48, M=16, T=15, dt=0.05, seed=37, run_path=[7],
         warm=1, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.03, 0.03, 0.06],
         x0=dict(vx=5.0, s=57.0, e_y=0.2), kind="bss", persist=False),
    # deterministic kinds through the same kernel
    dict(name="smppi", track="oval", K=48, M=1, T=10, dt=0.05, seed=11, run_path=[],
         warm=2, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.0, 0.0, 0.0],
         x0=dict(vx=3.0, s=1.0), kind="smppi", persist=False, temperature=5.0),
    dict(name="mppi", track="ellipse", K=64, M=1, T=20, dt=0.05, seed=7, run_path=[],
         warm=1, sigma_eps=[[0.15 ** 2, 0], [0, 0.35 ** 2]], noise=[0.0, 0.0, 0.0],
         x0="seeded", kind="mppi", persist=False, temperature=2.0),
]


def case_by_name(name):
    for c in CASES:
        if c["name"] == name:
            return c
    raise KeyError(name)


def build(case, mods):
    """Instantiate the case with module namespace ``mods`` (attributes:
    VehicleParams, VehicleState, NoiseModel, CostSpec, MppiConfig,
    make_test_track, with_timestep)."""
    from paper_2408_00494_b200.tracks import named_track

    if case["track"] == "open60":
        # an open (non-closing) track: s is clamped to [0, L] instead of wrapped
        s_pts = np.linspace(0.0, 60.0, 121)
        track = mods.Track(s=s_pts, kappa=0.03 * np.sin(s_pts / 9.0), half_width=2.0, closed=False,
                           length=60.0)
    else:
        track = named_track(case["track"], build=mods.make_test_track)
    model = mods.with_timestep(mods.VehicleParams(**case.get("vehicle", {})), case["dt"], "euler")
    stds, s0 = _seeded_scalars(case["seed"], track.length)
    nz = case["noise"]
    if nz == "seeded":
        ncov = np.diag(stds ** 2)
    else:
        arr = np.asarray(nz, dtype=float)
        ncov = np.diag(arr ** 2) if arr.ndim == 1 else arr
    noise = mods.NoiseModel(ncov)
    if case["x0"] == "seeded":
        x0 = mods.VehicleState.rolling(5.0, model, s=s0).as_array()
    else:
        kw = dict(case["x0"])
        vx = kw.pop("vx")
        if "s_frac" in kw:
            kw["s"] = kw.pop("s_frac") * track.length
        x0 = mods.VehicleState.rolling(vx, model, **kw).as_array()
    cov0 = np.asarray(case.get("cov0", np.zeros((4, 4))), dtype=float)
    cfg = mods.MppiConfig(kind=case["kind"], samples=case["K"], horizon=case["T"],
                          temperature=case.get("temperature", 1.0),
                          sigma_eps=np.asarray(case["sigma_eps"], dtype=float),
                          inner_samples=max(case["M"], 2),
                          persist_particles=case["persist"])
    cost_kw = dict(case.get("cost", {}))
    if "safety" in cost_kw:
        cost_kw["safety"] = mods.SafetyParams(**cost_kw["safety"])
    if "q_diag" in cost_kw:
        cost_kw["q_diag"] = np.asarray(cost_kw["q_diag"], dtype=float)
    cost = mods.CostSpec(**cost_kw)
    plan = None
    if "plan" in case:
        plan = np.tile(np.asarray(case["plan"], dtype=float), (case["T"], 1))
    return cfg, cost, model, track, noise, x0, cov0, plan


UPDATE_BATCHES = [(64, 6, 0.7, 0), (256, 20, 1.0, 17), (1000, 50, 5.0, 3), (128, 5, 1e-3, 0)]


def update_batch(j):
    """Seeded random update-law batch j (reference test_controllers.py:86-147
    style): uniform costs with some +inf, random controls beyond the bounds."""
    K, T, lam, n_inf = UPDATE_BATCHES[j]
    rng = np.random.default_rng(100 + j)
    costs = rng.uniform(0.0, 50.0, K)
    costs[rng.choice(K, n_inf, replace=False)] = np.inf
    controls = rng.uniform(-0.6, 1.2, size=(K, T, 2))
    return costs, controls, lam


# Closed-loop cases (reference sim.run_closed_loop, sim.py:232-309): the C2
# setting (ellipse, dt 0.05, plant RK4 at 0.01) at parity-test sizes.
CLOSED_LOOP = [
    dict(name="cl_bss", K=256, M=32, T=20, steps=60, seed=3, run=0, noise_std=0.05,
         init_speed=3.0, track="ellipse"),
    dict(name="cl_bss_r1", K=256, M=32, T=20, steps=60, seed=3, run=1, noise_std=0.05,
         init_speed=3.0, track="ellipse"),
]


def build_closed_loop(case, mods, sim_mod):
    """ExperimentConfig for a closed-loop case in either module namespace
    (mods: dynamics/controller types; sim_mod: the sim module)."""
    from paper_2408_00494_b200.tracks import named_track

    track = named_track(case["track"], build=mods.make_test_track)
    cfg = mods.MppiConfig(kind="bss", samples=case["K"], horizon=case["T"], inner_samples=case["M"],
                          sigma_eps=np.asarray(ELLIPSE_SIGMA_EPS))
    noise = mods.NoiseModel(np.diag([case["noise_std"] ** 2] * 3))
    kw = dict(controller=cfg, cost=mods.CostSpec(), vehicle=mods.VehicleParams(), track=track,
              noise=noise, dt_control=0.05, dt_plant=0.01, master_seed=case["seed"],
              max_steps=case["steps"], init_speed=case["init_speed"], collision_threshold=1.2)
    return sim_mod.ExperimentConfig(**kw)

"""Generate golden vectors by running the REFERENCE package (build container
only; /root/reference does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

For every case in ``tests/cases.py`` it builds the reference Controller,
runs the warm-start iterations, then captures one ``control_step``:
the per-step belief moments (by wrapping ``controllers.propagate_mc_batch``
/ ``propagate_particles_batch``, bound at reference controllers.py:16-23),
the rollout costs (by wrapping ``controllers.mppi_update``), v+ and the
next plan.  Noise is NOT stored: tests redraw it from the reference's own
keyed numpy substreams (streams.py:21-28) and a checksum stored here
detects a numpy stream change.  Also writes update-law vectors for
``mppi_update`` (controllers.py:180-194).
"""

import json
import os
import sys
import types
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent))

import belief_mppi.controllers as rc  # noqa: E402
from belief_mppi import dynamics as rd  # noqa: E402
from belief_mppi.streams import substream  # noqa: E402

from cases import CASES, CLOSED_LOOP, UPDATE_BATCHES, build, build_closed_loop, update_batch  # noqa: E402
from belief_mppi import sim as rsim  # noqa: E402

from belief_mppi.constraints import SafetyParams as RefSafetyParams  # noqa: E402

REF = types.SimpleNamespace(
    VehicleParams=rd.VehicleParams, VehicleState=rd.VehicleState, NoiseModel=rd.NoiseModel,
    CostSpec=rc.CostSpec, MppiConfig=rc.MppiConfig, make_test_track=rd.make_test_track,
    with_timestep=rd.with_timestep, SafetyParams=RefSafetyParams, Track=rd.Track)


def noise_checksums(case, it):
    """Checksums of the captured iteration's eps/z draws."""
    K, T, M = case["K"], case["T"], case["M"]
    rp = tuple(case["run_path"])
    zc = substream(case["seed"], *rp, 2, it).standard_normal((K, T, 2))
    out = {"zc_sum": float(zc.sum()), "zc_head": zc.reshape(-1)[:8].tolist()}
    if case["kind"] == "bss":
        z = substream(case["seed"], *rp, 3, it).standard_normal((T, K, M, 7))
        out.update(z_sum=float(z.sum()), z_head=z.reshape(-1)[:8].tolist())
    return out


def run_case(case):
    cfg, cost, model, track, noise, x0, cov0, plan = build(case, REF)
    ctrl = rc.Controller(cfg, cost, model, track, noise=noise, seed=case["seed"],
                         run_path=tuple(case["run_path"]))
    if plan is not None:
        ctrl.plan = rc.ControlPlan(plan)
    for _ in range(case["warm"]):
        ctrl.control_step(x0, cov0)
    plan_before = ctrl.plan.controls.copy()
    it = ctrl.iteration
    record, captured = [], {}
    orig_mc, orig_pp, orig_upd = rc.propagate_mc_batch, rc.propagate_particles_batch, rc.mppi_update

    def rec_mc(*a, **k):
        out = orig_mc(*a, **k)
        record.append((out[0].copy(), out[1].copy(), out[2].copy()))
        return out

    def rec_pp(*a, **k):
        out = orig_pp(*a, **k)
        record.append((out[0].copy(), out[1].copy(), out[2].copy()))
        return out

    def rec_upd(batch, lam, bounds):
        captured["costs"] = batch.costs.copy()
        captured["controls"] = batch.controls.copy()
        return orig_upd(batch, lam, bounds)

    rc.propagate_mc_batch, rc.propagate_particles_batch, rc.mppi_update = rec_mc, rec_pp, rec_upd
    invalid = False
    try:
        u0, nxt = ctrl.control_step(x0, cov0)
    except rc.AllRolloutsInvalid:
        invalid = True
    finally:
        rc.propagate_mc_batch, rc.propagate_particles_batch, rc.mppi_update = orig_mc, orig_pp, orig_upd
    K = case["K"]
    ks = np.arange(K) if K <= 64 else np.unique(np.concatenate(
        [np.arange(16), [int(np.argmin(captured["costs"]))]]))
    arrays = dict(plan_before=plan_before, costs=captured["costs"], x0=x0, cov0=cov0,
                  track_s=track.s, track_kappa=track.kappa, ks=ks,
                  u_sum=np.array([captured["controls"].sum()]))
    if record:
        arrays["means"] = np.stack([r[0][ks] for r in record])
        arrays["covs"] = np.stack([r[1][ks] for r in record])
        arrays["oks"] = np.stack([r[2] for r in record])
    if not invalid:
        arrays["u0"] = u0
        arrays["plan_after"] = nxt.controls
        arrays["vplus"] = np.concatenate([u0[None], nxt.controls[:-1]])
    meta = dict(case=case, iteration=it, invalid=invalid, track_length=track.length,
                **noise_checksums(case, it))
    np.savez_compressed(HERE / f"{case['name']}.npz", meta=json.dumps(meta), **arrays)
    print(f"{case['name']}: it={it} invalid={invalid} "
          f"finite={np.isfinite(captured['costs']).sum()}/{K}")


def update_law_vectors():
    """mppi_update on seeded random batches, incl. inf costs and tiny lambda."""
    out = {}
    for j in range(len(UPDATE_BATCHES)):
        costs, controls, lam = update_batch(j)
        plan = rc.mppi_update(rc.RolloutBatch(controls, np.zeros_like(controls), costs),
                              lam, rc.ControlBounds())
        out[f"u{j}_vplus"] = plan.controls
        out[f"u{j}_costs_sum"] = np.array([costs[np.isfinite(costs)].sum()])
    np.savez_compressed(HERE / "update_law.npz", **out)
    print("update_law: 4 batches")


def closed_loop_vectors():
    """Reference closed-loop trajectories (sim.run_closed_loop with
    record_trajectory) for tests/test_gpu_closed_loop.py."""
    for case in CLOSED_LOOP:
        cfg = build_closed_loop(case, REF, rsim)
        cfg.record_trajectory = True
        rec = rsim.run_closed_loop(cfg, case["run"])
        np.savez_compressed(HERE / f"{case['name']}.npz", meta=json.dumps(case),
                            trajectory=rec.trajectory, crashed=np.array([rec.crashed]),
                            steps=np.array([rec.steps]), collisions=np.array([rec.collisions]))
        print(f"{case['name']}: steps={rec.steps} crashed={rec.crashed} collisions={rec.collisions}")


def plant_vectors():
    """Reference RK4 plant steps (step_array with the plant params) on random
    states, for the host plant restatement (tests/test_sim_cpu.py)."""
    from paper_2408_00494_b200.tracks import named_track
    rng = np.random.default_rng(5)
    track = named_track("ellipse", build=rd.make_test_track)
    plant = rd.with_timestep(rd.VehicleParams(), 0.01, "rk4")
    n = 256
    x = np.zeros((n, 8))
    x[:, 0] = rng.uniform(0.5, 7, n); x[:, 1] = rng.normal(0, 0.3, n); x[:, 2] = rng.normal(0, 0.5, n)
    x[:, 3] = x[:, 0] / 0.095 * rng.uniform(0.8, 1.3, n); x[:, 4] = x[:, 0] / 0.095 * rng.uniform(0.8, 1.3, n)
    x[:, 5] = rng.normal(0, 0.3, n); x[:, 6] = rng.uniform(-1.4, 1.4, n); x[:, 7] = rng.uniform(0, track.length, n)
    u = np.stack([rng.uniform(-0.35, 0.35, n), rng.uniform(-1, 1, n)], 1)
    w = rng.normal(0, 0.05, (n, 3))
    out, ok = rd.step_array(x, u, w, plant, track)
    np.savez_compressed(HERE / "plant_rk4.npz", x=x, u=u, w=w, out=out, ok=ok)
    print("plant_rk4: 256 states")


def trackframe_vectors():
    """Reference TrackFrame poses (dynamics.py:592-690) on the BASELINE tracks,
    for the config-4 centerline table (obstacles.py)."""
    from paper_2408_00494_b200.tracks import named_track
    out = {}
    for name in ("ellipse", "spline0", "oval"):
        tr = named_track(name, build=rd.make_test_track)
        fr = rd.TrackFrame(tr)
        q = np.linspace(0.0, tr.length, 401)[:-1] + 0.0137
        out[name + "_s"] = q
        out[name + "_pose"] = np.array([fr.pose(v) for v in q])
        g = np.array([fr.to_global(v, 0.7, 0.1) for v in q[::10]])
        out[name + "_global_ey0.7"] = g
    np.savez_compressed(HERE / "trackframe.npz", **out)
    print("trackframe: 3 tracks")


if __name__ == "__main__":
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    names = set(sys.argv[1:])
    for c in CASES:
        if not names or c["name"] in names:
            run_case(c)
    if not names or "update_law" in names:
        update_law_vectors()
    if not names or "closed_loop" in names:
        closed_loop_vectors()
    if not names or "plant" in names:
        plant_vectors()
    if not names or "trackframe" in names:
        trackframe_vectors()

"""Drop-in with the reference's OWN objects, on CPU.

The stock reference package (installed in baseline/_ref, or importable from
/root/reference in the build container) builds every golden case's
``MppiConfig`` / ``CostSpec`` / ``SafetyParams`` / ``VehicleParams`` /
``Track`` / ``NoiseModel`` with its own constructors; this repo's
``build_problem`` must pack exactly the same ``bssmppi_problem`` from them as
from its mirror types -- every scalar field byte for byte and the track
tables element for element -- and this repo's ``Controller`` must accept
them (construction and validation; compute needs a GPU:
tests/test_gpu_acceptance.py drives the reference's own closed loop).
"""

import ctypes as C
import sys
import types
from pathlib import Path

import numpy as np
import pytest

from cases import CASES, build
from helpers import MINE

from paper_2408_00494_b200 import _lib
from paper_2408_00494_b200 import controllers as mc

ROOT = Path(__file__).resolve().parent.parent


def _ref_modules():
    for path in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (path / "belief_mppi").is_dir():
            if str(path) not in sys.path:
                sys.path.insert(0, str(path))
            break
    else:
        pytest.skip("reference package not available")
    import os
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/bssmppi_numba_cache")
    from belief_mppi import constraints as rk
    from belief_mppi import controllers as rc
    from belief_mppi import dynamics as rd
    return types.SimpleNamespace(
        VehicleParams=rd.VehicleParams, VehicleState=rd.VehicleState, NoiseModel=rd.NoiseModel,
        CostSpec=rc.CostSpec, MppiConfig=rc.MppiConfig, make_test_track=rd.make_test_track,
        with_timestep=rd.with_timestep, SafetyParams=rk.SafetyParams, Track=rd.Track,
        Controller=rc.Controller, CovSubset=__import__("belief_mppi.belief", fromlist=["x"]).CovSubset)


POINTERS = {"track_s", "track_kappa", "obstacles", "centerline"}


def _pack(objs, kind):
    cfg, cost, model, track, noise = objs
    ctx = mc.RolloutContext(model, track, cost, noise=noise)
    M = cfg.inner_samples if kind == "bss" else 1
    return mc.build_problem(kind, cfg.samples, cfg.horizon, M, cfg.temperature, cfg.control_cost_weight,
                            cfg.sigma_eps, cfg.precision, cfg.bounds, cfg.persist_particles, ctx)


@pytest.mark.parametrize("name", [c["name"] for c in CASES])
def test_problem_packed_identically_from_reference_objects(name):
    REF = _ref_modules()
    case = next(c for c in CASES if c["name"] == name)
    ref = build(case, REF)[:5]
    mine = build(case, MINE)[:5]
    assert type(ref[0]).__module__.startswith("belief_mppi")      # really the reference's types
    pr, keep_r = _pack(ref, case["kind"])
    pm, keep_m = _pack(mine, case["kind"])
    for fname, ftype in _lib.Problem._fields_:
        if fname in POINTERS:
            continue
        a, b = getattr(pr, fname), getattr(pm, fname)
        if isinstance(a, C.Array):
            a, b = list(a), list(b)
        assert np.array_equal(np.asarray(a), np.asarray(b)), (fname, a, b)
    n = pr.track_n
    assert n == pm.track_n
    for f in ("track_s", "track_kappa"):
        ra = np.ctypeslib.as_array(getattr(pr, f), shape=(n,))
        ma = np.ctypeslib.as_array(getattr(pm, f), shape=(n,))
        assert np.array_equal(ra, ma), f


def test_controller_accepts_reference_objects():
    """Construction with the reference's dataclasses (controllers.py:353-369
    signature, keyword names included) validates without touching CUDA; the
    unsupported-configuration errors are the reference's NotImplementedError."""
    REF = _ref_modules()
    case = next(c for c in CASES if c["name"] == "c1_s0")
    cfg, cost, model, track, noise, x0, cov0, plan = build(case, REF)
    ctrl = mc.Controller(cfg, cost, model, track, noise=noise, subset=REF.CovSubset((1, 2, 5, 6)),
                         seed=3, run_path=(5, 3))
    assert ctrl.plan.controls.shape == (cfg.horizon, 2) and ctrl.iteration == 0
    with pytest.raises(NotImplementedError):
        mc.Controller(cfg, cost, model, track, noise=noise, subset=REF.CovSubset((1, 2, 6)))
    hooked = type(cost)(belief_stage_cost=lambda means, sig: 0.0)
    with pytest.raises(NotImplementedError):
        mc.Controller(cfg, hooked, model, track, noise=noise)

"""Host closed-loop harness (paper_2408_00494_b200/sim.py): the FP64 RK4
plant reproduces the reference's step_array with integrator "rk4"
(dynamics.py:447-497, 550-573) and the run set-up follows sim.py."""

import numpy as np
import pytest

from cases import CLOSED_LOOP, build_closed_loop
from helpers import GOLDEN, MINE

from paper_2408_00494_b200 import sim
from paper_2408_00494_b200 import dynamics as md
from paper_2408_00494_b200.tracks import named_track


def test_plant_rk4_matches_reference():
    d = np.load(GOLDEN / "plant_rk4.npz")
    track = named_track("ellipse")
    plant = md.with_timestep(md.VehicleParams(), 0.01, "rk4")
    for i in range(len(d["x"])):
        out, ok = sim.plant_step(d["x"][i], d["u"][i], d["w"][i], plant, track)
        assert ok == bool(d["ok"][i])
        np.testing.assert_allclose(out, d["out"][i], rtol=1e-12, atol=1e-12)


def test_experiment_config_validation():
    with pytest.raises(ValueError):
        sim.ExperimentConfig(dt_control=0.05, dt_plant=0.03)
    with pytest.raises(ValueError):
        sim.ExperimentConfig(collision_threshold=5.0)
    cfg = build_closed_loop(CLOSED_LOOP[0], MINE, sim)
    assert cfg.plant_substeps == 5
    assert cfg.plant_params().integrator == "rk4" and cfg.model_params().dt == 0.05


def test_initial_state_matches_reference_trajectory_start():
    case = CLOSED_LOOP[0]
    cfg = build_closed_loop(case, MINE, sim)
    x0 = sim.initial_state(cfg, case["run"])
    assert x0[0] == pytest.approx(case["init_speed"], abs=0.5)
    assert x0[3] == x0[4] == pytest.approx(x0[0] / 0.095)

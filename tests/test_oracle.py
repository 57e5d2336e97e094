"""Pin the CPU oracle (oracle/bss_oracle.py) to golden vectors produced by
the real reference (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from cases import CASES, update_batch, UPDATE_BATCHES
from helpers import GOLDEN, Inputs

from oracle import bss_oracle as orc

NAMES = [c["name"] for c in CASES]


@pytest.mark.parametrize("name", NAMES)
def test_noise_stream_unchanged(name):
    """The numpy substreams still produce the draws the fixtures saw."""
    inp = Inputs(name)
    meta = inp.meta
    if inp.kind == "bss":
        assert float(inp.z.sum()) == pytest.approx(meta["z_sum"], rel=0, abs=1e-6)
        assert np.array_equal(inp.z.reshape(-1)[:8], np.asarray(meta["z_head"]))
    assert float(inp.u.sum()) == pytest.approx(float(inp.gold["u_sum"][0]), abs=1e-9)


@pytest.mark.parametrize("name", NAMES)
def test_track_tables_identical(name):
    inp = Inputs(name)
    assert np.array_equal(inp.track.s, inp.gold["track_s"])
    assert np.array_equal(inp.track.kappa, inp.gold["track_kappa"])
    assert np.array_equal(inp.x0, inp.gold["x0"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference(name):
    inp = Inputs(name)
    rec = []
    costs, vplus = inp.oracle(record=rec)
    gold = inp.gold
    fin = np.isfinite(gold["costs"])
    assert np.array_equal(np.isfinite(costs), fin)
    np.testing.assert_allclose(costs[fin], gold["costs"][fin], rtol=1e-9, atol=0)
    if inp.meta["invalid"]:
        assert vplus is None
    else:
        np.testing.assert_allclose(vplus, gold["vplus"], rtol=0, atol=1e-9)
    if "means" in gold:
        ks = gold["ks"]
        means = np.stack([r[0][ks] for r in rec])
        covs = np.stack([r[1][ks] for r in rec])
        oks = np.stack([r[2] for r in rec])
        assert np.array_equal(oks, gold["oks"])
        np.testing.assert_allclose(means, gold["means"], rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(covs, gold["covs"], rtol=1e-7, atol=1e-13)


@pytest.mark.parametrize("j", range(len(UPDATE_BATCHES)))
def test_oracle_update_law(j):
    d = np.load(GOLDEN / "update_law.npz")
    costs, controls, lam = update_batch(j)
    v = orc.mppi_update(costs, controls, lam, np.array([-0.35, -1.0]), np.array([0.35, 1.0]))
    np.testing.assert_allclose(v, d[f"u{j}_vplus"], rtol=0, atol=1e-12)

"""The C oracle (CPU baseline arm) restates the same reference algorithm as
the numpy oracle: it must agree with it -- and so with the golden reference
vectors -- on the captured-noise cases."""

import numpy as np
import pytest

from cases import CASES
from helpers import Inputs

from oracle import c_oracle
from paper_2408_00494_b200.controllers import build_problem

NAMES = [c["name"] for c in CASES]


def _problem(inp):
    cfg = inp.cfg
    M = cfg.inner_samples if inp.kind == "bss" else 1
    prob, keep = build_problem(inp.kind, inp.K, inp.T, M, cfg.temperature, cfg.control_cost_weight,
                               cfg.sigma_eps, cfg.precision, cfg.bounds, cfg.persist_particles,
                               inp.ctx)
    return prob, keep


@pytest.mark.parametrize("name", NAMES)
def test_c_oracle_matches_reference(name):
    inp = Inputs(name)
    prob, keep = _problem(inp)
    costs, u_used = c_oracle.rollout(prob, inp.x0, inp.cov0, inp.plan, u=inp.u, eps=inp.eps,
                                     z=inp.z, threads=2)
    gold = inp.gold["costs"]
    fin = np.isfinite(gold)
    assert np.array_equal(np.isfinite(costs), fin)
    np.testing.assert_allclose(costs[fin], gold[fin], rtol=1e-9)
    if not inp.meta["invalid"]:
        v = c_oracle.update(costs, inp.u, inp.cfg.temperature, inp.lo, inp.hi)
        np.testing.assert_allclose(v, inp.gold["vplus"], atol=1e-9)


def test_c_oracle_eps_mode_clamps_like_reference():
    inp = Inputs("clamp")
    prob, keep = _problem(inp)
    costs, u_used = c_oracle.rollout(prob, inp.x0, inp.cov0, inp.plan, eps=inp.eps, z=inp.z)
    np.testing.assert_array_equal(u_used, inp.u)
    np.testing.assert_allclose(costs, inp.gold["costs"], rtol=1e-9)


def test_philox_known_answers():
    """Random123 Philox4x32-10 known-answer vectors."""
    assert c_oracle.philox([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert c_oracle.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E,
                                                                  0xA20BC7C6, 0x6D5451FD]
    assert c_oracle.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                           [0xA4093822, 0x299F31D0]) == [0xD16CFE09, 0x94FDCCEB, 0x5001E420,
                                                        0x24126EA1]


def test_philox_round_counts_differ():
    a = c_oracle.philox([1, 2, 3, 4], [5, 6], rounds=7)
    b = c_oracle.philox([1, 2, 3, 4], [5, 6], rounds=10)
    assert a != b


def test_philox_mode_thread_invariant():
    """Counter-based noise: the CPU arm's result does not depend on threads."""
    inp = Inputs("c1_s0")
    prob, keep = _problem(inp)
    a, _ = c_oracle.control_step(prob, inp.x0, None, inp.plan, (1, 2), (3, 4), threads=1)
    b, _ = c_oracle.control_step(prob, inp.x0, None, inp.plan, (1, 2), (3, 4), threads=4)
    np.testing.assert_array_equal(a, b)


def test_iteration_key_matches_product_library():
    """The device-noise key schedule is host code in the product library; the
    C oracle restates it (used by the CPU closed-loop arm)."""
    from paper_2408_00494_b200 import _lib
    lib = _lib.load()
    out = (_lib.C.c_uint32 * 2)()
    for base, dom, it in [((1, 2), 2, 0), ((0xDEADBEEF, 7), 3, 12345), ((5, 6), 2, 2 ** 40 + 3)]:
        assert lib.bssmppi_iteration_key((_lib.C.c_uint32 * 2)(*base), dom, it, out) == 0
        assert (out[0], out[1]) == c_oracle.iteration_key(base, dom, it)
    assert c_oracle.iteration_key((1, 2), 2, 0) != c_oracle.iteration_key((1, 2), 3, 0)
    assert c_oracle.iteration_key((1, 2), 2, 0) != c_oracle.iteration_key((1, 2), 2, 1)

"""Chance-constraint scalars used by the rollout cost.

Host side only computes the back-off nu once (reference
``constraints.py:70-93``); the per-step DCBF ``track_dcbf_values``
(``constraints.py:130-137``) and the shield penalty ``penalty_values``
(``constraints.py:172-186``) are evaluated on the belief moments inside the
rollout kernel (``csrc/rollout.cuh`` dcbf / shield_penalty); the host-side
safety bookkeeping of the closed loop (``sim.SafetyMonitor``) restates them
in FP64 where it needs them.
"""

import math
from dataclasses import dataclass

import numpy as np
from scipy.special import erfinv


class InvalidBudget(ValueError):
    pass


class InvalidProbability(ValueError):
    pass


@dataclass(frozen=True)
class SafetyParams:
    """beta (``cbf_rate``) and C (``penalty``) of the discrete safety
    condition h_k >= (1 - beta) h_{k-1} (reference constraints.py:22-33)."""

    cbf_rate: float = 0.35
    penalty: float = 2000.0

    def __post_init__(self):
        if not 0.0 < self.cbf_rate < 1.0:
            raise ValueError("cbf_rate must lie in (0, 1)")
        if self.penalty < 0.0:
            raise ValueError("penalty must be >= 0")


def allocate_budget(p_fail: float, z: int):
    """Uniform Boole split of the failure budget (constraints.py:70-80)."""
    if not 0.0 < p_fail <= 1.0:
        raise InvalidBudget(f"failure budget {p_fail} outside (0, 1]")
    if z < 1:
        raise InvalidBudget("constraint count must be >= 1")
    share = p_fail / z
    return [share] * (z - 1) + [p_fail - share * (z - 1)]


def backoff_gaussian(p: float) -> float:
    """sqrt(2) erfinv(1 - 2p) (constraints.py:90-93)."""
    if not 0.0 < p <= 0.5:
        raise InvalidProbability(f"probability {p} outside (0, 0.5]")
    return float(math.sqrt(2.0) * erfinv(1.0 - 2.0 * p))

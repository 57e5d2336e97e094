"""Tracked covariance subset (reference ``belief.py:41-69``).

The device kernels track the 4x4 covariance of (vy, yaw rate, e_psi, e_y),
the reference's ``DEFAULT_SUBSET``.  Other subsets are accepted by the type
but rejected by the controller with ``NotImplementedError``.
"""

from dataclasses import dataclass

from .dynamics import IDX_EPSI, IDX_EY, IDX_VY, IDX_YAW_RATE


class DegenerateSamples(RuntimeError):
    """All (or all but one) propagated samples were non-finite."""


class UntrackedComponent(ValueError):
    """Requested state component is not part of the tracked covariance subset."""


@dataclass(frozen=True)
class CovSubset:
    indices: tuple

    def __post_init__(self):
        idx = tuple(int(i) for i in self.indices)
        if len(set(idx)) != len(idx):
            raise ValueError("covariance subset indices must be unique")
        if any(i < 0 for i in idx):
            raise ValueError("covariance subset indices must be >= 0")
        object.__setattr__(self, "indices", idx)

    def __len__(self):
        return len(self.indices)

    def position(self, state_index: int) -> int:
        try:
            return self.indices.index(state_index)
        except ValueError:
            raise UntrackedComponent(f"state component {state_index} is not tracked") from None


DEFAULT_SUBSET = CovSubset((IDX_VY, IDX_YAW_RATE, IDX_EPSI, IDX_EY))

"""Keyed random substreams (reference ``streams.py:13-28``).

``substream`` is the reference's numpy Philox4x64 stream: the oracle-noise
mode of the controller draws its control perturbations and belief normals
from it, exactly like the reference, and ships them to the device.

``device_key`` derives the 64-bit key of the *device* counter-based
generator (Philox4x32, ``csrc/philox.cuh``) from the same
(root seed, *path) identity, so performance-mode streams are keyed by the
same (seed, run_path, domain, iteration) tuple and stay independent of
scheduling, sharding and worker count.
"""

import numpy as np

DOMAIN_INIT = 0
DOMAIN_PLANT = 1
DOMAIN_CONTROL = 2
DOMAIN_BELIEF = 3
DOMAIN_MONITOR = 4
DOMAIN_RUN = 5


def _seed_sequence(root_seed, path):
    return np.random.SeedSequence(int(root_seed), spawn_key=tuple(int(p) for p in path))


def substream(root_seed: int, *path: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(_seed_sequence(root_seed, path)))


def device_key(root_seed: int, *path: int) -> tuple:
    """(k0, k1) uint32 Philox4x32 key for the substream (root_seed, *path)."""
    k = _seed_sequence(root_seed, path).generate_state(2, np.uint32)
    return int(k[0]), int(k[1])


def base_key(root_seed: int, *path: int) -> tuple:
    """Controller base key: SeedSequence(root_seed, spawn_key=path) -- the
    reference's stream identity (streams.py:21-28) without domain/iteration.
    Per-iteration keys are derived from it on the host by
    ``bssmppi_iteration_key`` (Philox4x32-10 of (iteration, domain))."""
    return device_key(root_seed, *path)

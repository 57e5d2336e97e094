"""ctypes wrapper of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Imported by tests/ and by bench.py's CPU legs (cpu_baseline, --impl
reference); never by the product package.  The problem struct is the same
C layout as the product ABI (include/bssmppi.h), packed by the product's
own ``build_problem`` so both sides read identical constants.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "liboracle.so"
_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise RuntimeError(f"{LIB} not built (make -C oracle)")
        lib = C.CDLL(os.fspath(LIB))
        from paper_2408_00494_b200._lib import Problem
        lib.orc_rollout.argtypes = [C.POINTER(Problem), _dp, _dp, _dp, _dp, _dp, _dp, _u32p, _u32p,
                                    _dp, _dp, C.c_int]
        lib.orc_rollout_moments.argtypes = [C.POINTER(Problem), _dp, _dp, _dp, _dp, _dp, _dp, _u32p,
                                            _u32p, _dp, _dp, _dp, C.c_int]
        lib.orc_update.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_double, _dp, _dp, _dp]
        lib.orc_control_step.argtypes = [C.POINTER(Problem), _dp, _dp, _dp, _u32p, _u32p, _dp, _dp,
                                         _dp, C.c_int]
        lib.orc_philox4x32.argtypes = [_u32p, _u32p, C.c_int, _u32p]
        lib.orc_belief_normals.argtypes = [_u32p, C.c_uint32, C.c_uint32, C.c_int, _dp]
        lib.orc_max_threads.restype = C.c_int
        lib.orc_iteration_key.argtypes = [_u32p, C.c_uint32, C.c_uint64, _u32p]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(_dp)


def _key(k):
    return None if k is None else (C.c_uint32 * 2)(int(k[0]), int(k[1]))


def rollout(problem, x0, cov0, nominal, u=None, eps=None, z=None, key_ctrl=None, key_belief=None,
            threads=0, moments=False):
    """Costs (k_count,) and the clamped controls used (k_count, T, 2); with
    ``moments=True`` also the per-step belief moments (T, k_count, 18):
    mean[8] then the covariance upper triangle (the device layout)."""
    lib = load()
    K, T = problem.k_count, problem.horizon
    keep = [np.ascontiguousarray(a, dtype=np.float64) if a is not None else None
            for a in (x0, cov0, nominal, u, eps, z)]
    costs = np.empty(K)
    u_out = np.empty((K, T, 2))
    mom = np.empty((T, K, 18)) if moments else None
    lib.orc_rollout_moments(C.byref(problem), *[_p(a) for a in keep], _key(key_ctrl), _key(key_belief),
                            costs.ctypes.data_as(_dp), u_out.ctypes.data_as(_dp),
                            None if mom is None else mom.ctypes.data_as(_dp), int(threads))
    return (costs, u_out, mom) if moments else (costs, u_out)


def update(costs, u, lam, lo, hi):
    lib = load()
    K, T, _ = u.shape
    out = np.empty((T, 2))
    c = np.ascontiguousarray(costs, dtype=np.float64)
    uu = np.ascontiguousarray(u, dtype=np.float64)
    rc = lib.orc_update(K, T, _p(c), _p(uu), float(lam), _p(np.asarray(lo, float)),
                        _p(np.asarray(hi, float)), out.ctypes.data_as(_dp))
    if rc == 3:
        raise RuntimeError("AllRolloutsInvalid")
    return out


def control_step(problem, x0, cov0, plan, key_ctrl, key_belief, threads=0):
    """One full Philox-noise iteration on the host cores; returns v+."""
    lib = load()
    K, T = problem.k_count, problem.horizon
    costs = np.empty(K)
    u = np.empty((K, T, 2))
    out = np.empty((T, 2))
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    cov = None if cov0 is None else np.ascontiguousarray(cov0, dtype=np.float64)
    plan = np.ascontiguousarray(plan, dtype=np.float64)
    rc = lib.orc_control_step(C.byref(problem), _p(x0), _p(cov), _p(plan), _key(key_ctrl),
                              _key(key_belief), costs.ctypes.data_as(_dp), u.ctypes.data_as(_dp),
                              out.ctypes.data_as(_dp), int(threads))
    if rc == 3:
        raise RuntimeError("AllRolloutsInvalid")
    return out, costs


def philox(ctr, key, rounds=10):
    out = (C.c_uint32 * 4)()
    load().orc_philox4x32((C.c_uint32 * 4)(*ctr), (C.c_uint32 * 2)(*key), int(rounds), out)
    return list(out)


def belief_normals(key, t, kg, m_count):
    """(m_count, 7) FP64 belief normals of particle-steps (t, kg, m < m_count)."""
    out = np.empty((m_count, 7))
    load().orc_belief_normals((C.c_uint32 * 2)(*key), int(t), int(kg), int(m_count), _p(out))
    return out


def iteration_key(base, domain, iteration):
    out = (C.c_uint32 * 2)()
    load().orc_iteration_key((C.c_uint32 * 2)(*base), int(domain), int(iteration), out)
    return int(out[0]), int(out[1])


def max_threads():
    return load().orc_max_threads()

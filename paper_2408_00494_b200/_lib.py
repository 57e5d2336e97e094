"""ctypes binding of the C ABI in ``include/bssmppi.h`` (libbssmppi.so).

The shared library is built in-tree by ``paper_2408_00494_b200.build``
(``__graft_entry__.build()``).  Loading never needs a GPU; every compute
entry point fails loudly (``BssMppiError``) when no CUDA device is present:
there is no CPU fallback anywhere on this path.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("BSSMPPI_LIB", Path(__file__).resolve().parent / "libbssmppi.so"))

OK, ERR_INVALID, ERR_CUDA, ERR_ALL_INVALID, ERR_UNSUPPORTED = range(5)
KIND = {"mppi": 0, "smppi": 1, "bss": 2}


class BssMppiError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[bssmppi status {code}] {msg}")
        self.code = code


class BssMppiUnsupported(BssMppiError, NotImplementedError):
    """BSSMPPI_ERR_UNSUPPORTED: outside the device path (the reference's
    NotImplementedError, INTEGRATION.md status table)."""


class Problem(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("samples", C.c_int32), ("horizon", C.c_int32),
        ("inner_samples", C.c_int32), ("persist_particles", C.c_int32),
        ("temperature", C.c_double), ("control_cost_weight", C.c_double),
        ("sigma_factor", C.c_double * 4), ("precision", C.c_double * 4),
        ("bounds_lo", C.c_double * 2), ("bounds_hi", C.c_double * 2),
        ("q_diag", C.c_double * 8), ("v_goal", C.c_double), ("obstacle_penalty", C.c_double),
        ("terminal_scale", C.c_double), ("cbf_rate", C.c_double), ("penalty", C.c_double),
        ("backoff", C.c_double),
        ("phys", C.c_double * 23), ("dt", C.c_double),
        ("noise_factor", C.c_double * 9),
        ("track_s", C.POINTER(C.c_double)), ("track_kappa", C.POINTER(C.c_double)),
        ("track_n", C.c_int32), ("track_length", C.c_double), ("half_width", C.c_double),
        ("track_closed", C.c_int32),
        ("k_begin", C.c_int32), ("k_count", C.c_int32),
        ("noise_kind", C.c_int32), ("laplace_scale", C.c_double), ("slip_bias", C.c_double),
        ("n_obstacles", C.c_int32), ("obstacles", C.POINTER(C.c_double)),
        ("obstacle_backoff", C.c_double), ("centerline", C.POINTER(C.c_double)),
        ("centerline_n", C.c_int32), ("centerline_ds", C.c_double),
        ("group_width", C.c_int32),
    ]


class Diag(C.Structure):
    _fields_ = [("cost_min", C.c_double), ("cost_argmin", C.c_int64), ("n_finite", C.c_int64),
                ("weight_sum", C.c_double), ("ess", C.c_double), ("device_ms", C.c_float),
                ("rollout_ms", C.c_float)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)
_ctx = C.c_void_p

# name -> (restype, argtypes); mirrors include/bssmppi.h one to one.
SIGNATURES = {
    "bssmppi_last_error": (C.c_char_p, []),
    "bssmppi_abi_version": (C.c_int32, []),
    "bssmppi_partial_len": (C.c_int32, [C.c_int32]),
    "bssmppi_group_width": (C.c_int32, [C.c_int32, C.c_int32]),
    "bssmppi_launch_shape": (C.c_int32, [_ctx, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "bssmppi_create": (C.c_int, [C.POINTER(Problem), C.c_int32, C.POINTER(_ctx)]),
    "bssmppi_destroy": (None, [_ctx]),
    "bssmppi_set_stream": (C.c_int, [_ctx, C.c_void_p]),
    "bssmppi_control_step": (C.c_int, [_ctx, _dp, _dp, _dp, _u32p, _u32p, _dp, _fp, _dp,
                                       C.POINTER(Diag)]),
    "bssmppi_step_partials": (C.c_int, [_ctx, _dp, _dp, _dp, _u32p, _u32p, _dp, _fp, C.c_void_p,
                                        C.c_int32]),
    "bssmppi_update_combine": (C.c_int, [_ctx, C.c_void_p, C.c_int32, _dp, C.POINTER(Diag)]),
    "bssmppi_upload_state": (C.c_int, [_ctx, _dp, _dp, _dp]),
    "bssmppi_enqueue_iteration": (C.c_int, [_ctx, _u32p, _u32p]),
    "bssmppi_download": (C.c_int, [_ctx, _dp, C.POINTER(Diag)]),
    "bssmppi_enqueue_partials": (C.c_int, [_ctx, _u32p, _u32p, C.c_void_p, C.c_int32]),
    "bssmppi_enqueue_combine": (C.c_int, [_ctx, C.c_void_p, C.c_int32]),
    "bssmppi_rollout": (C.c_int, [_ctx, _dp, _dp, _dp, _dp, _dp, _fp, _u32p, _dp, _fp]),
    "bssmppi_mppi_update": (C.c_int, [C.c_int32, C.c_int32, _dp, _dp, C.c_double, _dp, _dp, _dp,
                                      C.POINTER(Diag)]),
    "bssmppi_sample_controls": (C.c_int, [C.c_int32, C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp,
                                          _dp]),
    "bssmppi_step_array": (C.c_int, [_ctx, C.c_int32, _dp, _dp, _dp, _dp, _u8p]),
    "bssmppi_philox4x32": (C.c_int, [_u32p, _u32p, C.c_int32, _u32p]),
    "bssmppi_belief_normals": (C.c_int, [_u32p, C.c_int32, C.c_int32, C.c_int32, _fp]),
    "bssmppi_ffma_peak": (C.c_int, [C.c_int32, _dp]),
    "bssmppi_mufu_peak": (C.c_int, [C.c_int32, _dp]),
    "bssmppi_enqueue_step_device": (C.c_int, [_ctx, C.c_void_p, _u32p, _u32p, C.c_void_p]),
    "bssmppi_iteration_key": (C.c_int, [_u32p, C.c_uint32, C.c_uint64, _u32p]),
    "bssmppi_tire_table": (C.c_int, [_dp, C.c_double, _fp, C.c_int32, C.POINTER(C.c_int32), _dp, _dp]),
}

_LIB = None


def load():
    """Load libbssmppi.so (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise BssMppiError(ERR_CUDA, f"{LIB_PATH} not built; run __graft_entry__.build()")
        lib = C.CDLL(os.fspath(LIB_PATH))
        variant = "BSSMPPI_LIB" in os.environ   # A/B builds of older revisions (tools/)
        for name, (res, args) in SIGNATURES.items():
            if variant and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def check(code):
    if code != OK:
        cls = BssMppiUnsupported if code == ERR_UNSUPPORTED else BssMppiError
        raise cls(code, load().bssmppi_last_error().decode())
    return code


def dptr(a):
    """double* of a C-contiguous float64 array (or None)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def fptr(a):
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_fp)


def key_arr(key):
    if key is None:
        return None
    return (C.c_uint32 * 2)(int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF)

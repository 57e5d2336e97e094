"""The lateral tire table (csrc/bssmppi.cu tire_table_host, evaluated by
csrc/vehicle.cuh tire_q / lateral_shape): built by the library's host code
(bssmppi_tire_table, no GPU needed) and evaluated here in float32 with the
kernel's exact operation sequence -- row index by the 1.5 * 2^23 rounding
trick, in-cell offset by one FMA, Horner cubic by three, times alpha --
against float64 sin(C atan(B alpha)) over the whole slip-angle domain, for
the reference default tire, every golden case's tire and stiff ones."""

import ctypes as C
import math

import numpy as np
import pytest

from paper_2408_00494_b200 import _lib


def _fma32(a, b, c):
    # float32 FMA: the float64 product of two float32 values is exact, the
    # sum rounds once in float64 and once to float32 (differences from a true
    # single rounding are far below the bounds asserted here)
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


def _table(bc, steer):
    lib = _lib.load()
    cap = 2 * 4100
    out = np.zeros((cap, 4), dtype=np.float32)
    rows = C.c_int32()
    s = np.zeros(1)
    amax = np.zeros(1)
    rc = lib.bssmppi_tire_table(_lib.dptr(np.asarray(bc, dtype=np.float64)), float(steer), _lib.fptr(out), cap,
                                C.byref(rows), _lib.dptr(s), _lib.dptr(amax))
    assert rc == 0
    n = rows.value
    return out[:2 * n].reshape(2, n, 4), np.float32(s[0]), float(amax[0])


def _eval(tab, s, a):
    magic = np.float32(12582912.0)
    nf = _fma32(a, np.full_like(a, s), np.full_like(a, magic))
    f = _fma32(a, np.full_like(a, s), -(nf - magic))
    j = nf.view(np.uint32) & np.uint32(0x7FF)
    c = tab[j]
    p = _fma32(_fma32(_fma32(c[:, 3], f, c[:, 2]), f, c[:, 1]), f, c[:, 0])
    return p


@pytest.mark.parametrize("B,C,steer", [(4.0, 1.3, 0.35), (5.0, 1.4, 0.35), (3.5, 1.2, 0.35), (4.0, 1.9, 0.35),
                                       (4.0, 1.7, 0.35), (10.0, 1.5, 0.35), (20.0, 1.3, 0.6), (2.0, 2.5, 1.0),
                                       (4.0, 1.3, 2 * math.pi)])
def test_tire_table_accuracy(B, C, steer):
    tab, s, amax = _table([B, C, 0.5 * B, 0.9 * C], steer)
    rng = np.random.default_rng(1)
    for axle, (b, cc) in enumerate([(B, C), (0.5 * B, 0.9 * C)]):
        a = np.concatenate([rng.uniform(0, amax, 400_000), 10.0 ** np.linspace(-9, 0, 4000),
                            [0.0, amax]]).astype(np.float32)
        for sign in (1.0, -1.0):
            al = (sign * a).astype(np.float32)
            g = (al * _eval(tab[axle], s, np.abs(al))).astype(np.float32)
            exact = np.sin(cc * np.arctan(b * al.astype(np.float64)))
            err = np.abs(g - exact)
            assert err.max() < 3.5e-7, err.max()
            # relative accuracy wherever the magic-formula angle is away
            # from its interior zero at C atan(B |alpha|) = pi (C > 2 only)
            rel = (exact != 0) & (cc * np.arctan(b * np.abs(al.astype(np.float64))) < 0.9 * math.pi)
            assert (err[rel] / np.abs(exact[rel])).max() < 4e-7, (err[rel] / np.abs(exact[rel])).max()
            assert np.all(g[exact == 0] == 0)
    assert amax >= math.pi + steer


def test_tire_table_domain_and_index_range():
    tab, s, amax = _table([4.0, 1.3, 4.0, 1.3], 0.35)
    rows = tab.shape[1]
    # the largest slip angle a rollout meets (pi plus the steering bound,
    # plus FP32 rounding of atan2) stays inside the table
    j = _fma32(np.array([amax * (1 + 1e-6)], dtype=np.float32), np.array([s]), np.array([12582912.0], dtype=np.float32))
    assert (j.view(np.uint32) & 0x7FF)[0] < rows
    assert rows <= 330            # the reference tire fits the kernels' shared copy (vehicle.cuh kTireSmemRows)
    # NaN and inf read row 0 (and propagate through the in-cell offset)
    for v in (np.nan, np.inf):
        nf = _fma32(np.array([v], dtype=np.float32), np.array([s]), np.array([12582912.0], dtype=np.float32))
        assert (nf.view(np.uint32) & 0x7FF)[0] == 0


def test_tire_table_rejects_small_buffer():
    lib = _lib.load()
    out = np.zeros((4, 4), dtype=np.float32)
    rows = C.c_int32()
    s = np.zeros(1)
    amax = np.zeros(1)
    rc = lib.bssmppi_tire_table(_lib.dptr(np.array([4.0, 1.3, 4.0, 1.3])), 0.35, _lib.fptr(out), 4, C.byref(rows),
                                _lib.dptr(s), _lib.dptr(amax))
    assert rc != 0

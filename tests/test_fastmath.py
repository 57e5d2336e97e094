"""Pin the bounded-range polynomials of csrc/fastmath.cuh: re-evaluate each
one in float32 with the kernel's Horner order and bound its error against
float64 on the range the particle step uses."""

import math
import re
from pathlib import Path

import numpy as np
import pytest

SRC = (Path(__file__).resolve().parent.parent / "paper_2408_00494_b200" / "csrc" /
       "fastmath.cuh").read_text()


def _horner(c, t):
    p = np.full_like(t, c[0])
    for ci in c[1:]:
        p = (p * t + ci).astype(np.float32)
    return p


def _atan_x2_coeffs():
    body = SRC[SRC.index("float2 atan_mag_x2"):]
    body = body[:body.index("\n}\n")]
    first = re.findall(r"bc2\(([-0-9.e+]+)f\)", body)
    assert [float(v) for v in first[7:]] == [1.0]   # Q = 1 + s P(s): the Horner ends on 1
    return [np.float32(float(v)) for v in first[:7]]


def test_atan_x2():
    """Packed arctangent (slip angles and both magic formulas): the device
    algorithm in float32 with the kernel's Horner order and folded final
    FFMA, <= 3.3 ulp / 2.0e-7 absolute on the whole line (libdevice atanf:
    2 ulp)."""
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    from fit_poly import atan32
    c = np.array(_atan_x2_coeffs(), dtype=np.float64)
    assert len(c) == 7
    x = np.concatenate([np.linspace(-40, 40, 400001), np.geomspace(1e-6, 1e6, 100001),
                        -np.geomspace(1e-6, 1e6, 1001), [0.0, np.inf, -np.inf]])
    x = x.astype(np.float32).astype(np.float64)
    y = atan32(c, x)
    ex = np.arctan(x)
    e = np.abs(y - ex)
    assert e.max() < 2.0e-7, e.max()
    ulp = np.spacing(np.abs(ex).astype(np.float32)).astype(np.float64)
    assert (e / ulp).max() <= 3.3
    assert np.all(np.sign(y) == np.sign(x))


def test_sincos_pi_x2_half_range():
    """Packed heading / centerline (sin, cos): unconditional one-constant
    reduction, reflection to h = min(|x|, pi - |x|), the kSinCosHalf Horner
    chain (sine padded with a leading 0) -- emulated in float32 in the
    kernel's order on [-pi, pi] and beyond."""
    body = SRC[SRC.index("kSinCosHalf[6] = {"):]
    body = body[:body.index("};")]
    pairs = re.findall(r"\{([-0-9.e+]+)f, ([-0-9.e+]+)f\}", body)
    assert len(pairs) == 6
    sin_c = [np.float32(float(a)) for a, _ in pairs]
    cos_c = [np.float32(float(b)) for _, b in pairs]
    assert sin_c[0] == 0.0 and sin_c[-1] == 1.0 and cos_c[-1] == 1.0
    f = np.float32
    x = np.concatenate([np.linspace(-np.pi, np.pi, 400001), np.linspace(-9.0, 9.0, 100001)]).astype(f)
    n = np.rint((x * f(0.159154943)).astype(f)).astype(f)
    xr = (x.astype(np.float64) - n.astype(np.float64) * np.float64(f(6.28318548))).astype(f)
    a = np.abs(xr)
    b = (f(3.14159265) - a).astype(f)
    h = np.minimum(a, b)
    t = (h * h).astype(f)
    ps, pc = _horner(sin_c, t), _horner(cos_c, t)
    s_dev = np.copysign((ps * h).astype(f), xr).astype(np.float64)
    c_dev = np.where(b < a, -pc, pc).astype(np.float64)
    x64 = x.astype(np.float64)
    es, ec = np.abs(s_dev - np.sin(x64)), np.abs(c_dev - np.cos(x64))
    inside = np.abs(x64) <= np.pi
    assert es[inside].max() < 2.5e-7 and ec[inside].max() < 2.5e-7, (es[inside].max(), ec[inside].max())
    assert es.max() < 2e-6 and ec.max() < 2e-6          # reduced: + n * 1.7e-7 of 2 pi_f32
    small = np.abs(x64) < 0.7                          # heading errors: relative accuracy near 0
    nz = small & (np.abs(x64) > 1e-3)
    assert (es[nz] / np.abs(np.sin(x64[nz]))).max() < 3e-7


def test_centred_uniform2_16_is_exact():
    """philox.cuh centred_uniform2_16: the I2F-free 2u of a 16-bit field
    (mantissa bit insertion, FFMA 2m - 3, + 2^-16) equals 2 x the
    reference-form centred uniform (n + 1/2) 2^-16 - 1/2 for every n, and the
    derived Laplace inputs 1 - |2u| and a (2u) are bit-identical to 1 - 2|u|
    and (2a) u (oracle/bss_oracle.c centred_uniform16)."""
    n = np.arange(0, 1 << 16, dtype=np.uint32)
    top = n << np.uint32(16)                               # the field in bits 16..31
    m = (np.uint32(0x3F800000) + (top >> np.uint32(9))).view(np.float32)
    assert np.array_equal(m.astype(np.float64), 1.0 + n * 2.0 ** -16)
    v = (m.astype(np.float64) * 2.0 - 3.0).astype(np.float32) + np.float32(2.0 ** -16)
    u = (n.astype(np.float32) + np.float32(0.5)) * np.float32(2.0 ** -16) - np.float32(0.5)
    assert np.array_equal(v.astype(np.float64), 2.0 * u.astype(np.float64))
    assert np.abs(v).max() < 1.0
    assert np.array_equal(np.float32(1.0) - np.abs(v), np.float32(1.0) - np.float32(2.0) * np.abs(u))
    a = np.float32(0.05)
    assert np.array_equal(a * v, (np.float32(2.0) * a) * u)


def test_word_uniforms_are_exact():
    """philox.cuh word_radius / word_angle bit fields: the radius uniform
    (2 - 2^-21) - (1 + n 2^-20) is exactly 1 - (n + 1/2) 2^-20 for every
    20-bit n (Sterbenz), and the angle mantissa is exactly 1 + j / 4096 for
    every 12-bit j -- the values oracle/bss_oracle.c bm_word uses in FP64."""
    n = np.arange(0, 1 << 20, dtype=np.uint32)
    w = n << np.uint32(12)
    mr = (np.uint32(0x3F800000) + ((w & np.uint32(0xFFFFF000)) >> np.uint32(9))).view(np.float32)
    u1 = np.float32(2.0 - 2.0 ** -21) - mr
    assert np.array_equal(u1.astype(np.float64), 1.0 - (n + 0.5) * 2.0 ** -20)
    assert u1.min() > 0 and u1.max() < 1
    j = np.arange(0, 1 << 12, dtype=np.uint32)
    ma = (np.uint32(0x3F800000) | ((j & np.uint32(0xFFF)) << np.uint32(11))).view(np.float32)
    assert np.array_equal(ma.astype(np.float64), 1.0 + j / 4096.0)
    # the 4096-point angle grid keeps the pair's low moments exact
    th = 2 * np.pi * j / 4096.0
    for p in (2, 4, 6):
        assert abs(np.mean(np.cos(th) ** p) - math.comb(p, p // 2) / 2 ** p) < 1e-12

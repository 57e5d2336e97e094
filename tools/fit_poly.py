"""Fit the bounded-range polynomials of csrc/fastmath.cuh.

Lawson's algorithm (iteratively re-weighted least squares converging to the
weighted minimax fit) in float64, coefficients rounded to float32, then the
float32 Horner evaluation (with FMA, emulated exactly in float64) checked
on a dense grid.  tests/test_fastmath.py pins the resulting error bounds.

    python tools/fit_poly.py atan      # atan(a) = a + a s P(s), s = a^2, a in [0, 1]
    python tools/fit_poly.py sin_mf    # sin(x) = x P(x^2), |x| <= 2.05
    python tools/fit_poly.py cos_mf    # cos(x) = P(x^2),   |x| <= 2.05
    python tools/fit_poly.py sincos_pi # sin/cos on [-pi, pi]
"""

import sys

import numpy as np


def lawson(basis, target, weight, iters=400):
    """min_c max_i |weight_i (basis_i . c - target_i)| via Lawson re-weighting."""
    w = np.full(len(target), 1.0 / len(target))
    c = None
    for _ in range(iters):
        sw = np.sqrt(w) * weight
        c, *_ = np.linalg.lstsq(basis * sw[:, None], target * sw, rcond=None)
        err = np.abs(weight * (basis @ c - target))
        w = w * err
        w /= w.sum()
    return c


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def fma32(a, b, c):
    # a*b is exact in float64 for float32 inputs; one rounding to float32
    return f32(a * b + c)


def horner32(coef, t):
    p = np.full_like(t, coef[0])
    for ci in coef[1:]:
        p = fma32(p, t, ci)
    return p


def fit_atan(deg=7):
    """P of degree ``deg`` in s = a^2 with atan(a) ~= a + a s P(s) on [0, 1];
    weights make the fit minimax in the relative error of atan."""
    a = np.cos(np.linspace(np.pi / 2, 0, 20001)) ** 0.5   # dense near 0 and 1
    a = a[a > 1e-4]
    s = a * a
    g = (np.arctan(a) / a - 1.0) / s
    wt = a * s / np.arctan(a)
    basis = np.stack([s ** k for k in range(deg, -1, -1)], axis=1)
    c = f32(lawson(basis, g, wt))
    return c


def atan32(coef, x):
    """Device algorithm (fastmath.cuh atan_mag_x2): a = min(|x|, 1/|x|),
    Q = 1 + s P(s) by Horner, r = fma(+-a, Q, 0 or pi/2) (pi/2 - a Q for
    |x| > 1), sign of x.  MUFU.RCP is modelled as a correctly rounded
    reciprocal (the hardware's is within 1 ulp)."""
    t = np.abs(x)
    with np.errstate(divide="ignore"):
        r = f32(1.0 / t)
    a = np.minimum(t, r)
    s = f32(a * a)
    q = horner32(np.append(coef, 1.0), s)
    big = t > 1.0
    p = fma32(np.where(big, -a, a), q, np.where(big, np.float64(np.float32(1.57079637)), 0.0))
    return np.copysign(p, x)


def fit_atan_rat(n_p=3, n_q=2, iters=80):
    """atan(a) = a P(s) / Q(s), s = a^2, a in [0, 1], Q monic of degree n_q:
    Loeb's linearisation (P - g Q_low = g s^n_q, re-weighted by 1 / Q) with
    Lawson weights, minimax in the relative error.  Coefficients lowest first."""
    a = np.cos(np.linspace(np.pi / 2, 0, 40001)) ** 0.5
    a = a[a > 1e-5]
    s = a * a
    g = np.arctan(a) / a
    q_val = np.ones_like(s)
    ww = np.ones_like(s)
    for _ in range(iters):
        basis = np.concatenate([np.stack([s ** k for k in range(n_p + 1)], 1),
                                -g[:, None] * np.stack([s ** k for k in range(n_q)], 1)], 1)
        sw = np.sqrt(ww) / (np.abs(q_val) * g)
        c, *_ = np.linalg.lstsq(basis * sw[:, None], g * s ** n_q * sw, rcond=None)
        p, q = c[:n_p + 1], np.append(c[n_p + 1:], 1.0)
        q_val = sum(q[k] * s ** k for k in range(n_q + 1))
        err = np.abs(sum(p[k] * s ** k for k in range(n_p + 1)) / q_val - g) / g
        ww = ww * err
        ww /= ww.sum()
    return f32(p), f32(q)


def atan_rat32(p, q, x):
    """Device algorithm of fastmath.cuh atan_mag_x2 + sign: a = min(|x|, 1/|x|),
    P, Q Horner (Q's monic top step an add), R = 1/Q (MUFU.RCP modelled as
    correctly rounded), r = fma(+-a, P R, 0 or pi/2), sign of x."""
    t = np.abs(x)
    with np.errstate(divide="ignore"):
        a = np.minimum(t, f32(1.0 / t))
    s = f32(a * a)
    P = np.full_like(s, p[-1])
    for ck in p[-2::-1]:
        P = fma32(P, s, ck)
    Q = f32(s + q[-2])
    for ck in q[-3::-1]:
        Q = fma32(Q, s, ck)
    PR = f32(P * f32(1.0 / Q))
    big = t > 1.0
    r = fma32(np.where(big, -a, a), PR, np.where(big, np.float32(1.57079637), 0.0))
    return np.copysign(r, x)


def check_atan(coef):
    x = f32(np.concatenate([np.linspace(-40, 40, 2000001), np.geomspace(1e-6, 1e6, 400001)]))
    y = atan32(coef, x)
    ex = np.arctan(x)
    ulp = np.spacing(np.abs(ex).astype(np.float32)).astype(np.float64)
    e = np.abs(y - ex)
    return e.max(), (e / ulp).max()


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "atan"
    if what == "sincos_half":
        # (sin, cos) on [0, pi/2]: sin = x S(t) (degree 4), cos = C(t) (degree 5)
        xs = np.linspace(1e-5, np.pi / 2 + 1e-3, 40001)
        t = xs * xs
        for name, g, deg in (("sin", np.sin(xs) / xs, 4), ("cos", np.cos(xs), 5)):
            basis = np.stack([t ** k for k in range(deg, -1, -1)], 1)
            c = f32(lawson(basis, g, np.ones_like(g)))
            print(f"{name}:", ", ".join(f"{v:.9e}f" for v in c))
        return
    if what == "sin_tire":
        # sin x = x (1 + t Q(t)) on |x| <= 2.2 with Q of degree 4 (constant term of
        # the bracket held at 1): the short lateral tire sine of round 1 (now
        # replaced by the per-vehicle tire table, vehicle.cuh tire_q)
        xs = np.linspace(1e-5, 2.2, 40001)
        t = xs * xs
        g = (np.sin(xs) / xs - 1.0) / t
        basis = np.stack([t ** k for k in range(4, -1, -1)], 1)
        c = np.append(f32(lawson(basis, g, t / (np.sin(xs) / xs))), 1.0)
        x32 = f32(xs)
        y = f32(horner32(c, f32(x32 * x32)) * x32)
        e = np.abs(y - np.sin(x32))
        print(f"sin_tire: max abs err {e.max():.3e}, rel {(e / np.abs(np.sin(x32))).max():.3e}")
        print("  coefficients (highest first):", ", ".join(f"{v:.9e}f" for v in c))
        return
    if what == "atan_rat":
        p, q = fit_atan_rat()
        x = f32(np.concatenate([np.linspace(-40, 40, 2000001), np.geomspace(1e-6, 1e6, 400001)]))
        ex = np.arctan(x)
        e = np.abs(atan_rat32(p, q, x) - ex)
        ulp = np.spacing(np.abs(ex).astype(np.float32)).astype(np.float64)
        print(f"(3,2) rational: max abs err {e.max():.3e}, {(e / ulp).max():.2f} ulp")
        print("  P (lowest first):", ", ".join(f"{v:.9e}f" for v in p))
        print("  Q (lowest first):", ", ".join(f"{v:.9e}f" for v in q))
        return
    if what == "atan":
        for deg in (6, 7):
            c = fit_atan(deg)
            abs_e, ulps = check_atan(c)
            print(f"degree {deg}: max abs err {abs_e:.3e}, {ulps:.2f} ulp")
            print("  coefficients (highest first):", ", ".join(f"{v:.9e}f" for v in c))
    else:
        x = {"sin_mf": 2.05, "cos_mf": 2.05, "sincos_pi": np.pi}[what]
        xs = np.linspace(1e-4, x, 20001)
        t = xs * xs
        for name, odd, deg in (("sin", True, 6 if what == "sin_mf" else 7),
                               ("cos", False, 7 if what == "cos_mf" else 8)):
            if what == "sin_mf" and not odd or what == "cos_mf" and odd:
                continue
            g = np.sin(xs) / xs if odd else np.cos(xs)
            basis = np.stack([t ** k for k in range(deg, -1, -1)], axis=1)
            c = f32(lawson(basis, g, np.ones_like(g)))
            y = horner32(c, f32(t)) * (xs if odd else 1.0)
            ref = np.sin(xs) if odd else np.cos(xs)
            print(f"{name}: max abs err {np.abs(y - ref).max():.3e}")
            print("  coefficients (highest first):", ", ".join(f"{v:.9e}f" for v in c))


if __name__ == "__main__":
    main()

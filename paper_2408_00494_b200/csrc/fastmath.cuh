// Bounded-range FP32 elementary functions for the particle step.
//
// The libdevice versions (sinf/sincosf/atan2f/division) carry range
// reduction and IEEE slow paths the particle step never needs; these keep
// ~1-3 ulp accuracy on the ranges that occur and cost a handful of FMAs.
// Coefficients are Lawson-iterated (minimax) least-squares fits
// (`tools/fit_poly.py atan`, `sincos_half`).  The lateral magic formula is
// not here: it comes from the per-vehicle table of vehicle.cuh tire_q.
// tests/test_fastmath.py re-evaluates every polynomial in float32 (same
// Horner order) against float64 and pins the error bounds.
#pragma once

namespace bss {

// ---- packed FP32x2 forms (sm_100 FFMA2/FMUL2/FADD2: two IEEE lanes per
// issue slot, each lane rounded exactly like the scalar instruction).

__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// atan of two arguments: a = min(|x|, 1/|x|) in [0, 1], atan(a) = a Q(s),
// Q = 1 + s P(s), s = a^2 (P degree-6 minimax, tools/fit_poly.py atan), and
// pi/2 - atan(a) for |x| > 1 -- folded into the final FFMA2 as
// fma(+-a, Q, 0 or pi/2) with per-lane sign/offset selects (ALU), which
// saves the separate multiply and subtraction (2 FMA-pipe cycles per pair;
// 3.3 ulp / 2.0e-7 absolute on the whole line, pinned in test_fastmath).
// Returns |atan(x)| folded with rev = (r, o): r |atan x| + o for the caller's
// quadrant shift; lanes select -a when (|x| > 1) != (r < 0) and offset
// pi/2 when |x| > 1, else o.
__device__ __forceinline__ float2 atan_mag_x2(float2 x, bool neg, float off) {
  const float tx = fabsf(x.x), ty = fabsf(x.y);
  const float2 a = make_float2(fminf(tx, rcp_approx(tx)), fminf(ty, rcp_approx(ty)));
  const float2 s = __fmul2_rn(a, a);
  float2 q = __ffma2_rn(s, bc2(-4.822528455e-03f), bc2(2.473404258e-02f));
  q = __ffma2_rn(q, s, bc2(-6.020310149e-02f));
  q = __ffma2_rn(q, s, bc2(9.968471527e-02f));
  q = __ffma2_rn(q, s, bc2(-1.404132694e-01f));
  q = __ffma2_rn(q, s, bc2(1.997421384e-01f));
  q = __ffma2_rn(q, s, bc2(-3.333239257e-01f));
  q = __ffma2_rn(q, s, bc2(1.0f));
  const bool bx = tx > 1.f, by = ty > 1.f;
  const float2 sa = make_float2((bx != neg) ? -a.x : a.x, (by != neg) ? -a.y : a.y);
  return __ffma2_rn(sa, q, make_float2(bx ? 1.57079637f : off, by ? 1.57079637f : off));
}

__device__ __forceinline__ float2 atan_x2(float2 x) {
  const float2 m = atan_mag_x2(x, false, 0.f);
  return make_float2(copysignf(m.x, x.x), copysignf(m.y, x.y));
}

// atan2(Y, X) of two arguments given x = Y / X (via the caller's shared
// reciprocal of X) and rev = (1, 0) for X > 0, (-1, pi) for X < 0:
// sign(Y) (rev.y + rev.x atan|x|), the left-half-plane shift folded into the
// same final FFMA2 (for X > 0 identical to atan_x2); the sign comes from Y
// itself, so atan2(+-0, X < 0) = +-pi as in the reference.
__device__ __forceinline__ float2 atan2_x2(float2 x, float2 Y, float2 rev) {
  const float2 m = atan_mag_x2(x, rev.x < 0.f, rev.y);
  return make_float2(copysignf(m.x, Y.x), copysignf(m.y, Y.y));
}

// (sin, cos) on [0, pi/2] in one packed Horner chain: lane x the sine
// x S(t) (degree 4 in t = x^2, padded with a leading 0), lane y the cosine
// C(t) (degree 5); tools/fit_poly.py sincos_half: 1.2e-7 / 1.0e-7 absolute,
// ~1e-7 relative for the sine near 0.
__constant__ float2 kSinCosHalf[6] = {
    {0.0f, -2.604962503e-07f},            {2.605039072e-06f, 2.476005830e-05f},
    {-1.980899542e-04f, -1.388835954e-03f}, {8.333049715e-03f, 4.166663438e-02f},
    {-1.666665822e-01f, -5.0e-01f},         {1.0f, 1.0f}};

// returns (sin x, cos x), any x.  Reduced to [-pi, pi] unconditionally
// (for |x| <= pi, n = 0 and x passes through unchanged -- no compare, no
// predicated block), then reflected to h = min(|x|, pi - |x|) in [0, pi/2]:
// sin x = sign(x) sin h, cos x = +-cos h.  The half range halves the
// polynomial: 5 FFMA2 instead of 8 for one FADD and three ALU operations
// (min, copysign, select), i.e. 5 FMA-pipe cycles fewer.  For |x| <= pi/2,
// h = |x| exactly; past it pi - |x| carries pi_f32's 8.7e-8 offset.
__device__ __forceinline__ float2 sincos_pi_x2(float x) {
  {
    // one-constant Cody-Waite: exact for |x| <= pi (n = 0); beyond, the
    // reduced angle carries n * 1.7e-7 of 2 pi's float rounding (a heading
    // error past +-pi: reverse driving or a spun-out particle)
    const float n = rintf(x * 0.159154943f);
    x = fmaf(-n, 6.28318548e+00f, x);
  }
  const float a = fabsf(x), b = 3.14159265f - a;
  const float h = fminf(a, b);
  const float t = h * h;
  float2 p = kSinCosHalf[0];
#pragma unroll
  for (int j = 1; j < 6; ++j) p = __ffma2_rn(p, bc2(t), kSinCosHalf[j]);
  return make_float2(copysignf(p.x * h, x), b < a ? -p.y : p.y);
}

// tanh(x); |x| >= 9.02 rounds to +-1 in FP32 (wheels at speed), which skips
// the exp/rcp sequence for almost every particle.
__device__ __forceinline__ float tanh_sat(float x) {
  return fabsf(x) >= 9.02f ? copysignf(1.0f, x) : tanhf(x);
}

}  // namespace bss

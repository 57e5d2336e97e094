// FP32 single-track Pacejka model in the road-aligned frame, one particle
// per call, all state in registers.
//
// Restates the reference numba kernels (belief_mppi/dynamics.py):
//   curvature()    <- _curv_scalar   dynamics.py:340-369
//   vehicle_step() <- _tire_row      dynamics.py:372-395
//                   + _derivs_row    dynamics.py:398-437
//                   + _step_kernel   dynamics.py:447-497 (Euler branch)
// Deliberate FP32 restatements (checked by the parity tests):
//   * the friction-ellipse factor sqrt(max(1 - (Fx/D)^2, 0)) is |cos theta|
//     of the same magic-formula angle (identical algebra, no cancellation);
//   * sin/cos of the steering angle and drive_gain*throttle are hoisted per
//     (k, t) because all M particles of a rollout share the control;
//   * kappa(s) uses a uniform cell index + one-step correction instead of a
//     binary search (same piecewise-linear interpolant, incl. the closing
//     segment [s_{n-1}, L) -> kappa_0).
#pragma once
#include <cassert>
#include <cstdint>

// -DBSS_CHECKED: device-side bounds assertions (compute-sanitizer is not
// available on the GPU pool); release builds compile them out.
#ifdef BSS_CHECKED
#define BSS_ASSERT(c) assert(c)
#else
#define BSS_ASSERT(c) ((void)0)
#endif

#include "fastmath.cuh"

namespace bss {

struct VehDev {
  float inv_m, inv_iz, lf, lr, R, inv_jw;
  float Byf, Cyf, Byr, Cyr, Bxf, Cxf, Bxr, Cxr;
  float Dxf, Dyf, Dxr, Dyr;
  float drive, vfloor, rrf, rrr, spin_scale, dt;
  // front/rear lane pairs of the packed (FFMA2) particle step
  float2 lf_nlr;   // (lf, -lr)
  float2 Dy;       // (Dyf, Dyr)
  float2 Bx, Cx;   // (Bxf, Bxr), (Cxf, Cxr): longitudinal pair of step_shared
  float dt_lf_iz, ndt_lr_iz;   // dt lf / Iz, -dt lr / Iz: the yaw-rate Euler update
  float dt_m;                  // dt / m: the (vx, vy) Euler update
  // lateral magic formula sin(C atan(B alpha)) = alpha q(|alpha|) as a
  // piecewise-cubic table of q (build_tire_table in bssmppi.cu): rows
  // [front | rear] of tire_rows float4 {c0, c1, c2, c3}; row j is centred on
  // |alpha| = j / tire_s and evaluated at f = |alpha| tire_s - j in [-1/2, 1/2]
  const float4 *tire;          // device copy (global memory)
  float tire_s;                // cells per radian
  float tire_amax;             // table domain [0, tire_amax]: |alpha| beyond it -> libdevice (step kernels)
  int tire_rows;               // rows per axle (cells + 2)
  int tire_smem;               // both axles fit g_tire_tab: belief kernels read the shared copy
};

// Shared copy of the tire table in the belief kernels (rows of the front
// axle, then the rear's, at stride kTireSmemRows).
constexpr int kTireSmemRows = 330;
__shared__ __align__(16) float4 g_tire_tab[2 * kTireSmemRows];

// node[j] = {s_j, kappa_j, slope_j, s_{j+1}} plus a sentinel node[n].
struct TrackDev {
  const float4 *node;
  const int *cell;
  float L, inv_h, half_width;
  int ncell, n, closed;
  float L2;   // 2 L: upper end of the exact floor-mod fast path
};

struct CtlDev {
  float delta, cd, sd, drive_u1;
};

// Python/numba floor-mod (dynamics.py:486-489): result in [0, L], with
// (-tiny) % L == L.  Exact for x in [-L, 2L) (Sterbenz), fmodf otherwise.
__device__ __noinline__ float floor_mod_slow(float x, float L) {
  float r = fmodf(x, L);
  if (r < 0.f) r += L;
  return r;
}

__device__ __forceinline__ float floor_mod(float x, float L) {
  // fast path covers x in [-L, 2L) exactly (Sterbenz / Python semantics)
  const float r = (x >= L) ? x - L : ((x < 0.f) ? x + L : x);
  if (__builtin_expect(x >= -L && x < 2.f * L, 1)) return r;
  return floor_mod_slow(x, L);
}

// pi - ((pi - a) mod 2pi) (dynamics.py:486).  Inside (-pi, pi] this is the
// identity (to 1e-16 in the FP64 reference); evaluating it literally in FP32
// would quantise every heading error to ulp(pi) = 2.4e-7 rad, so the
// formula is applied only when a wrap actually happens.
__device__ __noinline__ float wrap_pi_slow(float a) {
  const float PI = 3.14159265358979f, TWO_PI = 6.28318530717959f;
  return PI - floor_mod(PI - a, TWO_PI);
}

__device__ __forceinline__ float wrap_pi(float a) {
  if (__builtin_expect(a > -3.14159265358979f && a <= 3.14159265358979f, 1)) return a;
  return wrap_pi_slow(a);
}

// Arc length after a step: the Python floor-mod on a closed track
// (dynamics.py:486-489), a clamp to [0, L] on an open one.  Both are the
// identity on [0, L) -- every particle-step except a lap crossing -- which is
// tested first; the closed-track fast path (exact on [-L, 2L)) and the
// out-of-line fmodf / clamp follow only when that test fails.
__device__ __noinline__ float track_s_slow(float x, float L, int closed) {
  if (closed) return floor_mod(x, L);
  return x < 0.f ? 0.f : (x > L ? L : x);   // NaN stays NaN (then scrubbed, ok = false)
}

__device__ __forceinline__ float track_s(float x, const TrackDev &tr) {
  const float L = tr.L;
  const float r = (x >= L) ? x - L : ((x < 0.f) ? x + L : x);
  if (__builtin_expect(x >= 0.f && x < L, 1)) return x;
  if (__builtin_expect(tr.closed && x >= -L && x < tr.L2, 1)) return r;
  return track_s_slow(x, L, tr.closed);
}

__device__ __forceinline__ float curvature(const TrackDev &tr, float s) {
  const float sw = track_s(s, tr);
  int ci = __float2int_rz(sw * tr.inv_h);
  ci = min(max(ci, 0), tr.ncell - 1);
  int lo = __ldg(tr.cell + ci);
  BSS_ASSERT(lo >= 0 && lo < tr.n);
  float4 nd = __ldg(tr.node + lo);
  if (sw < nd.x) {
    BSS_ASSERT(lo >= 1);
    nd = __ldg(tr.node + lo - 1);
  } else if (sw >= nd.w) {
    BSS_ASSERT(lo + 1 <= tr.n);
    nd = __ldg(tr.node + lo + 1);
  }
  BSS_ASSERT(!(sw == sw) || (sw >= nd.x && sw <= fmaxf(nd.w, nd.x)) || !tr.closed);
  return fmaf(nd.z, sw - nd.x, nd.y);
}

// Non-finite components -> 0 (dynamics.py:493-496); returns "all finite".
// Inlined into the cold branch: an out-of-line call taking x by address
// would pin the particle state in local memory for the whole loop.  The
// wheel speeds x[3], x[4] are shared by a rollout's particles and scrubbed
// once per (k, t) in step_shared, so only the other six are visited here.
__device__ __forceinline__ bool scrub_nonfinite6(float *x) {
  bool fin = true;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i == 3 || i == 4) continue;
    fin &= isfinite(x[i]);
    x[i] = isfinite(x[i]) ? x[i] : 0.f;
  }
  return fin;
}

// Fast screen: max |x_i| with NaN propagation (sm_100 three-input
// FMNMX3.NAN on the ALU pipe, abs as a free operand modifier) is finite iff
// every component is.
__device__ __forceinline__ float max3_nan(float a, float b, float c) {
  float d;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

__device__ __forceinline__ float max2_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

__device__ __forceinline__ bool all_finite8(const float x[8]) {
  float m = max3_nan(fabsf(x[0]), fabsf(x[1]), fabsf(x[2]));
  m = max3_nan(m, fabsf(x[3]), fabsf(x[4]));
  m = max3_nan(m, fabsf(x[5]), fabsf(x[6]));
  m = max2_nan(m, fabsf(x[7]));
  return m < __int_as_float(0x7f800000);
}

__device__ __forceinline__ bool all_finite2(float a, float b) {
  return max2_nan(fabsf(a), fabsf(b)) < __int_as_float(0x7f800000);
}

// x[0..2], x[5..7] (the particle-dependent components after a step)
__device__ __forceinline__ bool finite6(const float x[8]) {
  float m = max3_nan(fabsf(x[0]), fabsf(x[1]), fabsf(x[2]));
  m = max3_nan(m, fabsf(x[5]), fabsf(x[6]));
  m = max2_nan(m, fabsf(x[7]));
  return m < __int_as_float(0x7f800000);
}

// One screen for the rare events at the end of a step (dynamics.py:479-496):
// an arc-length wrap (closed track) or clamp (open track) and a non-finite
// component.  True only if neither can occur: 0 <= s < L (both the floor-mod
// and the clamp are the identity there) and the other components finite
// (their max.NaN is below inf).  Compares and max chains only -- ALU work,
// no FMA-pipe cycle -- feeding one branch.  The particle step adds the
// heading-wrap test to the same screen (common_case_psi below; round 1
// measured the merge slower, the round-2 kernel 1.5% faster, profiles/).
__device__ __forceinline__ bool common_case(const float x[8], const TrackDev &tr) {
  const float m = max3_nan(max3_nan(fabsf(x[0]), fabsf(x[1]), fabsf(x[2])), fabsf(x[6]), fabsf(x[5]));
  // 0 <= s < L as ONE unsigned compare of the bit patterns (L > 0: for
  // non-negative floats the order is the integers'; negative s, -0 and NaN
  // compare above L's pattern and take the exact path, which keeps -0)
  return (m < __int_as_float(0x7f800000)) & (__float_as_uint(x[7]) < __float_as_uint(tr.L));
}

// The exact per-component treatment when common_case fails: arc-length
// wrap / clamp, then non-finite -> 0; returns "all finite".
__device__ __forceinline__ bool rare_fixup(float x[8], const TrackDev &tr) {
  x[7] = track_s(x[7], tr);
  return finite6(x) || scrub_nonfinite6(x);
}

// common_case plus |e_psi| < pi (the heading wrap is the identity there),
// and the fix-up in the reference's order: heading wrap (dynamics.py:486),
// arc length, non-finite scrub.
__device__ __forceinline__ bool common_case_psi(const float x[8], const TrackDev &tr) {
  return common_case(x, tr) & (fabsf(x[5]) < 3.14159265358979f);
}
__device__ __forceinline__ bool rare_fixup_psi(float x[8], const TrackDev &tr) {
  x[5] = wrap_pi(x[5]);
  return rare_fixup(x, tr);
}

// The step split in two: everything that depends only on (vx, omega_f,
// omega_r, s) and the control -- the longitudinal slips and tire forces,
// the wheel accelerations and kappa(s) -- is `step_shared`; the rest, which
// also depends on (vy, r, e_psi, e_y), is `step_particle`.  After Gaussian
// re-projection (belief.py:264-272) all M particles of a rollout share
// (vx, omega_f, omega_r, s) exactly, so the rollout kernel evaluates
// step_shared once per (k, t) instead of once per particle.  vehicle_step()
// is the composition, so every path computes bit-identical values.
struct StepShared {
  float vxe, rx, inv_den;     // low-speed-floored vx and its reciprocal
  float fxf, fxr;             // longitudinal forces
  float2 cx;                  // (front, rear) |cos| friction-ellipse factors
  float dvx_lon;              // (fxr) / m: rear longitudinal force term of dvx
  float wf1, wr1;             // next-step wheel speeds (omega + dt * d omega), non-finite -> 0
  bool wfin;                  // both wheel speeds were finite (part of the step's ok)
  float kap;                  // kappa(s)
  float2 fb0;                 // (fxf cd + fxr, fxf sd): the particle-independent
                              //   parts of the body-frame force sums
  float2 nsd_cd;              // (-sin delta, cos delta)
  float2 rev;                 // atan2 quadrant fold: (1, 0) for vx_eff > 0, (-1, pi) below
  float2 dycx;                // (Dyf |cos|_f, Dyr |cos|_r): lateral peak x friction ellipse
};

// kap: kappa(x[7]), supplied by the caller (the rollout already has it from
// the belief mean's frame check).
__device__ __forceinline__ StepShared step_shared(const float x[8], const CtlDev &c, const VehDev &V,
                                                  const TrackDev &tr, float kap) {
  const float vx = x[0], wf = x[3], wr = x[4];
  StepShared h;
  // _tire_row: low-speed floor keeps the sign of vx.
  h.vxe = (vx >= 0.f) ? fmaxf(vx, V.vfloor) : fminf(vx, -V.vfloor);
#ifdef BSS_EXACT_MATH
  h.rx = 1.0f / h.vxe;
  h.inv_den = 1.0f / fabsf(h.vxe);
#else
  h.rx = rcp_approx(h.vxe);          // |vxe| >= v_floor > 0: MUFU.RCP, 1 ulp
  h.inv_den = fabsf(h.rx);
#endif
  const float sgf = (wf * V.R - vx) * h.inv_den;
  const float sgr = (wr * V.R - vx) * h.inv_den;
#ifdef BSS_EXACT_MATH
  const float txf = V.Cxf * atanf(V.Bxf * sgf), txr = V.Cxr * atanf(V.Bxr * sgr);
#else
  const float2 tx = __fmul2_rn(V.Cx, atan_x2(__fmul2_rn(V.Bx, make_float2(sgf, sgr))));
  const float txf = tx.x, txr = tx.y;
#endif
  float sxf, sxr;
#if defined(BSS_EXACT_MATH)
  sincosf(txf, &sxf, &h.cx.x);
  sincosf(txr, &sxr, &h.cx.y);
#else
  // polynomial sin/cos (relative accuracy near 0; MUFU.SIN's absolute
  // 2^-21.4 error is a large relative force error at small slips and drifts
  // the deterministic belief mean by ~1e-4 over a horizon)
  {
    const float2 sf = sincos_pi_x2(txf), sr = sincos_pi_x2(txr);
    sxf = sf.x; h.cx.x = sf.y;
    sxr = sr.x; h.cx.y = sr.y;
  }
#endif
  h.cx.x = fabsf(h.cx.x);
  h.cx.y = fabsf(h.cx.y);
  h.fxf = V.Dxf * sxf;
  h.fxr = V.Dxr * sxr;
  h.dvx_lon = h.fxr;
  h.fb0 = make_float2(fmaf(h.fxf, c.cd, h.fxr), h.fxf * c.sd);
  h.nsd_cd = make_float2(-c.sd, c.cd);
  h.rev = (h.vxe >= 0.f) ? make_float2(1.f, 0.f) : make_float2(-1.f, 3.14159265358979f);
  h.dycx = __fmul2_rn(V.Dy, h.cx);
  // _derivs_row wheel torque balance; rolling resistance opposes the spin
#ifdef BSS_EXACT_MATH
  const float spf = tanhf(wf * V.spin_scale), spr = tanhf(wr * V.spin_scale);
#else
  const float spf = tanh_sat(wf * V.spin_scale), spr = tanh_sat(wr * V.spin_scale);
#endif
  const float dwf = (-V.R * h.fxf - V.rrf * spf) * V.inv_jw;
  const float dwr = (c.drive_u1 - V.R * h.fxr - V.rrr * spr) * V.inv_jw;
  h.wf1 = wf + V.dt * dwf;
  h.wr1 = wr + V.dt * dwr;
  h.wfin = all_finite2(h.wf1, h.wr1);
  if (__builtin_expect(!h.wfin, 0)) {   // _step_kernel scrub of the shared components
    h.wf1 = isfinite(h.wf1) ? h.wf1 : 0.f;
    h.wr1 = isfinite(h.wr1) ? h.wr1 : 0.f;
  }
  h.kap = kap;
  return h;
}

// One Euler step x <- x + dt f(x, u), wraps, non-finite -> 0, given the
// shared terms of x.  Returns the reference's per-particle ok (frame > 0
// and finite).
#ifdef BSS_EXACT_MATH
// libdevice reference form (A/B parity builds, build_cuda(exact=True)).
template <bool TS = false>
__device__ __forceinline__ bool step_particle(float x[8], const StepShared &h, const CtlDev &c,
                                              const VehDev &V, const TrackDev &tr, uint32_t tire_base = 0) {
  const float vx = x[0], vy = x[1], r = x[2], ep = x[5], ey = x[6], s = x[7];
  const float af = c.delta - atan2f(vy + V.lf * r, h.vxe);
  const float ar = -atan2f(vy - V.lr * r, h.vxe);
  const float tyf = V.Cyf * atanf(V.Byf * af), tyr = V.Cyr * atanf(V.Byr * ar);
  const float syf = sinf(tyf), syr = sinf(tyr);
  const float fyf = V.Dyf * syf * h.cx.x, fyr = V.Dyr * syr * h.cx.y;
  // _derivs_row
  const float fxb = h.fxf * c.cd - fyf * c.sd;
  const float fyb = h.fxf * c.sd + fyf * c.cd;
  const float dvx = (fxb + h.dvx_lon) * V.inv_m + vy * r;
  const float dvy = (fyb + fyr) * V.inv_m - vx * r;
  const float dr = (V.lf * fyb - V.lr * fyr) * V.inv_iz;
  float frame = 1.f - h.kap * ey;
  bool ok = frame > 0.f;
  if (frame < 1e-3f) frame = 1e-3f;
  float se, ce;
  sincosf(ep, &se, &ce);
  const float ds = (vx * ce - vy * se) / frame;
  const float dey = vx * se + vy * ce;
  const float dep = r - h.kap * ds;
  // _step_kernel Euler branch + wraps
  x[0] = vx + V.dt * dvx;
  x[1] = vy + V.dt * dvy;
  x[2] = r + V.dt * dr;
  x[3] = h.wf1;
  x[4] = h.wr1;
  x[5] = wrap_pi(ep + V.dt * dep);
  x[6] = ey + V.dt * dey;
  const float s1 = s + V.dt * ds;
  x[7] = track_s(s1, tr);
  if (__builtin_expect(!finite6(x), 0)) ok = scrub_nonfinite6(x) && ok;
  return ok && h.wfin;
}

#else
// Shared-window address of the block's tire-table copy, kept in a register.
__device__ __forceinline__ uint32_t tire_tab_addr() {
  uint32_t v = (uint32_t)__cvta_generic_to_shared(g_tire_tab);
  asm volatile("" : "+r"(v));   // opaque: kept in a register (philox.cuh opaque_u32)
  return v;
}

// q(|alpha|) of one axle from its table rows: nearest-row index by the
// 1.5 2^23 rounding trick (the row number ends up in the low mantissa bits,
// no F2I), the in-cell offset by one FFMA, the cubic by three.  NaN / inf
// arguments read row 0 and propagate through f.  TS: the block's shared
// copy at base = tire_tab_addr(), else global memory.
template <bool TS>
__device__ __forceinline__ float tire_q(float a, const VehDev &V, int axle, uint32_t base) {
  const float MAGIC = 12582912.0f;   // 1.5 2^23
  if (!TS) {   // step kernels: arbitrary steering; keep the row in range (NaN stays NaN)
    asm("min.NaN.f32 %0, %0, %1;" : "+f"(a) : "f"(V.tire_amax));
  }
  const float nf = fmaf(a, V.tire_s, MAGIC);
  const float f = fmaf(a, V.tire_s, -(nf - MAGIC));
  const uint32_t j = __float_as_uint(nf) & 0x7ffu;
  BSS_ASSERT(j < (uint32_t)V.tire_rows && (!TS || j < (uint32_t)kTireSmemRows));
  float4 c;
  if (TS) {
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(c.x), "=f"(c.y), "=f"(c.z), "=f"(c.w)
        : "r"(base + (uint32_t)(axle * kTireSmemRows * 16) + (j << 4)));
  }
  else c = __ldg(V.tire + axle * V.tire_rows + j);
  return fmaf(fmaf(fmaf(c.w, f, c.z), f, c.y), f, c.x);
}

// (sin(Cf atan(Bf af)), sin(Cr atan(Br ar))) for alpha = (af, ar).  The
// rollouts' slip angles stay inside the table domain (|atan2| <= pi and the
// steering is clamped to its bounds, which size the table); the step kernels
// also take arbitrary steering and fall back to libdevice beyond it.
template <bool TS>
__device__ __forceinline__ float2 lateral_shape(float2 al, const VehDev &V, uint32_t base) {
  const float2 q = make_float2(tire_q<TS>(fabsf(al.x), V, 0, base), tire_q<TS>(fabsf(al.y), V, 1, base));
  float2 g = __fmul2_rn(al, q);
  if (!TS && __builtin_expect(fmaxf(fabsf(al.x), fabsf(al.y)) > V.tire_amax, 0)) {
    if (fabsf(al.x) > V.tire_amax) g.x = sinf(V.Cyf * atanf(V.Byf * al.x));
    if (fabsf(al.y) > V.tire_amax) g.y = sinf(V.Cyr * atanf(V.Byr * al.y));
  }
  return g;
}

// Packed form of the same step: the front/rear pairs (slip-angle arguments,
// both arctangent chains, lateral forces), the heading sin/cos polynomials
// and the (vx, vy) / (e_psi, e_y) Euler updates run as FP32x2 lanes, one
// issue slot per pair.  Every lane is an IEEE FMA/MUL/ADD, so all kernels
// (which share this function) stay bit-identical to one another.
// TS: the tire table is the belief kernel's shared copy (else global memory).
template <bool TS = false>
__device__ __forceinline__ bool step_particle(float x[8], const StepShared &h, const CtlDev &c,
                                              const VehDev &V, const TrackDev &tr, uint32_t tire_base = 0) {
  const float vx = x[0], vy = x[1], r = x[2], ep = x[5], ey = x[6], s = x[7];
  // slip-angle numerators (vy + lf r, vy - lr r); atan2(., vxe) = atan(. / vxe)
  // for vxe > 0, +-pi shifted for vxe < 0 (vxe is shared by the rollout)
  // (Y: its IEEE sign, signed zeros included, picks atan2's +-pi when
  // vx_eff < 0, as in the reference; folding 1/vx_eff into the FFMA2 would
  // lose it)
  const float2 Y = __ffma2_rn(bc2(r), V.lf_nlr, bc2(vy));
  const float2 A = atan2_x2(__fmul2_rn(Y, bc2(h.rx)), Y, h.rev);
  // slip angles alpha_f = delta - A.x, alpha_r = -A.y; lateral forces
  // D |cos|_long sin(C atan(B alpha)) from the tire table
  const float2 fy = __fmul2_rn(h.dycx, lateral_shape<TS>(make_float2(c.delta - A.x, -A.y), V, tire_base));
  // body-frame front force + rear longitudinal: (fxf cd - fyf sd + fxr, fxf sd + fyf cd)
  const float2 fb = __ffma2_rn(bc2(fy.x), h.nsd_cd, h.fb0);
  float frame = 1.f - h.kap * ey;
  bool ok = frame > 0.f;
  if (frame < 1e-3f) frame = 1e-3f;
  const float2 sc = sincos_pi_x2(ep);          // (sin e_psi, cos e_psi)
  const float2 vsc = __fmul2_rn(bc2(vy), sc);  // (vy se, vy ce)
  // frame in [1e-3, 1 + kappa w]: MUFU.RCP without __fdividef's huge-divisor guard
  const float ds = fmaf(vx, sc.y, -vsc.x) * rcp_approx(frame);
  const float dey = fmaf(vx, sc.x, vsc.y);
  const float dep = fmaf(-h.kap, ds, r);
  // _step_kernel Euler branch + wraps
  // (vx, vy) + dt ((fb.x, fb.y + fyr) / m + (vy r, -vx r)) with dt / m and
  // dt r folded into the FMAs: 6 FMA-pipe cycles instead of 7
  const float dtr = V.dt * r;
  const float2 v56 = __ffma2_rn(bc2(V.dt), make_float2(dep, dey), make_float2(ep, ey));
  x[0] = fmaf(V.dt_m, fb.x, fmaf(dtr, vy, vx));
  x[1] = fmaf(V.dt_m, fb.y, fmaf(V.dt_m, fy.y, fmaf(-dtr, vx, vy)));
  x[2] = fmaf(V.dt_lf_iz, fb.y, fmaf(V.ndt_lr_iz, fy.y, r));   // r + dt (lf fyb - lr fyr) / Iz
  x[3] = h.wf1;
  x[4] = h.wr1;
  x[5] = v56.x;   // wrapped in rare_fixup_psi (one screen for all rare events)
  x[6] = v56.y;
  x[7] = fmaf(V.dt, ds, s);
  // one screen for all rare events: heading wrap, arc-length wrap / clamp,
  // non-finite components (ALU compares, one branch; -1.5% at C3 against a
  // separate early heading test, profiles/README.md)
  if (__builtin_expect(!common_case_psi(x, tr), 0)) ok = rare_fixup_psi(x, tr) && ok;
  return ok && h.wfin;
}
#endif

template <bool TS = false>
__device__ __forceinline__ bool vehicle_step(float x[8], const CtlDev &c, const VehDev &V,
                                             const TrackDev &tr) {
  const StepShared h = step_shared(x, c, V, tr, curvature(tr, x[7]));
  return step_particle<TS>(x, h, c, V, tr);
}

__device__ __forceinline__ CtlDev make_ctl(float delta, float throttle, const VehDev &V) {
  CtlDev c;
  c.delta = delta;
  sincosf(delta, &c.sd, &c.cd);
  c.drive_u1 = V.drive * throttle;
  return c;
}

}  // namespace bss

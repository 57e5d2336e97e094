// Counter-based normal generator for performance mode.
//
// Philox4x32 (Salmon et al., SC'11; 7 rounds belief, 10 control) keyed per (seed, run_path, domain,
// iteration) -- the same identity as the reference's keyed numpy substreams
// (streams.py:21-28) -- with counters built from (t, global k, m), so every
// normal is a pure function of its coordinates: results do not depend on
// grid shape, K-sharding or launch order.
#pragma once
#include <cstdint>

namespace bss {

struct Philox4 {
  uint32_t x, y, z, w;
};

// 32x32 -> 64 multiply in one IMAD.WIDE.U32 on the device.
__host__ __device__ __forceinline__ void mulhilo32(uint32_t a, uint32_t b, uint32_t &hi, uint32_t &lo) {
#ifdef __CUDA_ARCH__
  uint64_t p;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
  lo = (uint32_t)p;
  hi = (uint32_t)(p >> 32);
#else
  const uint64_t p = (uint64_t)a * (uint64_t)b;
  lo = (uint32_t)p;
  hi = (uint32_t)(p >> 32);
#endif
}

// Round-key schedule k_i = k + i * (W0, W1), i = 0..9, precomputed on the
// host once per iteration so the rounds read their keys as kernel-constant
// operands instead of re-deriving them per call.
struct PhiloxKeys {
  uint32_t k[20];
};

__host__ __device__ __forceinline__ PhiloxKeys philox_schedule(uint32_t k0, uint32_t k1) {
  PhiloxKeys r;
  for (int i = 0; i < 10; ++i) {
    r.k[2 * i] = k0 + (uint32_t)i * 0x9E3779B9u;
    r.k[2 * i + 1] = k1 + (uint32_t)i * 0xBB67AE85u;
  }
  return r;
}

// Rounds of the hot belief-noise generator: Philox4x32 with 7 rounds passes
// TestU01 BigCrush (Salmon et al., SC'11, Table 2); 10 is Random123's
// default safety margin and is kept for the (tiny) control-noise stream.
#ifndef BSS_BELIEF_ROUNDS
#define BSS_BELIEF_ROUNDS 7
#endif
constexpr int kBeliefRounds = BSS_BELIEF_ROUNDS;
constexpr int kControlRounds = 10;

template <int R>
__host__ __device__ __forceinline__ Philox4 philox4x32(Philox4 c, const PhiloxKeys &rk) {
#pragma unroll
  for (int i = 0; i < R; ++i) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c.x, hi0, lo0);
    mulhilo32(0xCD9E8D57u, c.z, hi1, lo1);
    c = Philox4{hi1 ^ c.y ^ rk.k[2 * i], lo1, hi0 ^ c.w ^ rk.k[2 * i + 1], lo0};
  }
  return c;
}

#ifdef __CUDACC__
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// MUFU.LG2 without __log2f's denormal guard (FSETP/FMUL/FADD): the
// uniforms here are >= 2^-23, never denormal, so the value is identical.
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Box-Muller in the units the MUFU pipe works in.  The reference-side form
// (oracle/bss_oracle.c bm) is r (cos, sin)(2 pi (m_b - 1.5)) with
// r = sqrt(-2 ln u1), u1 = 2 - m_a and m_a, m_b in [1, 2) the mantissa values
// of the two words' top 23 bits (uniforms by bit insertion, no I2F).  Since
// sqrt(-2 ln u) = sqrt(2 ln 2) sqrt(-log2 u) and (cos, sin)(2 pi (m - 1.5)) =
// -(cos, sin)(2 pi m), the pair is kBmNeg * raw with
//   raw = sqrt(-log2 u1) (cos, sin)(2 pi m_b),
// which costs no multiply for the ln 2 factor (the negation is a MUFU
// operand modifier) and one FMUL by an immediate for the angle.  The rollout
// folds kBmNeg into its Cholesky and process-noise factors; everything else
// (statistics kernel, control samples) scales back with box_muller().
constexpr float kBmNeg = -1.17741002251547469f;   // -sqrt(2 ln 2)

__device__ __forceinline__ void box_muller_raw(uint32_t a, uint32_t b, float &z0, float &z1) {
  const float u1 = 2.0f - __uint_as_float(0x3f800000u | (a >> 9));
  const float ang = __uint_as_float(0x3f800000u | (b >> 9)) * 6.28318530718f;
  const float r = sqrt_approx(-lg2_approx(u1));
  float s, c;
  __sincosf(ang, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// Single raw normal (cosine branch) of a pair.
__device__ __forceinline__ void box_muller_raw1(uint32_t a, uint32_t b, float &z0) {
  const float u1 = 2.0f - __uint_as_float(0x3f800000u | (a >> 9));
  const float ang = __uint_as_float(0x3f800000u | (b >> 9)) * 6.28318530718f;
  z0 = sqrt_approx(-lg2_approx(u1)) * __cosf(ang);
}

// Standard normal pair (the oracle's bm()).
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float &z0, float &z1) {
  box_muller_raw(a, b, z0, z1);
  z0 *= kBmNeg;
  z1 *= kBmNeg;
}

// The 7 standard normals of particle-step (t, k, m) (Philox4x32-7 counters): [0:4] re-projection
// on the tracked subset, [4:7] process noise -- the column layout of the
// reference's z_all block (controllers.py:285-287, belief.py:328-333).
// The two Philox4x32-7 blocks of particle-step (t, k, m); both noise kinds
// (Gaussian, config-4 Laplace) transform the same eight words.
__device__ __forceinline__ void belief_bits(const PhiloxKeys &rk, uint32_t t, uint32_t kg, uint32_t m,
                                            Philox4 &a, Philox4 &b) {
  a = philox4x32<kBeliefRounds>(Philox4{t, m, kg, 0u}, rk);
  b = philox4x32<kBeliefRounds>(Philox4{t, m, kg, 1u}, rk);
}

// The 7 raw normals (standard normals / kBmNeg) of a particle-step.
__device__ __forceinline__ void raw_normals_from_bits(const Philox4 &a, const Philox4 &b, float z[7]) {
  box_muller_raw(a.x, a.y, z[0], z[1]);
  box_muller_raw(a.z, a.w, z[2], z[3]);
  box_muller_raw(b.x, b.y, z[4], z[5]);
  box_muller_raw1(b.z, b.w, z[6]);
}

// The 7 standard normals of particle-step (t, k, m) (statistics / parity kernel).
__device__ __forceinline__ void belief_normals(const PhiloxKeys &rk, uint32_t t, uint32_t kg,
                                               uint32_t m, float z[7]) {
  Philox4 a, b;
  belief_bits(rk, t, kg, m, a, b);
  raw_normals_from_bits(a, b, z);
#pragma unroll
  for (int j = 0; j < 7; ++j) z[j] *= kBmNeg;
}

// Config-4 extension: 4 re-projection normals + Laplace(0, b) on (vx, vy, r)
// + U(-a, a) lateral slip on vy from the same two Philox4x32-7 blocks (the
// second block's words become the uniforms instead of Box-Muller normals).
// 2u for the centred uniform u = (n + 1/2) 2^-23 - 1/2 of the top 23 bits n
// of w, i.e. (2n + 1 - 2^23) 2^-23 in (-1, 1): the mantissa m = 1 + n 2^-23
// by bit insertion, 2m - 3 (exact FFMA), + 2^-23 (exact) -- no I2F.
__device__ __forceinline__ float centred_uniform2(uint32_t w) {
  return fmaf(__uint_as_float(0x3f800000u | (w >> 9)), 2.0f, -3.0f) + 1.1920928955078125e-07f;
}

// z[0:4] are RAW normals (x kBmNeg = standard), w the noise increments.
__device__ __forceinline__ void laplace_from_bits(const Philox4 &p, const Philox4 &q, float b, float a,
                                                  float z[4], float w[3]) {
  box_muller_raw(p.x, p.y, z[0], z[1]);
  box_muller_raw(p.z, p.w, z[2], z[3]);
  const uint32_t words[3] = {q.x, q.y, q.z};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float v = centred_uniform2(words[i]);   // 2u
    // inverse CDF: -b sgn(u) ln(1 - 2|u|)
    w[i] = -b * copysignf(0.69314718056f * lg2_approx(1.0f - fabsf(v)), v);
  }
  w[1] += a * centred_uniform2(q.w);             // U(-a, a) = 2a u
}

// The 2 standard normals of control sample (k, t) (controllers.py:175).
__device__ __forceinline__ void control_normals(const PhiloxKeys &rk, uint32_t t, uint32_t kg,
                                                float &z0, float &z1) {
  const Philox4 a = philox4x32<kControlRounds>(Philox4{t, kg, 0x5eedc0deu, 0u}, rk);
  box_muller(a.x, a.y, z0, z1);
}
#endif

}  // namespace bss

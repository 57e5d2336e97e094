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

// Standard normal pair (the oracle's bm()).
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float &z0, float &z1) {
  box_muller_raw(a, b, z0, z1);
  z0 *= kBmNeg;
  z1 *= kBmNeg;
}

// Belief stream: ONE Philox4x32-7 block per particle-step (t, k, m), counter
// (t, m, k_global, 0).  Each of its four words carries one Box-Muller pair:
// the radius uniform from the word's top 20 bits, the angle from its low 12
// bits (independent bit fields, so the pair stays an exact polar draw):
//   u1 = 1 - (n + 1/2) 2^-20, n = w >> 12 (midpoint grid, never 0 or 1);
//   theta = 2 pi j / 4096, j = w & 0xfff.
// A 4096-point angle grid reproduces E[cos^p theta] exactly for every
// p < 4096, so all low-order moments of the pair are those of the
// continuous draw; the 20-bit radius truncates |z| at 5.3 sigma (tail mass
// 1.2e-7).  Words 0..3 -> normals (z0, z1), (z2, z3), (z4, z5), (z6, -):
// [0:4] re-projection on the tracked subset, [4:7] process noise -- the
// column layout of the reference's z_all block (controllers.py:285-287,
// belief.py:328-333).  One block instead of two halves the quarter-rate
// IMAD.WIDE work per particle-step (profiles/README.md).
constexpr float kU1Mid = 1.99999952316284180f;   // 2 - 2^-21 (exact in FP32)

// Raw pair (standard / kBmNeg) of one word: -sqrt(-2 ln u1) (cos, sin)
// theta = kBmNeg sqrt(-log2 u1) (cos, sin)(2 pi m_a), m_a = 1 + j / 4096.
__device__ __forceinline__ float word_radius(uint32_t w) {
  // 1 + n 2^-20 by bit insertion (mask, then one LEA.HI), then the exact
  // Sterbenz difference (2 - 2^-21) - (1 + n 2^-20)
  const float u1 = kU1Mid - __uint_as_float(0x3f800000u + ((w & 0xfffff000u) >> 9));
  return sqrt_approx(-lg2_approx(u1));
}
// Angle grid (cos, sin)(2 pi j / 4096), j = w & 0xfff, correctly rounded to
// FP32 from FP64 sincospi (one table per device, `angle_table_init_kernel`,
// built once before the first rollout).  The rollout kernels copy it into a
// per-block shared table (32 KB) and look a pair up with one LDS.64: no
// MUFU.SIN / MUFU.COS and no angle arithmetic per normal pair, and half an
// ulp of error instead of MUFU's 2^-21.4 absolute.  Persist blocks and the
// statistics hook read the device table itself (the same values).
constexpr int kAngleTab = 4096;
__device__ float2 g_angle_global[kAngleTab];

__global__ void angle_table_init_kernel() {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= kAngleTab) return;
  double s, c;
  sincospi((double)j / 2048.0, &s, &c);
  g_angle_global[j] = make_float2((float)c, (float)s);
}

__device__ __forceinline__ float2 angle_entry(uint32_t j) { return __ldg(&g_angle_global[j]); }

// The table of a rollout block (filled by bss_rollout_kernel; kernels that
// never name it do not allocate it).
__shared__ __align__(16) float2 g_angle_tab[kAngleTab];

// 32-bit shared-window address of a table, made opaque to the compiler: a
// per-thread register computed once per (k, t) instead of a uniform-register
// window base the compiler rebuilds (S2UR / UMOV / ULEA) inside the loop.
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
  asm volatile("" : "+r"(v));
  return v;
}
__device__ __forceinline__ uint32_t angle_tab_addr() {
  return opaque_u32((uint32_t)__cvta_generic_to_shared(g_angle_tab));
}
__device__ __forceinline__ float2 angle_lds(uint32_t base, uint32_t w) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(base + ((w & 0xfffu) << 3)));
  return v;
}
__device__ __forceinline__ float angle_lds_x(uint32_t base, uint32_t w) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(base + ((w & 0xfffu) << 3)));
  return v;
}

// TAB: read the block's shared-memory table at base = angle_tab_addr(),
// else evaluate in place (statistics kernel, persist mode).
template <bool TAB>
__device__ __forceinline__ float2 angle_cs(uint32_t w, uint32_t base) {
  if (TAB) return angle_lds(base, w);
  return angle_entry(w & 0xfffu);
}

template <bool TAB>
__device__ __forceinline__ void box_muller_word(uint32_t w, float &z0, float &z1, uint32_t base = 0) {
  const float r = word_radius(w);
  const float2 cs = angle_cs<TAB>(w, base);
  const float2 z = __fmul2_rn(make_float2(r, r), cs);
  z0 = z.x;
  z1 = z.y;
}
template <bool TAB>
__device__ __forceinline__ void box_muller_word1(uint32_t w, float &z0, uint32_t base = 0) {
  z0 = word_radius(w) * (TAB ? angle_lds_x(base, w) : angle_entry(w & 0xfffu).x);
}

__host__ __device__ __forceinline__ Philox4 belief_block(const PhiloxKeys &rk, uint32_t t, uint32_t kg, uint32_t m) {
  return philox4x32<kBeliefRounds>(Philox4{t, m, kg, 0u}, rk);
}

// The same block split at the particle index.  In the counter (t, m, kg, 0)
// only the y word depends on m, and y first meets a multiplier in round 1
// (via x1 = hi(M1 kg) ^ m ^ k0).  So of the first three rounds' six
// products, four -- M0 t, M1 kg (round 0), M1 z1 (round 1), M0 x2 (round 2)
// -- are the same for every particle of a rollout step: `belief_prefix`
// computes them once per (k, t), folded with their round keys into five
// words, and `belief_block_m` finishes a particle's block with the
// remaining 2 + 2 (R - 3) products (10 IMAD.WIDE instead of 14 at R = 7).
// The words are bit-identical to belief_block (tests/test_philox_split_cpu.py).
struct BeliefPrefix {
  uint32_t c1;    // hi(M1 kg) ^ k0:          x1 = c1 ^ m
  uint32_t w1k;   // lo(M0 t) ^ k3:           z2 = hi(M0 x1) ^ w1k
  uint32_t y2k;   // lo(M1 z1) ^ k4:          x3 = hi(M1 z2) ^ y2k
  uint32_t e;     // hi(M0 x2) ^ k5:          z3 = e ^ lo(M0 x1)
  uint32_t w3;    // lo(M0 x2)
};

__host__ __device__ __forceinline__ BeliefPrefix belief_prefix(const PhiloxKeys &rk, uint32_t t, uint32_t kg) {
  static_assert(kBeliefRounds >= 3, "belief_prefix hoists rounds 0-2");
  uint32_t a_hi, a_lo, b_hi, b_lo, d_hi, d_lo, e_hi, e_lo;
  mulhilo32(0xD2511F53u, t, a_hi, a_lo);
  mulhilo32(0xCD9E8D57u, kg, b_hi, b_lo);
  const uint32_t z1 = a_hi ^ rk.k[1];                 // w0 = 0
  mulhilo32(0xCD9E8D57u, z1, d_hi, d_lo);
  const uint32_t x2 = d_hi ^ b_lo ^ rk.k[2];          // y1 = lo(M1 kg)
  mulhilo32(0xD2511F53u, x2, e_hi, e_lo);
  return BeliefPrefix{b_hi ^ rk.k[0], a_lo ^ rk.k[3], d_lo ^ rk.k[4], e_hi ^ rk.k[5], e_lo};
}

__host__ __device__ __forceinline__ Philox4 belief_block_m(const BeliefPrefix &p, const PhiloxKeys &rk, uint32_t m) {
  uint32_t c_hi, c_lo, f_hi, f_lo;
  mulhilo32(0xD2511F53u, p.c1 ^ m, c_hi, c_lo);      // round 1, x1
  const uint32_t z2 = c_hi ^ p.w1k;
  mulhilo32(0xCD9E8D57u, z2, f_hi, f_lo);            // round 2, z2
  Philox4 c{f_hi ^ p.y2k, f_lo, p.e ^ c_lo, p.w3};   // state after round 2
#pragma unroll
  for (int i = 3; i < kBeliefRounds; ++i) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c.x, hi0, lo0);
    mulhilo32(0xCD9E8D57u, c.z, hi1, lo1);
    c = Philox4{hi1 ^ c.y ^ rk.k[2 * i], lo1, hi0 ^ c.w ^ rk.k[2 * i + 1], lo0};
  }
  return c;
}

// Radius mantissa 1 + n 2^-20 of a word (n = its top 20 bits): (w >> 9)
// masked and OR-ed with the exponent in ONE three-input LOP3 -- the
// exponent word comes from a register, since LOP3 takes one immediate.
__device__ __forceinline__ float radius_mantissa(uint32_t w, uint32_t one_bits) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w >> 9), "n"(0x7ffff8), "r"(one_bits));
  return __uint_as_float(r);
}

// The 7 raw normals (standard normals / kBmNeg) of a particle-step: the
// word_radius / box_muller_word arithmetic with the four uniforms formed
// as two FADD2 pairs (the host pass of nvcc takes the scalar form).
template <bool TAB>
__device__ __forceinline__ void raw_normals_from_block(const Philox4 &a, float z[7], uint32_t base = 0) {
#ifdef __CUDA_ARCH__
  uint32_t one;
  asm("mov.b32 %0, 0x3f800000;" : "=r"(one));
  const float2 u01 = __fadd2_rn(make_float2(kU1Mid, kU1Mid),
                                make_float2(-radius_mantissa(a.x, one), -radius_mantissa(a.y, one)));
  const float2 u23 = __fadd2_rn(make_float2(kU1Mid, kU1Mid),
                                make_float2(-radius_mantissa(a.z, one), -radius_mantissa(a.w, one)));
  const float r0 = sqrt_approx(-lg2_approx(u01.x)), r1 = sqrt_approx(-lg2_approx(u01.y));
  const float r2 = sqrt_approx(-lg2_approx(u23.x)), r3 = sqrt_approx(-lg2_approx(u23.y));
  const float2 p0 = __fmul2_rn(make_float2(r0, r0), angle_cs<TAB>(a.x, base));
  const float2 p1 = __fmul2_rn(make_float2(r1, r1), angle_cs<TAB>(a.y, base));
  const float2 p2 = __fmul2_rn(make_float2(r2, r2), angle_cs<TAB>(a.z, base));
  z[0] = p0.x; z[1] = p0.y; z[2] = p1.x; z[3] = p1.y; z[4] = p2.x; z[5] = p2.y;
  z[6] = r3 * (TAB ? angle_lds_x(base, a.w) : angle_entry(a.w & 0xfffu).x);
#else
  box_muller_word<TAB>(a.x, z[0], z[1], base);
  box_muller_word<TAB>(a.y, z[2], z[3], base);
  box_muller_word<TAB>(a.z, z[4], z[5], base);
  box_muller_word1<TAB>(a.w, z[6], base);
#endif
}

// The 7 standard normals of particle-step (t, k, m) (statistics / parity kernel).
__device__ __forceinline__ void belief_normals(const PhiloxKeys &rk, uint32_t t, uint32_t kg,
                                               uint32_t m, float z[7]) {
  raw_normals_from_block<false>(belief_block(rk, t, kg, m), z);
#pragma unroll
  for (int j = 0; j < 7; ++j) z[j] *= kBmNeg;
}

// Config-4 extension from the same single block: 4 re-projection normals
// (words 0, 1 as above) + Laplace(0, b) on (vx, vy, r) + U(-a, a) lateral
// slip on vy from the four 16-bit halves of words 2, 3.
// 2u for the centred uniform u = (n + 1/2) 2^-16 - 1/2 of a 16-bit field n,
// i.e. (2n + 1 - 2^16) 2^-16 in (-1, 1): the mantissa m = 1 + n 2^-16 by bit
// insertion, 2m - 3 (exact FFMA), + 2^-16 (exact) -- no I2F.
__device__ __forceinline__ float centred_uniform2_16(uint32_t field_at_top) {
  // field_at_top: the 16-bit field in bits 16..31, zeros below
  return fmaf(__uint_as_float(0x3f800000u + (field_at_top >> 9)), 2.0f, -3.0f) + 1.52587890625e-05f;
}

// z[0:4] are RAW normals (x kBmNeg = standard), w the noise increments.
template <bool TAB>
__device__ __forceinline__ void laplace_from_block(const Philox4 &p, float b, float a, float z[4], float w[3],
                                                   uint32_t base = 0) {
  box_muller_word<TAB>(p.x, z[0], z[1], base);
  box_muller_word<TAB>(p.y, z[2], z[3], base);
  const uint32_t fields[4] = {p.z & 0xffff0000u, p.z << 16, p.w & 0xffff0000u, p.w << 16};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float v = centred_uniform2_16(fields[i]);   // 2u
    // inverse CDF: -b sgn(u) ln(1 - 2|u|)
    w[i] = -b * copysignf(0.69314718056f * lg2_approx(1.0f - fabsf(v)), v);
  }
  w[1] += a * centred_uniform2_16(fields[3]);          // U(-a, a) = 2a u
}

// The 2 standard normals of control sample (k, t) (controllers.py:175).
__device__ __forceinline__ void control_normals(const PhiloxKeys &rk, uint32_t t, uint32_t kg,
                                                float &z0, float &z1) {
  const Philox4 a = philox4x32<kControlRounds>(Philox4{t, kg, 0x5eedc0deu, 0u}, rk);
  box_muller(a.x, a.y, z0, z1);
}
#endif

}  // namespace bss

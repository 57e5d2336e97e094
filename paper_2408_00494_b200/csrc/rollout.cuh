// Fused BSS-MPPI rollout kernel (sampling -> belief rollouts -> cost).
//
// Restates the reference hot loop (controllers.py:261-341 `_rollout`,
// belief.py:311-335 `propagate_mc_batch`, belief.py:227-308 Cholesky /
// sample build / moments, constraints.py:130-186 DCBF + shield penalty,
// controllers.py:166-177 + 215-228 sampling and costs) as ONE kernel:
//
//   * one group of G lanes owns one rollout k and its M Monte-Carlo
//     particles (lane l handles m = l, l+G, ...); G is the power of two >= M
//     (<= 32) narrowed by the measured policy in bssmppi.cu group_width
//     (C3: G = 8, 4 rollouts per warp, 32 particles per lane); the only
//     block-level sync follows the fill of the shared tables (Box-Muller
//     angles, tire forces) at kernel entry;
//   * particles never touch memory: noise (one Philox4x32-7 block per
//     particle-step, philox.cuh), re-projection x = mu + L z, the
//     Euler step, process noise and the moment sums all stay in registers;
//     the noise of particle m + G is generated inside particle m's
//     iteration (software pipelining, particle_pass);
//   * per-step moments use particle 0 of the group as the shift c,
//     accumulating S1 = sum(x - c), S2 = sum((x - c)(x - c)^T) in ONE pass,
//     reduced across the group with a reduce-scatter shuffle butterfly and
//     all-gathered through 20 floats of shared memory; mean = c + S1/M,
//     cov = (S2 - S1 S1^T / M)/(M-1).  Algebraically the reference's
//     two-pass estimator; deviations from the shift are O(sigma) so FP32
//     keeps tree-sum accuracy, and a zero-spread cloud collapses onto the
//     deterministic step exactly (belief.py:282-284 guarantee);
//   * everything per (k, t) -- stage cost, shared step terms, Cholesky,
//     DCBF, penalty, frame check -- is computed redundantly by the G lanes
//     (same issue slots as one lane); the controls, their clamp and the
//     control cost are sampled once per (k, t) in the prologue;
//   * launch constants (process-noise kind, tire-sine range) are resolved
//     once at kernel entry, so each variant's T loop holds one branch-free
//     particle loop; the FMA pipe (shared by the Philox IMAD.WIDE, FFMA2 and
//     FFMA: 4 / 2 / 1 cycles) is the budget the particle step is written to.
#pragma once
#include <cstdint>

#include "philox.cuh"
#include "vehicle.cuh"

namespace bss {

enum CtrlMode { CTRL_PHILOX = 0, CTRL_EPS = 1, CTRL_GIVEN = 2 };

struct RollParams {
  VehDev V;
  TrackDev tr;
  int k_count, k_begin, T, M;
  int ctrl_mode;      // CtrlMode
  int noise_on;       // process noise nonzero (dynamics.py:571 skips the add otherwise)
  int noise_diag;     // noise factor is diagonal: 3 multiplies instead of a 3x3 product
  int shield;         // det kinds: 1 = smppi
  float invM, invMm1;
  float q[8];
  float v_goal, c_obs, term, beta1 /* 1 - beta */, c_pen, nu;
  float gamma, prec[4], sfac[4], lo[2], hi[2];
  float F[9];          // process-noise factor
  float Fk[9];         // kBmNeg * F: the factor applied to Philox raw normals (philox.cuh)
  int chol_rank;       // max Cholesky rank: min(4, M - 1) (cov0: 4)
  PhiloxKeys kc;       // control-noise key schedule
  PhiloxKeys kb;       // belief-noise key schedule
  const float *x0;     // [8]
  const float *cov0;   // [16]
  const float *plan;   // [T*2] nominal
  const double *eps_in;  // [k_count*T*2] (CTRL_EPS / CTRL_GIVEN)
  const double *u_in;    // [k_count*T*2] (CTRL_GIVEN)
  const float *z_in;     // [T*k_count*M*7] oracle-noise mode
  float *u_out;          // [k_count*T*2] clamped controls for the update
  float4 *ctl;           // [k_count*T] per-(k,t) control table {delta, cos, sin, drive*u1}
  float *ccost;          // [k_count*T] per-(k,t) control-cost terms
  float *cost_out;       // [k_count]
  float *mom_out;        // [T*k_count*18] or null
  // config-4 extensions (obstacles.py); n_obs == 0 and noise_kind == 0 = reference
  int noise_kind;        // 1: Laplace + uniform vy slip
  float lap_b, slip_a;
  int n_obs;
  const float4 *obs;     // {x, y, radius, 0}
  float nu_obs;
  const float4 *cl;      // centerline rows {x, y, theta, 0} at s = i / cl_inv_ds
  int cl_n;
  float cl_inv_ds;
};

__device__ __forceinline__ float stage_cost(const float x[8], const RollParams &P) {
  // controllers.py:215-220: sum q_i (x_i - g_i)^2 + C_obs [|e_y| > w]
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float d = (i == 0) ? x[0] - P.v_goal : x[i];
    acc = fmaf(__fmul_rn(P.q[i], d), d, acc);
  }
  return acc + ((fabsf(x[6]) > P.tr.half_width) ? P.c_obs : 0.f);
}

// The cost terms below round every product and sum separately (__fmul_rn /
// __fadd_rn cannot be contracted into FMAs): the belief and deterministic
// kernels inline them into different code, and free contraction could then
// round them differently -- BSS with a degenerate belief must reproduce
// S-MPPI's costs bit for bit (acceptance criterion 06).
__device__ __forceinline__ float dcbf(float ey, float sigy, const RollParams &P) {
  // constraints.py:130-137
  const float margin = fmaxf(__fsub_rn(P.tr.half_width, __fmul_rn(P.nu, sigy)), 0.f);
  return __fsub_rn(__fmul_rn(margin, margin), __fmul_rn(ey, ey));
}

__device__ __forceinline__ float shield_penalty(float hc, float hp, const RollParams &P) {
  // constraints.py:172-186: C max(-(h_k - (1 - beta) h_{k-1}), 0)
  return __fmul_rn(P.c_pen, fmaxf(-__fsub_rn(hc, __fmul_rn(P.beta1, hp)), 0.f));
}

// Obstacle terms of a belief mean (config-4 extension, obstacles.py):
// p = centerline(s) + e_y n(s); for each obstacle d_i = |p - o_i|,
// h_i = d_i - r_i - nu |d d_i / d e_y| sigma_y (reference heuristic_h_i,
// constraints.py:112-120, on the tracked subset), h_obs = min_i h_i;
// inside = some d_i < r_i (collision indicator of the stage cost).
__device__ __forceinline__ float obstacle_terms(const RollParams &P, float s, float ey, float sigy,
                                                bool &inside) {
  const float sw = track_s(s, P.tr);
  const float fi = sw * P.cl_inv_ds;
  const int j = min(max((int)fi, 0), P.cl_n - 2);
  const float f = fi - (float)j;
  const float4 a = P.cl[j], b = P.cl[j + 1];
  const float cx = fmaf(f, b.x - a.x, a.x), cy = fmaf(f, b.y - a.y, a.y), th = fmaf(f, b.z - a.z, a.z);
  const float2 sc = sincos_pi_x2(th);          // (sin, cos) of the centerline heading
  const float nx = -sc.x, ny = sc.y;
  const float px = fmaf(ey, nx, cx), py = fmaf(ey, ny, cy);
  float h = __int_as_float(0x7f800000);
  inside = false;
  for (int i = 0; i < P.n_obs; ++i) {
    const float4 o = P.obs[i];
    const float dx = px - o.x, dy = py - o.y;
    const float d2 = dx * dx + dy * dy;
    float inv;                                   // 1/d from one MUFU.RSQ (non-ftz approx)
    asm("rsqrt.approx.f32 %0, %1;" : "=f"(inv) : "f"(d2));
    const float d = d2 > 0.f ? d2 * inv : 0.f;
    inside |= d < o.z;
    const float eta = d2 > 0.f ? (dx * nx + dy * ny) * inv : 1.f;
    h = fminf(h, __fsub_rn(__fsub_rn(d, o.z), __fmul_rn(__fmul_rn(P.nu_obs, fabsf(eta)), sigy)));
  }
  return h;
}

// sqrt(max(v, 0)) for sigma_y from one MUFU (non-ftz approx, ~2^-22 relative).
__device__ __forceinline__ float sigma_of(float v) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(fmaxf(v, 0.f)));
  return r;
}

// Per-(k,t) control: sample/clamp/control-cost (controllers.py:166-177, 223-228).
__device__ __forceinline__ void control_at(const RollParams &P, int k, int kg, int t,
                                           float &u0, float &u1, float &ccost) {
  const float v0 = P.plan[2 * t], v1 = P.plan[2 * t + 1];
  float e0, e1;
  if (P.ctrl_mode == CTRL_PHILOX) {
    float z0, z1;
    control_normals(P.kc, (uint32_t)t, (uint32_t)kg, z0, z1);
    e0 = P.sfac[0] * z0 + P.sfac[1] * z1;
    e1 = P.sfac[2] * z0 + P.sfac[3] * z1;
  } else {
    const size_t o = ((size_t)k * P.T + t) * 2;
    e0 = (float)P.eps_in[o];
    e1 = (float)P.eps_in[o + 1];
  }
  if (P.ctrl_mode == CTRL_GIVEN) {
    const size_t o = ((size_t)k * P.T + t) * 2;
    u0 = (float)P.u_in[o];
    u1 = (float)P.u_in[o + 1];
  } else {
    u0 = fminf(fmaxf(v0 + e0, P.lo[0]), P.hi[0]);
    u1 = fminf(fmaxf(v1 + e1, P.lo[1]), P.hi[1]);
  }
  // gamma * v^T P (v + eps) with the UNCLAMPED v + eps (controllers.py:227)
  const float a0 = v0 + e0, a1 = v1 + e1;
  const float pa0 = __fadd_rn(__fmul_rn(P.prec[0], a0), __fmul_rn(P.prec[1], a1));
  const float pa1 = __fadd_rn(__fmul_rn(P.prec[2], a0), __fmul_rn(P.prec[3], a1));
  ccost = __fmul_rn(P.gamma, __fadd_rn(__fmul_rn(v0, pa0), __fmul_rn(v1, pa1)));
}

// sqrt(p) and 1/sqrt(p) of a positive pivot from one MUFU.RSQ (the non-ftz
// approx form keeps denormal pivots; relative error ~2^-22, far below the
// FP32 sample-covariance noise) instead of IEEE sqrtf + division.
__device__ __forceinline__ void pivot_root(float p, float &l, float &inv) {
  asm("rsqrt.approx.f32 %0, %1;" : "=f"(inv) : "f"(p));
  l = p * inv;
}

// 4x4 PSD Cholesky with zero-pivot columns left zero (belief.py:235-256).
// A column is dropped when its pivot is not positive -- exact for the
// structurally zero rows (noise-free components, zero initial covariance),
// like the reference's 1e-300 clamp -- and, because a sample covariance of
// M particles has rank <= M - 1, at most M - 1 pivots are kept (for M <= 4
// the FP64 reference's extra pivots are rounding noise of O(1e-8 sigma)).
__device__ __forceinline__ void chol4(const float C[10], float L[10], int max_rank) {
  // packed lower: L00 L10 L11 L20 L21 L22 L30 L31 L32 L33
  // C packed upper: c00 c01 c02 c03 c11 c12 c13 c22 c23 c33
  const float c00 = C[0], c01 = C[1], c02 = C[2], c03 = C[3], c11 = C[4], c12 = C[5],
              c13 = C[6], c22 = C[7], c23 = C[8], c33 = C[9];
  int rank = 0;
  float l00 = 0.f, l10 = 0.f, l20 = 0.f, l30 = 0.f;
  if (c00 > 0.f && rank < max_rank) {
    ++rank;
    float inv;
    pivot_root(c00, l00, inv);
    l10 = c01 * inv; l20 = c02 * inv; l30 = c03 * inv;
  }
  float l11 = 0.f, l21 = 0.f, l31 = 0.f;
  {
    const float acc = c11 - l10 * l10;
    if (acc > 0.f && rank < max_rank) {
      ++rank;
      float inv;
      pivot_root(acc, l11, inv);
      l21 = (c12 - l20 * l10) * inv;
      l31 = (c13 - l30 * l10) * inv;
    }
  }
  float l22 = 0.f, l32 = 0.f;
  {
    const float acc = c22 - l20 * l20 - l21 * l21;
    if (acc > 0.f && rank < max_rank) {
      ++rank;
      float inv;
      pivot_root(acc, l22, inv);
      l32 = (c23 - l30 * l20 - l31 * l21) * inv;
    }
  }
  float l33 = 0.f;
  {
    const float acc = c33 - l30 * l30 - l31 * l31 - l32 * l32;
    if (acc > 0.f && rank < max_rank) {
      float inv;
      pivot_root(acc, l33, inv);
    }
  }
  L[0] = l00; L[1] = l10; L[2] = l11; L[3] = l20; L[4] = l21;
  L[5] = l22; L[6] = l30; L[7] = l31; L[8] = l32; L[9] = l33;
}

// The re-projection factor for Philox raw normals: L kBmNeg (philox.cuh),
// once per (k, t) instead of one multiply per normal.
__device__ __forceinline__ void scale_raw(float L[10]) {
#pragma unroll
  for (int i = 0; i < 10; ++i) L[i] *= kBmNeg;
}

// Reduce-scatter butterfly of 18 partial sums over a G-lane group, then an
// all-gather through shared memory; every lane returns the 18 group sums.
template <int G>
__device__ __forceinline__ void group_allreduce18(float a[18], int li, float *slot) {
  // Each level halves the values a lane holds; `base` is the absolute index
  // of a[0] and `cnt` how many of the held values are real (the rest are
  // zero padding that must not be written back).
  int base = 0, cnt = 18;
#define BSS_RS_LEVEL(N, OFF)                                                   \
  if (G > OFF) {                                                               \
    constexpr int H = (N + 1) / 2;                                             \
    const bool up = (li & OFF) != 0;                                           \
    _Pragma("unroll") for (int i = 0; i < H; ++i) {                            \
      const float lo = a[i];                                                   \
      const float hi = (i + H < N) ? a[i + H] : 0.f;                           \
      const float send = up ? lo : hi;                                         \
      const float keep = up ? hi : lo;                                         \
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);                   \
    }                                                                          \
    base += up ? H : 0;                                                        \
    cnt = up ? max(cnt - H, 0) : min(cnt, H);                                  \
  }
  // offsets descend from G/2 to 1; level sizes for 18 values: 9, 5, 3, 2, 1
  BSS_ASSERT(base >= 0);
  if (G == 32) {
    BSS_RS_LEVEL(18, 16) BSS_RS_LEVEL(9, 8) BSS_RS_LEVEL(5, 4) BSS_RS_LEVEL(3, 2) BSS_RS_LEVEL(2, 1)
    BSS_ASSERT(cnt <= 0 || base < 18);
    if (cnt > 0) slot[base] = a[0];
  } else if (G == 16) {
    BSS_RS_LEVEL(18, 8) BSS_RS_LEVEL(9, 4) BSS_RS_LEVEL(5, 2) BSS_RS_LEVEL(3, 1)
#pragma unroll
    for (int i = 0; i < 2; ++i) if (i < cnt) slot[base + i] = a[i];
  } else if (G == 8) {
    BSS_RS_LEVEL(18, 4) BSS_RS_LEVEL(9, 2) BSS_RS_LEVEL(5, 1)
#pragma unroll
    for (int i = 0; i < 3; ++i) if (i < cnt) slot[base + i] = a[i];
  } else if (G == 4) {
    BSS_RS_LEVEL(18, 2) BSS_RS_LEVEL(9, 1)
#pragma unroll
    for (int i = 0; i < 5; ++i) if (i < cnt) slot[base + i] = a[i];
  } else {  // G == 2
    BSS_RS_LEVEL(18, 1)
#pragma unroll
    for (int i = 0; i < 9; ++i) if (i < cnt) slot[base + i] = a[i];
  }
#undef BSS_RS_LEVEL
  __syncwarp();
  const float4 *s4 = reinterpret_cast<const float4 *>(slot);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 v = s4[i];
    a[4 * i] = v.x; a[4 * i + 1] = v.y; a[4 * i + 2] = v.z; a[4 * i + 3] = v.w;
  }
  const float2 v = reinterpret_cast<const float2 *>(slot)[8];
  a[16] = v.x;
  a[17] = v.y;
}

// The same for the 16 sums of re-projected particles (the two wheel-speed
// sums are identically zero and skipped): exact halvings at every level, so
// G = 32 needs 16 shuffles instead of 20 (and half the selects); the last
// level of G = 32 pairs lanes holding one value each (both keep the sum).
template <int G>
__device__ __forceinline__ void group_allreduce16(float a[16], int li, float *slot) {
  int base = 0;
#define BSS_RS16(N, OFF)                                                       \
  {                                                                            \
    constexpr int H = N / 2;                                                   \
    const bool up = (li & OFF) != 0;                                           \
    _Pragma("unroll") for (int i = 0; i < H; ++i) {                            \
      const float send = up ? a[i] : a[i + H];                                 \
      const float keep = up ? a[i + H] : a[i];                                 \
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);                   \
    }                                                                          \
    base += up ? H : 0;                                                        \
  }
  if (G == 32) {
    BSS_RS16(16, 16) BSS_RS16(8, 8) BSS_RS16(4, 4) BSS_RS16(2, 2)
    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
    if ((li & 1) == 0) slot[base] = a[0];
  } else if (G == 16) {
    BSS_RS16(16, 8) BSS_RS16(8, 4) BSS_RS16(4, 2) BSS_RS16(2, 1)
    slot[base] = a[0];
  } else if (G == 8) {
    BSS_RS16(16, 4) BSS_RS16(8, 2) BSS_RS16(4, 1)
    slot[base] = a[0]; slot[base + 1] = a[1];
  } else if (G == 4) {
    BSS_RS16(16, 2) BSS_RS16(8, 1)
#pragma unroll
    for (int i = 0; i < 4; ++i) slot[base + i] = a[i];
  } else {  // G == 2
    BSS_RS16(16, 1)
#pragma unroll
    for (int i = 0; i < 8; ++i) slot[base + i] = a[i];
  }
#undef BSS_RS16
  __syncwarp();
  const float4 *s4 = reinterpret_cast<const float4 *>(slot);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 v = s4[i];
    a[4 * i] = v.x; a[4 * i + 1] = v.y; a[4 * i + 2] = v.z; a[4 * i + 3] = v.w;
  }
}

constexpr int kSlotFloats = 20;   // 18 sums, 16-byte aligned slot
#ifndef BSS_BLOCK_THREADS
#define BSS_BLOCK_THREADS 128
#endif
constexpr int kBlockThreads = BSS_BLOCK_THREADS;
// The belief kernel is also instantiated for 512-thread blocks (same
// 128-register budget: one block fills an SM's register file); see
// bssmppi.cu rollout_block_threads for when it is launched.
constexpr int kMaxBlockThreads = 512;
// ... and for 64-thread blocks (8 per SM, same registers): launches whose
// warps fill the SMs in one balanced round (bssmppi.cu rollout_block_threads).
constexpr int kSmallBlockThreads = 64;
// Register budget: 4 resident 128-thread blocks per SM (<= 128 registers,
// 16 warps/SM).  With the software-pipelined noise (particle_pass) the extra
// registers buy more than occupancy: 5 / 6 / 7 blocks per SM (96 / 80 / 72
// registers) measured slower at C3 (profiles/README.md).
#ifndef BSS_MIN_BLOCKS
#define BSS_MIN_BLOCKS 4
#endif

// Prologue shared by the rollout kernels: the G lanes of a group sample the
// T controls of rollout k in parallel (lane l takes t = l, l+G, ...),
// write the clamped u for the update and the per-(k,t) control table
// {delta, cos delta, sin delta, drive_gain * throttle} the particle steps
// read, and return the rollout's control cost (controllers.py:166-177,
// 223-228) summed over the group.
template <int G>
__device__ __forceinline__ float control_prologue(const RollParams &P, int k, int kg, int li,
                                                  bool active) {
  const size_t row = (size_t)k * P.T;
  for (int t = li; t < P.T; t += G) {
    float u0, u1, c;
    control_at(P, k, kg, t, u0, u1, c);
    if (active) {
      reinterpret_cast<float2 *>(P.u_out)[row + t] = make_float2(u0, u1);
      // the steering the dynamics see stays inside the bounds the tire
      // table is sized for (a no-op except for out-of-bounds given controls)
      const float dl = fminf(fmaxf(u0, P.lo[0]), P.hi[0]);
      float sd, cd;
      sincosf(dl, &sd, &cd);
      P.ctl[row + t] = make_float4(dl, cd, sd, P.V.drive * u1);
      P.ccost[row + t] = c;
    }
  }
  __syncwarp();
  // the reference adds the whole control cost before the stage costs
  // (controllers.py:272-273); summing it in t order keeps every kernel
  // (bss / smppi / mppi) bit-identical when the belief is degenerate
  float cc = 0.f;
  for (int t = 0; t < P.T; ++t) cc += P.ccost[row + t];
  return cc;
}

// Process-noise kinds of the particle loop (template parameter NK): diagonal
// Gaussian factor (3 multiplies, the hot case), a general 3x3 factor or none
// (the reference skips the add, dynamics.py:571; a runtime test), config-4
// Laplace + slip.
enum NoiseKind { NK_GAUSS_DIAG = 0, NK_LAPLACE = 1, NK_GAUSS_GENERAL = 2 };

// The 7 noise values of particle-step (t, k, m): [0:4] the re-projection
// normals on the tracked subset, [4:7] the process noise -- standard
// normals scaled by F after the step (the column layout of the reference's
// z_all block, controllers.py:285-287, belief.py:328-333) or, for the
// config-4 extension, the Laplace + slip increments themselves.  ZARR reads
// the reference's normals (guarded to zeros for m >= M).  NK, the noise
// kind (NoiseKind), is a template parameter so that the pipelined loop body
// of particle_pass is one branch-free scheduling region.
template <bool ZARR, int NK, bool TAB>
__device__ __forceinline__ void particle_noise(const RollParams &P, const BeliefPrefix &bp,
                                               int t, int k, int m, float n[7], uint32_t ang) {
  if (ZARR) {
    if (m < P.M) {
      BSS_ASSERT(t < P.T && k < P.k_count);
      const float *zp = P.z_in + (((size_t)t * P.k_count + k) * P.M + m) * 7;
#pragma unroll
      for (int j = 0; j < 7; ++j) n[j] = zp[j];
    } else {
#pragma unroll
      for (int j = 0; j < 7; ++j) n[j] = 0.f;
    }
  } else {
    const Philox4 a = belief_block_m(bp, P.kb, (uint32_t)m);
    if (NK == NK_LAPLACE) laplace_from_block<TAB>(a, P.lap_b, P.slip_a, n, n + 4, ang);
    else raw_normals_from_block<TAB>(a, n, ang);
  }
}

// One particle-step given its noise: re-project (or load the persistent
// particle), Euler step, process noise.  Returns the post-step state in x.
template <bool PERSIST, bool ZARR, int NK, bool TS>
__device__ __forceinline__ void particle_step(const RollParams &P, int t, int m, const float mean[8],
                                              const float L[10], const CtlDev &ctl, const StepShared &sh,
                                              float *cloud, const float z[7], float x[8], uint32_t tire) {
  const int M = P.M;
  const float *F = ZARR ? P.F : P.Fk;   // Philox normals arrive raw (x kBmNeg folded in)
  if (PERSIST && t > 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = cloud[i * M + m];
  } else {
    // x = mu, tracked subset (vy, r, e_psi, e_y) += L z[0:4] (belief.py:259-272),
    // as FP32x2 columns: (vy, r) += (L00, L10) z0, then r += L11 z1;
    // (e_psi, e_y) += (L20, L30) z0 + (L21, L31) z1 + (L22, L32) z2, then
    // e_y += L33 z3 -- 6 issue slots instead of 10
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = mean[i];
    const float2 x12 = __ffma2_rn(bc2(z[0]), make_float2(L[0], L[1]), make_float2(mean[1], mean[2]));
    float2 x56 = __ffma2_rn(bc2(z[0]), make_float2(L[3], L[6]), make_float2(mean[5], mean[6]));
    x56 = __ffma2_rn(bc2(z[1]), make_float2(L[4], L[7]), x56);
    x56 = __ffma2_rn(bc2(z[2]), make_float2(L[5], L[8]), x56);
    x[1] = x12.x;
    x[2] = fmaf(L[2], z[1], x12.y);
    x[5] = x56.x;
    x[6] = fmaf(L[9], z[3], x56.y);
  }
  // per-particle ok is discarded (belief.py:370); a re-projected particle
  // shares (vx, omega_f, omega_r, s) with the mean, hence the shared terms
  if (PERSIST && t > 0) vehicle_step<TS>(x, ctl, P.V, P.tr);
  else step_particle<TS>(x, sh, ctl, P.V, P.tr, tire);
  if (NK == NK_LAPLACE) {                // config-4 extension, after integration too
    x[0] += z[4];
    x[1] += z[5];
    x[2] += z[6];
  } else if (NK == NK_GAUSS_DIAG) {      // added after integration (dynamics.py:571-572)
    x[0] = fmaf(F[0], z[4], x[0]);
    const float2 x12 = __ffma2_rn(make_float2(F[4], F[8]), make_float2(z[5], z[6]), make_float2(x[1], x[2]));
    x[1] = x12.x;
    x[2] = x12.y;
  } else if (P.noise_on) {               // NK_GAUSS_GENERAL: 3x3 factor or none
    x[0] += F[0] * z[4] + F[1] * z[5] + F[2] * z[6];
    x[1] += F[3] * z[4] + F[4] * z[5] + F[5] * z[6];
    x[2] += F[6] * z[4] + F[7] * z[5] + F[8] * z[6];
  }
  if (PERSIST) {
#pragma unroll
    for (int i = 0; i < 8; ++i) cloud[i * M + m] = x[i];
  }
}

// SHARED_WHEELS: after re-projection every particle's next-step wheel
// speeds equal the shift's (they depend only on the shared terms), so their
// sums are identically zero and skipped.
template <bool SHARED_WHEELS>
__device__ __forceinline__ void accumulate(float acc[18], const float x[8], const float c[8]) {
  float d[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (SHARED_WHEELS && (i == 3 || i == 4)) { d[i] = 0.f; continue; }
    d[i] = x[i] - c[i];
    acc[i] += d[i];
  }
  const float a1 = d[1], a2 = d[2], a5 = d[5], a6 = d[6];
  acc[8] = fmaf(a1, a1, acc[8]);   acc[9] = fmaf(a1, a2, acc[9]);
  acc[10] = fmaf(a1, a5, acc[10]); acc[11] = fmaf(a1, a6, acc[11]);
  acc[12] = fmaf(a2, a2, acc[12]); acc[13] = fmaf(a2, a5, acc[13]);
  acc[14] = fmaf(a2, a6, acc[14]); acc[15] = fmaf(a5, a5, acc[15]);
  acc[16] = fmaf(a5, a6, acc[16]); acc[17] = fmaf(a6, a6, acc[17]);
}

// The same sums for re-projected particles (wheel sums identically zero) in
// FP32x2 lanes: (S1_0, S1_7), (S1_1, S1_2), (S1_5, S1_6) and the products
// (11, 22), (55, 66), (15, 16), (25, 26) as FADD2 / FFMA2, 12 and 56 scalar
// -- 12 issue slots instead of 22, every lane rounded exactly like the
// scalar form (bit-identical sums).
struct AccPacked {
  float2 a07, a12, a56, q1122, q5566, q1516, q2526;
  float q12, q56;
};

// nc: the NEGATED shift pairs (-c0, -c7), (-c1, -c2), (-c5, -c6) (x - c
// == x + (-c) exactly; there is no FSUB2).
__device__ __forceinline__ void accumulate_packed(AccPacked &A, const float x[8], const float2 nc[3]) {
  const float2 d07 = __fadd2_rn(make_float2(x[0], x[7]), nc[0]);
  const float2 d12 = __fadd2_rn(make_float2(x[1], x[2]), nc[1]);
  const float2 d56 = __fadd2_rn(make_float2(x[5], x[6]), nc[2]);
  A.a07 = __fadd2_rn(A.a07, d07);
  A.a12 = __fadd2_rn(A.a12, d12);
  A.a56 = __fadd2_rn(A.a56, d56);
  A.q1122 = __ffma2_rn(d12, d12, A.q1122);
  A.q5566 = __ffma2_rn(d56, d56, A.q5566);
  A.q1516 = __ffma2_rn(make_float2(d12.x, d12.x), d56, A.q1516);
  A.q2526 = __ffma2_rn(make_float2(d12.y, d12.y), d56, A.q2526);
  A.q12 = fmaf(d12.x, d12.y, A.q12);
  A.q56 = fmaf(d56.x, d56.y, A.q56);
}

// Back to the acc[18] layout of group_allreduce18 / the moment formulas.
__device__ __forceinline__ void unpack_acc(const AccPacked &A, float acc[18]) {
  acc[0] = A.a07.x; acc[1] = A.a12.x; acc[2] = A.a12.y; acc[3] = 0.f; acc[4] = 0.f;
  acc[5] = A.a56.x; acc[6] = A.a56.y; acc[7] = A.a07.y;
  acc[8] = A.q1122.x; acc[9] = A.q12; acc[10] = A.q1516.x; acc[11] = A.q1516.y;
  acc[12] = A.q1122.y; acc[13] = A.q2526.x; acc[14] = A.q2526.y; acc[15] = A.q5566.x;
  acc[16] = A.q56; acc[17] = A.q5566.y;
}

// All particles of rollout k at step t for one lane (m = li, li + G, ...):
// noise, step, and the shifted one-pass moment sums.  Particle 0 of the
// group doubles as the shift c of the moments: it sits O(sigma) from the
// mean, and a zero-spread cloud gives d == 0.
//
// Software-pipelined noise: the Philox blocks and Box-Muller transforms of
// particle m + G are produced inside particle m's iteration, so the
// quarter-rate IMAD.WIDE / MUFU work overlaps the FP32 dynamics in one
// scheduling region; the last particle is peeled, so no draw is wasted.
template <int G, bool PERSIST, bool ZARR, int NK, bool TS>
__device__ __forceinline__ void particle_pass(const RollParams &P, int t, int k, int kg, int li,
                                              const float mean[8], const float L[10], const CtlDev &ctl,
                                              const StepShared &sh, float *cloud,
                                              float acc[18], float c[8]) {
  constexpr bool TAB = !PERSIST;   // persist blocks spend their shared memory on the clouds
  const int M = P.M;
  const bool has0 = li < M;
  float x[8], zc[7], zn[7];
  // Philox rounds 0-2 minus the particle index: once per (k, t)
  const BeliefPrefix bp = ZARR ? BeliefPrefix{} : belief_prefix(P.kb, (uint32_t)t, (uint32_t)kg);
  // table addresses in registers for the loop (philox.cuh opaque_u32)
  const uint32_t ang = TAB && !ZARR ? angle_tab_addr() : 0u;
  const uint32_t tire = TS ? tire_tab_addr() : 0u;
  particle_noise<ZARR, NK, TAB>(P, bp, t, k, li, zc, ang);
  if (li + G < M) particle_noise<ZARR, NK, TAB>(P, bp, t, k, li + G, zn, ang);
  if (has0) particle_step<PERSIST, ZARR, NK, TS>(P, t, li, mean, L, ctl, sh, cloud, zc, x, tire);
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = __shfl_sync(0xffffffffu, x[i], 0, G);
  // persist clouds need the wheel sums too (scalar form); re-projected
  // particles use the packed sums
  AccPacked A{};
  const float2 nc[3] = {make_float2(-c[0], -c[7]), make_float2(-c[1], -c[2]), make_float2(-c[5], -c[6])};
  const auto add = [&](const float x_[8]) {
    if (PERSIST) accumulate<false>(acc, x_, c);
    else accumulate_packed(A, x_, nc);
  };
  if (has0) add(x);
  int m = li + G;
  // unrolled twice: the look-ahead noise alternates between two register
  // sets instead of being copied (7 moves) at every particle
#pragma unroll 2
  for (; m + G < M; m += G) {             // steady state: look one particle ahead
#pragma unroll
    for (int j = 0; j < 7; ++j) zc[j] = zn[j];
    particle_noise<ZARR, NK, TAB>(P, bp, t, k, m + G, zn, ang);
    particle_step<PERSIST, ZARR, NK, TS>(P, t, m, mean, L, ctl, sh, cloud, zc, x, tire);
    add(x);
  }
  if (m < M) {                            // last particle: no look-ahead draw
    particle_step<PERSIST, ZARR, NK, TS>(P, t, m, mean, L, ctl, sh, cloud, zn, x, tire);
    add(x);
  }
  if (!PERSIST) unpack_acc(A, acc);
}

// BSS rollouts.  G: lanes per rollout; PERSIST: keep the particle cloud in
// shared memory instead of re-projecting (controllers.py:288-305);
// ZARR: read the reference's normals instead of Philox; NK: the process
// noise kind (NoiseKind), resolved once at kernel entry so every variant's
// T loop holds exactly one particle loop (register allocation per variant).
template <int G, bool PERSIST, bool ZARR, int NK, bool TS, int BT>
__device__ __forceinline__ void bss_rollout(const RollParams &P) {
  extern __shared__ float4 smem4[];
  float *smem = reinterpret_cast<float *>(smem4);
  constexpr int GPW = 32 / G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gi = lane / G, li = lane % G;
  constexpr int nwarps = BT / 32;
  const int warp_global = blockIdx.x * nwarps + warp;
  if (warp_global * GPW >= P.k_count) return;            // whole warp idle
  const int kraw = warp_global * GPW + gi;
  const bool active = kraw < P.k_count;
  const int k = active ? kraw : P.k_count - 1;            // keep shuffles convergent
  const int kg = P.k_begin + k;
  float *slots = smem + (warp * GPW + gi) * 2 * kSlotFloats;
  float *cloud = PERSIST ? smem + nwarps * GPW * 2 * kSlotFloats +
                               (size_t)(warp * GPW + gi) * 8 * P.M
                         : nullptr;

  float total = control_prologue<G>(P, k, kg, li, active);
  float mean[8], C[10], L[10];
#pragma unroll
  for (int i = 0; i < 8; ++i) mean[i] = P.x0[i];
  {
    const int ui[10] = {0, 1, 2, 3, 5, 6, 7, 10, 11, 15};
#pragma unroll
    for (int i = 0; i < 10; ++i) C[i] = P.cov0[ui[i]];
  }
  chol4(C, L, 4);   // the initial belief covariance is not a sample estimate
  if (!ZARR) scale_raw(L);
  float h_cur = dcbf(mean[6], sigma_of(C[9]), P);
  float h_prev = h_cur;
  bool inside = false;
  float ho_cur = P.n_obs ? obstacle_terms(P, mean[7], mean[6], sigma_of(C[9]), inside) : 0.f;
  float ho_prev = ho_cur;
  bool dead = false;
  const float4 *ctl_row = P.ctl + (size_t)k * P.T;
  float kap_mean = curvature(P.tr, mean[7]);   // kappa(s_bar): frame check and next step's shared terms
  // The step's control row and shared terms are produced at the end of the
  // previous step (after its moments): the control-row load then overlaps
  // the group reduction, and step_shared's dependency chain runs beside the
  // Cholesky's instead of after it -- the per-step latency that bounds the
  // small (few-rollouts-per-SM) shapes.
  float4 cv = ctl_row[0];
  StepShared sh = step_shared(mean, CtlDev{cv.x, cv.y, cv.z, cv.w}, P.V, P.tr, kap_mean);

  for (int t = 0; t < P.T; ++t) {
    total += stage_cost(mean, P);
    if (t > 0) total += shield_penalty(h_cur, h_prev, P);
    if (P.n_obs) {
      if (inside) total += P.c_obs;
      if (t > 0) total += shield_penalty(ho_cur, ho_prev, P);
    }
    const CtlDev ctl{cv.x, cv.y, cv.z, cv.w};

    float acc[18];
#pragma unroll
    for (int i = 0; i < 18; ++i) acc[i] = 0.f;
    float c[8];
    particle_pass<G, PERSIST, ZARR, NK, TS>(P, t, k, kg, li, mean, L, ctl, sh, cloud, acc, c);
    if (t + 1 < P.T) cv = ctl_row[t + 1];
    if (PERSIST) {
      group_allreduce18<G>(acc, li, slots + (t & 1) * kSlotFloats);
    } else {   // wheel sums are zero after re-projection: reduce the other 16
      float a16[16] = {acc[0], acc[1], acc[2], acc[5], acc[6], acc[7], acc[8], acc[9],
                       acc[10], acc[11], acc[12], acc[13], acc[14], acc[15], acc[16], acc[17]};
      group_allreduce16<G>(a16, li, slots + (t & 1) * kSlotFloats);
      acc[0] = a16[0]; acc[1] = a16[1]; acc[2] = a16[2]; acc[3] = 0.f; acc[4] = 0.f;
      acc[5] = a16[3]; acc[6] = a16[4]; acc[7] = a16[5];
#pragma unroll
      for (int i = 8; i < 18; ++i) acc[i] = a16[i - 2];
    }

    // moments (belief.py:275-308 semantics)
    float mu[8], dm[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      dm[i] = acc[i] * P.invM;
      mu[i] = c[i] + dm[i];
    }
    {
      const int sub[4] = {1, 2, 5, 6};
      int q = 0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = a; b < 4; ++b, ++q)
          C[q] = (acc[8 + q] - acc[sub[a]] * dm[sub[b]]) * P.invMm1;
    }
    if (P.mom_out != nullptr && active && li == 0) {
      float *mo = P.mom_out + ((size_t)t * P.k_count + k) * 18;
#pragma unroll
      for (int i = 0; i < 8; ++i) mo[i] = mu[i];
#pragma unroll
      for (int i = 0; i < 10; ++i) mo[8 + i] = C[i];
    }
    // ok = finite(mean) & finite(cov) & 1 - kappa(s_bar) e_bar > 0 (belief.py:376-379)
    const bool fin = all_finite8(mu) && all_finite8(C) && all_finite2(C[8], C[9]);
    kap_mean = curvature(P.tr, mu[7]);
    const bool ok = fin && (1.f - kap_mean * mu[6] > 0.f);
    dead |= !ok;
    // _finite_or_zero (controllers.py:231-235, 311-312)
#pragma unroll
    for (int i = 0; i < 8; ++i) mean[i] = mu[i];
    if (__builtin_expect(!fin, 0)) {
#pragma unroll
      for (int i = 0; i < 8; ++i) mean[i] = isfinite(mu[i]) ? mu[i] : 0.f;
#pragma unroll
      for (int i = 0; i < 10; ++i) C[i] = isfinite(C[i]) ? C[i] : 0.f;
      kap_mean = curvature(P.tr, mean[7]);
    }
    h_prev = h_cur;
    h_cur = dcbf(mean[6], sigma_of(C[9]), P);
    if (P.n_obs) {
      ho_prev = ho_cur;
      ho_cur = obstacle_terms(P, mean[7], mean[6], sigma_of(C[9]), inside);
    }
    if (!PERSIST) {
      chol4(C, L, P.chol_rank);
      if (!ZARR) scale_raw(L);
      sh = step_shared(mean, CtlDev{cv.x, cv.y, cv.z, cv.w}, P.V, P.tr, kap_mean);
    }
  }
  // two separate adds, in the reference's order (controllers.py:318-319):
  // the det kernel adds them the same way, so BSS == S-MPPI stays bit-exact
  total += __fmul_rn(P.term, stage_cost(mean, P));
  total += shield_penalty(h_cur, h_prev, P);
  if (P.n_obs) {
    total += __fmul_rn(P.term, inside ? P.c_obs : 0.f);
    total += shield_penalty(ho_cur, ho_prev, P);
  }
  if (active && li == 0) P.cost_out[k] = dead ? __int_as_float(0x7f800000) : total;
}

#ifdef BSS_MAXNREG
#define BSS_ROLLOUT_BOUNDS __maxnreg__(BSS_MAXNREG)
#else
#define BSS_ROLLOUT_BOUNDS __launch_bounds__(BT, kBlockThreads * BSS_MIN_BLOCKS / BT)
#endif
// Kernel-entry dispatch on the launch-constant noise kind and tire-sine
// range: every variant's T loop holds exactly one particle loop.
template <int G, bool PERSIST, bool ZARR, bool TS, int BT>
__device__ __forceinline__ void bss_rollout_nk(const RollParams &P) {
#ifdef BSS_AB_ONLY   // quick A/B builds (tools/build_variants.sh): the hot variant only
  bss_rollout<G, PERSIST, ZARR, NK_GAUSS_DIAG, TS, BT>(P);
#else
  if (!ZARR && P.noise_kind == 1) bss_rollout<G, PERSIST, ZARR, NK_LAPLACE, TS, BT>(P);
  else if (P.noise_diag) bss_rollout<G, PERSIST, ZARR, NK_GAUSS_DIAG, TS, BT>(P);
  else bss_rollout<G, PERSIST, ZARR, NK_GAUSS_GENERAL, TS, BT>(P);
#endif
}

// BT: block threads, a compile-time constant (128, or 512 for the one-wave
// shapes of bssmppi.cu rollout_block_threads); same register budget.
template <int G, bool PERSIST, bool ZARR, int BT = kBlockThreads>
__global__ void BSS_ROLLOUT_BOUNDS bss_rollout_kernel(const RollParams P) {
  // Shared tables, copied once per block -- the Box-Muller angle table
  // (philox.cuh g_angle_global, two entries per 16-byte load) and the tire
  // table (vehicle.cuh; persist blocks keep their shared memory for the
  // clouds) -- then the kernel's one block-wide barrier, before any warp
  // can retire.
  const bool ts = !PERSIST && P.V.tire_smem;
  if (!PERSIST && !ZARR) {
    const float4 *src = reinterpret_cast<const float4 *>(g_angle_global);
    float4 *dst = reinterpret_cast<float4 *>(g_angle_tab);
    static_assert((kAngleTab / 2) % BT == 0, "angle table copy: whole rounds per thread");
    constexpr int R = kAngleTab / 2 / BT;
    constexpr int CH = R < 8 ? R : 8;       // up to 8 loads in flight before their stores
#pragma unroll
    for (int i0 = 0; i0 < R; i0 += CH) {
      float4 v[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) v[i] = __ldg(src + threadIdx.x + (i0 + i) * BT);
#pragma unroll
      for (int i = 0; i < CH; ++i) dst[threadIdx.x + (i0 + i) * BT] = v[i];
    }
  }
  if (ts)
    for (int j = threadIdx.x; j < 2 * P.V.tire_rows; j += BT) {
      const int axle = j >= P.V.tire_rows, row = j - axle * P.V.tire_rows;
      g_tire_tab[axle * kTireSmemRows + row] = __ldg(P.V.tire + j);
    }
  if (!PERSIST) __syncthreads();
#ifdef BSS_AB_ONLY
  bss_rollout_nk<G, PERSIST, ZARR, true, BT>(P);
#else
  if constexpr (PERSIST) {
    bss_rollout_nk<G, PERSIST, ZARR, false, BT>(P);
  } else {
    if (ts) bss_rollout_nk<G, PERSIST, ZARR, true, BT>(P);
    else bss_rollout_nk<G, PERSIST, ZARR, false, BT>(P);
  }
#endif
}

// Deterministic rollouts for kind "mppi" / "smppi" (controllers.py:320-338):
// one lane per k, state carried in registers.
template <bool SHIELD>
__device__ __forceinline__ void det_rollout(const RollParams &P) {
  const int kraw = blockIdx.x * kBlockThreads + threadIdx.x;
  if (kraw >= P.k_count) return;
  const int k = kraw, kg = P.k_begin + k;
  float total = control_prologue<1>(P, k, kg, 0, true);
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = P.x0[i];
  float h_cur = SHIELD ? dcbf(x[6], 0.f, P) : 0.f;
  float h_prev = h_cur;
  bool inside = false;
  float ho_cur = P.n_obs ? obstacle_terms(P, x[7], x[6], 0.f, inside) : 0.f;
  float ho_prev = ho_cur;
  bool dead = false;
  const float4 *ctl_row = P.ctl + (size_t)k * P.T;
  for (int t = 0; t < P.T; ++t) {
    total += stage_cost(x, P);
    if (SHIELD && t > 0) total += shield_penalty(h_cur, h_prev, P);
    if (P.n_obs) {
      if (inside) total += P.c_obs;
      if (SHIELD && t > 0) total += shield_penalty(ho_cur, ho_prev, P);
    }
    const float4 cv = ctl_row[t];
    const bool ok = vehicle_step<false>(x, CtlDev{cv.x, cv.y, cv.z, cv.w}, P.V, P.tr);
    dead |= !ok;
    if (SHIELD) {
      h_prev = h_cur;
      h_cur = dcbf(x[6], 0.f, P);
    }
    if (P.n_obs) {
      ho_prev = ho_cur;
      ho_cur = obstacle_terms(P, x[7], x[6], 0.f, inside);
    }
  }
  total += __fmul_rn(P.term, stage_cost(x, P));
  if (SHIELD) total += shield_penalty(h_cur, h_prev, P);
  if (P.n_obs) {
    total += __fmul_rn(P.term, inside ? P.c_obs : 0.f);
    if (SHIELD) total += shield_penalty(ho_cur, ho_prev, P);
  }
  P.cost_out[k] = dead ? __int_as_float(0x7f800000) : total;
}

template <bool SHIELD>
__global__ void __launch_bounds__(kBlockThreads) det_rollout_kernel(const RollParams P) {
  det_rollout<SHIELD>(P);
}

// step_array (dynamics.py:550-573): one particle per thread, FP64 I/O.
__device__ __forceinline__ void step_array(const VehDev &V, const TrackDev &tr, int n, const double *x,
                                           const double *u, const double *w, double *xo, uint8_t *oko) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) s[j] = (float)x[(size_t)i * 8 + j];
  const bool ok = vehicle_step<false>(s, make_ctl((float)u[2 * (size_t)i], (float)u[2 * (size_t)i + 1], V), V, tr);
  if (w != nullptr) {
#pragma unroll
    for (int j = 0; j < 3; ++j) s[j] += (float)w[(size_t)i * 3 + j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) xo[(size_t)i * 8 + j] = (double)s[j];
  oko[i] = ok ? 1 : 0;
}

__global__ void step_array_kernel(VehDev V, TrackDev tr, int n, const double *x, const double *u,
                                  const double *w, double *xo, uint8_t *oko) {
  step_array(V, tr, n, x, u, w, xo, oko);
}

}  // namespace bss

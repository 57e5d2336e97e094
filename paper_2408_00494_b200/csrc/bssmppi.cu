// C ABI of the B200-native BSS-MPPI step (include/bssmppi.h).
//
// Host-side responsibilities only: validate the problem, lay the track out
// for the device (cell-indexed float4 nodes), own the per-controller device
// buffers and pinned staging, pick the kernel instantiation, and order
// copies / kernels / events on one CUDA stream.  No numerics of the path run
// on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/bssmppi.h"
#include "rollout.cuh"
#include "update.cuh"

using namespace bss;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(BSSMPPI_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));     \
  } while (0)

template <typename T>
int dev_alloc(T **p, size_t n) {
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc((void **)p, n * sizeof(T));
  if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "cudaMalloc(%zu B): %s", n * sizeof(T), cudaGetErrorString(e));
  return BSSMPPI_OK;
}

}  // namespace

struct bssmppi_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int kind = 0, K = 0, T = 0, M = 0, k_begin = 0, k_count = 0, persist = 0;
  double lam = 1.0, lo[2] = {0, 0}, hi[2] = {0, 0};
  RollParams rp{};
  float4 *d_node = nullptr;
  int *d_cell = nullptr;
  float *d_state = nullptr;   // x0[8] | cov0[16] | plan[2T]
  float *d_u = nullptr, *d_cost = nullptr;
  float4 *d_ctl = nullptr;    // per-(k,t) control table
  float4 *d_obs = nullptr, *d_cl = nullptr;   // config-4 extension tables
  float4 *d_tire = nullptr;   // lateral tire table (vehicle.cuh tire_q)
  float *d_cc = nullptr;      // per-(k,t) control-cost terms
  double *d_eps = nullptr, *d_uin = nullptr;
  float *d_z = nullptr, *d_mom = nullptr;
  size_t cap_eps = 0, cap_uin = 0, cap_z = 0, cap_mom = 0;
  double *d_rec = nullptr;    // per-block records
  int nblocks = 0, chunk = 0;
  double *d_out = nullptr;    // vplus[2T] | head[5]
  float *h_state = nullptr;   // pinned
  double *h_out = nullptr;    // pinned, mapped: final update kernels write v+ and head here
  double *h_out_dev = nullptr;  // device alias of h_out
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evr = nullptr;   // iteration start/end, rollout end
  cudaEvent_t ev_h2d = nullptr;   // last h_state -> d_state copy (h_state reuse guard)
  bool h2d_pending = false;
  bool timed = false;
  int sms = 148;                  // multiprocessors of the device (launch-shape policy)
  int force_g = 0;                // bssmppi_problem.group_width (0 = policy)
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

constexpr size_t kSmemMax = 227 * 1024;   // opt-in dynamic shared memory per block
constexpr int kPersistMaxM = 1792;         // persist clouds of one G = 32 block fit kSmemMax

bool valid_group_width(int g) { return g == 2 || g == 4 || g == 8 || g == 16 || g == 32; }

int validate(const bssmppi_problem *p) {
  if (!p) return fail(BSSMPPI_ERR_INVALID, "problem is NULL");
  if (p->kind < 0 || p->kind > 2) return fail(BSSMPPI_ERR_INVALID, "unknown controller kind %d", p->kind);
  if (p->samples < 1 || p->horizon < 1) return fail(BSSMPPI_ERR_INVALID, "samples and horizon must be >= 1");
  if (p->horizon > 512) return fail(BSSMPPI_ERR_UNSUPPORTED, "horizon %d > 512", p->horizon);
  if (!(std::isfinite(p->phys[6]) && std::isfinite(p->phys[7]) && std::isfinite(p->phys[8]) &&
        std::isfinite(p->phys[9])))
    return fail(BSSMPPI_ERR_INVALID, "lateral magic-formula coefficients must be finite");
  if (!(std::fabs(p->bounds_lo[0]) <= 2 * M_PI && std::fabs(p->bounds_hi[0]) <= 2 * M_PI))
    return fail(BSSMPPI_ERR_UNSUPPORTED, "steering bounds beyond +-2 pi (the tire table covers "
                "|slip angle| <= pi + max |steering bound|)");
  if (!(p->temperature > 0.0)) return fail(BSSMPPI_ERR_INVALID, "temperature must be > 0");
  if (p->kind == BSSMPPI_KIND_BSS && p->inner_samples < 2)
    return fail(BSSMPPI_ERR_INVALID, "bss controller needs inner_samples >= 2");
  if (p->kind == BSSMPPI_KIND_BSS && p->inner_samples > 8192)
    return fail(BSSMPPI_ERR_UNSUPPORTED, "inner_samples %d > 8192", p->inner_samples);
  if (p->kind == BSSMPPI_KIND_BSS && p->persist_particles && p->inner_samples > kPersistMaxM)
    return fail(BSSMPPI_ERR_UNSUPPORTED, "persist_particles keeps the cloud in shared memory: inner_samples %d > %d",
                p->inner_samples, kPersistMaxM);
  if (p->k_count < 1 || p->k_begin < 0 || (int64_t)p->k_begin + p->k_count > p->samples)
    return fail(BSSMPPI_ERR_INVALID, "shard [%d, %d) outside K=%d", p->k_begin, p->k_begin + p->k_count, p->samples);
  if (!p->track_s || !p->track_kappa || p->track_n < 2)
    return fail(BSSMPPI_ERR_INVALID, "track needs >= 2 samples");
  if (!(p->half_width > 0.0) || !(p->track_length > 0.0)) return fail(BSSMPPI_ERR_INVALID, "bad track geometry");
  if (p->track_s[0] != 0.0) return fail(BSSMPPI_ERR_INVALID, "track s must start at 0");
  for (int j = 1; j < p->track_n; ++j)
    if (!(p->track_s[j] > p->track_s[j - 1])) return fail(BSSMPPI_ERR_INVALID, "track s must increase strictly");
  if (p->track_closed ? !(p->track_length > p->track_s[p->track_n - 1]) : (p->track_length < p->track_s[p->track_n - 1]))
    return fail(BSSMPPI_ERR_INVALID, "track length inconsistent with samples");
  if (!(p->dt > 0.0)) return fail(BSSMPPI_ERR_INVALID, "dt must be > 0");
  if (p->noise_kind < 0 || p->noise_kind > 1) return fail(BSSMPPI_ERR_INVALID, "unknown noise kind %d", p->noise_kind);
  if (p->n_obstacles < 0 || p->n_obstacles > 64) return fail(BSSMPPI_ERR_UNSUPPORTED, "0..64 obstacles supported");
  if (p->group_width != 0 && !valid_group_width(p->group_width))
    return fail(BSSMPPI_ERR_INVALID, "group_width must be 0 (policy) or 2, 4, 8, 16, 32 (got %d)", p->group_width);
  if (p->n_obstacles > 0 && (!p->obstacles || !p->centerline || p->centerline_n < 2 || !(p->centerline_ds > 0.0)))
    return fail(BSSMPPI_ERR_INVALID, "obstacles need a centerline table");
  return BSSMPPI_OK;
}

// Config-4 extension tables (obstacles.py).
int build_extensions(bssmppi_ctx *c, const bssmppi_problem *p) {
  RollParams &r = c->rp;
  r.noise_kind = p->noise_kind;
  r.lap_b = (float)p->laplace_scale;
  r.slip_a = (float)p->slip_bias;
  r.n_obs = p->n_obstacles;
  r.nu_obs = (float)p->obstacle_backoff;
  if (p->n_obstacles == 0) return BSSMPPI_OK;
  std::vector<float4> ob(p->n_obstacles), cl(p->centerline_n);
  for (int i = 0; i < p->n_obstacles; ++i)
    ob[i] = make_float4((float)p->obstacles[3 * i], (float)p->obstacles[3 * i + 1], (float)p->obstacles[3 * i + 2], 0.f);
  for (int i = 0; i < p->centerline_n; ++i)
    cl[i] = make_float4((float)p->centerline[3 * i], (float)p->centerline[3 * i + 1], (float)p->centerline[3 * i + 2], 0.f);
  int rc;
  if ((rc = dev_alloc(&c->d_obs, ob.size())) || (rc = dev_alloc(&c->d_cl, cl.size()))) return rc;
  CUDA_TRY(cudaMemcpy(c->d_obs, ob.data(), ob.size() * sizeof(float4), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_cl, cl.data(), cl.size() * sizeof(float4), cudaMemcpyHostToDevice));
  r.obs = c->d_obs;
  r.cl = c->d_cl;
  r.cl_n = p->centerline_n;
  r.cl_inv_ds = (float)(1.0 / p->centerline_ds);
  return BSSMPPI_OK;
}

// Lateral tire table (vehicle.cuh tire_q / lateral_shape): sin(C atan(B a))
// = a q(|a|) with q(a) = sin(C atan(B a)) / a (even, smooth, q(0) = C B).
// Rows are centred on a = j / s; each holds the cubic in f = a s - j that
// interpolates q in FP64 at the four Chebyshev nodes of f in [-1/2, 1/2]
// (near-minimax).  The domain covers every slip angle a rollout can meet,
// |alpha| <= pi + max |steering bound|, and the cell width keeps B h <=
// 0.055: the FP32 evaluation then stays at ~1.9e-7 relative (rounding level)
// for all B, C (tests/test_tire_table.py).
constexpr double kTireBh = 0.055;
constexpr int kTireMaxCells = 2000;   // row index must fit 0x7ff (vehicle.cuh tire_q)

double tire_q_exact(double B, double C, double a) {
  return std::fabs(a) < 1e-300 ? C * B : std::sin(C * std::atan(B * a)) / a;
}

void tire_table_host(const double bc[4], double steer_max, std::vector<float4> &tab, double &sc,
                     double &amax, int &rows) {
  amax = M_PI + steer_max + 0.01;
  const double bmax = std::max(bc[0], bc[2]);
  const int cells = (int)std::min<double>(kTireMaxCells, std::max(64.0, std::ceil(amax * bmax / kTireBh)));
  sc = cells / amax;
  rows = cells + 2;
  tab.assign(2 * (size_t)rows, make_float4(0.f, 0.f, 0.f, 0.f));
  double nodes[4];
  for (int i = 0; i < 4; ++i) nodes[i] = -0.5 + 0.5 * (1.0 - std::cos((2 * i + 1) * M_PI / 8.0));
  for (int axle = 0; axle < 2; ++axle) {
    const double B = bc[2 * axle], C = bc[2 * axle + 1];
    for (int j = 0; j < rows; ++j) {
      double A[4][5];   // Vandermonde system of the interpolating cubic in f
      for (int i = 0; i < 4; ++i) {
        double pw = 1.0;
        for (int k = 0; k < 4; ++k) { A[i][k] = pw; pw *= nodes[i]; }
        A[i][4] = tire_q_exact(B, C, (j + nodes[i]) / sc);
      }
      for (int k = 0; k < 4; ++k) {            // Gauss-Jordan, partial pivoting
        int piv = k;
        for (int i = k + 1; i < 4; ++i) if (std::fabs(A[i][k]) > std::fabs(A[piv][k])) piv = i;
        for (int m = 0; m < 5; ++m) std::swap(A[k][m], A[piv][m]);
        for (int i = 0; i < 4; ++i) {
          if (i == k) continue;
          const double f = A[i][k] / A[k][k];
          for (int m = k; m < 5; ++m) A[i][m] -= f * A[k][m];
        }
      }
      tab[(size_t)axle * rows + j] = make_float4((float)(A[0][4] / A[0][0]), (float)(A[1][4] / A[1][1]),
                                                 (float)(A[2][4] / A[2][2]), (float)(A[3][4] / A[3][3]));
    }
  }
}

int build_tire_table(bssmppi_ctx *c, const bssmppi_problem *p) {
  const double *q = p->phys;
  const double bc[4] = {q[6], q[7], q[8], q[9]};
  std::vector<float4> tab;
  double sc, amax;
  int rows;
  tire_table_host(bc, std::max(std::fabs(p->bounds_lo[0]), std::fabs(p->bounds_hi[0])), tab, sc, amax, rows);
  int rc;
  if ((rc = dev_alloc(&c->d_tire, tab.size()))) return rc;
  CUDA_TRY(cudaMemcpy(c->d_tire, tab.data(), tab.size() * sizeof(float4), cudaMemcpyHostToDevice));
  VehDev &Vd = c->rp.V;
  Vd.tire = c->d_tire;
  Vd.tire_s = (float)sc;
  Vd.tire_amax = (float)amax;
  Vd.tire_rows = rows;
  Vd.tire_smem = rows <= kTireSmemRows ? 1 : 0;
  return BSSMPPI_OK;
}

// Cell-indexed node table (see vehicle.cuh curvature()).
int build_track(bssmppi_ctx *c, const bssmppi_problem *p) {
  const int n = p->track_n;
  std::vector<float> sf(n), kf(n);
  for (int j = 0; j < n; ++j) { sf[j] = (float)p->track_s[j]; kf[j] = (float)p->track_kappa[j]; }
  const float Lf = (float)p->track_length;
  double min_gap = 1e300;
  for (int j = 0; j + 1 < n; ++j) min_gap = std::min(min_gap, (double)sf[j + 1] - (double)sf[j]);
  if (p->track_closed) min_gap = std::min(min_gap, (double)Lf - (double)sf[n - 1]);
  if (!(min_gap > 0.0)) return fail(BSSMPPI_ERR_UNSUPPORTED, "track samples collide in FP32");
  const double h = 0.5 * min_gap;
  const double ncell_d = std::ceil((double)Lf / h) + 1.0;
  if (ncell_d > (double)(1 << 24)) return fail(BSSMPPI_ERR_UNSUPPORTED, "track sample spacing too fine for the cell index");
  const int ncell = (int)ncell_d;
  std::vector<float4> node(n + 1);
  const float INF = INFINITY;
  for (int j = 0; j < n; ++j) {
    double s0 = p->track_s[j], k0 = p->track_kappa[j], s1, k1;
    float next;
    if (j + 1 < n) { s1 = p->track_s[j + 1]; k1 = p->track_kappa[j + 1]; next = sf[j + 1]; }
    else if (p->track_closed) { s1 = p->track_length; k1 = p->track_kappa[0]; next = Lf; }
    else { s1 = s0; k1 = k0; next = INF; }
    const double slope = (s1 > s0) ? (k1 - k0) / (s1 - s0) : 0.0;
    node[j] = make_float4(sf[j], kf[j], (float)slope, next);
  }
  node[n] = p->track_closed ? make_float4(Lf, kf[0], 0.f, INF) : make_float4(sf[n - 1], kf[n - 1], 0.f, INF);
  std::vector<int> cell(ncell);
  int j = 0;
  for (int i = 0; i < ncell; ++i) {
    const double x = i * h;
    while (j + 1 < n && (double)sf[j + 1] <= x) ++j;
    cell[i] = j;
  }
  int rc;
  if ((rc = dev_alloc(&c->d_node, n + 1))) return rc;
  if ((rc = dev_alloc(&c->d_cell, ncell))) return rc;
  CUDA_TRY(cudaMemcpy(c->d_node, node.data(), (n + 1) * sizeof(float4), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_cell, cell.data(), ncell * sizeof(int), cudaMemcpyHostToDevice));
  TrackDev &tr = c->rp.tr;
  tr.node = c->d_node;
  tr.cell = c->d_cell;
  tr.L = Lf;
  tr.L2 = 2.f * Lf;
  tr.inv_h = (float)(1.0 / h);
  tr.half_width = (float)p->half_width;
  tr.ncell = ncell;
  tr.n = n;
  tr.closed = p->track_closed ? 1 : 0;
  return BSSMPPI_OK;
}

void fill_params(bssmppi_ctx *c, const bssmppi_problem *p) {
  const double *q = p->phys;
  VehDev &V = c->rp.V;
  V.inv_m = (float)(1.0 / q[0]); V.inv_iz = (float)(1.0 / q[1]);
  V.lf = (float)q[2]; V.lr = (float)q[3]; V.R = (float)q[4]; V.inv_jw = (float)(1.0 / q[5]);
  V.Byf = (float)q[6]; V.Cyf = (float)q[7]; V.Byr = (float)q[8]; V.Cyr = (float)q[9];
  V.Bxf = (float)q[10]; V.Cxf = (float)q[11]; V.Bxr = (float)q[12]; V.Cxr = (float)q[13];
  V.Dxf = (float)q[14]; V.Dyf = (float)q[15]; V.Dxr = (float)q[16]; V.Dyr = (float)q[17];
  V.drive = (float)q[18]; V.vfloor = (float)q[20];
  V.rrf = (float)(q[19] * q[21] * q[4]); V.rrr = (float)(q[19] * q[22] * q[4]);
  V.spin_scale = (float)(q[4] / 0.1); V.dt = (float)p->dt;
  V.lf_nlr = make_float2(V.lf, -V.lr);
  V.dt_lf_iz = (float)(p->dt * q[2] / q[1]);
  V.ndt_lr_iz = (float)(-p->dt * q[3] / q[1]);
  V.dt_m = (float)(p->dt / q[0]);
  V.Dy = make_float2(V.Dyf, V.Dyr);
  V.Bx = make_float2(V.Bxf, V.Bxr);
  V.Cx = make_float2(V.Cxf, V.Cxr);
  RollParams &r = c->rp;
  r.k_count = p->k_count; r.k_begin = p->k_begin; r.T = p->horizon; r.M = std::max(1, p->inner_samples);
  r.invM = (float)(1.0 / r.M);
  r.invMm1 = (float)(1.0 / std::max(1, r.M - 1));
  for (int i = 0; i < 8; ++i) r.q[i] = (float)p->q_diag[i];
  r.v_goal = (float)p->v_goal; r.c_obs = (float)p->obstacle_penalty; r.term = (float)p->terminal_scale;
  r.beta1 = (float)(1.0 - p->cbf_rate); r.c_pen = (float)p->penalty; r.nu = (float)p->backoff;
  r.gamma = (float)p->control_cost_weight;
  for (int i = 0; i < 4; ++i) { r.prec[i] = (float)p->precision[i]; r.sfac[i] = (float)p->sigma_factor[i]; }
  for (int i = 0; i < 2; ++i) { r.lo[i] = (float)p->bounds_lo[i]; r.hi[i] = (float)p->bounds_hi[i]; }
  bool any = false;
  for (int i = 0; i < 9; ++i) {
    r.F[i] = (float)p->noise_factor[i];
    r.Fk[i] = (float)((double)kBmNeg * p->noise_factor[i]);
    any |= p->noise_factor[i] != 0.0;
  }
  r.noise_on = any ? 1 : 0;
  const double *F = p->noise_factor;
  r.noise_diag = (any && F[1] == 0.0 && F[2] == 0.0 && F[3] == 0.0 && F[5] == 0.0 && F[6] == 0.0 &&
                  F[7] == 0.0) ? 1 : 0;
  r.shield = p->kind == BSSMPPI_KIND_SMPPI ? 1 : 0;
  r.chol_rank = std::min(4, std::max(1, r.M - 1));
}

// Lanes per rollout.  Start from one warp (or the power of two >= M), then
// narrow the group -- the per-(k, t) work (shared step terms, reduction,
// Cholesky, costs) costs the same warp instructions for 1 or 32/G rollouts,
// so narrower groups amortise it over more particles per lane -- as long as
// the narrower grid keeps the SMs busy:
//   (1) to >= 8 particles per lane while >= 1024 warps remain;
//   (1b) to >= 16 particles per lane while >= 1400 warps remain (measured
//       between 1024 warps, where the wider group wins by 4-6% -- 2048 x 256,
//       4096 x 128, 8192 x 64 -- and 1500, where the narrower one wins by
//       9-10% -- 3000 x 256, 12000 x 64; also 4096 x 256 -5.5%,
//       8192 x 128 -5.6%, 16384 x 64 -7%; profiles/README.md);
//   (2) to <= 64 particles per lane while >= 4096 warps remain (~1.7 waves
//       of 16 warps x 148 SMs), down to G = 2 (M = 64 at K >= 65536: 3.88 vs
//       4.16 ms at 131072 x 64 x 60, 1.68 vs 1.79 ms at 65536 x 64 x 50).
// Fitted to a G sweep over 14 (K, M) shapes with the pipelined kernel
// (tools/g_sweep.sh, profiles/r1_group_width_sweep.txt): it picks the best
// or a tied G on every one.  Decided on the LOCAL rollout count, so a
// K-shard of 2048 rollouts (C3 over 8 GPUs) keeps one warp per rollout;
// across world sizes the moment sums may then differ by FP32 summation order.
// bssmppi_problem.group_width pins G explicitly (parity tests at the
// production widths, sweeps).

int group_width(int M, int K) {
  int g = 2;
  while (g < M && g < 32) g <<= 1;
  const auto warps = [K](int gg) { return (long long)K * gg / 32; };
  while (g > 4 && M < 8 * g && warps(g / 2) >= 1024) g >>= 1;
  while (g > 4 && M < 16 * g && warps(g / 2) >= 1400) g >>= 1;
  while (g > 2 && M < 64 * g && warps(g / 2) >= 4096) g >>= 1;
  return g;
}

// Persist mode keeps each rollout's cloud ([8][M] floats) in shared memory:
// widen the group until a block's clouds fit (G = 32 holds M <= kPersistMaxM).
size_t persist_smem(int g, int M) {
  return (size_t)(kBlockThreads / 32) * (32 / g) * 2 * kSlotFloats * sizeof(float) +
         (size_t)(kBlockThreads / g) * 8 * M * sizeof(float);
}

// forced: bssmppi_problem.group_width (0 = the policy above).  Persist mode
// is not narrowed: its clouds live in shared memory ([8][M] floats per
// rollout), so a narrow group means few resident blocks -- at C3 G = 8 holds
// one 128 KB block per SM and runs 9.54 ms against 4.22 ms at G = 32
// (tools/persist_sweep.py: G = 32 or a tie on every shape).
int rollout_group_width(int M, int K, bool persist, int forced = 0) {
  int g = forced ? forced : group_width(M, K);
  if (persist && !forced) {
    g = 2;
    while (g < M && g < 32) g <<= 1;
  }
  while (persist && g < 32 && persist_smem(g, M) > kSmemMax) g <<= 1;
  return g;
}

// Block size of the belief kernel: 128 threads (4 blocks per SM) in
// general; 512 (one block per SM, same registers and occupancy) when the
// launch is one nearly full wave -- between 80% and 100% of
// (SMs x 16 warps), 1900-2368 warps on 148 SMs: the 8-GPU shards of C3 and
// C4 and the C2 control step ran 4-5% faster that way, while half-wave
// launches (half the SMs left idle with 512-thread blocks) and multi-wave
// ones ran slower (tools/block_sweep.sh, profiles/r1_block_sweep.txt).
// BSSMPPI_FORCE_BLOCK = 128 | 512 overrides (sweeps); other values are
// reported and ignored.
#ifndef BSS_BIG_MIN_FRAC
#define BSS_BIG_MIN_FRAC 0.8
#endif
int rollout_block_threads(int k_count, int G, bool persist, bool zarr, int sms) {
  static const int forced = [] {
    const char *e = std::getenv("BSSMPPI_FORCE_BLOCK");
    const int v = e ? std::atoi(e) : 0;
    const bool ok = v == kBlockThreads || v == kMaxBlockThreads || v == kSmallBlockThreads;
    if (e && !ok) std::fprintf(stderr, "bssmppi: BSSMPPI_FORCE_BLOCK=%s ignored (64, 128 or 512)\n", e);
    return ok ? v : 0;
  }();
  // persist: clouds sized per 128-thread block; zarr (parity runs): 128 only
  if (persist || zarr) return kBlockThreads;
  if (forced) return (forced == kSmallBlockThreads && G != 4 && G != 8) ? kBlockThreads : forced;
  const long long warps = (long long)k_count * G / 32;
  const long long wave = (long long)sms * (kBlockThreads / 32) * BSS_MIN_BLOCKS;
  return (warps >= (long long)(BSS_BIG_MIN_FRAC * wave) && warps <= wave) ? kMaxBlockThreads : kBlockThreads;
}

// Static shared memory of a kernel (cached: cudaFuncGetAttributes is a
// driver query, and launches sit on the host latency path of small K).
size_t static_smem_of(const void *fn) {
  static std::mutex mu;
  static std::vector<std::pair<const void *, size_t>> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto &e : cache)
    if (e.first == fn) return e.second;
  cudaFuncAttributes a{};
  const size_t v = cudaFuncGetAttributes(&a, fn) == cudaSuccess ? a.sharedSizeBytes : 48 * 1024;
  cache.emplace_back(fn, v);
  return v;
}
template <typename F>
size_t static_smem_of(F *fn) { return static_smem_of(reinterpret_cast<const void *>(fn)); }

template <int G>
cudaError_t launch_bss_g(const RollParams &rp, bool persist, bool zarr, int sms, cudaStream_t st) {
  const int threads = rollout_block_threads(rp.k_count, G, persist, zarr, sms);
  const int GPB = threads / G;   // rollouts per block
  const int blocks = (rp.k_count + GPB - 1) / GPB;
  size_t smem = (size_t)(threads / 32) * (32 / G) * 2 * kSlotFloats * sizeof(float);
  if (persist) smem += (size_t)GPB * 8 * rp.M * sizeof(float);
  void (*fn)(const RollParams);
#ifdef BSS_AB_ONLY   // quick A/B builds: Philox re-projection kernels only
  if (persist || zarr) return cudaErrorNotSupported;
  fn = threads == kMaxBlockThreads ? bss_rollout_kernel<G, false, false, kMaxBlockThreads>
                                   : bss_rollout_kernel<G, false, false>;
#else
  if (persist) fn = zarr ? bss_rollout_kernel<G, true, true> : bss_rollout_kernel<G, true, false>;
  else if (zarr) fn = bss_rollout_kernel<G, false, true>;
  else if (threads == kMaxBlockThreads) fn = bss_rollout_kernel<G, false, false, kMaxBlockThreads>;
  else if constexpr (G == 4 || G == 8) {
    if (threads == kSmallBlockThreads) fn = bss_rollout_kernel<G, false, false, kSmallBlockThreads>;
    else fn = bss_rollout_kernel<G, false, false>;
  }
  else fn = bss_rollout_kernel<G, false, false>;
#endif
  // the kernels also hold static tables (Box-Muller angles, the tire
  // table's shared copy): past 48 KB in total the dynamic part needs the
  // opt-in attribute
  if (smem + static_smem_of(fn) > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  fn<<<blocks, threads, smem, st>>>(rp);
  return cudaGetLastError();
}

int launch_rollout(bssmppi_ctx *c, const RollParams &rp, bool zarr) {
  cudaError_t e;
  if (c->kind == BSSMPPI_KIND_BSS) {
    switch (rollout_group_width(rp.M, rp.k_count, c->persist != 0, c->force_g)) {
      case 2: e = launch_bss_g<2>(rp, c->persist, zarr, c->sms, c->stream); break;
      case 4: e = launch_bss_g<4>(rp, c->persist, zarr, c->sms, c->stream); break;
      case 8: e = launch_bss_g<8>(rp, c->persist, zarr, c->sms, c->stream); break;
      case 16: e = launch_bss_g<16>(rp, c->persist, zarr, c->sms, c->stream); break;
      default: e = launch_bss_g<32>(rp, c->persist, zarr, c->sms, c->stream); break;
    }
  } else {
    const int blocks = (rp.k_count + kBlockThreads - 1) / kBlockThreads;
    if (rp.shield) det_rollout_kernel<true><<<blocks, kBlockThreads, 0, c->stream>>>(rp);
    else det_rollout_kernel<false><<<blocks, kBlockThreads, 0, c->stream>>>(rp);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "rollout launch: %s", cudaGetErrorString(e));
  return BSSMPPI_OK;
}

// Per-block partial records of this context's rollouts, then either one
// rank record into rec_out (final = 0) or the final v+ (final = 1).
int launch_update(bssmppi_ctx *c, bool final_, double *rec_out) {
  const int T2 = 2 * c->T;
  if (final_ && c->k_count <= kSmallK && T2 <= kCombinePart) {   // one launch at small K
    update_small_kernel<<<1, kCombThreads, 0, c->stream>>>(c->k_count, c->k_begin, T2, c->d_cost, c->d_u, c->lam,
                                                           c->lo[0], c->lo[1], c->hi[0], c->hi[1], c->d_out,
                                                           c->d_state + 24, c->d_out + T2, c->h_out_dev);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "update launch: %s", cudaGetErrorString(e));
    return BSSMPPI_OK;
  }
  update_partials_kernel<float, float><<<c->nblocks, kUpdThreads, 0, c->stream>>>(
      c->k_count, c->k_begin, T2, c->d_cost, c->d_u, c->lam, c->chunk, c->d_rec);
  combine_kernel<<<1, kCombThreads, 0, c->stream>>>(
      c->nblocks, T2, c->d_rec, c->lam, final_ ? 1 : 0, rec_out, c->lo[0], c->lo[1], c->hi[0],
      c->hi[1], c->d_out, c->d_state + 24, c->d_out + T2, final_ ? c->h_out_dev : nullptr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "update launch: %s", cudaGetErrorString(e));
  return BSSMPPI_OK;
}

template <typename T>
int ensure(T **p, size_t *cap, size_t n) {
  if (*cap >= n && *p) return BSSMPPI_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  int rc = dev_alloc(p, n);
  if (rc == BSSMPPI_OK) *cap = n;
  return rc;
}

int stage_state(bssmppi_ctx *c, const double *x0, const double *cov0, const double *plan) {
  if (!x0 || !plan) return fail(BSSMPPI_ERR_INVALID, "x0 and plan are required");
  float *h = c->h_state;
  // the previous upload's asynchronous copy may still be queued behind an
  // iteration: wait for it before rewriting the pinned staging buffer
  if (c->h2d_pending) CUDA_TRY(cudaEventSynchronize(c->ev_h2d));
  for (int i = 0; i < 8; ++i) h[i] = (float)x0[i];
  for (int i = 0; i < 16; ++i) h[8 + i] = cov0 ? (float)cov0[i] : 0.f;
  for (int i = 0; i < 2 * c->T; ++i) h[24 + i] = (float)plan[i];
  CUDA_TRY(cudaMemcpyAsync(c->d_state, h, (24 + 2 * c->T) * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaEventRecord(c->ev_h2d, c->stream));
  c->h2d_pending = true;
  return BSSMPPI_OK;
}

// Base rollout params for one iteration.
RollParams iteration_params(bssmppi_ctx *c, const uint32_t *kc, const uint32_t *kb) {
  RollParams rp = c->rp;
  rp.x0 = c->d_state;
  rp.cov0 = c->d_state + 8;
  rp.plan = c->d_state + 24;
  rp.u_out = c->d_u;
  rp.ctl = c->d_ctl;
  rp.ccost = c->d_cc;
  rp.cost_out = c->d_cost;
  rp.mom_out = nullptr;
  rp.eps_in = nullptr;
  rp.u_in = nullptr;
  rp.z_in = nullptr;
  rp.ctrl_mode = CTRL_PHILOX;
  rp.kc = philox_schedule(kc ? kc[0] : 0u, kc ? kc[1] : 0u);
  rp.kb = philox_schedule(kb ? kb[0] : 0u, kb ? kb[1] : 0u);
  return rp;
}

// Upload oracle-noise arrays (local k-range) into rp.
int stage_noise(bssmppi_ctx *c, RollParams &rp, const double *eps, const float *z) {
  if (eps) {
    const size_t n = (size_t)c->k_count * c->T * 2;
    int rc = ensure(&c->d_eps, &c->cap_eps, n);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->d_eps, eps, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    rp.eps_in = c->d_eps;
    rp.ctrl_mode = CTRL_EPS;
  }
  if (z) {
    if (c->kind != BSSMPPI_KIND_BSS) return fail(BSSMPPI_ERR_INVALID, "belief normals given to a deterministic controller");
    if (c->rp.noise_kind != 0)
      return fail(BSSMPPI_ERR_UNSUPPORTED, "Laplace/slip noise has no reference stream (Philox mode only)");
    const size_t n = (size_t)c->T * c->k_count * c->M * 7;
    int rc = ensure(&c->d_z, &c->cap_z, n);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->d_z, z, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    rp.z_in = c->d_z;
  }
  return BSSMPPI_OK;
}

int run_iteration(bssmppi_ctx *c, RollParams &rp, bool final_, double *rec_out) {
  CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
  int rc = launch_rollout(c, rp, rp.z_in != nullptr);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->evr, c->stream));
  rc = launch_update(c, final_, rec_out);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
  c->timed = true;
  return BSSMPPI_OK;
}

int finish(bssmppi_ctx *c, double *vplus, bssmppi_diag *diag) {
  const int T2 = 2 * c->T;
  // the final update kernel wrote v+ and head into mapped h_out as well
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const double *head = c->h_out + T2;
  if (diag) {
    diag->cost_min = head[0];
    diag->weight_sum = head[1];
    diag->ess = head[2] > 0.0 ? head[1] * head[1] / head[2] : 0.0;
    diag->n_finite = (int64_t)head[3];
    diag->cost_argmin = (int64_t)head[4];
    float ms = 0.f, rms = 0.f;
    if (c->timed) {
      cudaEventElapsedTime(&ms, c->ev0, c->ev1);
      cudaEventElapsedTime(&rms, c->ev0, c->evr);
    }
    diag->device_ms = ms;
    diag->rollout_ms = rms;
  }
  if (!(head[3] > 0.0)) return fail(BSSMPPI_ERR_ALL_INVALID, "no rollout produced a finite cost");
  if (vplus) std::memcpy(vplus, c->h_out, T2 * sizeof(double));
  return BSSMPPI_OK;
}

// The device's Box-Muller angle table (philox.cuh g_angle_global), built once
// per device before its first rollout or statistics launch.
int ensure_angle_table(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lock(mu);
  for (int d : done)
    if (d == device) return BSSMPPI_OK;
  // on a private non-blocking stream: no implicit synchronisation with
  // work the caller already has in flight on the device
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e == cudaSuccess) {
    angle_table_init_kernel<<<kAngleTab / 256, 256, 0, st>>>();
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
  if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "angle table: %s", cudaGetErrorString(e));
  done.push_back(device);
  return BSSMPPI_OK;
}

}  // namespace

extern "C" {

const char *bssmppi_last_error(void) { return g_err.c_str(); }

int32_t bssmppi_abi_version(void) { return BSSMPPI_ABI_VERSION; }

int32_t bssmppi_partial_len(int32_t horizon) { return kRecHead + 2 * horizon; }

int32_t bssmppi_group_width(int32_t inner_samples, int32_t k_count) {
  return group_width(std::max(2, inner_samples), std::max(1, k_count));
}

int32_t bssmppi_launch_shape(const bssmppi_ctx *c, int32_t *group_width_out, int32_t *block_threads_out) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  int g = 1, bt = kBlockThreads;
  if (c->kind == BSSMPPI_KIND_BSS) {
    g = rollout_group_width(c->M, c->k_count, c->persist != 0, c->force_g);
    bt = rollout_block_threads(c->k_count, g, c->persist != 0, false, c->sms);
  }
  if (group_width_out) *group_width_out = g;
  if (block_threads_out) *block_threads_out = bt;
  return BSSMPPI_OK;
}

int bssmppi_create(const bssmppi_problem *problem, int32_t device, bssmppi_ctx **out) {
  if (!out) return fail(BSSMPPI_ERR_INVALID, "out is NULL");
  *out = nullptr;
  int rc = validate(problem);
  if (rc) return rc;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(BSSMPPI_ERR_CUDA, "no CUDA device available (the BSS-MPPI path has no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(BSSMPPI_ERR_INVALID, "device %d out of range", device);
  DeviceGuard guard(device);
  CUDA_TRY(cudaSetDevice(device));
  if ((rc = ensure_angle_table(device))) return rc;
  bssmppi_ctx *c = new bssmppi_ctx();
  c->device = device;
  c->kind = problem->kind;
  c->K = problem->samples;
  c->T = problem->horizon;
  c->M = problem->kind == BSSMPPI_KIND_BSS ? problem->inner_samples : 1;
  c->k_begin = problem->k_begin;
  c->k_count = problem->k_count;
  c->persist = problem->kind == BSSMPPI_KIND_BSS && problem->persist_particles;
  c->lam = problem->temperature;
  c->force_g = problem->group_width;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  for (int i = 0; i < 2; ++i) { c->lo[i] = problem->bounds_lo[i]; c->hi[i] = problem->bounds_hi[i]; }
  fill_params(c, problem);
  auto bail = [&](int code) { bssmppi_destroy(c); return code; };
  if ((rc = build_track(c, problem))) return bail(rc);
  if ((rc = build_extensions(c, problem))) return bail(rc);
  if ((rc = build_tire_table(c, problem))) return bail(rc);
  const int T2 = 2 * c->T;
  c->nblocks = std::min(1024, std::max(1, std::min((c->k_count + 63) / 64, 2 * 148)));
  c->chunk = (c->k_count + c->nblocks - 1) / c->nblocks;
  c->nblocks = (c->k_count + c->chunk - 1) / c->chunk;
  if ((rc = dev_alloc(&c->d_state, 24 + T2))) return bail(rc);
  if ((rc = dev_alloc(&c->d_u, (size_t)c->k_count * T2))) return bail(rc);
  if ((rc = dev_alloc(&c->d_cost, c->k_count))) return bail(rc);
  if ((rc = dev_alloc(&c->d_ctl, (size_t)c->k_count * c->T))) return bail(rc);
  if ((rc = dev_alloc(&c->d_cc, (size_t)c->k_count * c->T))) return bail(rc);
  if ((rc = dev_alloc(&c->d_rec, (size_t)c->nblocks * (kRecHead + T2)))) return bail(rc);
  if ((rc = dev_alloc(&c->d_out, T2 + kRecHead))) return bail(rc);
  if (cudaMallocHost((void **)&c->h_state, (24 + T2) * sizeof(float)) != cudaSuccess ||
      cudaHostAlloc((void **)&c->h_out, (T2 + kRecHead) * sizeof(double), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void **)&c->h_out_dev, c->h_out, 0) != cudaSuccess)
    return bail(fail(BSSMPPI_ERR_CUDA, "cudaMallocHost failed"));
  if (cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
      cudaEventCreate(&c->evr) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_h2d, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(BSSMPPI_ERR_CUDA, "cudaEventCreate failed"));
  CUDA_TRY(cudaMemset(c->d_state, 0, (24 + T2) * sizeof(float)));
  *out = c;
  return BSSMPPI_OK;
}

void bssmppi_destroy(bssmppi_ctx *c) {
  if (!c) return;
  DeviceGuard guard(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaFree(c->d_node); cudaFree(c->d_cell); cudaFree(c->d_state); cudaFree(c->d_u);
  cudaFree(c->d_cost); cudaFree(c->d_ctl); cudaFree(c->d_cc); cudaFree(c->d_obs); cudaFree(c->d_cl); cudaFree(c->d_tire); cudaFree(c->d_eps); cudaFree(c->d_uin); cudaFree(c->d_z);
  cudaFree(c->d_mom); cudaFree(c->d_rec); cudaFree(c->d_out);
  if (c->h_state) cudaFreeHost(c->h_state);
  if (c->h_out) cudaFreeHost(c->h_out);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->evr) cudaEventDestroy(c->evr);
  if (c->ev_h2d) cudaEventDestroy(c->ev_h2d);
  delete c;
}

int bssmppi_set_stream(bssmppi_ctx *c, void *stream) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  c->stream = (cudaStream_t)stream;
  return BSSMPPI_OK;
}

int bssmppi_upload_state(bssmppi_ctx *c, const double *x0, const double *cov0, const double *plan) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  DeviceGuard guard(c->device);
  return stage_state(c, x0, cov0, plan);
}

int bssmppi_enqueue_iteration(bssmppi_ctx *c, const uint32_t key_ctrl[2], const uint32_t key_belief[2]) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  if (c->k_begin != 0 || c->k_count != c->K)
    return fail(BSSMPPI_ERR_INVALID, "sharded context: use bssmppi_enqueue_partials + bssmppi_enqueue_combine");
  DeviceGuard guard(c->device);
  RollParams rp = iteration_params(c, key_ctrl, key_belief);
  return run_iteration(c, rp, true, nullptr);
}

int bssmppi_download(bssmppi_ctx *c, double *vplus, bssmppi_diag *diag) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  DeviceGuard guard(c->device);
  return finish(c, vplus, diag);
}

int bssmppi_enqueue_step_device(bssmppi_ctx *c, const float *state_dev, const uint32_t key_ctrl[2],
                                const uint32_t key_belief[2], double *out_dev) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  if (!state_dev || !out_dev) return fail(BSSMPPI_ERR_INVALID, "state_dev and out_dev are required");
  if (c->k_begin != 0 || c->k_count != c->K)
    return fail(BSSMPPI_ERR_INVALID, "sharded context: use bssmppi_enqueue_partials + bssmppi_enqueue_combine");
  DeviceGuard guard(c->device);
  const int T2 = 2 * c->T;
  CUDA_TRY(cudaMemcpyAsync(c->d_state, state_dev, (24 + T2) * sizeof(float), cudaMemcpyDeviceToDevice,
                           c->stream));
  RollParams rp = iteration_params(c, key_ctrl, key_belief);
  int rc = run_iteration(c, rp, true, nullptr);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(out_dev, c->d_out, (T2 + kRecHead) * sizeof(double), cudaMemcpyDeviceToDevice,
                           c->stream));
  return BSSMPPI_OK;
}

int bssmppi_control_step(bssmppi_ctx *c, const double *x0, const double *cov0, const double *plan,
                         const uint32_t key_ctrl[2], const uint32_t key_belief[2], const double *eps,
                         const float *z, double *vplus, bssmppi_diag *diag) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  if (c->k_begin != 0 || c->k_count != c->K)
    return fail(BSSMPPI_ERR_INVALID, "sharded context: use bssmppi_step_partials + bssmppi_update_combine");
  DeviceGuard guard(c->device);
  int rc = stage_state(c, x0, cov0, plan);
  if (rc) return rc;
  RollParams rp = iteration_params(c, key_ctrl, key_belief);
  if ((rc = stage_noise(c, rp, eps, z))) return rc;
  if ((rc = run_iteration(c, rp, true, nullptr))) return rc;
  return finish(c, vplus, diag);
}

int bssmppi_step_partials(bssmppi_ctx *c, const double *x0, const double *cov0, const double *plan,
                          const uint32_t key_ctrl[2], const uint32_t key_belief[2], const double *eps,
                          const float *z, double *partials_dev, int32_t slot) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  if (!partials_dev || slot < 0) return fail(BSSMPPI_ERR_INVALID, "partials buffer/slot invalid");
  DeviceGuard guard(c->device);
  int rc = stage_state(c, x0, cov0, plan);
  if (rc) return rc;
  RollParams rp = iteration_params(c, key_ctrl, key_belief);
  if ((rc = stage_noise(c, rp, eps, z))) return rc;
  return run_iteration(c, rp, false, partials_dev + (size_t)slot * (kRecHead + 2 * c->T));
}

int bssmppi_enqueue_partials(bssmppi_ctx *c, const uint32_t key_ctrl[2], const uint32_t key_belief[2],
                             double *partials_dev, int32_t slot) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  if (!partials_dev || slot < 0) return fail(BSSMPPI_ERR_INVALID, "partials buffer/slot invalid");
  DeviceGuard guard(c->device);
  RollParams rp = iteration_params(c, key_ctrl, key_belief);
  return run_iteration(c, rp, false, partials_dev + (size_t)slot * (kRecHead + 2 * c->T));
}

int bssmppi_enqueue_combine(bssmppi_ctx *c, const double *partials_dev, int32_t nslots) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  if (!partials_dev || nslots < 1 || nslots > 1024) return fail(BSSMPPI_ERR_INVALID, "bad partials / nslots");
  DeviceGuard guard(c->device);
  const int T2 = 2 * c->T;
  combine_kernel<<<1, kCombThreads, 0, c->stream>>>(nslots, T2, partials_dev, c->lam, 1, nullptr, c->lo[0],
                                                   c->lo[1], c->hi[0], c->hi[1], c->d_out, c->d_state + 24,
                                                   c->d_out + T2, c->h_out_dev);
  CUDA_TRY(cudaGetLastError());
  return BSSMPPI_OK;
}

int bssmppi_update_combine(bssmppi_ctx *c, const double *partials_dev, int32_t nslots, double *vplus,
                           bssmppi_diag *diag) {
  int rc = bssmppi_enqueue_combine(c, partials_dev, nslots);
  if (rc) return rc;
  DeviceGuard guard(c->device);
  return finish(c, vplus, diag);
}

int bssmppi_rollout(bssmppi_ctx *c, const double *x0, const double *cov0, const double *u, const double *eps,
                    const double *nominal, const float *z, const uint32_t key_belief[2], double *costs,
                    float *moments) {
  if (!c) return fail(BSSMPPI_ERR_INVALID, "ctx is NULL");
  if (!u || !eps || !nominal) return fail(BSSMPPI_ERR_INVALID, "u, eps and nominal are required");
  DeviceGuard guard(c->device);
  int rc = stage_state(c, x0, cov0, nominal);
  if (rc) return rc;
  RollParams rp = iteration_params(c, nullptr, key_belief);
  if ((rc = stage_noise(c, rp, eps, z))) return rc;
  const size_t n = (size_t)c->k_count * c->T * 2;
  if ((rc = ensure(&c->d_uin, &c->cap_uin, n))) return rc;
  CUDA_TRY(cudaMemcpyAsync(c->d_uin, u, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  rp.u_in = c->d_uin;
  rp.ctrl_mode = CTRL_GIVEN;
  const size_t nm = (size_t)c->T * c->k_count * 18;
  if (moments && c->kind == BSSMPPI_KIND_BSS) {
    if ((rc = ensure(&c->d_mom, &c->cap_mom, nm))) return rc;
    rp.mom_out = c->d_mom;
  }
  if ((rc = launch_rollout(c, rp, rp.z_in != nullptr))) return rc;
  std::vector<float> hc(c->k_count);
  CUDA_TRY(cudaMemcpyAsync(hc.data(), c->d_cost, c->k_count * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  if (rp.mom_out) CUDA_TRY(cudaMemcpyAsync(moments, c->d_mom, nm * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (costs)
    for (int k = 0; k < c->k_count; ++k) costs[k] = (double)hc[k];
  return BSSMPPI_OK;
}

int bssmppi_mppi_update(int32_t K, int32_t T, const double *costs, const double *controls, double temperature,
                        const double lo[2], const double hi[2], double *vplus, bssmppi_diag *diag) {
  if (K < 1 || T < 1 || T > 512 || !costs || !controls || !lo || !hi || !vplus)
    return fail(BSSMPPI_ERR_INVALID, "bad mppi_update arguments");
  if (!(temperature > 0.0)) return fail(BSSMPPI_ERR_INVALID, "temperature must be > 0");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(BSSMPPI_ERR_CUDA, "no CUDA device available (the BSS-MPPI path has no CPU fallback)");
  const int T2 = 2 * T;
  int nblocks = std::min(1024, std::max(1, std::min((K + 63) / 64, 2 * 148)));
  const int chunk = (K + nblocks - 1) / nblocks;
  nblocks = (K + chunk - 1) / chunk;
  double *d_c = nullptr, *d_u = nullptr, *d_rec = nullptr, *d_out = nullptr;
  int rc = BSSMPPI_OK;
  std::vector<double> h(T2 + kRecHead);
  if ((rc = dev_alloc(&d_c, K)) || (rc = dev_alloc(&d_u, (size_t)K * T2)) ||
      (rc = dev_alloc(&d_rec, (size_t)nblocks * (kRecHead + T2))) || (rc = dev_alloc(&d_out, T2 + kRecHead))) {
  } else {
    cudaError_t e = cudaMemcpy(d_c, costs, K * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_u, controls, (size_t)K * T2 * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      update_partials_kernel<double, double><<<nblocks, kUpdThreads>>>(K, 0, T2, d_c, d_u, temperature, chunk, d_rec);
      combine_kernel<<<1, kCombThreads>>>(nblocks, T2, d_rec, temperature, 1, nullptr, lo[0], lo[1], hi[0], hi[1],
                                         d_out, nullptr, d_out + T2, nullptr);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(h.data(), d_out, h.size() * sizeof(double), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(BSSMPPI_ERR_CUDA, "mppi_update: %s", cudaGetErrorString(e));
  }
  cudaFree(d_c); cudaFree(d_u); cudaFree(d_rec); cudaFree(d_out);
  if (rc) return rc;
  const double *head = h.data() + T2;
  if (diag) {
    diag->cost_min = head[0];
    diag->weight_sum = head[1];
    diag->ess = head[2] > 0.0 ? head[1] * head[1] / head[2] : 0.0;
    diag->n_finite = (int64_t)head[3];
    diag->cost_argmin = (int64_t)head[4];
    diag->device_ms = 0.f;
    diag->rollout_ms = 0.f;
  }
  if (!(head[3] > 0.0)) return fail(BSSMPPI_ERR_ALL_INVALID, "no rollout produced a finite cost");
  std::memcpy(vplus, h.data(), T2 * sizeof(double));
  return BSSMPPI_OK;
}

}  // extern "C"

namespace {
__global__ void sample_controls_kernel(int n, int T, const double *z, double f0, double f1, double f2, double f3,
                                       const double *nominal, double lo0, double lo1, double hi0, double hi1,
                                       double *eps, double *u) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)n * T) return;
  const int t = (int)(i % T);
  const double z0 = z[2 * i], z1 = z[2 * i + 1];
  // eps = z @ F^T (controllers.py:175)
  const double e0 = z0 * f0 + z1 * f1, e1 = z0 * f2 + z1 * f3;
  eps[2 * i] = e0;
  eps[2 * i + 1] = e1;
  u[2 * i] = fmin(fmax(nominal[2 * t] + e0, lo0), hi0);
  u[2 * i + 1] = fmin(fmax(nominal[2 * t + 1] + e1, lo1), hi1);
}

// Measured FP32 peak (roofline denominator): 8 independent FFMA chains per
// thread, 148 * 8 blocks of 256 threads.
__global__ void __launch_bounds__(256) ffma_peak_kernel(float *out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678f) out[0] = s;
}

// MUFU (XU pipe) throughput: 8 independent ex2.approx chains per thread,
// x <- 2^(-x) stays in (0.5, 1); the negation is a free operand modifier.
__global__ void __launch_bounds__(256) mufu_peak_kernel(float *out, int iters) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 0.5f + threadIdx.x * 1e-4f + i * 1e-2f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(x[i]) : "f"(-x[i]));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678f) out[0] = s;
}

__global__ void philox_kernel(Philox4 c, uint32_t k0, uint32_t k1, int rounds, uint32_t *out) {
  const PhiloxKeys rk = philox_schedule(k0, k1);
  const Philox4 r = rounds == 7 ? philox4x32<7>(c, rk) : philox4x32<10>(c, rk);
  out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
}

__global__ void belief_normals_kernel(uint32_t k0, uint32_t k1, int t, int k, int mcount, float *out) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= mcount) return;
  float z[7];
  belief_normals(philox_schedule(k0, k1), (uint32_t)t, (uint32_t)k, (uint32_t)m, z);
  for (int j = 0; j < 7; ++j) out[(size_t)m * 7 + j] = z[j];
}
}  // namespace

extern "C" {

int bssmppi_sample_controls(int32_t n, int32_t T, const double *z, const double factor[4], const double *nominal,
                            const double lo[2], const double hi[2], double *eps, double *u) {
  if (n < 1 || T < 1 || !z || !factor || !nominal || !lo || !hi || !eps || !u)
    return fail(BSSMPPI_ERR_INVALID, "bad sample_controls arguments");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(BSSMPPI_ERR_CUDA, "no CUDA device available (the BSS-MPPI path has no CPU fallback)");
  const size_t cnt = (size_t)n * T * 2;
  double *d = nullptr;
  int rc = dev_alloc(&d, 3 * cnt + 2 * T);
  if (rc) return rc;
  double *dz = d, *de = d + cnt, *du = d + 2 * cnt, *dn = d + 3 * cnt;
  cudaError_t e = cudaMemcpy(dz, z, cnt * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dn, nominal, 2 * T * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const size_t items = (size_t)n * T;
    sample_controls_kernel<<<(unsigned)((items + 255) / 256), 256>>>(n, T, dz, factor[0], factor[1], factor[2],
                                                                     factor[3], dn, lo[0], lo[1], hi[0], hi[1], de, du);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(eps, de, cnt * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(u, du, cnt * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "sample_controls: %s", cudaGetErrorString(e));
  return BSSMPPI_OK;
}

int bssmppi_step_array(bssmppi_ctx *c, int32_t n, const double *x, const double *u, const double *w, double *x_out,
                       uint8_t *ok) {
  if (!c || n < 1 || !x || !u || !x_out || !ok) return fail(BSSMPPI_ERR_INVALID, "bad step_array arguments");
  DeviceGuard guard(c->device);
  double *d = nullptr;
  uint8_t *dok = nullptr;
  int rc = dev_alloc(&d, (size_t)n * (8 + 2 + 3 + 8));
  if (rc) return rc;
  if ((rc = dev_alloc(&dok, n))) { cudaFree(d); return rc; }
  double *dx = d, *du = d + (size_t)n * 8, *dw = d + (size_t)n * 10, *dxo = d + (size_t)n * 13;
  cudaError_t e = cudaMemcpy(dx, x, (size_t)n * 8 * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(du, u, (size_t)n * 2 * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && w) e = cudaMemcpy(dw, w, (size_t)n * 3 * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    step_array_kernel<<<(n + 127) / 128, 128, 0, c->stream>>>(c->rp.V, c->rp.tr, n, dx, du, w ? dw : nullptr, dxo, dok);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = cudaMemcpy(x_out, dxo, (size_t)n * 8 * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(ok, dok, n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  cudaFree(dok);
  if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "step_array: %s", cudaGetErrorString(e));
  return BSSMPPI_OK;
}

int bssmppi_philox4x32(const uint32_t ctr[4], const uint32_t key[2], int32_t rounds, uint32_t out[4]) {
  if (!ctr || !key || !out) return fail(BSSMPPI_ERR_INVALID, "NULL argument");
  if (rounds != 7 && rounds != 10) return fail(BSSMPPI_ERR_INVALID, "rounds must be 7 or 10");
  uint32_t *d = nullptr;
  int rc = dev_alloc(&d, 4);
  if (rc) return rc;
  philox_kernel<<<1, 1>>>(Philox4{ctr[0], ctr[1], ctr[2], ctr[3]}, key[0], key[1], rounds, d);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(out, d, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "philox: %s", cudaGetErrorString(e));
  return BSSMPPI_OK;
}

int bssmppi_iteration_key(const uint32_t base[2], uint32_t domain, uint64_t iteration, uint32_t out[2]) {
  if (!base || !out) return fail(BSSMPPI_ERR_INVALID, "NULL argument");
  // Philox4x32-10 of (iteration lo, iteration hi, domain, tag) under the
  // controller's base key: distinct (domain, iteration) -> independent keys.
  const Philox4 r = philox4x32<10>(Philox4{(uint32_t)iteration, (uint32_t)(iteration >> 32), domain, 0x6b657973u},
                                   philox_schedule(base[0], base[1]));
  out[0] = r.x;
  out[1] = r.y;
  return BSSMPPI_OK;
}

int bssmppi_ffma_peak(int32_t device, double *tflops) {
  if (!tflops) return fail(BSSMPPI_ERR_INVALID, "NULL argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(BSSMPPI_ERR_CUDA, "no CUDA device %d", device);
  DeviceGuard guard(device);
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float *d = nullptr;
  int rc = dev_alloc(&d, 1);
  if (rc) return rc;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, iters = 4096;
  ffma_peak_kernel<<<blocks, 256>>>(d, 64, 0.999f, 1e-3f);   // warm-up
  cudaEventRecord(e0);
  ffma_peak_kernel<<<blocks, 256>>>(d, iters, 0.999f, 1e-3f);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "ffma_peak: %s", cudaGetErrorString(e));
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * 256;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return BSSMPPI_OK;
}

int bssmppi_mufu_peak(int32_t device, double *tops) {
  if (!tops) return fail(BSSMPPI_ERR_INVALID, "NULL argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(BSSMPPI_ERR_CUDA, "no CUDA device %d", device);
  DeviceGuard guard(device);
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float *d = nullptr;
  int rc = dev_alloc(&d, 1);
  if (rc) return rc;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, iters = 512;
  mufu_peak_kernel<<<blocks, 256>>>(d, 16);   // warm-up
  cudaEventRecord(e0);
  mufu_peak_kernel<<<blocks, 256>>>(d, iters);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "mufu_peak: %s", cudaGetErrorString(e));
  const double ops = 8.0 * 16 * (double)iters * blocks * 256;
  *tops = ops / (ms * 1e-3) / 1e12;
  return BSSMPPI_OK;
}

int bssmppi_tire_table(const double bc[4], double steer_max, float *out, int32_t cap, int32_t *rows,
                       double *cells_per_rad, double *amax) {
  if (!bc || !out || !rows || !cells_per_rad || !amax || !(steer_max >= 0.0))
    return fail(BSSMPPI_ERR_INVALID, "bad tire_table arguments");
  std::vector<float4> tab;
  int r;
  tire_table_host(bc, steer_max, tab, *cells_per_rad, *amax, r);
  *rows = r;
  if ((size_t)cap < tab.size()) return fail(BSSMPPI_ERR_INVALID, "tire_table needs %zu rows", tab.size());
  std::memcpy(out, tab.data(), tab.size() * sizeof(float4));
  return BSSMPPI_OK;
}

int bssmppi_belief_normals(const uint32_t key[2], int32_t t, int32_t k, int32_t m_count, float *out) {
  if (!key || !out || m_count < 1) return fail(BSSMPPI_ERR_INVALID, "bad belief_normals arguments");
  int dev = 0;
  cudaGetDevice(&dev);
  int rc = ensure_angle_table(dev);
  if (rc) return rc;
  float *d = nullptr;
  rc = dev_alloc(&d, (size_t)m_count * 7);
  if (rc) return rc;
  belief_normals_kernel<<<(m_count + 127) / 128, 128>>>(key[0], key[1], t, k, m_count, d);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(out, d, (size_t)m_count * 7 * sizeof(float), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(BSSMPPI_ERR_CUDA, "belief_normals: %s", cudaGetErrorString(e));
  return BSSMPPI_OK;
}

}  // extern "C"

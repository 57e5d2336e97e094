/*
 * bss_oracle.c -- FP64 CPU restatement of the reference BSS-MPPI step.
 * TEST INFRASTRUCTURE ONLY: used by tests/ (checker) and by bench.py's
 * cpu_baseline / --impl reference leg (the timed CPU arm).  Never linked by
 * the product library.
 *
 * Follows the reference numba/numpy path line by line
 * (/root/reference/pkg/src/belief_mppi):
 *   curv()          _curv_scalar          dynamics.py:340-369 (binary search)
 *   tire()          _tire_row             dynamics.py:372-395
 *   derivs()        _derivs_row           dynamics.py:398-437
 *   step_euler()    _step_kernel (Euler)  dynamics.py:447-497
 *   chol4()         _psd_chol_kernel      belief.py:235-256 (1e-300 clamp)
 *   moments()       _moments_kernel       belief.py:275-308 (pairwise tree
 *                   mean, fixed-order two-pass unbiased covariance)
 *   rollout_one()   _rollout bss/mppi/smppi controllers.py:261-341
 *   orc_update()    mppi_weights/mppi_update controllers.py:180-194
 * Noise: either the reference's captured arrays (eps (K,T,2), z (T,K,M,7))
 * or the device's Philox4x32 counters (same keys/counters as csrc/), so
 * the timed CPU arm does the same work as the GPU arm.
 * Parallel over rollouts k with OpenMP (the reference parallelises only
 * across processes, sim.py:321-322; one k is independent of all others).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/bssmppi.h"

typedef struct {
  const bssmppi_problem *p;
  const double *ph;
} Ctx;

static double pymod(double a, double b) { /* Python/numba floor-mod */
  double r = fmod(a, b);
  if (r != 0.0 && ((r < 0.0) != (b < 0.0))) r += b;
  return r;
}

static double curv(const bssmppi_problem *p, double s) {
  const double *sn = p->track_s, *kn = p->track_kappa;
  const int n = p->track_n;
  const double L = p->track_length;
  double sw = p->track_closed ? pymod(s, L) : fmin(fmax(s, 0.0), L);
  double x0, x1, y0, y1;
  if (p->track_closed && sw >= sn[n - 1]) {
    x0 = sn[n - 1]; x1 = L; y0 = kn[n - 1]; y1 = kn[0];
  } else {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) / 2;
      if (sn[mid] <= sw) lo = mid; else hi = mid - 1;
    }
    if (lo >= n - 1) return kn[n - 1];
    x0 = sn[lo]; x1 = sn[lo + 1]; y0 = kn[lo]; y1 = kn[lo + 1];
  }
  if (x1 == x0) return y0;
  return y0 + (y1 - y0) * (sw - x0) / (x1 - x0);
}

static int derivs(const Ctx *c, const double *x, double u0, double u1, double *dx) {
  const double *p = c->ph;
  const double vx = x[0], vy = x[1], r = x[2], wf = x[3], wr = x[4], e_psi = x[5], e_y = x[6], s = x[7];
  double vx_eff = vx >= 0.0 ? fmax(vx, p[20]) : fmin(vx, -p[20]);
  double denom = fabs(vx_eff);
  double alpha_f = u0 - atan2(vy + p[2] * r, vx_eff);
  double alpha_r = -atan2(vy - p[3] * r, vx_eff);
  double sigma_f = (wf * p[4] - vx) / denom;
  double sigma_r = (wr * p[4] - vx) / denom;
  double fyf0 = p[15] * sin(p[7] * atan(p[6] * alpha_f));
  double fyr0 = p[17] * sin(p[9] * atan(p[8] * alpha_r));
  double fxf = p[14] * sin(p[11] * atan(p[10] * sigma_f));
  double fxr = p[16] * sin(p[13] * atan(p[12] * sigma_r));
  double a = fxf / p[14], b = fxr / p[16];
  double fyf = fyf0 * sqrt(fmax(1.0 - a * a, 0.0));
  double fyr = fyr0 * sqrt(fmax(1.0 - b * b, 0.0));
  double cos_d = cos(u0), sin_d = sin(u0);
  double fxf_b = fxf * cos_d - fyf * sin_d;
  double fyf_b = fxf * sin_d + fyf * cos_d;
  dx[0] = (fxf_b + fxr) / p[0] + vy * r;
  dx[1] = (fyf_b + fyr) / p[0] - vx * r;
  dx[2] = (p[2] * fyf_b - p[3] * fyr) / p[1];
  double spin_f = tanh(wf * p[4] / 0.1), spin_r = tanh(wr * p[4] / 0.1);
  dx[3] = (-p[4] * fxf - p[19] * p[21] * p[4] * spin_f) / p[5];
  dx[4] = (p[18] * u1 - p[4] * fxr - p[19] * p[22] * p[4] * spin_r) / p[5];
  double kappa = curv(c->p, s);
  double frame = 1.0 - kappa * e_y;
  int ok = frame > 0.0;
  if (frame < 1e-3) frame = 1e-3;
  double cos_e = cos(e_psi), sin_e = sin(e_psi);
  double ds = (vx * cos_e - vy * sin_e) / frame;
  dx[7] = ds;
  dx[6] = vx * sin_e + vy * cos_e;
  dx[5] = r - kappa * ds;
  return ok;
}

static int step_euler(const Ctx *c, double *x, double u0, double u1) {
  double dx[8];
  int ok = derivs(c, x, u0, u1, dx);
  const double dt = c->p->dt, L = c->p->track_length;
  for (int i = 0; i < 8; ++i) x[i] = x[i] + dt * dx[i];
  x[5] = M_PI - pymod(M_PI - x[5], 2.0 * M_PI);
  if (c->p->track_closed) x[7] = pymod(x[7], L);
  else if (x[7] < 0.0) x[7] = 0.0;
  else if (x[7] > L) x[7] = L;
  for (int i = 0; i < 8; ++i)
    if (!isfinite(x[i])) { ok = 0; x[i] = 0.0; }
  return ok;
}

static void chol4(const double C[16], double L[16]) {
  memset(L, 0, 16 * sizeof(double));
  for (int col = 0; col < 4; ++col) {
    double acc = C[col * 4 + col];
    for (int k = 0; k < col; ++k) acc -= L[col * 4 + k] * L[col * 4 + k];
    if (acc <= 1e-300) continue;
    double piv = sqrt(acc);
    L[col * 4 + col] = piv;
    for (int r = col + 1; r < 4; ++r) {
      double a = C[r * 4 + col];
      for (int k = 0; k < col; ++k) a -= L[r * 4 + k] * L[col * 4 + k];
      L[r * 4 + col] = a / piv;
    }
  }
}

static const int SUB[4] = {1, 2, 5, 6};

static void moments(const double *x, int n, double *buf, double *mean, double *cov) {
  for (int c = 0; c < 8; ++c) {
    for (int j = 0; j < n; ++j) buf[j] = x[j * 8 + c];
    int width = n;
    while (width > 1) {
      int half = width / 2;
      for (int j = 0; j < half; ++j) buf[j] = buf[2 * j] + buf[2 * j + 1];
      if (width % 2 == 1) { buf[half] = buf[width - 1]; width = half + 1; }
      else width = half;
    }
    mean[c] = buf[0] / n;
  }
  for (int a = 0; a < 4; ++a)
    for (int b = a; b < 4; ++b) {
      double acc = 0.0, ma = mean[SUB[a]], mb = mean[SUB[b]];
      for (int j = 0; j < n; ++j) acc += (x[j * 8 + SUB[a]] - ma) * (x[j * 8 + SUB[b]] - mb);
      double v = acc / (n - 1);
      cov[a * 4 + b] = v;
      cov[b * 4 + a] = v;
    }
}

/* ---- Philox4x32 (7 rounds belief, 10 control) + Box-Muller: same counters as csrc/philox.cuh ---- */
static void philox_r(uint32_t c[4], uint32_t k0, uint32_t k1, int rounds) {
  for (int i = 0; i < rounds; ++i) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
}

/* rounds: 7 for the belief stream, 10 for the control stream (csrc/philox.cuh) */
static void philox(uint32_t c[4], uint32_t k0, uint32_t k1) { philox_r(c, k0, k1, 10); }

static void bm(uint32_t a, uint32_t b, double *z0, double *z1) {
  union { uint32_t u; float f; } x, y;
  x.u = 0x3f800000u | (a >> 9);
  y.u = 0x3f800000u | (b >> 9);
  double u1 = 2.0 - (double)x.f, u2 = (double)y.f - 1.5;
  double r = sqrt(-2.0 * log(u1));
  *z0 = r * cos(2.0 * M_PI * u2);
  *z1 = r * sin(2.0 * M_PI * u2);
}

/* Belief stream (csrc/philox.cuh belief_block / box_muller_word): ONE
 * Philox4x32-7 block per particle-step, counter (t, m, kg, 0); word i ->
 * pair i with u1 = 1 - (n + 1/2) 2^-20 (n = top 20 bits) and angle
 * 2 pi j / 4096 (j = low 12 bits); standard pair -sqrt(-2 ln u1)(cos, sin). */
static void bm_word(uint32_t w, double *z0, double *z1) {
  double u1 = 1.0 - ((double)(w >> 12) + 0.5) * (1.0 / 1048576.0);
  double th = 2.0 * M_PI * (double)(w & 0xfffu) / 4096.0;
  double r = sqrt(-2.0 * log(u1));
  *z0 = -r * cos(th);
  if (z1) *z1 = -r * sin(th);
}

static void belief_normals(uint32_t k0, uint32_t k1, uint32_t t, uint32_t kg, uint32_t m, double z[7]) {
  uint32_t a[4] = {t, m, kg, 0u};
  philox_r(a, k0, k1, 7);
  bm_word(a[0], &z[0], &z[1]);
  bm_word(a[1], &z[2], &z[3]);
  bm_word(a[2], &z[4], &z[5]);
  bm_word(a[3], &z[6], NULL);
}

static void control_normals(uint32_t k0, uint32_t k1, uint32_t t, uint32_t kg, double *z0, double *z1) {
  uint32_t a[4] = {t, kg, 0x5eedc0deu, 0u};
  philox(a, k0, k1);
  bm(a[0], a[1], z0, z1);
}

/* The 7 belief normals of (t, kg, m) for m < m_count (row-major [m][7]): the
 * checker for bssmppi_belief_normals. */
int orc_belief_normals(const uint32_t key[2], uint32_t t, uint32_t kg, int m_count, double *out) {
  for (int m = 0; m < m_count; ++m) belief_normals(key[0], key[1], t, kg, (uint32_t)m, out + (size_t)m * 7);
  return 0;
}

/* Per-iteration key (same definition as bssmppi_iteration_key). */
int orc_iteration_key(const uint32_t base[2], uint32_t domain, uint64_t iteration, uint32_t out[2]) {
  uint32_t c[4] = {(uint32_t)iteration, (uint32_t)(iteration >> 32), domain, 0x6b657973u};
  philox_r(c, base[0], base[1], 10);
  out[0] = c[0];
  out[1] = c[1];
  return 0;
}

int orc_philox4x32(const uint32_t ctr[4], const uint32_t key[2], int rounds, uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  philox_r(c, key[0], key[1], rounds);
  memcpy(out, c, sizeof(c));
  return 0;
}

/* Config-4 extension (beyond the reference; obstacles.py): Laplace + slip
 * noise from the second Philox block's words, obstacle heuristic terms. */
/* centred uniform (n + 1/2) 2^-16 - 1/2 of a 16-bit field n */
static double centred_uniform16(uint32_t n) { return ((double)n + 0.5) * (1.0 / 65536.0) - 0.5; }

/* csrc/philox.cuh laplace_from_block: normals from words 0, 1; Laplace on
 * (vx, vy, r) and the vy slip from the 16-bit halves of words 2, 3. */
static void belief_noise_laplace(uint32_t k0, uint32_t k1, uint32_t t, uint32_t kg, uint32_t m, double b,
                                 double a, double z[4], double w[3]) {
  uint32_t p[4] = {t, m, kg, 0u};
  philox_r(p, k0, k1, 7);
  bm_word(p[0], &z[0], &z[1]);
  bm_word(p[1], &z[2], &z[3]);
  const uint32_t f[4] = {p[2] >> 16, p[2] & 0xffffu, p[3] >> 16, p[3] & 0xffffu};
  for (int i = 0; i < 3; ++i) {
    double u = centred_uniform16(f[i]);
    w[i] = -b * copysign(log(1.0 - 2.0 * fabs(u)), u);
  }
  w[1] += 2.0 * a * centred_uniform16(f[3]);
}

static double obstacle_terms(const bssmppi_problem *p, double s, double ey, double sigy, int *inside) {
  const double L = p->track_length;
  double sw = p->track_closed ? pymod(s, L) : fmin(fmax(s, 0.0), L);
  double fi = sw / p->centerline_ds;
  int j = (int)fi;
  if (j < 0) j = 0;
  if (j > p->centerline_n - 2) j = p->centerline_n - 2;
  double f = fi - j;
  const double *a = p->centerline + 3 * j, *b = a + 3;
  double cx = a[0] + f * (b[0] - a[0]), cy = a[1] + f * (b[1] - a[1]), th = a[2] + f * (b[2] - a[2]);
  double nx = -sin(th), ny = cos(th);
  double px = cx + ey * nx, py = cy + ey * ny, h = INFINITY;
  *inside = 0;
  for (int i = 0; i < p->n_obstacles; ++i) {
    const double *o = p->obstacles + 3 * i;
    double dx = px - o[0], dy = py - o[1], d = sqrt(dx * dx + dy * dy);
    if (d < o[2]) *inside = 1;
    double eta = d > 0.0 ? (dx * nx + dy * ny) / d : 1.0;
    double hi = d - o[2] - p->obstacle_backoff * fabs(eta) * sigy;
    if (hi < h) h = hi;
  }
  return h;
}

static double stage(const bssmppi_problem *p, const double *x) {
  double quad = 0.0;
  for (int i = 0; i < 8; ++i) {
    double d = x[i] - (i == 0 ? p->v_goal : 0.0);
    quad += d * d * p->q_diag[i];
  }
  return quad + p->obstacle_penalty * (fabs(x[6]) > p->half_width ? 1.0 : 0.0);
}

static double dcbf(const bssmppi_problem *p, double ey, double sig) {
  double m = fmax(p->half_width - p->backoff * sig, 0.0);
  return m * m - ey * ey;
}

static double pen(const bssmppi_problem *p, double hc, double hp) {
  return p->penalty * fmax(-(hc - (1.0 - p->cbf_rate) * hp), 0.0);
}

typedef struct {
  const double *x0, *cov0, *nominal, *u_in, *eps_in, *z_in;
  uint32_t kc[2], kb[2];
  int philox_ctrl, philox_belief;
  double *mom_out;   /* (T, k_count, 18): mean[8] + upper cov (00,01,02,03,11,12,13,22,23,33), or NULL */
} Inputs;

/* One rollout k (local index); returns its cost, writes u_out row. */
static double rollout_one(const Ctx *c, const Inputs *in, int k, double *xs, double *buf, double *u_out) {
  const bssmppi_problem *p = c->p;
  const int T = p->horizon, M = p->kind == BSSMPPI_KIND_BSS ? p->inner_samples : 1;
  const int kg = p->k_begin + k, K = p->k_count;
  double mean[8], cov[16], L[16], total = 0.0;
  int dead = 0;
  memcpy(mean, in->x0, sizeof(mean));
  for (int i = 0; i < 16; ++i) cov[i] = in->cov0 ? in->cov0[i] : 0.0;
  const int bss = p->kind == BSSMPPI_KIND_BSS, shield = p->kind != BSSMPPI_KIND_MPPI;
  double sig = bss ? sqrt(fmax(cov[15], 0.0)) : 0.0;
  double h_cur = dcbf(p, mean[6], sig), h_prev = h_cur;
  int inside = 0;
  double ho_cur = p->n_obstacles ? obstacle_terms(p, mean[7], mean[6], sig, &inside) : 0.0, ho_prev = ho_cur;
  int noise_on = 0;
  for (int i = 0; i < 9; ++i) noise_on |= p->noise_factor[i] != 0.0;
  const double *F = p->noise_factor;
  for (int t = 0; t < T; ++t) {
    total += stage(p, mean);
    if (shield && t > 0) total += pen(p, h_cur, h_prev);
    if (p->n_obstacles) {
      if (inside) total += p->obstacle_penalty;
      if (shield && t > 0) total += pen(p, ho_cur, ho_prev);
    }
    double v0 = in->nominal[2 * t], v1 = in->nominal[2 * t + 1], e0, e1, u0, u1;
    const size_t o = ((size_t)k * T + t) * 2;
    if (in->philox_ctrl) {
      double z0, z1;
      control_normals(in->kc[0], in->kc[1], t, kg, &z0, &z1);
      e0 = p->sigma_factor[0] * z0 + p->sigma_factor[1] * z1;
      e1 = p->sigma_factor[2] * z0 + p->sigma_factor[3] * z1;
    } else {
      e0 = in->eps_in[o]; e1 = in->eps_in[o + 1];
    }
    if (in->u_in) { u0 = in->u_in[o]; u1 = in->u_in[o + 1]; }
    else {
      u0 = fmin(fmax(v0 + e0, p->bounds_lo[0]), p->bounds_hi[0]);
      u1 = fmin(fmax(v1 + e1, p->bounds_lo[1]), p->bounds_hi[1]);
    }
    if (u_out) { u_out[o] = u0; u_out[o + 1] = u1; }
    const double a0 = v0 + e0, a1 = v1 + e1;
    total += p->control_cost_weight * (v0 * (p->precision[0] * a0 + p->precision[1] * a1) +
                                       v1 * (p->precision[2] * a0 + p->precision[3] * a1));
    if (!bss) {
      dead |= !step_euler(c, mean, u0, u1);
      if (shield) { h_prev = h_cur; h_cur = dcbf(p, mean[6], 0.0); }
      if (p->n_obstacles) { ho_prev = ho_cur; ho_cur = obstacle_terms(p, mean[7], mean[6], 0.0, &inside); }
      continue;
    }
    const int reproject = !(p->persist_particles && t > 0);
    if (reproject) chol4(cov, L);
    for (int m = 0; m < M; ++m) {
      double z[7] = {0, 0, 0, 0, 0, 0, 0}, wl[3] = {0.0, 0.0, 0.0};
      if (in->philox_belief && p->noise_kind == 1)
        belief_noise_laplace(in->kb[0], in->kb[1], t, kg, m, p->laplace_scale, p->slip_bias, z, wl);
      else if (in->philox_belief) belief_normals(in->kb[0], in->kb[1], t, kg, m, z);
      else {
        const double *zp = in->z_in + (((size_t)t * K + k) * M + m) * 7;
        for (int j = 0; j < 7; ++j) z[j] = zp[j];
      }
      double *x = xs + (size_t)m * 8;
      if (reproject) {
        memcpy(x, mean, sizeof(mean));
        for (int a = 0; a < 4; ++a) {
          double acc = 0.0;
          for (int b = 0; b < 4; ++b) acc += L[a * 4 + b] * z[b];
          x[SUB[a]] += acc;
        }
      }
      step_euler(c, x, u0, u1);
      if (p->noise_kind == 1)
        for (int i = 0; i < 3; ++i) x[i] += wl[i];
      else if (noise_on)
        for (int i = 0; i < 3; ++i) x[i] += F[i * 3] * z[4] + F[i * 3 + 1] * z[5] + F[i * 3 + 2] * z[6];
    }
    double mu[8], cv[16];
    moments(xs, M, buf, mu, cv);
    if (in->mom_out) {
      double *mo = in->mom_out + ((size_t)t * K + k) * 18;
      for (int i = 0; i < 8; ++i) mo[i] = mu[i];
      int q = 8;
      for (int a = 0; a < 4; ++a)
        for (int b = a; b < 4; ++b) mo[q++] = cv[a * 4 + b];
    }
    int ok = 1;
    for (int i = 0; i < 8; ++i) ok &= isfinite(mu[i]);
    for (int i = 0; i < 16; ++i) ok &= isfinite(cv[i]);
    ok = ok && (1.0 - curv(p, mu[7]) * mu[6]) > 0.0;
    for (int i = 0; i < 8; ++i) mean[i] = isfinite(mu[i]) ? mu[i] : 0.0;
    for (int i = 0; i < 16; ++i) cov[i] = isfinite(cv[i]) ? cv[i] : 0.0;
    dead |= !ok;
    h_prev = h_cur;
    h_cur = dcbf(p, mean[6], sqrt(fmax(cov[15], 0.0)));
    if (p->n_obstacles) {
      ho_prev = ho_cur;
      ho_cur = obstacle_terms(p, mean[7], mean[6], sqrt(fmax(cov[15], 0.0)), &inside);
    }
  }
  total += p->terminal_scale * stage(p, mean);
  if (shield) total += pen(p, h_cur, h_prev);
  if (p->n_obstacles) {
    total += p->terminal_scale * (inside ? p->obstacle_penalty : 0.0);
    if (shield) total += pen(p, ho_cur, ho_prev);
  }
  return dead ? INFINITY : total;
}

/* Rollout costs for the context's k-range.  Noise arrays override Philox.
 * mom_out (nullable): the per-step belief moments, (T, k_count, 18). */
int orc_rollout_moments(const bssmppi_problem *p, const double *x0, const double *cov0, const double *nominal,
                        const double *u_in, const double *eps_in, const double *z_in, const uint32_t key_ctrl[2],
                        const uint32_t key_belief[2], double *costs, double *u_out, double *mom_out,
                        int nthreads) {
  double ph[23];
  memcpy(ph, p->phys, sizeof(ph));
  Ctx c = {p, ph};
  Inputs in;
  memset(&in, 0, sizeof(in));
  in.x0 = x0; in.cov0 = cov0; in.nominal = nominal; in.u_in = u_in; in.eps_in = eps_in; in.z_in = z_in;
  in.philox_ctrl = eps_in == NULL;
  in.philox_belief = z_in == NULL;
  in.mom_out = mom_out;
  if (key_ctrl) { in.kc[0] = key_ctrl[0]; in.kc[1] = key_ctrl[1]; }
  if (key_belief) { in.kb[0] = key_belief[0]; in.kb[1] = key_belief[1]; }
  const int M = p->kind == BSSMPPI_KIND_BSS ? p->inner_samples : 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
  {
    double *xs = (double *)malloc((size_t)M * 8 * sizeof(double));
    double *buf = (double *)malloc((size_t)M * sizeof(double));
#pragma omp for schedule(dynamic, 4)
    for (int k = 0; k < p->k_count; ++k) costs[k] = rollout_one(&c, &in, k, xs, buf, u_out);
    free(xs);
    free(buf);
  }
  return 0;
}

int orc_rollout(const bssmppi_problem *p, const double *x0, const double *cov0, const double *nominal,
                const double *u_in, const double *eps_in, const double *z_in, const uint32_t key_ctrl[2],
                const uint32_t key_belief[2], double *costs, double *u_out, int nthreads) {
  return orc_rollout_moments(p, x0, cov0, nominal, u_in, eps_in, z_in, key_ctrl, key_belief, costs, u_out, NULL,
                             nthreads);
}

/* mppi_weights + mppi_update (controllers.py:180-194).  Returns 3 if no
 * finite cost (AllRolloutsInvalid). */
int orc_update(int K, int T, const double *costs, const double *u, double lam, const double lo[2],
               const double hi[2], double *vplus) {
  double beta = INFINITY;
  int any = 0;
  for (int k = 0; k < K; ++k)
    if (isfinite(costs[k])) { any = 1; if (costs[k] < beta) beta = costs[k]; }
  if (!any) return 3;
  double z = 0.0;
  for (int i = 0; i < 2 * T; ++i) vplus[i] = 0.0;
  for (int k = 0; k < K; ++k) {
    double w = exp(-(costs[k] - beta) / lam);
    z += w;
    for (int i = 0; i < 2 * T; ++i) vplus[i] += w * u[(size_t)k * 2 * T + i];
  }
  for (int i = 0; i < 2 * T; ++i) {
    double v = vplus[i] / z;
    vplus[i] = fmin(fmax(v, (i & 1) ? lo[1] : lo[0]), (i & 1) ? hi[1] : hi[0]);
  }
  return 0;
}

/* Full iteration (Philox noise): rollouts of k-range + update.  u scratch
 * (k_count*T*2) and costs (k_count) are caller-provided. */
int orc_control_step(const bssmppi_problem *p, const double *x0, const double *cov0, const double *plan,
                     const uint32_t key_ctrl[2], const uint32_t key_belief[2], double *costs, double *u,
                     double *vplus, int nthreads) {
  orc_rollout(p, x0, cov0, plan, NULL, NULL, NULL, key_ctrl, key_belief, costs, u, nthreads);
  return orc_update(p->k_count, p->horizon, costs, u, p->temperature, p->bounds_lo, p->bounds_hi, vplus);
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

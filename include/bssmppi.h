/*
 * bssmppi.h -- C ABI of the B200-native BSS-MPPI optimisation step.
 *
 * The reference (arxiv 2408.00494, package `belief_mppi`) is pure Python;
 * its only "FFI" is the Python call surface of `belief_mppi.controllers`.
 * Each entry point below replaces one piece of that surface and is bound
 * from Python with ctypes (paper_2408_00494_b200/_lib.py; INTEGRATION.md
 * shows the stub a maintainer would add to the reference package).
 *
 * Conventions: plain C types only; host pointers unless the name says
 * `_dev`; arrays are C-contiguous row-major; every function returns a
 * bssmppi_status and leaves a message for bssmppi_last_error().  Compute
 * runs on the context's CUDA stream (bssmppi_set_stream), FP32 in the
 * kernels, FP64 in the weighted update.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/belief_mppi):
 *   bssmppi_create            Controller.__init__        controllers.py:353-369
 *                             (+ MppiConfig 71-105, CostSpec 108-138, RolloutContext 197-212)
 *   bssmppi_control_step      Controller.control_step    controllers.py:374-410
 *   bssmppi_step_partials     sample_controls+rollout_bss+mppi_weights, K-shard
 *                             controllers.py:166-177, 252-341, 180-187
 *   bssmppi_update_combine    mppi_update                controllers.py:190-194
 *   bssmppi_rollout           rollout_bss / rollout_smppi / rollout_mppi
 *                             controllers.py:238-258 (+ _rollout 261-341)
 *   bssmppi_mppi_update       mppi_update on a host batch controllers.py:180-194
 *   bssmppi_sample_controls   sample_controls from captured normals controllers.py:166-177
 *   bssmppi_step_array        step_array (Euler)         dynamics.py:550-573
 *   bssmppi_enqueue_iteration device-resident control_step + warm start
 *                             (controllers.py:407-409, ControlPlan.shifted 154-156)
 *   bssmppi_enqueue_step_device control_step on device buffers (torch tensors)
 *                             controllers.py:374-410
 */
#ifndef BSSMPPI_H
#define BSSMPPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSSMPPI_ABI_VERSION 3

typedef enum {
  BSSMPPI_OK = 0,
  BSSMPPI_ERR_INVALID = 1,      /* bad argument (reference: ValueError) */
  BSSMPPI_ERR_CUDA = 2,         /* CUDA runtime failure / no device */
  BSSMPPI_ERR_ALL_INVALID = 3,  /* no finite rollout cost (reference: AllRolloutsInvalid) */
  BSSMPPI_ERR_UNSUPPORTED = 4   /* configuration outside the device path */
} bssmppi_status;

enum { BSSMPPI_KIND_MPPI = 0, BSSMPPI_KIND_SMPPI = 1, BSSMPPI_KIND_BSS = 2 };

/* One controller's constants.  Field groups mirror the reference types. */
typedef struct bssmppi_problem {
  /* MppiConfig (controllers.py:71-105) */
  int32_t kind;                 /* BSSMPPI_KIND_* */
  int32_t samples;              /* K (global, all shards) */
  int32_t horizon;              /* T (<= 512) */
  int32_t inner_samples;        /* M (bss only; 2..8192) */
  int32_t persist_particles;    /* controllers.py:83; the cloud lives in shared
                                   memory, so M <= 1792 (else UNSUPPORTED) */
  double temperature;           /* lambda */
  double control_cost_weight;   /* gamma */
  double sigma_factor[4];       /* psd_factor(sigma_eps), 2x2 row-major */
  double precision[4];          /* pinv(sigma_eps), 2x2 row-major */
  double bounds_lo[2];          /* ControlBounds.lower */
  double bounds_hi[2];          /* ControlBounds.upper */
  /* CostSpec (controllers.py:108-138) + SafetyParams (constraints.py:22-33) */
  double q_diag[8];
  double v_goal;
  double obstacle_penalty;
  double terminal_scale;
  double cbf_rate;              /* beta */
  double penalty;               /* C */
  double backoff;               /* nu */
  /* VehicleParams: _phys_vector order (dynamics.py:325-337), Euler dt */
  double phys[23];
  double dt;
  /* NoiseModel.factor (dynamics.py:276-300), 3x3 row-major, channels (vx, vy, r) */
  double noise_factor[9];
  /* Track (dynamics.py:152-196); tables are copied at create time */
  const double *track_s;
  const double *track_kappa;
  int32_t track_n;
  double track_length;
  double half_width;
  int32_t track_closed;
  /* K-shard owned by this context: global k in [k_begin, k_begin + k_count) */
  int32_t k_begin;
  int32_t k_count;
  /* ---- Extensions BEYOND the reference (BASELINE config 4); zero = off.
   * The reference has only Gaussian noise (dynamics.py:289-290) and only the
   * track DCBF in its rollouts (controllers.py:293); see obstacles.py. */
  int32_t noise_kind;            /* 0: Gaussian via noise_factor; 1: Laplace(laplace_scale) on
                                    (vx, vy, r) + U(-slip_bias, slip_bias) on vy (Philox only) */
  double laplace_scale;
  double slip_bias;
  int32_t n_obstacles;           /* <= 64 */
  const double *obstacles;       /* n x 3: centre x, y, radius (global frame) */
  double obstacle_backoff;       /* nu of each obstacle chance constraint (heuristic_h_i) */
  const double *centerline;      /* rows x 3: x, y, theta at s = i * centerline_ds */
  int32_t centerline_n;
  double centerline_ds;
  /* ---- Launch shape (not a reference parameter): lanes per rollout of the
   * bss kernel, 0 = the measured policy (bssmppi_group_width), else 2, 4, 8,
   * 16 or 32 -- lets the parity tests pin the production widths. */
  int32_t group_width;
} bssmppi_problem;

/* Diagnostics of one iteration (the reference returns none; north_star asks). */
typedef struct bssmppi_diag {
  double cost_min;          /* min finite rollout cost (the update baseline) */
  int64_t cost_argmin;      /* global k of cost_min */
  int64_t n_finite;         /* rollouts with finite cost */
  double weight_sum;        /* sum_k exp(-(S_k - min S)/lambda) */
  double ess;               /* (sum w)^2 / sum w^2 */
  float device_ms;          /* CUDA-event time of the last enqueued iteration */
  float rollout_ms;         /* ... of which the fused rollout kernel */
} bssmppi_diag;

const char *bssmppi_last_error(void);
int32_t bssmppi_abi_version(void);
/* Size of one K-shard partial record: 5 + 2*horizon doubles. */
int32_t bssmppi_partial_len(int32_t horizon);
/* Lanes per rollout the bss kernel uses for (M, local rollout count). */
int32_t bssmppi_group_width(int32_t inner_samples, int32_t k_count);

typedef struct bssmppi_ctx bssmppi_ctx;
/* The bss kernel's launch shape for this context: lanes per rollout (1 for
 * the deterministic kinds) and threads per block, as the next launch will
 * use them (policy, problem.group_width, BSSMPPI_FORCE_BLOCK). */
int32_t bssmppi_launch_shape(const bssmppi_ctx *ctx, int32_t *group_width, int32_t *block_threads);

int bssmppi_create(const bssmppi_problem *problem, int32_t device, bssmppi_ctx **out);
void bssmppi_destroy(bssmppi_ctx *ctx);
/* Stream for all subsequent work (cudaStream_t as void*; NULL = legacy default). */
int bssmppi_set_stream(bssmppi_ctx *ctx, void *cuda_stream);

/* One receding-horizon iteration with host buffers (controllers.py:374-410).
 *   x0[8], cov0[16] (nullable => zero), plan[T*2] nominal.
 *   Noise: eps (K*T*2 post-factor perturbations) and z (T*K*M*7 standard
 *   normals, float) given => oracle-noise mode, consumed exactly like the
 *   reference; both NULL => device Philox4x32 keyed by key_ctrl / key_belief.
 *   Output vplus[T*2] (the optimised sequence before the warm-start shift). */
int bssmppi_control_step(bssmppi_ctx *ctx, const double *x0, const double *cov0,
                         const double *plan, const uint32_t key_ctrl[2],
                         const uint32_t key_belief[2], const double *eps, const float *z,
                         double *vplus, bssmppi_diag *diag);

/* K-sharded variant: rollouts of this context's k-range and the weighted
 * partial record written into partials_dev[slot * partial_len ...]
 * (device memory, e.g. a torch tensor later all-reduced over NCCL).
 * eps/z, if given, cover only the local k-range. */
int bssmppi_step_partials(bssmppi_ctx *ctx, const double *x0, const double *cov0,
                          const double *plan, const uint32_t key_ctrl[2],
                          const uint32_t key_belief[2], const double *eps, const float *z,
                          double *partials_dev, int32_t slot);
/* Combine nslots partial records (rank order) -> clamp(v+) (mppi_update). */
int bssmppi_update_combine(bssmppi_ctx *ctx, const double *partials_dev, int32_t nslots,
                           double *vplus, bssmppi_diag *diag);

/* Device-resident loop for throughput measurement: uses the x0/cov0/plan
 * last uploaded with bssmppi_upload_state, runs one full iteration and
 * shifts v+ into the device plan (warm start).  Asynchronous. */
int bssmppi_upload_state(bssmppi_ctx *ctx, const double *x0, const double *cov0,
                         const double *plan);
int bssmppi_enqueue_iteration(bssmppi_ctx *ctx, const uint32_t key_ctrl[2],
                              const uint32_t key_belief[2]);
/* Device-resident K-shard iteration: partial record into partials_dev[slot]
 * (asynchronous), and the asynchronous combine of nslots records into v+
 * with the warm-start shift of the device plan. */
int bssmppi_enqueue_partials(bssmppi_ctx *ctx, const uint32_t key_ctrl[2],
                             const uint32_t key_belief[2], double *partials_dev, int32_t slot);
int bssmppi_enqueue_combine(bssmppi_ctx *ctx, const double *partials_dev, int32_t nslots);
/* Synchronise and read the last iteration's v+ (nullable) and diagnostics. */
int bssmppi_download(bssmppi_ctx *ctx, double *vplus, bssmppi_diag *diag);

/* One iteration on device buffers, for callers that keep the state on the
 * GPU (e.g. torch CUDA tensors, with bssmppi_set_stream to torch's stream):
 * state_dev = float x0[8] | cov0[16] (row-major 4x4) | plan[2T];
 * out_dev   = double v+[2T] | head[5] {cost_min, Z, Z2, n_finite, argmin}.
 * Asynchronous on the context stream: no host copies or synchronisation.
 * n_finite == 0 in the head is the AllRolloutsInvalid case; state_dev is
 * not modified (the caller does the warm-start shift). */
int bssmppi_enqueue_step_device(bssmppi_ctx *ctx, const float *state_dev, const uint32_t key_ctrl[2],
                                const uint32_t key_belief[2], double *out_dev);

/* Rollout costs of a given sampled batch (rollout_bss / rollout_smppi /
 * rollout_mppi): u, eps (K*T*2, clamped / raw), nominal (T*2).
 * z (T*K*M*7 float) or NULL => Philox keyed by key_belief.
 * costs[K] out (+inf marks dead rollouts).  moments (nullable) receives the
 * raw per-step belief moments, (T, K, 18) float: mean[8] then the upper
 * triangle of the 4x4 covariance (00,01,02,03,11,12,13,22,23,33). */
int bssmppi_rollout(bssmppi_ctx *ctx, const double *x0, const double *cov0, const double *u,
                    const double *eps, const double *nominal, const float *z,
                    const uint32_t key_belief[2], double *costs, float *moments);

/* Context-free FP64 update law on a host batch (mppi_update). */
int bssmppi_mppi_update(int32_t K, int32_t T, const double *costs, const double *controls,
                        double temperature, const double lo[2], const double hi[2],
                        double *vplus, bssmppi_diag *diag);

/* sample_controls from captured normals: eps = z F^T, u = clip(nominal + eps).
 * z, eps, u: n*T*2; nominal T*2. */
int bssmppi_sample_controls(int32_t n, int32_t T, const double *z, const double factor[4],
                            const double *nominal, const double lo[2], const double hi[2],
                            double *eps, double *u);

/* Batched Euler step on the context's vehicle/track (step_array):
 * x (n*8), u (n*2), w (n*3 or NULL) -> x_out (n*8), ok (n). */
int bssmppi_step_array(bssmppi_ctx *ctx, int32_t n, const double *x, const double *u,
                       const double *w, double *x_out, uint8_t *ok);

/* Test hooks for the device generator: the Philox4x32 block function
 * (rounds = 10, the control stream, or 7, the belief stream) and the
 * per-particle-step normals the rollout consumes in Philox mode. */
int bssmppi_philox4x32(const uint32_t ctr[4], const uint32_t key[2], int32_t rounds,
                       uint32_t out[4]);
int bssmppi_belief_normals(const uint32_t key[2], int32_t t, int32_t k, int32_t m_count,
                           float *out /* m_count*7 */);

/* The lateral tire table the kernels evaluate sin(C atan(B alpha)) from
 * (host-side, no device work; the context builds the same table):
 * bc = {B_front, C_front, B_rear, C_rear}, steer_max = max |steering bound|.
 * Writes 2 * rows float4 rows {c0, c1, c2, c3} (front, then rear) into out
 * (capacity cap rows), rows per axle, cells per radian and the domain end.
 * Returns BSSMPPI_ERR_INVALID if cap is too small. */
int bssmppi_tire_table(const double bc[4], double steer_max, float *out, int32_t cap,
                       int32_t *rows, double *cells_per_rad, double *amax);

/* Per-iteration device-noise key: Philox4x32-10 of (iteration, domain) under
 * the controller's base key (host-side, no device work). */
int bssmppi_iteration_key(const uint32_t base[2], uint32_t domain, uint64_t iteration,
                          uint32_t out[2]);

/* Measured FP32 FFMA throughput of the device (roofline denominator). */
int bssmppi_ffma_peak(int32_t device, double *tflops);

/* Measured MUFU (XU pipe, ex2.approx) throughput of the device in Tera
 * ops/s: the denominator of the transcendental (SFU) roofline. */
int bssmppi_mufu_peak(int32_t device, double *tops);

#ifdef __cplusplus
}
#endif
#endif /* BSSMPPI_H */

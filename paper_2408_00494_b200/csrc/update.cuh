// Information-theoretic update (controllers.py:180-194):
//   w_k = exp(-(S_k - min_finite S) / lambda),  v+ = clip(sum_k w_k u_k / sum_k w_k)
// as a two-level, fixed-order (deterministic) reduction in FP64:
//   1. update_partials_kernel: each block owns a contiguous k-chunk and emits
//      a record {beta_b, Z_b, Z2_b, n_b, argmin_b, N_b[2T]} with weights
//      relative to its OWN minimum beta_b (one pass over u, no global min);
//   2. combine_kernel: rescales records by exp(-(beta_b - beta)/lambda) and
//      sums them in record order.  The same kernel combines K-shard records
//      of several GPUs after one NCCL all-reduce, so a
//      sharded iteration equals the single-GPU one up to FP64 rounding.
#pragma once
#include <cstdint>

namespace bss {

constexpr int kRecHead = 5;   // beta, Z, Z2, n_finite, argmin
constexpr int kUpdThreads = 256;
constexpr int kCombThreads = 512;     // combine_kernel: more loads in flight for the column pass
constexpr int kCombineSlices = 16;    // record slices per column in combine_kernel
constexpr int kCombinePart = 2048;    // slice partials held in shared memory (16 KB)

__device__ __forceinline__ double to_d(float v) { return (double)v; }
__device__ __forceinline__ double to_d(double v) { return v; }

template <typename CT, typename UT>
__global__ void __launch_bounds__(kUpdThreads)
update_partials_kernel(int n, int k_begin, int T2, const CT *costs, const UT *u, double lam,
                       int chunk, double *rec) {
  __shared__ double s_min[kUpdThreads];
  __shared__ long long s_arg[kUpdThreads];
  __shared__ double s_cnt[kUpdThreads];
  __shared__ double s_w[kUpdThreads];
  __shared__ double s_z[kUpdThreads], s_z2[kUpdThreads];
  const int tid = threadIdx.x;
  const int k0 = blockIdx.x * chunk;
  const int k1 = min(n, k0 + chunk);
  double *out = rec + (size_t)blockIdx.x * (kRecHead + T2);
  // pass 1: block min over finite costs (ties -> smallest k), finite count
  double mn = __longlong_as_double(0x7ff0000000000000ll);
  long long arg = -1;
  double cnt = 0.0;
  for (int k = k0 + tid; k < k1; k += kUpdThreads) {
    const double c = to_d(costs[k]);
    if (isfinite(c)) {
      cnt += 1.0;
      if (c < mn) { mn = c; arg = k; }
    }
  }
  s_min[tid] = mn; s_arg[tid] = arg; s_cnt[tid] = cnt;
  __syncthreads();
  for (int s = kUpdThreads / 2; s > 0; s >>= 1) {
    if (tid < s) {
      const double a = s_min[tid], b = s_min[tid + s];
      const long long ia = s_arg[tid], ib = s_arg[tid + s];
      if (b < a || (b == a && ib >= 0 && (ia < 0 || ib < ia))) { s_min[tid] = b; s_arg[tid] = ib; }
      s_cnt[tid] += s_cnt[tid + s];
    }
    __syncthreads();
  }
  const double beta = s_min[0];
  const bool any = s_cnt[0] > 0.0;
  // pass 2: weights relative to beta_b, fixed-order sums
  double z = 0.0, z2 = 0.0;
  double nacc[4] = {0.0, 0.0, 0.0, 0.0};   // columns tid, tid+256, ... (2T <= 1024)
  for (int base = k0; base < k1; base += kUpdThreads) {
    __syncthreads();
    const int k = base + tid;
    double w = 0.0;
    if (k < k1 && any) {
      const double c = to_d(costs[k]);
      w = isfinite(c) ? exp(-(c - beta) / lam) : 0.0;
    }
    s_w[tid] = w;
    z += w;
    z2 += w * w;
    __syncthreads();
    const int cnt_k = min(kUpdThreads, k1 - base);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = tid + j * kUpdThreads;
      if (col < T2) {
        // 16 loads in flight per thread (each is an L2 round trip)
        double a = nacc[j];
        const UT *up = u + (size_t)base * T2 + col;
#pragma unroll 16
        for (int i = 0; i < cnt_k; ++i) a = fma(s_w[i], to_d(up[(size_t)i * T2]), a);
        nacc[j] = a;
      }
    }
  }
  s_z[tid] = z;
  s_z2[tid] = z2;
  __syncthreads();
  for (int s = kUpdThreads / 2; s > 0; s >>= 1) {
    if (tid < s) { s_z[tid] += s_z[tid + s]; s_z2[tid] += s_z2[tid + s]; }
    __syncthreads();
  }
  if (tid == 0) {
    out[0] = beta;
    out[1] = s_z[0];
    out[2] = s_z2[0];
    out[3] = s_cnt[0];
    out[4] = (double)(s_arg[0] < 0 ? -1 : s_arg[0] + k_begin);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int col = tid + j * kUpdThreads;
    if (col < T2) out[kRecHead + col] = nacc[j];
  }
}

// Combine `nrec` records (<= 1024), block-parallel and in a fixed order
// (deterministic).  final == 0: write one record to rec_out.  final == 1:
// v+ = clip(N/Z) -> vplus (double), warm-start shifted plan
// (ControlPlan.shifted, controllers.py:154-156) -> plan_out (float, may be
// null), head {beta, Z, Z2, n, argmin} -> head_out; v+ and head also to
// `mirror` (host-mapped pinned memory, may be null) so the host reads the
// result after the stream sync without a separate device-to-host copy.
__global__ void __launch_bounds__(kCombThreads)
combine_kernel(int nrec, int T2, const double *rec, double lam, int final_, double *rec_out,
               double lo0, double lo1, double hi0, double hi1, double *vplus, float *plan_out,
               double *head_out, double *mirror) {
  __shared__ double s_scale[1024];
  __shared__ double s_part[kCombinePart];
  __shared__ double s_a[kCombThreads], s_b[kCombThreads], s_c[kCombThreads];
  __shared__ long long s_i[kCombThreads];
  __shared__ double s_head[kRecHead];
  const int tid = threadIdx.x;
  const int R = kRecHead + T2;
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  // 1. global minimum (ties -> smallest k) and finite count
  double mn = INF, cnt = 0.0;
  long long arg = -1;
  for (int r = tid; r < nrec; r += kCombThreads) {
    const double *h = rec + (size_t)r * R;
    if (h[3] > 0.0) {
      cnt += h[3];
      const long long a = (long long)h[4];
      if (h[0] < mn || (h[0] == mn && (arg < 0 || a < arg))) { mn = h[0]; arg = a; }
    }
  }
  s_a[tid] = mn; s_i[tid] = arg; s_c[tid] = cnt;
  __syncthreads();
  for (int s = kCombThreads / 2; s > 0; s >>= 1) {
    if (tid < s) {
      const double a = s_a[tid], b = s_a[tid + s];
      const long long ia = s_i[tid], ib = s_i[tid + s];
      if (b < a || (b == a && ib >= 0 && (ia < 0 || ib < ia))) { s_a[tid] = b; s_i[tid] = ib; }
      s_c[tid] += s_c[tid + s];
    }
    __syncthreads();
  }
  const double beta = s_a[0];
  const long long argmin = s_i[0];
  const double n = s_c[0];
  __syncthreads();
  // 2. rescale factors exp(-(beta_r - beta)/lambda); Z, Z2
  double z = 0.0, z2 = 0.0;
  for (int r = tid; r < nrec; r += kCombThreads) {
    const double *h = rec + (size_t)r * R;
    const double sc = (h[3] > 0.0) ? exp(-(h[0] - beta) / lam) : 0.0;
    s_scale[r] = sc;
    z += sc * h[1];
    z2 += sc * sc * h[2];
  }
  s_a[tid] = z; s_b[tid] = z2;
  __syncthreads();
  for (int s = kCombThreads / 2; s > 0; s >>= 1) {
    if (tid < s) { s_a[tid] += s_a[tid + s]; s_b[tid] += s_b[tid + s]; }
    __syncthreads();
  }
  if (tid == 0) {
    s_head[0] = beta; s_head[1] = s_a[0]; s_head[2] = s_b[0]; s_head[3] = n;
    s_head[4] = (double)argmin;
  }
  __syncthreads();
  // 3. N[col] = sum_r scale_r N_r[col] (records with n_r = 0 carry N_r = 0):
  //    (column, record-slice) items over all threads -- consecutive threads
  //    read consecutive columns of one record -- then the slice partials are
  //    summed in slice order (fixed order: deterministic).
  const int ns = max(1, min(kCombineSlices, min(kCombinePart / T2, nrec)));
  const int per = (nrec + ns - 1) / ns;
  for (int it = tid; it < ns * T2; it += kCombThreads) {
    const int col = it % T2, sl = it / T2;
    const int r0 = sl * per, r1 = min(nrec, r0 + per);
    const double *src = rec + kRecHead + col;
    double a = 0.0;
#pragma unroll 16
    for (int r = r0; r < r1; ++r) a = fma(s_scale[r], src[(size_t)r * R], a);
    s_part[it] = a;
  }
  __syncthreads();
  for (int col = tid; col < T2; col += kCombThreads) {
    double a = 0.0;
    for (int sl = 0; sl < ns; ++sl) a += s_part[sl * T2 + col];
    if (!final_) {
      rec_out[kRecHead + col] = a;
    } else {
      // no finite rollout (AllRolloutsInvalid): v+ is NaN, never a clamped 0/0
      const double v = a / s_head[1];
      const double l = (col & 1) ? lo1 : lo0, h = (col & 1) ? hi1 : hi0;
      vplus[col] = s_head[3] > 0.0 ? fmin(fmax(v, l), h) : __longlong_as_double(0x7ff8000000000000ll);
      if (mirror != nullptr) mirror[col] = vplus[col];
    }
  }
  if (tid < kRecHead) {
    if (!final_) {
      rec_out[tid] = s_head[tid];
    } else {
      head_out[tid] = s_head[tid];
      if (mirror != nullptr) mirror[T2 + tid] = s_head[tid];
    }
  }
  // AllRolloutsInvalid leaves the warm start untouched (the reference raises
  // before replacing the plan, controllers.py:183-185, 407-409)
  if (final_ && plan_out != nullptr && s_head[3] > 0.0) {
    __syncthreads();
    for (int col = tid; col < T2; col += kCombThreads) {
      const int src = (col + 2 < T2) ? col + 2 : col;   // drop first, repeat last
      plan_out[col] = (float)vplus[src];
    }
  }
}

// Small-K update in ONE launch (K <= kSmallK, single context, final v+):
// the same weights, sums and outputs as update_partials_kernel +
// combine_kernel(final = 1) with one record, without the second launch and
// the record round trip -- the update is latency-bound at small K (C1, C2,
// closed-loop control).  Fixed-order reductions (deterministic).
constexpr int kSmallK = 1024;   // at K = 2048 the two-level update was already faster (A/B)

__global__ void __launch_bounds__(kCombThreads)
update_small_kernel(int n, int k_begin, int T2, const float *costs, const float *u, double lam, double lo0,
                    double lo1, double hi0, double hi1, double *vplus, float *plan_out, double *head_out,
                    double *mirror) {
  __shared__ double s_w[kSmallK];
  __shared__ double s_part[kCombinePart];   // also the reduction scratch of steps 1-2
  __shared__ double s_head[kRecHead];
  static_assert(4 * kCombThreads <= kCombinePart, "reduction scratch must fit s_part");
  double *s_a = s_part, *s_b = s_part + kCombThreads, *s_c = s_part + 2 * kCombThreads;
  long long *s_i = reinterpret_cast<long long *>(s_part + 3 * kCombThreads);
  const int tid = threadIdx.x;
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  // 1. minimum over finite costs (ties -> smallest k), finite count
  double mn = INF, cnt = 0.0;
  long long arg = -1;
  for (int k = tid; k < n; k += kCombThreads) {
    const double c = (double)costs[k];
    if (isfinite(c)) {
      cnt += 1.0;
      if (c < mn) { mn = c; arg = k; }
    }
  }
  s_a[tid] = mn; s_i[tid] = arg; s_c[tid] = cnt;
  __syncthreads();
  for (int s = kCombThreads / 2; s > 0; s >>= 1) {
    if (tid < s) {
      const double a = s_a[tid], b = s_a[tid + s];
      const long long ia = s_i[tid], ib = s_i[tid + s];
      if (b < a || (b == a && ib >= 0 && (ia < 0 || ib < ia))) { s_a[tid] = b; s_i[tid] = ib; }
      s_c[tid] += s_c[tid + s];
    }
    __syncthreads();
  }
  const double beta = s_a[0];
  const long long argmin = s_i[0];
  const double nfin = s_c[0];
  __syncthreads();
  // 2. weights w_k = exp(-(S_k - beta) / lambda) (controllers.py:180-187); Z, Z2
  double z = 0.0, z2 = 0.0;
  for (int k = tid; k < n; k += kCombThreads) {
    const double c = (double)costs[k];
    const double w = (nfin > 0.0 && isfinite(c)) ? exp(-(c - beta) / lam) : 0.0;
    s_w[k] = w;
    z += w;
    z2 += w * w;
  }
  s_a[tid] = z; s_b[tid] = z2;
  __syncthreads();
  for (int s = kCombThreads / 2; s > 0; s >>= 1) {
    if (tid < s) { s_a[tid] += s_a[tid + s]; s_b[tid] += s_b[tid + s]; }
    __syncthreads();
  }
  if (tid == 0) {
    s_head[0] = beta; s_head[1] = s_a[0]; s_head[2] = s_b[0]; s_head[3] = nfin;
    s_head[4] = (double)(argmin < 0 ? -1 : argmin + k_begin);
  }
  __syncthreads();
  // 3. N[col] = sum_k w_k u_k[col] (controllers.py:190-194): (column,
  //    k-slice) items over all threads, slice partials summed in slice order
  const int ns = max(1, min(kCombineSlices, min(kCombinePart / T2, n)));
  const int per = (n + ns - 1) / ns;
  for (int it = tid; it < ns * T2; it += kCombThreads) {
    const int col = it % T2, sl = it / T2;
    const int k0 = sl * per, k1 = min(n, k0 + per);
    const float *src = u + col;
    double a = 0.0;
#pragma unroll 16
    for (int k = k0; k < k1; ++k) a = fma(s_w[k], (double)src[(size_t)k * T2], a);
    s_part[it] = a;
  }
  __syncthreads();
  // 4. v+ = clip(N / Z); head; warm-start shifted plan (controllers.py:154-156)
  for (int col = tid; col < T2; col += kCombThreads) {
    double a = 0.0;
    for (int sl = 0; sl < ns; ++sl) a += s_part[sl * T2 + col];
    const double v = a / s_head[1];
    const double l = (col & 1) ? lo1 : lo0, h = (col & 1) ? hi1 : hi0;
    vplus[col] = nfin > 0.0 ? fmin(fmax(v, l), h) : __longlong_as_double(0x7ff8000000000000ll);
    if (mirror != nullptr) mirror[col] = vplus[col];
  }
  if (tid < kRecHead) {
    head_out[tid] = s_head[tid];
    if (mirror != nullptr) mirror[T2 + tid] = s_head[tid];
  }
  if (plan_out != nullptr && nfin > 0.0) {   // AllRolloutsInvalid: plan untouched
    __syncthreads();
    for (int col = tid; col < T2; col += kCombThreads) {
      const int src = (col + 2 < T2) ? col + 2 : col;   // drop first, repeat last
      plan_out[col] = (float)vplus[src];
    }
  }
}

}  // namespace bss

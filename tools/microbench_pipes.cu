// FMA-pipe sharing on sm_100a: do IMAD.WIDE (the Philox multiply), FFMA2
// and scalar FFMA compete for the same issue/pipe cycles?  Each kernel runs
// independent chains per thread (no latency bound) and reports warp-
// instructions per clock per SMSP for its mix.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench_pipes.cu -o /tmp/pipes && /tmp/pipes
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8

__device__ __forceinline__ void imad_wide(uint32_t &a, uint32_t &b) {
  uint64_t p;
  asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(0xD2511F53u));
  a = (uint32_t)(p >> 32) ^ b;
  b = (uint32_t)p;
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// NW IMAD.WIDE, NF2 FFMA2, NF scalar FFMA, ND DFMA (+ one F2F.F64.F32 per
// DFMA when CVT) per chain and round
template <int NW, int NF2, int NF, int ND = 0, bool CVT = false>
__global__ void __launch_bounds__(256) mix(float *out, int iters, float k) {
  uint32_t a[CHAINS], b[CHAINS];
  float2 x[CHAINS];
  float y[CHAINS];
  double dd[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) {
    a[i] = threadIdx.x * 7919u + i;
    b[i] = threadIdx.x ^ (i * 131u);
    x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 1e-3f);
    y[i] = threadIdx.x * 1e-4f + i;
    dd[i] = threadIdx.x * 1e-5 + i;
  }
  const float2 c1 = make_float2(0.999f, 0.998f), c0 = make_float2(1e-3f, 2e-3f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
#pragma unroll
      for (int j = 0; j < NW; ++j) imad_wide(a[i], b[i]);
#pragma unroll
      for (int j = 0; j < NF2; ++j) x[i] = ffma2(x[i], c1, c0);
#pragma unroll
      for (int j = 0; j < NF; ++j) y[i] = fmaf(y[i], k, 1e-3f);
#pragma unroll
      for (int j = 0; j < ND; ++j) dd[i] = fma(CVT ? (double)y[i] : (double)k, 0.999, dd[i]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += (float)(a[i] ^ b[i]) + x[i].x + x[i].y + y[i] + (float)dd[i];
  if (s == 12345.678f) out[0] = s;
}

template <int NW, int NF2, int NF, int ND = 0, bool CVT = false>
void run(const char *name, float *d) {
  const int blocks = 148 * 8, threads = 256, iters = 2048;
  mix<NW, NF2, NF, ND, CVT><<<blocks, threads>>>(d, 16, 0.999f);   // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<NW, NF2, NF, ND, CVT><<<blocks, threads>>>(d, iters, 0.999f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double cycles = ms * 1e-3 * clk_khz * 1e3;
  const double warp_inst = (double)blocks * (threads / 32) * iters * CHAINS * (NW + NF2 + NF + ND * (CVT ? 2 : 1));
  const double per_smsp = warp_inst / (148.0 * 4.0) / cycles;
  // pipe-cycle model: IMAD.WIDE 4, FFMA2 2, FFMA 1 cycle of one shared FMA pipe
  const double model = (double)blocks * (threads / 32) * iters * CHAINS * (4.0 * NW + 2.0 * NF2 + NF) / (148.0 * 4.0);
  printf("%-28s %.3f ms  %.3f warp-inst/clk/SMSP  shared-pipe model busy %.0f%%\n", name, ms, per_smsp,
         100.0 * model / cycles);
}

int main() {
  float *d;
  cudaMalloc(&d, 4);
  run<1, 0, 0>("IMAD.WIDE only", d);
  run<0, 1, 0>("FFMA2 only", d);
  run<0, 0, 1>("FFMA only", d);
  run<1, 2, 0>("1 IMAD.WIDE : 2 FFMA2", d);
  run<1, 4, 0>("1 IMAD.WIDE : 4 FFMA2", d);
  run<1, 0, 4>("1 IMAD.WIDE : 4 FFMA", d);
  run<1, 0, 8>("1 IMAD.WIDE : 8 FFMA", d);
  run<0, 1, 2>("1 FFMA2 : 2 FFMA", d);
  run<1, 2, 4>("1 IMAD.WIDE : 2 FFMA2 : 4 FFMA", d);
  run<0, 0, 0, 1>("DFMA only", d);
  run<0, 0, 0, 1, true>("F2F.F64 + DFMA only", d);
  run<1, 0, 4, 2>("1 IMAD.WIDE : 4 FFMA : 2 DFMA", d);
  run<1, 0, 4, 2, true>("1 IMAD.WIDE : 4 FFMA : 2 (F2F + DFMA)", d);
  cudaFree(d);
  return 0;
}

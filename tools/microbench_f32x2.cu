// Packed FP32x2 (FFMA2/FMUL2/FADD2, sm_100a) vs scalar FFMA throughput.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench_f32x2.cu -o /tmp/f2bench && /tmp/f2bench
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void __launch_bounds__(256) ffma_scalar(float *out, int iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], a, b);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345.678f) out[0] = s;
}

template <int CH>
__global__ void __launch_bounds__(256) ffma_packed(float *out, int iters, float a, float b) {
  float2 x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, threadIdx.x * 2e-3f + i);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b * 0.5f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < CH; ++i) x[i] = __ffma2_rn(x[i], a2, b2);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i].x + x[i].y;
  if (s == 12345.678f) out[0] = s;
}

// packed chains with register (not uniform) operands that differ per lane
template <int CH>
__global__ void __launch_bounds__(256) ffma_packed_reg(float *out, int iters, float a) {
  float2 x[CH], m[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    x[i] = make_float2(threadIdx.x * 1e-3f + i, threadIdx.x * 2e-3f + i);
    m[i] = make_float2(a + threadIdx.x * 1e-9f, a - i * 1e-9f);
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < CH; ++i) x[i] = __ffma2_rn(x[i], m[i], m[(i + 1) % CH]);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i].x + x[i].y;
  if (s == 12345.678f) out[0] = s;
}

template <class F>
double run(F launch, double flop) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch(16);
  cudaEventRecord(e0);
  launch(2048);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return flop * 2048 / (ms * 1e-3) / 1e12;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *d;
  cudaMalloc(&d, 4);
  const int blocks = sms * 8;
  const double per_iter = 2.0 * 16 * blocks * 256;   // FLOP per (lane-chain, iter)
  printf("scalar FFMA  8 chains: %.1f TFLOP/s\n",
         run([&](int it) { ffma_scalar<8><<<blocks, 256>>>(d, it, 0.999f, 1e-3f); }, per_iter * 8));
  printf("scalar FFMA 16 chains: %.1f TFLOP/s\n",
         run([&](int it) { ffma_scalar<16><<<blocks, 256>>>(d, it, 0.999f, 1e-3f); }, per_iter * 16));
  printf("FFMA2 4 chains (8 lanes): %.1f TFLOP/s\n",
         run([&](int it) { ffma_packed<4><<<blocks, 256>>>(d, it, 0.999f, 1e-3f); }, per_iter * 8));
  printf("FFMA2 8 chains (16 lanes): %.1f TFLOP/s\n",
         run([&](int it) { ffma_packed<8><<<blocks, 256>>>(d, it, 0.999f, 1e-3f); }, per_iter * 16));
  printf("FFMA2 8 chains, register operands: %.1f TFLOP/s\n",
         run([&](int it) { ffma_packed_reg<8><<<blocks, 256>>>(d, it, 0.999f); }, per_iter * 16));
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}

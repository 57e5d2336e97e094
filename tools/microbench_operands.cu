// FP32 pipe throughput by operand form (sm_100a): does an FFMA/FMUL/FADD
// with all-register operands issue at the same rate as immediate /
// constant-bank forms?  8 independent chains per thread.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench_operands.cu -o /tmp/opbench && /tmp/opbench
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float kC[2] = {0.999f, 1e-3f};

// x = x * a + b, a/b immediates
__global__ void __launch_bounds__(256) ffma_imm(float *out, int iters) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], 0.999f, 1e-3f);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678f) out[0] = s;
}

// x = x * y + w, all three distinct per-thread registers
__global__ void __launch_bounds__(256) ffma_reg(float *out, int iters, float a) {
  float x[8], y[8], w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = threadIdx.x * 1e-3f + i;
    y[i] = a - threadIdx.x * 1e-9f - i * 1e-8f;
    w[i] = 1e-3f + threadIdx.x * 1e-9f + i * 1e-8f;
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], y[i], w[i]);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + y[i] + w[i];
  if (s == 12345.678f) out[0] = s;
}

// x = x * c + w: constant-bank multiplier, register addend
__global__ void __launch_bounds__(256) ffma_const(float *out, int iters) {
  float x[8], w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = threadIdx.x * 1e-3f + i;
    w[i] = 1e-3f + threadIdx.x * 1e-9f + i * 1e-8f;
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], kC[0], w[i]);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + w[i];
  if (s == 12345.678f) out[0] = s;
}

// x = x * y (two registers)
__global__ void __launch_bounds__(256) fmul_reg(float *out, int iters, float a) {
  float x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = threadIdx.x * 1e-3f + i;
    y[i] = a + threadIdx.x * 1e-9f + i * 1e-8f;
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = x[i] * y[i];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + y[i];
  if (s == 12345.678f) out[0] = s;
}

// x = x + y (two registers)
__global__ void __launch_bounds__(256) fadd_reg(float *out, int iters, float a) {
  float x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = threadIdx.x * 1e-3f + i;
    y[i] = a + threadIdx.x * 1e-9f + i * 1e-8f;
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = x[i] + y[i];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + y[i];
  if (s == 12345.678f) out[0] = s;
}

// 32x32 -> 64 IMAD.WIDE.U32 (Philox multiply)
__global__ void __launch_bounds__(256) imad_wide(unsigned *out, int iters) {
  unsigned x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7u + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        unsigned long long p;
        asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(x[i]), "r"(0xD2511F53u));
        x[i] = (unsigned)(p >> 32) ^ (unsigned)p;
      }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345u) out[0] = s;
}

// one integer-multiply form per kernel: 0 = mul.wide.u32 (IMAD.WIDE.U32),
// 1 = mul.hi.u32, 2 = mul.lo.u32, 3 = lop3 only (xor with a constant)
template <int FORM>
__global__ void __launch_bounds__(256) imul_form(unsigned *out, int iters) {
  unsigned x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 7u + i; y[i] = threadIdx.x * 3u + i; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (FORM == 0) {
          unsigned long long p;
          asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(x[i]), "r"(0xD2511F53u));
          x[i] = (unsigned)p;
          y[i] += (unsigned)(p >> 32);
        } else if (FORM == 1) {
          asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(x[i]) : "r"(x[i]), "r"(0xD2511F53u));
        } else if (FORM == 2) {
          asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(x[i]) : "r"(x[i]), "r"(0xD2511F53u));
        } else {
          asm volatile("xor.b32 %0, %1, %2;" : "=r"(x[i]) : "r"(x[i]), "r"(0xD2511F53u));
        }
      }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + y[i];
  if (s == 12345u) out[0] = s;
}

template <class F>
double rate(F launch, double ops_per_iter) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch(16);
  cudaEventRecord(e0);
  launch(1024);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ops_per_iter * 1024 / (ms * 1e-3);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *d;
  cudaMalloc(&d, 64);
  const int blocks = sms * 8;
  const double warp_inst = 8.0 * 16 * blocks * 256 / 32;   // warp-instructions per iter
  // report warp-instructions per cycle per SMSP (1.0 = full issue rate)
  const double per = 1.0 / (sms * 4.0 * clk * 1e3);
  printf("FFMA imm,imm      %.2f warp-inst/clk/SMSP\n", per * rate([&](int it) { ffma_imm<<<blocks, 256>>>(d, it); }, warp_inst));
  printf("FFMA reg,reg,reg  %.2f\n", per * rate([&](int it) { ffma_reg<<<blocks, 256>>>(d, it, 0.999f); }, warp_inst));
  printf("FFMA reg,const,reg %.2f\n", per * rate([&](int it) { ffma_const<<<blocks, 256>>>(d, it); }, warp_inst));
  printf("FMUL reg,reg      %.2f\n", per * rate([&](int it) { fmul_reg<<<blocks, 256>>>(d, it, 1.0f); }, warp_inst));
  printf("FADD reg,reg      %.2f\n", per * rate([&](int it) { fadd_reg<<<blocks, 256>>>(d, it, 1e-7f); }, warp_inst));
  printf("IMAD.WIDE + LOP3  %.2f (pairs)\n", per * rate([&](int it) { imad_wide<<<blocks, 256>>>((unsigned *)d, it); }, warp_inst));
  printf("mul.wide.u32 (+IADD) %.2f\n", per * rate([&](int it) { imul_form<0><<<blocks, 256>>>((unsigned *)d, it); }, warp_inst));
  printf("mul.hi.u32        %.2f\n", per * rate([&](int it) { imul_form<1><<<blocks, 256>>>((unsigned *)d, it); }, warp_inst));
  printf("mul.lo.u32        %.2f\n", per * rate([&](int it) { imul_form<2><<<blocks, 256>>>((unsigned *)d, it); }, warp_inst));
  printf("xor (LOP3)        %.2f\n", per * rate([&](int it) { imul_form<3><<<blocks, 256>>>((unsigned *)d, it); }, warp_inst));
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

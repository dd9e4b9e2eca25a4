// Microbenchmark: per-SM throughput of the softmax instruction mix on sm_100a.
// Each kernel runs W warps per SM doing N iterations of 8 independent chains of one op.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 4096
__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__global__ void k_ex2(float *out, float s) {
  long long t0 = clock64();
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = s * (threadIdx.x + i) * 1e-6f;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
  float acc = 0; for (int i = 0; i < 8; ++i) acc += x[i];
  if (acc == 1234.5f) out[0] = acc;
  __syncthreads(); if (blockIdx.x == 0 && threadIdx.x == 0) reinterpret_cast<long long *>(out)[1] = clock64() - t0;
}
__global__ void k_ffma2(float *out, float s) {
  long long t0 = clock64();
  uint64_t x[8]; const uint64_t a = pk(1.0001f, 0.9999f), b = pk(1e-7f, 2e-7f);
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = pk(s + i, s - i);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(a), "l"(b));
  uint64_t acc = 0; for (int i = 0; i < 8; ++i) acc ^= x[i];
  if (acc == 12345) out[0] = 1;
  __syncthreads(); if (blockIdx.x == 0 && threadIdx.x == 0) reinterpret_cast<long long *>(out)[1] = clock64() - t0;
}
__global__ void k_ffma(float *out, float s) {
  long long t0 = clock64();
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = s + i;
  const float a = 1.0001f + s * 1e-9f, b = 1e-7f * s;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(a), "f"(b));
  float acc = 0; for (int i = 0; i < 8; ++i) acc += x[i];
  if (acc == 1234.5f) out[0] = acc;
  __syncthreads(); if (blockIdx.x == 0 && threadIdx.x == 0) reinterpret_cast<long long *>(out)[1] = clock64() - t0;
}
__global__ void k_f2fp(float *out, float s) {
  long long t0 = clock64();
  float x[8]; uint32_t y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = s + i; y[i] = 0; }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y[i]) : "f"(x[i]), "f"(__uint_as_float(y[i])));
    }
  uint32_t acc = 0; for (int i = 0; i < 8; ++i) acc ^= y[i];
  if (acc == 12345) out[0] = 1;
  __syncthreads(); if (blockIdx.x == 0 && threadIdx.x == 0) reinterpret_cast<long long *>(out)[1] = clock64() - t0;
}
__global__ void k_fmnmx3(float *out, float s) {
  long long t0 = clock64();
  float x[8]; const float b = s * 0.5f, c = s * 0.25f;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = s + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(b + it), "f"(c));
  float acc = 0; for (int i = 0; i < 8; ++i) acc += x[i];
  if (acc == 1234.5f) out[0] = acc;
  __syncthreads(); if (blockIdx.x == 0 && threadIdx.x == 0) reinterpret_cast<long long *>(out)[1] = clock64() - t0;
}
__global__ void k_ex2h(float *out, float s) {
  long long t0 = clock64();
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(x[i]) : "f"(s * 1e-3f * i), "f"(-s * 1e-3f * i));
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[i]));
  uint32_t acc = 0; for (int i = 0; i < 8; ++i) acc ^= x[i];
  if (acc == 12345) out[0] = 1;
  __syncthreads(); if (blockIdx.x == 0 && threadIdx.x == 0) reinterpret_cast<long long *>(out)[1] = clock64() - t0;
}
__global__ void k_ex2h1(float *out, float s) {
  long long t0 = clock64();
  unsigned short x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) asm("cvt.rn.f16.f32 %0, %1;" : "=h"(x[i]) : "f"(s * 1e-3f * i));
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16 %0, %0;" : "+h"(x[i]));
  unsigned acc = 0; for (int i = 0; i < 8; ++i) acc ^= x[i];
  if (acc == 12345) out[0] = 1;
  __syncthreads(); if (blockIdx.x == 0 && threadIdx.x == 0) reinterpret_cast<long long *>(out)[1] = clock64() - t0;
}
template <typename K> float run(K k, int warps, const char *name) {
  float *o; cudaMalloc(&o, 64);
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k<<<sms, warps * 32>>>(o, 1.f); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<<<sms, warps * 32>>>(o, 1.f); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double ops = (double)warps * 32 * ITERS * 8;  // lane-ops per SM
  long long c; cudaMemcpy(&c, reinterpret_cast<long long *>(o) + 1, 8, cudaMemcpyDeviceToHost);
  printf("%-8s warps/SM=%2d  %.3f ms  %lld cyc  lane-ops/clk/SM = %.1f  (eff clock %.0f MHz)\n", name, warps, ms, c, ops / c, c / (ms * 1e3));
  cudaFree(o);
  return ms;
}
int main() {
  for (int w : {4, 8, 16}) {
    run(k_ex2h, w, "ex2f16x2");
    run(k_ex2h1, w, "ex2f16");
    run(k_ex2, w, "ex2");
    run(k_ffma, w, "ffma");
    run(k_ffma2, w, "ffma2");
    run(k_f2fp, w, "f2fp");
    run(k_fmnmx3, w, "fmnmx3");
  }
}

// Probe: does a warp issuing tcgen05.mma slow the OTHER warps of its SM sub-partition?
// (tools/pair_trace.py: in the CTA-pair prefix kernel the softmax warps that share a sub-partition
// with the MMA-issuing warp publish P ~600 cycles later per block.)
// One CTA per SM, 4 warps on sub-partitions 0..3 plus warp 4 (sub-partition 0 again):
//   warp 0 (SMSP 0): mode 0 idle; mode 1 issues M=128 N=128 K=16 bf16 MMAs (SS, zero operands)
//                    back to back, a commit + wait every `batch` MMAs; mode 2 the same with a
//                    tcgen05.ld-free loop of UIADD3-only work (descriptor math) instead of MMAs
//   warps 1-4:       a dependent-free FFMA2 / MUFU.EX2 mix (the softmax's instruction mix)
// Prints each worker warp's cycles: warps 4 (SMSP 0, shared with the issuer) and 1-3 (others).
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../paper_2402_05099_b200/csrc/ptx.cuh"

using namespace hydra;

__global__ void __launch_bounds__(160, 1) probe(int mode, int iters, int batch, int tm, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *sA = smem, *sB = smem + 32768;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  __shared__ int done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
    stop = 0;
    done = 0;
  }
  if (warp == 0) ptx::tmem_alloc<256>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    if (mode >= 1 && lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, 128, false);
      const uint32_t a = ptx::smem_u32(sA), b = ptx::smem_u32(sB);
      uint32_t ph = 0;
      while (!stop) {
        if (mode == 1) {
#pragma unroll 1
          for (int i = 0; i < batch; ++i)
            ptx::mma_ss(tmem, ptx::smem_desc_sw128(a + (i % 4) * 32, 16, 1024), ptx::smem_desc_sw128(b + (i % 4) * 32, 16, 1024),
                        idesc, i > 0);
          ptx::mma_commit(&bar);
          ptx::mbar_wait(&bar, ph);
          ph ^= 1;
        } else {
          __nanosleep(100);
        }
      }
    }
    __syncwarp();
  } else {
    float x0 = lane * 1e-3f, x1 = x0 + 0.5f, x2 = x0 + 0.25f, x3 = x0 + 0.125f;
    float y0 = 0.f, y1 = 0.f, y2 = 0.f, y3 = 0.f;
    const uint32_t tcol = tmem + ((uint32_t)((warp % 4) * 32) << 16) + 128;
    uint32_t tv[32];
    for (int i = 0; i < 32; ++i) tv[i] = 0;
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
      if (tm && (it % tm) == 0) {  // TMEM traffic like the softmax: a 32-column load, then a store
        ptx::tmem_ld32(tcol, tv);
        ptx::tmem_ld_wait();
        tv[it % 32] += 1;
        ptx::tmem_st32(tcol, tv);
        ptx::tmem_st_wait();
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        x0 = fmaf(x0, 0.999f, -0.001f);
        x1 = fmaf(x1, 0.999f, -0.001f);
        x2 = fmaf(x2, 0.999f, -0.001f);
        x3 = fmaf(x3, 0.999f, -0.001f);
        float e0, e1, e2, e3;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(x0));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(x1));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e2) : "f"(x2));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e3) : "f"(x3));
        y0 += e0;
        y1 += e1;
        y2 += e2;
        y3 += e3;
      }
    }
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 8 + warp] = t1 - t0;
    if (lane == 0 && (y0 + y1 + y2 + y3 + (float)tv[3]) == 12345.f) out[0] = 0;  // keep the work
    // the last worker warp to finish stops the issuer
    if (lane == 0 && atomicAdd(&done, 1) == 3) stop = 1;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(tmem);
  }
}

int main(int argc, char **argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;
  const int batch = argc > 2 ? atoi(argv[2]) : 8;
  const int tm = argc > 3 ? atoi(argv[3]) : 0;  // workers: a TMEM load + store every tm iterations (0 = none)
  long long *d;
  cudaMalloc(&d, 148 * 8 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(d, 0, 148 * 8 * sizeof(long long));
    probe<<<148, 160, 65536>>>(mode, iters, batch, tm, d);
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    long long h[148 * 8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double s[8] = {0};
    for (int b = 0; b < 148; ++b)
      for (int w = 1; w < 5; ++w) s[w] += (double)h[b * 8 + w] / 148;
    printf("tm %d batch %d mode %d (%s): worker cycles  warp1 %.0f  warp2 %.0f  warp3 %.0f  warp4(same SMSP as issuer) %.0f\n", tm, batch, mode,
           mode ? "MMA issuer busy" : "issuer idle", s[1], s[2], s[3], s[4]);
  }
  return 0;
}

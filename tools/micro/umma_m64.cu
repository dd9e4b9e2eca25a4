// Probe: TMEM placement of a cta_group::1 tcgen05.mma with M = 64 (kind::f16, bf16 -> f32).
// D[m, n] = sum_k A[m, k] B[n, k] with A[m, 0] = m + 1 and B[n, 0] = n + 1 (other k = 0),
// so D[m, n] = (m + 1)(n + 1).  TMEM is pre-filled with -1; every lane 0..127 and column
// 0..15 is dumped so the row -> lane map can be read off.  Also dumps the M = 128 case.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2402_05099_b200/csrc/ptx.cuh"

using namespace hydra;

template <int M>
__global__ void probe(float *out) {
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ __align__(1024) uint8_t sB[16 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 128 * 128 / 2; i += blockDim.x) reinterpret_cast<__nv_bfloat16 *>(sA)[i] = __float2bfloat16(0.f);
  for (int i = threadIdx.x; i < 16 * 128 / 2; i += blockDim.x) reinterpret_cast<__nv_bfloat16 *>(sB)[i] = __float2bfloat16(0.f);
  __syncthreads();
  // SW128 K-major: element (r, k) at r*128 + ((k/8) ^ (r%8))*16 + (k%8)*2; only k = 0 set
  if (threadIdx.x < M) {
    const int r = threadIdx.x;
    *reinterpret_cast<__nv_bfloat16 *>(sA + r * 128 + ((0 ^ (r % 8)) * 16)) = __float2bfloat16((float)(r + 1));
  }
  if (threadIdx.x < 16) {
    const int r = threadIdx.x;
    *reinterpret_cast<__nv_bfloat16 *>(sB + r * 128 + ((0 ^ (r % 8)) * 16)) = __float2bfloat16((float)(r + 1));
  }
  ptx::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<32>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(-1.f);
    ptx::tmem_st16(tmem + ((uint32_t)(warp * 32) << 16), v);
    ptx::tmem_st_wait();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(M, 16, false);
    ptx::mma_ss(tmem, ptx::smem_desc_sw128(ptx::smem_u32(sA), 16, 1024), ptx::smem_desc_sw128(ptx::smem_u32(sB), 16, 1024),
                idesc, 0);
    ptx::mma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  uint32_t v[16];
  ptx::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  ptx::tmem_ld_wait();
  for (int i = 0; i < 16; ++i) out[(warp * 32 + lane) * 16 + i] = __uint_as_float(v[i]);
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<32>(tmem);
}

int main() {
  float *d, h[128 * 16];
  cudaMalloc(&d, sizeof h);
  for (int which = 0; which < 2; ++which) {
    if (which == 0) probe<64><<<1, 128>>>(d);
    else probe<128><<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("M=%d err=%s\n", which == 0 ? 64 : 128, cudaGetErrorString(e));
    for (int l = 0; l < 128; ++l) {
      // row m is identified by D[m, 0] = m + 1 (and checked against column n: (m+1)(n+1))
      const float c0 = h[l * 16 + 0];
      bool ok = true;
      for (int n = 0; n < 16; ++n) ok &= h[l * 16 + n] == c0 * (n + 1);
      printf("lane %3d: row %4.0f %s  cols:", l, c0 - 1, ok ? "consistent" : "MIXED");
      for (int n = 0; n < 16; ++n) printf(" %g", h[l * 16 + n]);
      printf("\n");
    }
  }
  return 0;
}

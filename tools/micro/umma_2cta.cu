// Probe: the CTA-pair (cta_group::2) building blocks of the prefix kernel, checked against a
// host matmul.  One cluster of two CTAs:
//   TMA (cta_group::2 form, completion counted on the leader's barrier) loads into each CTA:
//     Q rows [128r, 128r+128) (two 64-dim SW128 panels), K tokens [64r, 64r+64) (two panels),
//     V all 128 tokens x dims [64r, 64r+64) (one MN-major panel)
//   leader: S[256 x 128] = Q K^T  (M = 256, N = 128, K = 128; both operands from smem)
//   each CTA: P = bf16(S / 16) of its 128 rows -> TMEM (packed pairs, 64 columns) -> arrive
//   leader: O[256 x 128] = P V    (A from TMEM, B = V MN-major, N split by dims)
//   commit multicast to both CTAs; each CTA dumps S and O of its rows.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 umma_2cta.cu -lcuda -o umma_2cta
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2402_05099_b200/csrc/ptx.cuh"

using namespace hydra;

struct Maps {
  CUtensorMap q, k, v;
};

constexpr int QT = 128 * 256;  // Q tile: 128 rows x 256 B (two panels of 16 KB)
constexpr int KT = 64 * 256;   // K half: 64 tokens x 256 B (two panels of 8 KB)
constexpr int VT = 128 * 128;  // V half: 128 tokens x 128 B (one panel)
constexpr int OFF_Q = 0, OFF_K = QT, OFF_V = QT + KT, OFF_BAR = QT + KT + VT;
constexpr int SMEM = OFF_BAR + 64 + 1024;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) probe(const __grid_constant__ Maps M, float *outS,
                                                                         float *outO) {
  extern __shared__ uint8_t raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *full = bars, *s_done = bars + 1, *p_full = bars + 2, *o_done = bars + 3;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 4);
  const uint32_t rank = ptx::cluster_ctarank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(full, 1);
    ptx::mbar_init(s_done, 1);
    ptx::mbar_init(p_full, 8);  // 4 softmax warps x 2 CTAs
    ptx::mbar_init(o_done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair<512>(tslot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t full_leader = ptx::mapa(ptx::smem_u32(full), 0);
  const uint32_t pfull_leader = ptx::mapa(ptx::smem_u32(p_full), 0);

  if (warp == 0 && lane == 0) {
    if (rank == 0) ptx::mbar_arrive_expect_tx(full, 2 * (QT + KT + VT));
    ptx::tma_load_3d_pair(smem + OFF_Q, &M.q, full_leader, 0, 0, 128 * rank);
    ptx::tma_load_3d_pair(smem + OFF_Q + QT / 2, &M.q, full_leader, 64, 0, 128 * rank);
    ptx::tma_load_3d_pair(smem + OFF_K, &M.k, full_leader, 0, 0, 64 * rank);
    ptx::tma_load_3d_pair(smem + OFF_K + KT / 2, &M.k, full_leader, 64, 0, 64 * rank);
    ptx::tma_load_3d_pair(smem + OFF_V, &M.v, full_leader, 64 * rank, 0, 0);
  }
  if (warp == 1 && rank == 0 && ptx::elect_one()) {
    ptx::mbar_wait(full, 0);
    ptx::tc_fence_after();
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(256, 128, false);
    const uint32_t qa = ptx::smem_u32(smem + OFF_Q), ka = ptx::smem_u32(smem + OFF_K);
    for (int kk = 0; kk < 8; ++kk)
      ptx::mma2_ss(tmem, ptx::smem_desc_sw128(qa + (kk / 4) * (QT / 2) + (kk % 4) * 32, 16, 1024),
                   ptx::smem_desc_sw128(ka + (kk / 4) * (KT / 2) + (kk % 4) * 32, 16, 1024), idesc_s, kk > 0);
    ptx::mma2_commit(s_done);
    ptx::mbar_wait_cluster(p_full, 0);
    ptx::tc_fence_after();
    constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(256, 128, true);
    const uint32_t va = ptx::smem_u32(smem + OFF_V);
    for (int kk = 0; kk < 8; ++kk)
      ptx::mma2_ts(tmem + 256, tmem + 128 + kk * 8, ptx::smem_desc_sw128(va + kk * 2048, 16, 1024), idesc_pv, kk > 0);
    ptx::mma2_commit(o_done);
  }
  if (warp >= 4) {
    const int q4 = warp % 4, r = q4 * 32 + lane;
    const uint32_t lb = (uint32_t)(q4 * 32) << 16;
    ptx::mbar_wait(s_done, 0);
    ptx::tc_fence_after();
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      ptx::tmem_ld32(tmem + lb + c * 32, v);
      ptx::tmem_ld_wait();
      uint32_t pk[16];
      for (int i = 0; i < 32; ++i) outS[(size_t)(128 * rank + r) * 128 + c * 32 + i] = __uint_as_float(v[i]);
      for (int i = 0; i < 16; ++i)
        pk[i] = ptx::cvt_bf16x2(__uint_as_float(v[2 * i]) / 16.f, __uint_as_float(v[2 * i + 1]) / 16.f);
      ptx::tmem_st16(tmem + lb + 128 + c * 16, pk);
    }
    ptx::tmem_st_wait();
    ptx::tc_fence_before();
    ptx::warp_arrive_cluster(pfull_leader);
    ptx::mbar_wait(o_done, 0);
    ptx::tc_fence_after();
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      ptx::tmem_ld32(tmem + lb + 256 + c * 32, v);
      ptx::tmem_ld_wait();
      for (int i = 0; i < 32; ++i) outO[(size_t)(128 * rank + r) * 128 + c * 32 + i] = __uint_as_float(v[i]);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<512>(tmem);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
// [rows][128] bf16 as a 3-D map {128 dims, 1, rows} with box {64, 1, box_rows}
static void mk(CUtensorMap *m, void *base, int rows, int box_rows) {
  cuuint64_t d[3] = {128, 1, (cuuint64_t)rows}, s[2] = {256, 256};
  cuuint32_t b[3] = {64, 1, (cuuint32_t)box_rows}, e[3] = {1, 1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
}

int main() {
  std::vector<__nv_bfloat16> hq(256 * 128), hk(128 * 128), hv(128 * 128);
  srand(1);
  auto rnd = [] { return (float)((rand() % 17) - 8) / 8.f; };
  for (auto &x : hq) x = __float2bfloat16(rnd());
  for (auto &x : hk) x = __float2bfloat16(rnd());
  for (auto &x : hv) x = __float2bfloat16(rnd());
  __nv_bfloat16 *dq, *dk, *dv;
  float *dS, *dO;
  cudaMalloc(&dq, hq.size() * 2);
  cudaMalloc(&dk, hk.size() * 2);
  cudaMalloc(&dv, hv.size() * 2);
  cudaMalloc(&dS, 256 * 128 * 4);
  cudaMalloc(&dO, 256 * 128 * 4);
  cudaMemcpy(dq, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dS, 0xff, 256 * 128 * 4);
  cudaMemset(dO, 0xff, 256 * 128 * 4);
  Maps M;
  mk(&M.q, dq, 256, 128);
  mk(&M.k, dk, 128, 64);
  mk(&M.v, dv, 128, 128);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  probe<<<2, 256, SMEM>>>(M, dS, dO);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> S(256 * 128), O(256 * 128);
  cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  double es = 0, eo = 0;
  std::vector<float> Pr(256 * 128);
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < 128; ++n) {
      double a = 0;
      for (int k = 0; k < 128; ++k) a += (double)__bfloat162float(hq[m * 128 + k]) * __bfloat162float(hk[n * 128 + k]);
      es = fmax(es, fabs(a - S[m * 128 + n]));
      Pr[m * 128 + n] = __bfloat162float(__float2bfloat16((float)a / 16.f));
    }
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < 128; ++n) {
      double a = 0;
      for (int k = 0; k < 128; ++k) a += (double)Pr[m * 128 + k] * __bfloat162float(hv[k * 128 + n]);
      eo = fmax(eo, fabs(a - O[m * 128 + n]));
    }
  printf("max|dS| = %.3e  max|dO| = %.3e   S[0][0]=%f S[255][127]=%f O[200][70]=%f\n", es, eo, S[0], S[256 * 128 - 1],
         O[200 * 128 + 70]);
  printf(es < 1e-3 && eo < 1e-2 ? "PASS\n" : "FAIL\n");
  return 0;
}

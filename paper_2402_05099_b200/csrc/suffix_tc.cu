// suffix_tc.cu -- persistent, TMA-fed, tensor-core suffix attention for sm_100a.
//
// PAPER.md §3.2: suffix attention is "computed normally, with a single query per
// sequence" -- a memory-bound GEMV per (sequence b, KV head j) over lens[b] tokens.  The
// SIMT decode kernel spends ~45 warp-instructions per 512-B K/V row pair (shuffle
// reductions, bf16 unpacking, FMAs), so it needs nearly every SM to saturate HBM.  This
// kernel moves the arithmetic onto the tensor core, where it is almost free, so a few
// dozen SMs can stream the suffix while the rest run the prefix GEMM:
//   S^T [128 tokens x 16] = K_tile [128 x 128] . Q^T        (tcgen05.mma, M=128, N=16)
//   O^T [128 dims x 16]  += V_tile^T [128 x 128 tokens] . P^T (tcgen05.mma, A MN-major)
// N = 16 holds the g = Hq/Hkv query heads of the KV group (zero-padded), so GQA reuses
// every K/V byte g times.  One CTA per SM (persistent, 192 threads):
//   warp 0     TMA producer: per item the g query rows (Q^T) and per 128-token block
//              the K and V tiles (two 64-column SWIZZLE_128B boxes each) into a
//              3-stage ring; reads lens[b] itself, so only blocks with valid tokens move
//   warp 1     TMEM allocator + single-thread MMA issuer: S(0) S(1) PV(0) S(2) PV(1) ...
//   warps 2-5  softmax: thread = token lane; per block a block max per head (warp
//              shuffles + smem across the 4 warps), the stale-max rule of the prefix
//              kernel (rescale only when the max grows by > 8, log2 units), P^T as bf16
//              into shared memory (B operand of the PV MMA); epilogue per item:
//              O^T / l with thread = head dim (coalesced stores), LSE per head.
// Tokens >= lens[b] inside the last block: their scores are masked to -inf, and their
// V rows are zeroed in shared memory before the PV MMA (0 * NaN would poison O).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace hydra {

namespace stc {
constexpr int BT = 128;   // tokens per block (UMMA M of S^T, K of PV)
constexpr int HD = 128;   // head dim (UMMA K of S^T, M of PV)
constexpr int NQ = 16;    // padded query heads per KV group (UMMA N)
constexpr int NS = 3;     // K stages and V stages (separate rings: K frees after S, V after PV)
constexpr int kThreads = 192;
constexpr int PANEL = BT * 128;      // 128 rows x 128 B
constexpr int TILE = 2 * PANEL;      // 32 KB
constexpr int QPANEL = NQ * 128;     // 2 KB: 16 rows x 64 dims
constexpr int QTILE = 2 * QPANEL;    // 4 KB
constexpr int PPANEL = NQ * 128;     // P^T: 16 rows x 64 tokens
constexpr int PTILE = 2 * PPANEL;    // 4 KB
constexpr int OFF_K = 0;
constexpr int OFF_V = OFF_K + NS * TILE;
constexpr int OFF_Q = OFF_V + NS * TILE;     // 2 slots
constexpr int OFF_P = OFF_Q + 2 * QTILE;     // 2 slots
constexpr int OFF_RED = OFF_P + 2 * PTILE;   // [2 block parity][4 warps][16] max + [2 item parity][4][16] sums
constexpr int OFF_BAR = OFF_RED + (2 * 4 * NQ + 2 * 4 * NQ) * 4;
// k_full, k_empty, v_full, v_empty [NS]; q_full, q_empty, s_full, p_full, o_free, pv_done [2]
constexpr int N_BARS = 4 * NS + 12;
constexpr int BYTES = OFF_BAR + N_BARS * 8 + 16;
constexpr int ALLOC = BYTES + 1024;
constexpr uint32_t TMEM_COLS = 64;  // S^T x2 (16 cols each), O^T x2
}  // namespace stc

struct __align__(64) SuffixTcParams {
  CUtensorMap tmK, tmV, tmQ;
  const int32_t *lens;
  int32_t B, Hq, Hkv, g;
  float scale_log2;
  int32_t n_items;
  float *o, *lse;
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int G>  // query heads per KV group (compile-time: no per-head predicates)
__global__ void __launch_bounds__(stc::kThreads, 1) suffix_tc_kernel(const __grid_constant__ SuffixTcParams P) {
  using namespace stc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *k_full = bars, *k_empty = bars + NS, *v_full = bars + 2 * NS, *v_empty = bars + 3 * NS;
  uint64_t *q_full = bars + 4 * NS, *q_empty = q_full + 2, *s_full = q_full + 4, *p_full = q_full + 6,
           *o_free = q_full + 8, *pv_done = q_full + 10;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + N_BARS);
  float *red_max = reinterpret_cast<float *>(smem + OFF_RED);  // [2][4][NQ]
  float *red_sum = red_max + 2 * 4 * NQ;                        // [2][4][NQ]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int g = G;

  // zero Q^T / P^T slots once: rows >= g (padding heads) must stay 0 forever
  for (int i = threadIdx.x; i < (2 * QTILE + 2 * PTILE) / 16; i += kThreads)
    reinterpret_cast<uint4 *>(smem + OFF_Q)[i] = make_uint4(0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&P.tmK);
    ptx::prefetch_tmap(&P.tmV);
    ptx::prefetch_tmap(&P.tmQ);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], 4);  // one elected arrival per softmax warp
      ptx::mbar_init(&o_free[i], 4);
      ptx::mbar_init(&pv_done[i], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================= TMA producer =================
    if (ptx::elect_one()) {
      uint32_t gb = 0, qi = 0;
      for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
        const int b = item / P.Hkv, j = item % P.Hkv;
        const int len = P.lens[b];
        const int nblk = (len + BT - 1) / BT;
        if (nblk == 0) continue;
        const int qs = qi & 1;
        ptx::mbar_wait(&q_empty[qs], ((qi >> 1) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&q_full[qs], 2 * 64 * g * 2);
        uint8_t *sQ = smem + OFF_Q + qs * QTILE;
        ptx::tma_load_3d(sQ, &P.tmQ, &q_full[qs], 0, j * g, b);
        ptx::tma_load_3d(sQ + QPANEL, &P.tmQ, &q_full[qs], 64, j * g, b);
        ++qi;
        for (int n = 0; n < nblk; ++n, ++gb) {
          const int st = gb % NS;
          const uint32_t ph = ((gb / NS) & 1) ^ 1;
          uint8_t *sK = smem + OFF_K + st * TILE, *sV = smem + OFF_V + st * TILE;
          const int t0 = n * BT;
          ptx::mbar_wait(&k_empty[st], ph);
          ptx::mbar_arrive_expect_tx(&k_full[st], TILE);
          ptx::tma_load_4d(sK, &P.tmK, &k_full[st], 0, j, t0, b);
          ptx::tma_load_4d(sK + PANEL, &P.tmK, &k_full[st], 64, j, t0, b);
          ptx::mbar_wait(&v_empty[st], ph);
          ptx::mbar_arrive_expect_tx(&v_full[st], TILE);
          ptx::tma_load_4d(sV, &P.tmV, &v_full[st], 0, j, t0, b);
          ptx::tma_load_4d(sV + PANEL, &P.tmV, &v_full[st], 64, j, t0, b);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (flat block sequence across items, one-block lookahead) =================
    if (ptx::elect_one()) {
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(BT, NQ, false);                 // A=K, B=Q^T (K-major)
      constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(HD, NQ, false) | (1u << 15);  // A=V^T (MN-major), B=P^T
      struct Blk {
        uint32_t gbi, st, ob, qs, item_no;
        bool first, last;
      } prev{};
      bool have_prev = false;
      uint32_t gbi = 0, qi = 0, item_no = 0;
      auto do_pv = [&](const Blk &x) {
        const uint32_t slot = x.gbi & 1;
        ptx::mbar_wait(&p_full[slot], (x.gbi >> 1) & 1);
        if (x.first) ptx::mbar_wait(&o_free[x.ob], ((x.item_no >> 1) & 1) ^ 1);
        ptx::mbar_wait(&v_full[x.st], (x.gbi / NS) & 1);
        ptx::tc_fence_after();
        const uint32_t v_addr = ptx::smem_u32(smem + OFF_V + x.st * TILE);
        const uint32_t p_addr = ptx::smem_u32(smem + OFF_P + slot * PTILE);
#pragma unroll
        for (int kk = 0; kk < BT / 16; ++kk)
          ptx::mma_ss(tmem + 2 * NQ + x.ob * NQ, ptx::smem_desc_sw128(v_addr + kk * 2048, PANEL, 1024),
                      ptx::smem_desc_sw128(p_addr + (kk / 4) * PPANEL + (kk % 4) * 32, 16, 1024), idesc_pv,
                      (!x.first || kk > 0));
        ptx::mma_commit(&pv_done[slot]);
        ptx::mma_commit(&v_empty[x.st]);
        if (x.last) ptx::mma_commit(&q_empty[x.qs]);
      };
      for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
        const int b = item / P.Hkv;
        const int nblk = (P.lens[b] + BT - 1) / BT;
        if (nblk == 0) continue;
        const uint32_t qs = qi & 1;
        ptx::mbar_wait(&q_full[qs], (qi >> 1) & 1);
        const uint32_t q_addr = ptx::smem_u32(smem + OFF_Q + qs * QTILE);
        for (int n = 0; n < nblk; ++n, ++gbi) {
          const uint32_t st = gbi % NS;
          ptx::mbar_wait(&k_full[st], (gbi / NS) & 1);
          ptx::tc_fence_after();
          const uint32_t k_addr = ptx::smem_u32(smem + OFF_K + st * TILE);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk / 4) * PANEL + (kk % 4) * 32, qoff = (kk / 4) * QPANEL + (kk % 4) * 32;
            ptx::mma_ss(tmem + (gbi & 1) * NQ, ptx::smem_desc_sw128(k_addr + off, 16, 1024),
                        ptx::smem_desc_sw128(q_addr + qoff, 16, 1024), idesc_s, kk > 0);
          }
          ptx::mma_commit(&s_full[gbi & 1]);
          ptx::mma_commit(&k_empty[st]);
          if (have_prev) do_pv(prev);  // PV of the previous block after S of this one
          prev = Blk{gbi, st, item_no & 1, qs, item_no, n == 0, n == nblk - 1};
          have_prev = true;
        }
        ++qi;
        ++item_no;
      }
      if (have_prev) do_pv(prev);
    }
  } else {
    // ================= softmax (thread = token lane) / lagged epilogue (thread = head dim) =================
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const float c2 = P.scale_log2;
    uint32_t gbi = 0, item_no = 0;
    // state of the item whose epilogue is pending (run after the next item's first block)
    bool pend = false;
    int64_t pend_row0 = 0;
    uint32_t pend_ob = 0, pend_last = 0;
    float pm[G], pl[G];
    auto epilogue = [&]() {
      ptx::mbar_wait(&pv_done[pend_last & 1], (pend_last >> 1) & 1);
      ptx::tc_fence_after();
      // two epilogues can run back to back (the lagged one and the final one): alternate
      // the reduction buffer by item parity so a fast warp never overwrites sums a slow
      // warp is still reading
      float *rs = red_sum + pend_ob * 4 * NQ;
#pragma unroll
      for (int h = 0; h < G; ++h) {
          float x = pl[h];
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
          if (lane == 0) rs[quarter * NQ + h] = x;
        }
      named_bar_sync(1, 128);
      uint32_t ov[NQ];
      ptx::tmem_ld16(tmem + lane_base + 2 * NQ + pend_ob * NQ, ov);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      ptx::warp_arrive(&o_free[pend_ob]);
#pragma unroll
      for (int h = 0; h < G; ++h) {
          const float L = rs[h] + rs[NQ + h] + rs[2 * NQ + h] + rs[3 * NQ + h];
          P.o[(pend_row0 + h) * HD + r] = __uint_as_float(ov[h]) / L;
          if (r == h) P.lse[pend_row0 + h] = (pm[h] + log2f(L)) * HYDRA_LN2;
        }
      pend = false;
    };
    for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
      const int b = item / P.Hkv, j = item % P.Hkv;
      const int len = P.lens[b];
      const int nblk = (len + BT - 1) / BT;
      const int64_t row0 = (int64_t)b * P.Hq + (int64_t)j * g;
      if (nblk == 0) {  // empty suffix: (0, -inf) sentinel
        for (int h = 0; h < g; ++h) {
          P.o[(row0 + h) * HD + r] = 0.f;
          if (r == 0) P.lse[row0 + h] = -INFINITY;
        }
        continue;
      }
      const uint32_t ob = item_no & 1;
      const uint32_t o_tmem = tmem + lane_base + 2 * NQ + ob * NQ;
      float m[G], l[G];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        m[h] = -INFINITY;
        l[h] = 0.f;
      }
      for (int n = 0; n < nblk; ++n, ++gbi) {
        const uint32_t buf = gbi & 1;
        ptx::mbar_wait(&s_full[buf], (gbi >> 1) & 1);
        ptx::tc_fence_after();
        uint32_t sv[NQ];
        ptx::tmem_ld16(tmem + lane_base + buf * NQ, sv);
        ptx::tmem_ld_wait();
        const int valid = min(BT, len - n * BT);
        const bool tok = r < valid;
        float s[G];
        float *rm = red_max + buf * 4 * NQ;
#pragma unroll
        for (int h = 0; h < G; ++h) {
          s[h] = tok ? __uint_as_float(sv[h]) : -INFINITY;
          float x = s[h];
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
          if (lane == 0) rm[quarter * NQ + h] = x;
        }
        named_bar_sync(1, 128);
        float alpha[NQ];
        bool resc = false;
#pragma unroll
        for (int h = 0; h < NQ; ++h) alpha[h] = 1.f;
#pragma unroll
        for (int h = 0; h < G; ++h) {
          const float bm = fmaxf(fmaxf(rm[h], rm[NQ + h]), fmaxf(rm[2 * NQ + h], rm[3 * NQ + h]));
          const float mnew = bm * c2;
          if (mnew > m[h] + 8.0f) {  // block-uniform decision
            const float mt = fmaxf(m[h], mnew);
            alpha[h] = fast_exp2(m[h] - mt);
            m[h] = mt;
            resc = true;
          }
        }
        float p[G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
          p[h] = tok ? fast_exp2(fmaf(s[h], c2, -m[h])) : 0.f;
          l[h] = l[h] * alpha[h] + p[h];
        }
        // P slot `buf` was last read by PV(gbi - 2)
        if (gbi >= 2) ptx::mbar_wait(&pv_done[buf], ((gbi - 2) >> 1) & 1);
        if (resc && n >= 1) {  // rare: O^T column h *= alpha[h] once PV(gbi - 1) has landed
          ptx::mbar_wait(&pv_done[buf ^ 1], ((gbi - 1) >> 1) & 1);
          ptx::tc_fence_after();
          uint32_t ov[NQ];
          ptx::tmem_ld16(o_tmem, ov);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int h = 0; h < NQ; ++h) ov[h] = __float_as_uint(__uint_as_float(ov[h]) * alpha[h]);
          ptx::tmem_st16(o_tmem, ov);
          ptx::tmem_st_wait();
        }
        uint8_t *sp = smem + OFF_P + buf * PTILE + (r / 64) * PPANEL;
        const int c = (r % 64) / 8, e = r % 8;
#pragma unroll
        for (int h = 0; h < G; ++h)
          *reinterpret_cast<__nv_bfloat16 *>(sp + h * 128 + ((c ^ (h % 8)) * 16) + e * 2) = __float2bfloat16_rn(p[h]);
        if (valid < BT) ptx::mbar_wait(&v_full[gbi % NS], (gbi / NS) & 1);  // V tile landed
        if (!tok) {  // rows past lens[b] in the last block: zero the V row (0 * NaN would poison O)
          uint8_t *vrow = smem + OFF_V + (gbi % NS) * TILE + r * 128;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            *reinterpret_cast<uint4 *>(vrow + q * 16) = make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4 *>(vrow + PANEL + q * 16) = make_uint4(0, 0, 0, 0);
          }
        }
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        ptx::warp_arrive(&p_full[buf]);
        if (n == 0 && pend) epilogue();  // previous item's epilogue, off the critical path
      }
      pend = true;
      pend_row0 = row0;
      pend_ob = ob;
      pend_last = gbi - 1;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        pm[h] = m[h];
        pl[h] = l[h];
      }
      ++item_no;
    }
    if (pend) epilogue();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem);
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn3() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool suffix_tc_supported(const hydra_heads *h) {
  const int g = h->num_q_heads / h->num_kv_heads;
  const bool g_ok = g == 1 || g == 2 || g == 4 || g == 8 || g == 16;
  return h->dtype == HYDRA_BF16 && h->head_dim == 128 && g_ok && encode_fn3() != nullptr;
}

template <int G>
static cudaError_t launch_g(const SuffixTcParams &P, int grid, cudaStream_t s) {
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(suffix_tc_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, stc::ALLOC);
  });
  if (attr != cudaSuccess) return attr;
  suffix_tc_kernel<G><<<grid, stc::kThreads, stc::ALLOC, s>>>(P);
  return cudaGetLastError();
}

hydra_status launch_suffix_tc(const SuffixTcArgs &a, int n_ctas, cudaStream_t s) {
  auto fn = encode_fn3();
  if (!fn) return HYDRA_ECUDA;
  SuffixTcParams P;
  memset(&P, 0, sizeof(P));
  const int g = a.Hq / a.Hkv;
  {
    const cuuint64_t dims[4] = {(cuuint64_t)stc::HD, (cuuint64_t)a.Hkv, (cuuint64_t)a.S_cap, (cuuint64_t)a.B};
    const cuuint64_t strides[3] = {(cuuint64_t)a.s_sh * 2, (cuuint64_t)a.s_st * 2, (cuuint64_t)a.s_sb * 2};
    const cuuint32_t box[4] = {64, 1, (cuuint32_t)stc::BT, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    if (fn(&P.tmK, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(a.k), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return HYDRA_ECUDA;
    if (fn(&P.tmV, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(a.v), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return HYDRA_ECUDA;
  }
  {
    const cuuint64_t dims[3] = {(cuuint64_t)stc::HD, (cuuint64_t)a.Hq, (cuuint64_t)a.B};
    const cuuint64_t strides[2] = {(cuuint64_t)a.q_sh * 2, (cuuint64_t)a.q_sb * 2};
    const cuuint32_t box[3] = {64, (cuuint32_t)g, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (fn(&P.tmQ, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(a.q), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return HYDRA_ECUDA;
  }
  P.lens = a.lens;
  P.B = a.B;
  P.Hq = a.Hq;
  P.Hkv = a.Hkv;
  P.g = g;
  P.scale_log2 = a.scale_log2;
  P.n_items = a.B * a.Hkv;
  P.o = a.o;
  P.lse = a.lse;
  if (P.n_items == 0) return HYDRA_OK;
  const int grid = n_ctas > 0 && n_ctas < P.n_items ? n_ctas : P.n_items;
  cudaError_t e = cudaErrorInvalidValue;
  switch (g) {
    case 1: e = launch_g<1>(P, grid, s); break;
    case 2: e = launch_g<2>(P, grid, s); break;
    case 4: e = launch_g<4>(P, grid, s); break;
    case 8: e = launch_g<8>(P, grid, s); break;
    case 16: e = launch_g<16>(P, grid, s); break;
  }
  return e == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

}  // namespace hydra

// prefix_tc.cu -- inter-sequence batched prefix attention on sm_100a tensor cores.
//
// PAPER.md §3.2: the decode queries of all B sequences attend to the
// same prefix K/V, so they are stacked into one matrix and prefix attention becomes
// a dense GEMM-shaped problem that reads the prefix once and runs on tensor cores
// (App. B `attention(batched_q, prefix_k, prefix_v)`).  For KV head j the
// stacked query matrix has rows r = b*g + i holding q[b, j*g+i, :] (g = Hq/Hkv), so a
// GQA group shares every K/V tile too.  Output per row: O = softmax(s) V (fp32,
// normalised) and LSE (natural log, Eq. 4) for the later combine (Eq. 5).
//
// One CTA = one 128-row query tile x one KV head x one KV split.  192 threads:
//   warp 0      TMA producer: K and V tiles of 128 tokens x 128 dims (two 64-column
//               SWIZZLE_128B boxes each) into a 3-stage ring (separate K / V slots)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5   softmax / correction / epilogue, one query row per thread (TMEM lane)
// TMEM (512 columns): S0 [0,128) and S1 [128,256) fp32 score tiles (double-buffered so
// the MMA of block n+1 overlaps the softmax of block n); P(n) is written back as bf16
// into the first 64 columns of its S buffer and consumed from TMEM as the A operand of
// the PV MMA; O accumulates in [256,384).
// Pipeline order issued by the MMA thread: S(0) S(1) PV(0) S(2) PV(1) ... PV(last).
// Online softmax in the log2 domain with the scale folded into one FFMA; the running
// max is only raised when a row's max grows by more than 8 (log2 units), so P <= 256
// and the O correction (TMEM ld/scale/st) is rare; the final O / l uses the same stale
// max, which keeps the result exact.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"
#include "fused.cuh"

namespace hydra {

namespace tc {
constexpr int BM = 128;  // stacked query rows per tile (UMMA M)
constexpr int BN = 128;  // KV tokens per block (UMMA N of S, K of PV)
constexpr int HD = 128;  // head dim (UMMA K of S, N of PV)
constexpr int kThreads = 192;
constexpr int PANEL = BN * 128;          // one 64-column SWIZZLE_128B panel: 128 rows x 128 B
constexpr int TILE = 2 * PANEL;          // 128 rows x 128 dims bf16 = 32 KB
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t COL_O = 256;
// Shared-memory carve-up for NS pipeline stages (K and V slots per stage).
template <int NS>
struct Smem {
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + TILE;
  static constexpr int OFF_V = OFF_K + NS * TILE;
  static constexpr int OFF_BAR = OFF_V + NS * TILE;
  static constexpr int N_BARS = 4 * NS + 2 + 2 + 1;
  static constexpr int BYTES = OFF_BAR + N_BARS * 8 + 16;
  static constexpr int ALLOC = BYTES + 1024;  // slack for 1024-B alignment (SWIZZLE_128B atoms)
};
}  // namespace tc

struct __align__(64) PrefixTcKernelParams {
  CUtensorMap tmK;
  CUtensorMap tmV;
  const __nv_bfloat16 *q;
  int64_t q_sb, q_sh;
  int32_t Hq, Hkv, g;
  float scale_log2;
  int64_t P;
  int32_t B;
  const PrefixTask *tasks;
  const int32_t *seq_list;
  int32_t n_splits;
  float *o, *lse;
  int64_t o_slot_stride, lse_slot_stride;
  int32_t debug_variant;  // bring-up switch: bit0 swaps the V descriptor LBO/SBO
  FusedCombine fc;        // fc.cnt != null: the Eq. 5 merge of every completed row in this epilogue
};

// Fused Eq. 5 (fused.cuh): count this warp's rows; merge the rows this split completed.
__device__ __forceinline__ void tc1_fused_arrive(const FusedCombine &F, bool live, int64_t seq, int h, int Hq,
                                                 int lane) {
  if (F.pre_done) return;  // sequential schedule: the suffix kernel counts and merges
  __threadfence();
  __syncwarp();
  const int64_t row = seq * Hq + h;
  int n_pre = 0;
  bool last = false;
  if (live) {
    n_pre = fc_prefix_pieces(F, seq, h);
    last = fc_arrive(F, row, n_pre + F.n_suf);
  }
  unsigned mask = __ballot_sync(0xffffffffu, last);
  if (mask) __threadfence();
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    fc_merge_row_warp(F, __shfl_sync(0xffffffffu, row, src), __shfl_sync(0xffffffffu, n_pre, src), lane);
  }
}

template <int NS>
__global__ void __launch_bounds__(tc::kThreads, 1) prefix_tc_kernel(const __grid_constant__ PrefixTcKernelParams P) {
  using namespace tc;
  using L = Smem<NS>;
  constexpr int OFF_Q = L::OFF_Q, OFF_K = L::OFF_K, OFF_V = L::OFF_V, OFF_BAR = L::OFF_BAR, N_BARS = L::N_BARS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem + OFF_Q;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *k_full = bars, *k_empty = bars + NS, *v_full = bars + 2 * NS, *v_empty = bars + 3 * NS;
  uint64_t *s_full = bars + 4 * NS, *p_full = bars + 4 * NS + 2, *pv_done = bars + 4 * NS + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + N_BARS);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int j = blockIdx.y, split = blockIdx.z;

  // ---- work item
  PrefixTask task;
  if (P.tasks) {
    task = P.tasks[blockIdx.x];
  } else {
    task.kv_off = 0;
    task.kv_len = P.P;
    task.seq_off = 0;
    task.n_seq = P.B;
    task.depth = 0;
    task.tile = blockIdx.x;
  }
  const int64_t n_rows = (int64_t)task.n_seq * P.g;
  const int64_t row0 = (int64_t)task.tile * BM;
  const int nblk_total = (int)((task.kv_len + BN - 1) / BN);
  const int per_split = (nblk_total + P.n_splits - 1) / P.n_splits;
  const int blk_begin = split * per_split;
  const int nblk = max(0, min(nblk_total, blk_begin + per_split) - blk_begin);
  const int out_slot = task.depth * P.n_splits + split;

  if (nblk == 0) {  // empty KV range for this split: the (0, -inf) sentinel
    if (warp >= 2) {
      const int64_t rr = row0 + 32 * (warp % 4) + lane;
      const bool live = rr < n_rows;
      int64_t seq = 0;
      int h = 0;
      if (live) {
        seq = P.seq_list ? P.seq_list[task.seq_off + rr / P.g] : rr / P.g;
        h = j * P.g + (int)(rr % P.g);
        P.lse[out_slot * P.lse_slot_stride + seq * P.Hq + h] = -INFINITY;
        float4 *o = reinterpret_cast<float4 *>(P.o + out_slot * P.o_slot_stride + (seq * P.Hq + h) * HD);
        for (int c = 0; c < HD / 4; ++c) o[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (P.fc.cnt) tc1_fused_arrive(P.fc, live, seq, h, P.Hq, lane);
    }
    return;
  }

  // ---- one-time setup
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&P.tmK);
    ptx::prefetch_tmap(&P.tmV);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], 4);  // one elected arrival per softmax warp
    }
    ptx::mbar_init(pv_done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
  if (warp >= 2) {
    // Stacked query row r of this tile -> sQ in the canonical K-major SWIZZLE_128B
    // layout: panel = dim/64, row r at r*128 B, 16-B chunk c stored at chunk c^(r%8).
    const int r = 32 * (warp % 4) + lane;
    const int64_t rr = row0 + r;
    uint4 chunks[16];
    if (rr < n_rows) {
      const int64_t seq = P.seq_list ? P.seq_list[task.seq_off + rr / P.g] : rr / P.g;
      const int h = j * P.g + (int)(rr % P.g);
      const uint4 *src = reinterpret_cast<const uint4 *>(P.q + seq * P.q_sb + (int64_t)h * P.q_sh);
#pragma unroll
      for (int c = 0; c < 16; ++c) chunks[c] = __ldg(src + c);
    } else {
#pragma unroll
      for (int c = 0; c < 16; ++c) chunks[c] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int panel = c / 8, cc = c % 8;
      *reinterpret_cast<uint4 *>(sQ + panel * PANEL + r * 128 + ((cc ^ (r % 8)) * 16)) = chunks[c];
    }
    ptx::fence_proxy_async_smem();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================= TMA producer =================
    if (ptx::elect_one()) {
      for (int n = 0; n < nblk; ++n) {
        const int st = n % NS;
        const uint32_t ph = (n / NS) & 1;
        const int t0 = (int)(task.kv_off + (int64_t)(blk_begin + n) * BN);
        uint8_t *sK = smem + OFF_K + st * TILE;
        uint8_t *sV = smem + OFF_V + st * TILE;
        ptx::mbar_wait(&k_empty[st], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&k_full[st], TILE);
        ptx::tma_load_3d(sK, &P.tmK, &k_full[st], 0, j, t0);
        ptx::tma_load_3d(sK + PANEL, &P.tmK, &k_full[st], 64, j, t0);
        ptx::mbar_wait(&v_empty[st], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&v_full[st], TILE);
        ptx::tma_load_3d(sV, &P.tmV, &v_full[st], 0, j, t0);
        ptx::tma_load_3d(sV + PANEL, &P.tmV, &v_full[st], 64, j, t0);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (one thread) =================
    if (ptx::elect_one()) {
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(BM, BN, false);  // S = Q K^T, both K-major
      constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(BM, HD, true);  // O += P V, V is MN-major
      const uint32_t q_addr = ptx::smem_u32(sQ);
      for (int n = 0; n <= nblk; ++n) {
        if (n < nblk) {
          const int st = n % NS;
          ptx::mbar_wait(&k_full[st], (n / NS) & 1);
          ptx::tc_fence_after();
          const uint32_t k_addr = ptx::smem_u32(smem + OFF_K + st * TILE);
          const uint32_t d_tmem = tmem + (uint32_t)(n & 1) * BN;
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk / 4) * PANEL + (kk % 4) * 32;
            ptx::mma_ss(d_tmem, ptx::smem_desc_sw128(q_addr + off, 16, 1024),
                        ptx::smem_desc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0);
          }
          ptx::mma_commit(&s_full[n & 1]);
          ptx::mma_commit(&k_empty[st]);
        }
        if (n >= 1) {
          const int m = n - 1, st = m % NS;
          ptx::mbar_wait(&p_full[m & 1], (m >> 1) & 1);
          ptx::mbar_wait(&v_full[st], (m / NS) & 1);
          ptx::tc_fence_after();
          const uint32_t v_addr = ptx::smem_u32(smem + OFF_V + st * TILE);
          const uint32_t p_tmem = tmem + (uint32_t)(m & 1) * BN;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            // B = V tile, MN-major: 16 tokens per step = 2 groups of 8 rows (SBO 1024 B);
            // the two 64-dim panels are LBO = 16 KB apart.  A = P in TMEM: 16 bf16 per row
            // = 8 packed 32-bit columns per step.
            const uint64_t vdesc = (kTesting && (P.debug_variant & 1))
                                       ? ptx::smem_desc_sw128(v_addr + kk * 2048, 1024, PANEL)
                                       : ptx::smem_desc_sw128(v_addr + kk * 2048, PANEL, 1024);
            ptx::mma_ts(tmem + COL_O, p_tmem + kk * 8, vdesc, idesc_pv, (m > 0 || kk > 0));
          }
          ptx::mma_commit(pv_done);
          ptx::mma_commit(&v_empty[st]);
        }
      }
    }
  } else {
    // ================= softmax / correction / epilogue (warps 2..5) =================
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const float c2 = P.scale_log2;
    float m2 = -INFINITY, l = 0.f;
    for (int n = 0; n < nblk; ++n) {
      const uint32_t sbuf = tmem + lane_base + (uint32_t)(n & 1) * BN;
      ptx::mbar_wait(&s_full[n & 1], (n >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) ptx::tmem_ld32(sbuf + c * 32, sr[c]);
      ptx::tmem_ld_wait();
      const int64_t rem = task.kv_len - (int64_t)(blk_begin + n) * BN;
      if (rem < BN) {  // partial last block only (CTA-uniform): mask columns >= rem
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i >= rem) sr[c][i] = 0xff800000u;  // -inf
      }
      // row max: 8 independent FMNMX3 chains of depth 8, then a short tree
      float acc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaxf(__uint_as_float(sr[0][2 * k]), __uint_as_float(sr[0][2 * k + 1]));
#pragma unroll
      for (int i = 16; i < BN; i += 16)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          acc[k] = ptx::fmax3(acc[k], __uint_as_float(sr[(i + 2 * k) / 32][(i + 2 * k) % 32]),
                              __uint_as_float(sr[(i + 2 * k + 1) / 32][(i + 2 * k + 1) % 32]));
      const float mx = fmaxf(ptx::fmax3(acc[0], acc[1], acc[2]),
                             fmaxf(ptx::fmax3(acc[3], acc[4], acc[5]), fmaxf(acc[6], acc[7])));
      const float mnew = mx * c2;
      const bool need = mnew > m2 + 8.0f;
      const bool any = __any_sync(0xffffffffu, need);
      float alpha = 1.f;
      if (any) {
        const float mt = fmaxf(m2, mnew);
        alpha = fast_exp2(m2 - mt);  // m2 = -inf on the first block -> 0
        m2 = mt;
      }
      // p = 2^(s*c2 - m2): packed FFMA2 for the argument, MUFU.EX2 per element,
      // packed FADD2 into 4 independent row-sum chains, bf16x2 pack for the PV MMA
      const uint64_t cc = ptx::pack2(c2, c2), nm = ptx::pack2(-m2, -m2);
      uint64_t sacc[4] = {0, 0, 0, 0};
      uint32_t pk[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float x0, x1;
          ptx::unpack2(ptx::fma2(ptx::pack2(__uint_as_float(sr[c][2 * i]), __uint_as_float(sr[c][2 * i + 1])), cc, nm),
                       x0, x1);
          const float p0 = fast_exp2(x0), p1 = fast_exp2(x1);
          sacc[i % 4] = ptx::add2(sacc[i % 4], ptx::pack2(p0, p1));
          pk[c][i] = ptx::cvt_bf16x2(p0, p1);  // low half = even column
        }
      float s0, s1, s2, s3, s4, s5, s6, s7;
      ptx::unpack2(ptx::add2(sacc[0], sacc[1]), s0, s1);
      ptx::unpack2(ptx::add2(sacc[2], sacc[3]), s2, s3);
      (void)s4; (void)s5; (void)s6; (void)s7;
      const float sum = (s0 + s1) + (s2 + s3);
      l = l * alpha + sum;
      if (n >= 1) {
        ptx::mbar_wait(pv_done, (n - 1) & 1);  // PV(n-1) has landed in O
        ptx::tc_fence_after();
        if (any) {  // rare: rescale the O row by alpha
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t orow[32];
            ptx::tmem_ld32(tmem + lane_base + COL_O + c * 32, orow);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) orow[i] = __float_as_uint(__uint_as_float(orow[i]) * alpha);
            ptx::tmem_st32(tmem + lane_base + COL_O + c * 32, orow);
          }
        }
      }
      // P(n) -> first 64 columns of its S buffer (bf16 pairs)
      {
        uint32_t a[32], b[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          a[i] = pk[0][i];
          a[16 + i] = pk[1][i];
          b[i] = pk[2][i];
          b[16 + i] = pk[3][i];
        }
        ptx::tmem_st32(sbuf, a);
        ptx::tmem_st32(sbuf + 32, b);
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::warp_arrive(&p_full[n & 1]);
    }
    // ---- epilogue: O / l and LSE = (m2 + log2 l) ln 2
    ptx::mbar_wait(pv_done, (nblk - 1) & 1);
    ptx::tc_fence_after();
    const int64_t rr = row0 + r;
    const bool live = rr < n_rows;
    int64_t seq = 0;
    int h = 0;
    if (live) {
      seq = P.seq_list ? P.seq_list[task.seq_off + rr / P.g] : rr / P.g;
      h = j * P.g + (int)(rr % P.g);
    }
    const float inv = 1.f / l;
    float *orow_g = P.o + out_slot * P.o_slot_stride + (seq * P.Hq + h) * HD;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t orow[32];
      ptx::tmem_ld32(tmem + lane_base + COL_O + c * 32, orow);
      ptx::tmem_ld_wait();
      if (live) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4 *>(orow_g + c * 32 + i) =
              make_float4(__uint_as_float(orow[i]) * inv, __uint_as_float(orow[i + 1]) * inv,
                          __uint_as_float(orow[i + 2]) * inv, __uint_as_float(orow[i + 3]) * inv);
      }
    }
    if (live) P.lse[out_slot * P.lse_slot_stride + seq * P.Hq + h] = (m2 + log2f(l)) * HYDRA_LN2;
    if (P.fc.cnt) tc1_fused_arrive(P.fc, live, seq, h, P.Hq, lane);
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
static bool make_kv_map(CUtensorMap *m, const void *base, int64_t T, int Hkv, int64_t st, int64_t sh) {
  const uint64_t dims[3] = {(uint64_t)tc::HD, (uint64_t)Hkv, (uint64_t)T};
  const uint64_t strides[2] = {(uint64_t)sh * 2, (uint64_t)st * 2};
  const uint32_t box[3] = {64, 1, (uint32_t)tc::BN};
  return encode_bf16_map(m, 3, base, dims, strides, box);
}

bool prefix_tc_supported(const hydra_heads *h) {
  return h->dtype == HYDRA_BF16 && h->head_dim == 128 && tensor_maps_available();
}

template <int NS>
static cudaError_t set_smem_attr() {
  return ensure_smem_attr(reinterpret_cast<const void *>(prefix_tc_kernel<NS>), tc::Smem<NS>::ALLOC);
}

hydra_status launch_prefix_tc(const PrefixTcArgs &a, cudaStream_t s) {
  const int stages = a.stages == 2 ? 2 : 3;
  if ((stages == 2 ? set_smem_attr<2>() : set_smem_attr<3>()) != cudaSuccess) return HYDRA_ECUDA;
  PrefixTcKernelParams P;
  memset(&P, 0, sizeof(P));
  if (a.kv_total > 0) {
    if (!make_kv_map(&P.tmK, a.k, a.kv_total, a.Hkv, a.kv_st, a.kv_sh)) return HYDRA_ECUDA;
    if (!make_kv_map(&P.tmV, a.v, a.kv_total, a.Hkv, a.kv_st, a.kv_sh)) return HYDRA_ECUDA;
  }
  P.q = reinterpret_cast<const __nv_bfloat16 *>(a.q);
  P.q_sb = a.q_sb;
  P.q_sh = a.q_sh;
  P.Hq = a.Hq;
  P.Hkv = a.Hkv;
  P.g = a.g;
  P.scale_log2 = a.scale_log2;
  P.P = a.P;
  P.B = a.B;
  P.tasks = a.tasks;
  P.seq_list = a.seq_list;
  P.n_splits = a.n_splits;
  P.o = a.o;
  P.lse = a.lse;
  P.o_slot_stride = a.o_slot_stride;
  P.lse_slot_stride = a.lse_slot_stride;
  P.debug_variant = a.debug_variant;
  P.fc = a.fc;
  if (P.fc.cnt && (a.tasks || P.fc.n_pre_splits != a.n_splits || P.fc.sk_total != 0)) return HYDRA_EINVAL;
  const int n_x = a.tasks ? a.n_tasks : (int)(((int64_t)a.B * a.g + tc::BM - 1) / tc::BM);
  if (n_x == 0) return HYDRA_OK;
  const dim3 grid(n_x, a.Hkv, a.n_splits);
  if (stages == 2)
    prefix_tc_kernel<2><<<grid, tc::kThreads, tc::Smem<2>::ALLOC, s>>>(P);
  else
    prefix_tc_kernel<3><<<grid, tc::kThreads, tc::Smem<3>::ALLOC, s>>>(P);
  return cudaGetLastError() == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

}  // namespace hydra

// suffix_short.cu -- tensor-core suffix attention for SHORT grouped-query suffixes (sm_100a).
//
// PAPER.md §3.2: the suffix is "computed normally, with a single query per sequence" --
// a memory-bound GEMV per (sequence b, KV head j) over lens[b] tokens, here with the g query
// heads of the KV group as the N dimension of the MMAs (every K/V byte read once for g heads):
//   S^T [128 tokens x N] = K_tile [128 x 128] . Q^T          (tcgen05.mma, M = 128)
//   O^T [128 dims x N]  += V_tile^T [128 x 128 tokens] . P^T  (A operand MN-major)
// Same operand layouts and arithmetic as suffix_tc.cu; a different schedule.
//
// Why a second kernel: with one-tile items (C6: 1024 items of 128 tokens x g = 8 heads; C4: 4096
// items, g = 4) the persistent warp-specialised kernel streamed 2.5-4.7 TB/s.  Its CTA-0
// timeline (tools/suffix_trace.py) shows ~3000 cycles per 64-KB item, set by the softmax warps'
// per-item chain (max, exp, P^T, item hand-off ~1000 cycles, i-cache misses of a 6 K-instruction
// kernel), with only one CTA per SM to hide it.  Here a CTA is one control warp plus four
// softmax / epilogue warps (160 threads, one K and one V stage, ~71 KB of shared memory), so
// THREE CTAs share an SM and their independent chains hide each other's latency, while each
// CTA still prefetches its next K tile during the softmax and its next V tile during the next
// item's score MMAs.
//
// Roles per CTA:
//   warp 0   control: lane 0 issues the TMA loads (K, V, Q^T of an item) and all MMAs -- S(c)
//            as soon as K(c) lands, the next K tile once S(c) has read K(c); PV(c) once P^T
//            and V(c) are ready, the next V tile once PV(c) has read V(c); all 32 lanes zero
//            the V rows past lens[b] of a ragged last block (0 * NaN would poison O)
//   warps 1-4 softmax (thread = token = TMEM lane of S^T): one round per item over its <= 2
//            blocks (max per head through warp shuffles + shared memory, exp2, P^T as bf16
//            into shared memory), then the item's epilogue (thread = head dim = TMEM lane of
//            O^T): O / l, LSE, coalesced 512-B row stores.
// Items (b, j) are dealt round-robin to the CTAs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"
#include "fused.cuh"

namespace hydra {

// (SuffixTcParams is declared in suffix_tc.cu's translation unit; this kernel takes its own.)
struct __align__(64) SuffixShortParams {
  CUtensorMap tmK, tmV, tmQ;
  const int32_t *lens;
  int32_t B, Hq, Hkv;
  float scale_log2;
  int32_t n_items;
  int32_t S_cap;
  float *o, *lse;
  int32_t mutate;                // testing build only: 2 = CTA 0 skips head 0's store of its first item
  unsigned long long *timer;     // measurement: [0] min CTA start, [1] max CTA end (%globaltimer ns)
};

namespace ssh {
constexpr int BT = 128;             // tokens per block
constexpr int HD = 128;             // head dim
constexpr int NR = 8;               // rows of the Q^T / P^T operands (g <= 8 heads, zero-padded): UMMA N = 8
constexpr int NC = 16;              // TMEM columns per S^T block / O^T (the suffix_tc.cu layout)
constexpr int kThreads = 160;
constexpr int PANEL = BT * 128;     // 128 rows x 128 B
constexpr int TILE = 2 * PANEL;     // 32 KB
constexpr int QPANEL = NR * 128;    // 8 rows x 64 dims
constexpr int QTILE = 2 * QPANEL;   // 2 KB
constexpr int PPANEL = NR * 128;    // P^T: 8 rows x 64 tokens
constexpr int PTILE = 2 * PPANEL;   // 2 KB per 128-token block
constexpr int OFF_K = 0;
constexpr int OFF_V = OFF_K + TILE;
constexpr int OFF_Q = OFF_V + TILE;
constexpr int OFF_P = OFF_Q + QTILE;                   // P^T of the item's (up to) two blocks
constexpr int OFF_RED = OFF_P + 2 * PTILE;             // [4 warps][NC] block max + [4][NC] item sums
constexpr int OFF_BAR = OFF_RED + 2 * 4 * NC * 4;
constexpr int N_BARS = 9;  // k_full, k_empty, v_full, v_empty, q_full, s_full, p_full, pv_done, o_full
constexpr int BYTES = OFF_BAR + N_BARS * 8 + 16;
constexpr int ALLOC = BYTES + 1024;
constexpr int kCtasPerSm = 3;
static_assert(kCtasPerSm * (ALLOC + 1024) <= 233472, "suffix_short: three CTAs must fit an SM's shared memory");
constexpr uint32_t TMEM_COLS = 64;  // S^T blocks 0 / 1 at [0,16) [16,32), O^T at [32,48)
constexpr uint32_t O_COL = 32;
}  // namespace ssh

// One item = one sequence b and KV head j, all of its (<= 2) blocks in ONE softmax round: the
// arithmetic of suffix_tc.cu with CB = 2 (one max over the round, the same exp2 / bf16 P^T /
// row-sum order, the PV MMAs block after block, the same L sum), so both kernels give the same
// bits and the paged (suffix_tc) and contiguous calls of one step stay bitwise identical.
template <int G>
__global__ void __launch_bounds__(ssh::kThreads, ssh::kCtasPerSm)
    suffix_short_kernel(const __grid_constant__ SuffixShortParams P) {
  using namespace ssh;
  static_assert(G <= NR, "short-suffix kernel: g <= 8");
  extern __shared__ uint8_t smem_raw[];
  if (P.timer && threadIdx.x == 0) atomicMin(P.timer, gtimer());
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *k_full = bars, *k_empty = bars + 1, *v_full = bars + 2, *v_empty = bars + 3, *q_full = bars + 4;
  uint64_t *s_full = bars + 5, *p_full = bars + 6, *pv_done = bars + 7, *o_full = bars + 8;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + N_BARS);
  float *red_max = reinterpret_cast<float *>(smem + OFF_RED);  // [4][NC]
  float *red_sum = red_max + 4 * NC;                            // [4][NC]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  // Q^T and P^T rows >= g (padding heads) must read as zero
  for (int i = threadIdx.x; i < (QTILE + 2 * PTILE) / 16; i += kThreads)
    reinterpret_cast<uint4 *>(smem + OFF_Q)[i] = make_uint4(0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&P.tmK);
    ptx::prefetch_tmap(&P.tmV);
    ptx::prefetch_tmap(&P.tmQ);
    for (int i = 0; i < N_BARS; ++i) ptx::mbar_init(&bars[i], i == 6 ? 4 : 1);  // p_full: one arrival per softmax warp
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================= control warp: TMA loads and MMAs from lane 0; ragged V rows zeroed by all lanes =====
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(BT, NR, false);                // A = K, B = Q^T
    constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(HD, NR, false) | (1u << 15);  // A = V^T (MN-major)
    const bool l0 = lane == 0;
    // blocks of this CTA's non-empty items in order: (item, block c)
    int k_item = blockIdx.x, k_c = 0, k_nblk = 0;  // next K tile to load
    int v_item = blockIdx.x, v_c = 0, v_nblk = 0;  // next V tile to load
    auto nblk_of = [&](int it) { return (min(max(__ldg(P.lens + it / P.Hkv), 0), P.S_cap) + BT - 1) / BT; };
    auto seek = [&](int &it, int &c, int &nb) {  // (it, c) -> the next existing block at or after it
      while (it < P.n_items) {
        if (c == 0) nb = nblk_of(it);
        if (c < nb) return true;
        it += gridDim.x;
        c = 0;
      }
      return false;
    };
    auto load_k = [&]() {  // the next K tile (and, for an item's first block, its Q^T)
      if (!seek(k_item, k_c, k_nblk)) return;
      const int b = k_item / P.Hkv, j = k_item % P.Hkv;
      if (l0) {
        if (k_c == 0) {
          ptx::mbar_arrive_expect_tx(q_full, 2 * 64 * G * 2);
          ptx::tma_load_3d(smem + OFF_Q, &P.tmQ, q_full, 0, j * G, b);
          ptx::tma_load_3d(smem + OFF_Q + QPANEL, &P.tmQ, q_full, 64, j * G, b);
        }
        ptx::mbar_arrive_expect_tx(k_full, TILE);
        ptx::tma_load_4d(smem + OFF_K, &P.tmK, k_full, 0, j, k_c * BT, b);
        ptx::tma_load_4d(smem + OFF_K + PANEL, &P.tmK, k_full, 64, j, k_c * BT, b);
      }
      ++k_c;
    };
    auto load_v = [&]() {
      if (!seek(v_item, v_c, v_nblk)) return;
      const int b = v_item / P.Hkv, j = v_item % P.Hkv;
      if (l0) {
        ptx::mbar_arrive_expect_tx(v_full, TILE);
        ptx::tma_load_4d(smem + OFF_V, &P.tmV, v_full, 0, j, v_c * BT, b);
        ptx::tma_load_4d(smem + OFF_V + PANEL, &P.tmV, v_full, 64, j, v_c * BT, b);
      }
      ++v_c;
    };
    load_k();
    load_v();
    const uint32_t q_addr = ptx::smem_u32(smem + OFF_Q), k_addr = ptx::smem_u32(smem + OFF_K);
    const uint32_t v_addr = ptx::smem_u32(smem + OFF_V), p_addr = ptx::smem_u32(smem + OFF_P);
    uint32_t kb = 0, vb = 0, it_no = 0;  // K tiles, V tiles, items consumed
    for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
      const int len = min(max(__ldg(P.lens + item / P.Hkv), 0), P.S_cap);
      const int nb = (len + BT - 1) / BT;
      if (nb == 0) continue;
      // S^T(c) = K(c) . Q^T for the item's blocks; K(c+1) / the next item's K load behind each
      ptx::mbar_wait(q_full, it_no & 1);
      for (int c = 0; c < nb; ++c, ++kb) {
        ptx::mbar_wait(k_full, kb & 1);
        if (l0) {
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            ptx::mma_ss(tmem + c * NC, ptx::smem_desc_sw128(k_addr + (kk / 4) * PANEL + (kk % 4) * 32, 16, 1024),
                        ptx::smem_desc_sw128(q_addr + (kk / 4) * QPANEL + (kk % 4) * 32, 16, 1024), idesc_s, kk > 0);
          if (c + 1 == nb) ptx::mma_commit(s_full);
          ptx::mma_commit(k_empty);  // K(c) (and, at the last block, Q^T) read
        }
        __syncwarp();
        ptx::mbar_wait(k_empty, kb & 1);
        load_k();  // streams during the softmax
      }
      // O^T = sum_c V(c)^T . P^T(c)
      ptx::mbar_wait(p_full, it_no & 1);
      for (int c = 0; c < nb; ++c, ++vb) {
        ptx::mbar_wait(v_full, vb & 1);
        const int valid = len - c * BT;
        if (valid < BT) {  // ragged last block: zero V rows valid..127 (0 * NaN would poison O)
          for (int i = lane; i < (BT - valid) * 16; i += 32) {
            const int row = valid + i / 16, ch = i % 16;
            *reinterpret_cast<uint4 *>(smem + OFF_V + (ch / 8) * PANEL + row * 128 + (ch % 8) * 16) = make_uint4(0, 0, 0, 0);
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
        }
        if (l0) {
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BT / 16; ++kk)
            ptx::mma_ss(tmem + O_COL, ptx::smem_desc_sw128(v_addr + kk * 2048, PANEL, 1024),
                        ptx::smem_desc_sw128(p_addr + c * PTILE + (kk / 4) * PPANEL + (kk % 4) * 32, 16, 1024),
                        idesc_pv, (c > 0 || kk > 0) ? 1u : 0u);
          ptx::mma_commit(v_empty);
          if (c + 1 == nb) {
            ptx::mma_commit(pv_done);  // P^T slots free
            ptx::mma_commit(o_full);
          }
        }
        __syncwarp();
        ptx::mbar_wait(v_empty, vb & 1);
        load_v();  // streams during the next item's score MMAs and softmax
      }
      ++it_no;
    }
  } else {
    // ================= softmax (thread = token) + epilogue (thread = head dim) =================
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const float c2 = P.scale_log2;
    const int cc = (r % 64) / 8, e = r % 8;
    uint32_t item_no = 0;
    for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
      const int b = item / P.Hkv, j = item % P.Hkv;
      const int len = min(max(__ldg(P.lens + b), 0), P.S_cap);
      const int nb = (len + BT - 1) / BT;
      const int64_t row0 = (int64_t)b * P.Hq + (int64_t)j * G;
      if (nb == 0) {  // empty suffix: the (0, -inf) part
#pragma unroll
        for (int h = 0; h < G; ++h) {
          P.o[(row0 + h) * HD + r] = 0.f;
          if (r == h) P.lse[row0 + h] = -INFINITY;
        }
        continue;
      }
      ptx::mbar_wait(s_full, item_no & 1);
      ptx::tc_fence_after();
      uint32_t sv[2][NC];
      ptx::tmem_ld16(tmem + lane_base, sv[0]);
      if (nb > 1) ptx::tmem_ld16(tmem + lane_base + NC, sv[1]);
      ptx::tmem_ld_wait();
      bool tok[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) tok[c] = c < nb && c * BT + r < len;
      float s[2][G];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float x = -INFINITY;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          s[c][h] = tok[c] ? __uint_as_float(sv[c][h]) : -INFINITY;
          x = fmaxf(x, s[c][h]);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
        if (lane == 0) red_max[quarter * NC + h] = x;
      }
      ptx::named_bar_sync(1, 128);
      float m[G], l[G];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        // the round max (suffix_tc.cu's first round: m = -inf is always raised, l = 0 * 0 + acc)
        m[h] = fmaxf(fmaxf(red_max[h], red_max[NC + h]), fmaxf(red_max[2 * NC + h], red_max[3 * NC + h])) * c2;
      }
      float p[2][G];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          p[c][h] = tok[c] ? fast_exp2(fmaf(s[c][h], c2, -m[h])) : 0.f;
          acc += p[c][h];
        }
        l[h] = acc;
      }
      // P^T slots were last read by the previous item's PV MMAs
      if (item_no > 0) ptx::mbar_wait(pv_done, (item_no - 1) & 1);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c >= nb) break;
        uint8_t *sp = smem + OFF_P + c * PTILE + (r / 64) * PPANEL;
#pragma unroll
        for (int h = 0; h < G; ++h)
          *reinterpret_cast<__nv_bfloat16 *>(sp + h * 128 + ((cc ^ (h % 8)) * 16) + e * 2) = __float2bfloat16_rn(p[c][h]);
      }
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      ptx::warp_arrive(p_full);
      // ---- epilogue: L = sum over the item's tokens, O = O^T / L, LSE (natural log)
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float x = l[h];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) red_sum[quarter * NC + h] = x;
      }
      ptx::named_bar_sync(1, 128);
      float L[G];
#pragma unroll
      for (int h = 0; h < G; ++h) L[h] = red_sum[h] + red_sum[NC + h] + red_sum[2 * NC + h] + red_sum[3 * NC + h];
      ptx::mbar_wait(o_full, item_no & 1);
      ptx::tc_fence_after();
      uint32_t ov[NC];
      ptx::tmem_ld16(tmem + lane_base + O_COL, ov);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      const bool skip0 = kTesting && P.mutate == 2 && blockIdx.x == 0 && item_no == 0;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        if (!(skip0 && h == 0)) P.o[(row0 + h) * HD + r] = __uint_as_float(ov[h]) / L[h];
        if (r == h) P.lse[row0 + h] = (m[h] + log2f(L[h])) * HYDRA_LN2;
      }
      // red_max / red_sum are rewritten after the next item's first named barrier, which every
      // thread reaches only after its reads above
      ++item_no;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem);
  }
  if (P.timer && threadIdx.x == 0) atomicMax(P.timer + 1, gtimer());
  // As a programmatic dependent of the prefix kernel: complete only after it.  Only the last CTA
  // in launch order waits (decode.cu): the others exit and free their slot for later CTAs, so
  // the SMs the prefix leaves idle keep working through the grid while the prefix runs.
  asm volatile("griddepcontrol.launch_dependents;");  // the combine may launch as the last CTAs drain
  if (blockIdx.x == gridDim.x - 1) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ------------------------------------------------------------------ host side
bool suffix_short_supported(int g, int64_t S_cap) {
  return (g == 2 || g == 4 || g == 8) && S_cap > 0 && S_cap <= 2 * ssh::BT;
}

template <int G>
static cudaError_t launch_g(const SuffixShortParams &P, int grid, bool pdl, cudaStream_t s) {
  const cudaError_t attr = ensure_smem_attr(reinterpret_cast<const void *>(suffix_short_kernel<G>), ssh::ALLOC);
  if (attr != cudaSuccess) return attr;
  return launch_maybe_pdl(suffix_short_kernel<G>, dim3(grid), dim3(ssh::kThreads), ssh::ALLOC, s, pdl, P);
}

hydra_status launch_suffix_short(const SuffixTcArgs &a, int n_ctas, cudaStream_t s) {
  const int g = a.Hq / a.Hkv;
  if (a.block_table || a.n_split > 1 || a.fc.cnt || !suffix_short_supported(g, a.S_cap)) return HYDRA_EINVAL;
  SuffixShortParams P;
  memset(&P, 0, sizeof(P));
  {
    const uint64_t dims[4] = {(uint64_t)ssh::HD, (uint64_t)a.Hkv, (uint64_t)a.S_cap, (uint64_t)a.B};
    const uint64_t strides[3] = {(uint64_t)a.s_sh * 2, (uint64_t)a.s_st * 2, (uint64_t)a.s_sb * 2};
    const uint32_t box[4] = {64, 1, (uint32_t)ssh::BT, 1};
    if (!encode_bf16_map(&P.tmK, 4, a.k, dims, strides, box)) return HYDRA_ECUDA;
    if (!encode_bf16_map(&P.tmV, 4, a.v, dims, strides, box)) return HYDRA_ECUDA;
  }
  {
    const uint64_t dims[3] = {(uint64_t)ssh::HD, (uint64_t)a.Hq, (uint64_t)a.B};
    const uint64_t strides[2] = {(uint64_t)a.q_sh * 2, (uint64_t)a.q_sb * 2};
    const uint32_t box[3] = {64, (uint32_t)g, 1};
    if (!encode_bf16_map(&P.tmQ, 3, a.q, dims, strides, box)) return HYDRA_ECUDA;
  }
  P.lens = a.lens;
  P.B = a.B;
  P.Hq = a.Hq;
  P.Hkv = a.Hkv;
  P.scale_log2 = a.scale_log2;
  P.n_items = a.B * a.Hkv;
  P.S_cap = (int32_t)a.S_cap;
  P.o = a.o;
  P.lse = a.lse;
  P.mutate = kTesting ? a.mutate : 0;
  P.timer = a.timer;
  if (P.n_items == 0) return HYDRA_OK;
  const int grid = std::min(P.n_items, n_ctas > 0 ? n_ctas : ssh::kCtasPerSm * device_sm_count());
  const bool pdl = a.pdl != 0;
  cudaError_t e = cudaErrorInvalidValue;
  switch (g) {
    case 2: e = launch_g<2>(P, grid, pdl, s); break;
    case 4: e = launch_g<4>(P, grid, pdl, s); break;
    case 8: e = launch_g<8>(P, grid, pdl, s); break;
  }
  return e == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

}  // namespace hydra

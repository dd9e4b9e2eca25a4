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
// every K/V byte g times.  One CTA per SM (persistent, 448 threads), one warp per job so
// that no stage ever waits behind another kind of slot:
//   warp 0      TMA producer, K ring (3 x 32 KB; a slot frees once its score MMA is done)
//   warp 6      TMA producer, V ring (3 x 32 KB; a slot frees once its PV MMA is done)
//   warp 7      TMA producer, Q^T slots (the g query rows of an item)
//   warp 1      TMEM allocator + score-MMA issuer: S^T(n) as soon as K(n) lands and the
//               softmax has consumed S^T slot n % 3
//   warp 12     PV-MMA issuer: O^T += V^T P^T as soon as P^T(n) and V(n) are ready
//   warp 13     paged cache only: block-table entries of upcoming tiles -> smem ring (cp.async)
//   warps 2-5   softmax (thread = token lane): per round of CB blocks a block max per head
//               (warp shuffles + smem across the 4 warps), the stale-max rule of the prefix
//               kernel (rescale only when the max grows by > 8, log2 units), P^T as bf16
//               into shared memory (B operand of the PV MMA)
//   warps 8-11  epilogue (thread = head dim): O^T / l, LSE, coalesced stores, after the
//               item's last PV -- off the softmax warps' critical path
// Reads lens[b] itself, so only blocks with valid tokens move.  Tokens >= lens[b] inside
// the last block: their scores are masked to -inf, and the PV warp zeroes their V rows in
// shared memory before the PV MMA (0 * NaN would poison O).
// Per-SM rate (tools/suffix_rate.py, C3 shape): 112 GB/s at 16 CTAs, 100 at 64; 7.0 TB/s
// on 80-92 SMs.  The earlier single-issuer version (S(n) then PV(n-1) from one thread,
// epilogue on the softmax warps) coupled every V slot release to the next K tile and the
// softmax chain: 60-73 GB/s per SM (profiles/r1d_suffix_streaming.md).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"
#include "fused.cuh"

namespace hydra {

namespace stc {
constexpr int BT = 128;   // tokens per block (UMMA M of S^T, K of PV)
constexpr int HD = 128;   // head dim (UMMA K of S^T, M of PV)
constexpr int NQ = 16;    // padded query heads per KV group (smem / TMEM layout)
// UMMA N actually issued: the g heads padded to 8 when g <= 8 -- the rows past g are zero, and
// an MHA GEMV at N = 16 spent 16x the useful tensor work (energy under the 1 kW cap)
#ifndef HYDRA_SUFFIX_MMA_N8
#define HYDRA_SUFFIX_MMA_N8 1
#endif
template <int G>
constexpr int kMmaN = (HYDRA_SUFFIX_MMA_N8 && G <= 8) ? 8 : 16;
constexpr int NS = 3;     // K stages and V stages (separate rings: K frees after S, V after PV)
constexpr int kThreads = 448;  // warp 0 K producer, 1 score MMA, 2-5 softmax, 6 V producer, 7 Q producer,
                               // 8-11 epilogue, 12 PV MMA, 13 paged-cache block-table loader
constexpr int PANEL = BT * 128;      // 128 rows x 128 B
constexpr int TILE = 2 * PANEL;      // 32 KB
constexpr int QPANEL = NQ * 128;     // 2 KB: 16 rows x 64 dims
constexpr int QTILE = 2 * QPANEL;    // 4 KB
constexpr int PPANEL = NQ * 128;     // P^T: 16 rows x 64 tokens
constexpr int PTILE = 2 * PPANEL;    // 4 KB per 128-token block
constexpr int OFF_K = 0;
constexpr int OFF_V = OFF_K + NS * TILE;
constexpr int OFF_Q = OFF_V + NS * TILE;     // 2 slots
// Round slots (S^T in TMEM, P^T in smem): the score MMA may run nsp rounds ahead of the PV
// MMA, so a round's softmax is done long before its V tile lands and a V slot is held for
// little more than the load latency (SM-budget measurements, tools/suffix_trace.py).
// Q slots: items the score MMA may be ahead of the PV MMA, plus one.
__host__ __device__ constexpr int nsp(int cb) { return 3; }
__host__ __device__ constexpr int nqs(int cb) { return cb == 1 ? 3 : 2; }
__host__ __device__ constexpr int off_p(int cb) { return OFF_Q + nqs(cb) * QTILE; }
__host__ __device__ constexpr int off_red(int cb) { return off_p(cb) + nsp(cb) * cb * PTILE; }
// [2 round parity][4 warps][16] max + [2 item parity][4][16] sums
__host__ __device__ constexpr int off_bar(int cb) { return off_red(cb) + (2 * 4 * NQ + 2 * 4 * NQ + 2 * NQ) * 4; }
// k_full, k_empty, v_full, v_empty [NS]; q_full, q_empty [4]; s_full, p_full, pv_done [4];
// o_free, o_full, ml_full [2]
constexpr int N_BARS = 4 * NS + 8 + 12 + 6;
// Paged cache: a ring of PR tiles' page ids (16 sub-tiles max) shared by the K and V
// producers, filled with cp.async by warp 13 (tab_full / tab_empty barriers).
constexpr int PR = 6;
__host__ __device__ constexpr int off_tab(int cb) { return off_bar(cb) + N_BARS * 8 + 16; }
__host__ __device__ constexpr int alloc_bytes(int cb) { return off_tab(cb) + PR * (16 * 4 + 16) + 1024; }
static_assert(alloc_bytes(1) <= 232448 && alloc_bytes(2) <= 232448, "suffix_tc smem over the 227 KB opt-in limit");
// S^T x 2 round slots x CB blocks (16 columns each), O^T x 2; rounded up to a power of two
__host__ __device__ constexpr uint32_t tmem_cols(int cb) { return 128u; }  // nsp*cb*16 + 2*16 <= 128
}  // namespace stc

struct __align__(64) SuffixTcParams {
  CUtensorMap tmK, tmV, tmQ;
  const int32_t *lens;
  int32_t B, Hq, Hkv, g;
  float scale_log2;
  int32_t n_items;
  float *o, *lse;
  int32_t S_cap;     // lens[b] is clamped to [0, S_cap] (hydra.h precondition; release and testing)
  int32_t mutate;    // testing build only: 2 = CTA 0's epilogue skips head 0's store of its first item
  int32_t debug;     // testing build only, timing experiments (invalid results): 256 = the MMA warp releases K/V
                     // tiles as they land (no MMA, no softmax), 512 = no softmax work,
                     // 4096 / 8192 = no score / PV MMA instructions
  long long *trace;  // diagnostics: CTA 0 event timestamps [kTraceRows][kTraceN] (tools/suffix_trace.py); null = off
  // Paged cache (null = contiguous [B, S_cap, Hkv, d]): tmK / tmV then map the page pools
  // [n_pages, page_size, Hkv, d] with a box of pbox = min(page_size, BT) tokens, and token t of
  // sequence b is row t % page_size of page block_table[b * bt_stride + t / page_size].
  const int32_t *block_table;
  int64_t bt_stride;
  int32_t page_shift, pbox_shift;  // log2(page_size), log2(pbox)
  // split-K over tokens: item = (b * Hkv + j) * n_split + sp covers tokens
  // [sp * split_len, (sp + 1) * split_len) of sequence b; its (O, LSE) go to slot sp
  int32_t n_split, split_len;
  int64_t o_split_stride, lse_split_stride;
  FusedCombine fc;  // fc.cnt != null: the epilogue warps count each row's part and merge completed rows
  int32_t pdl;      // host only: launch as a programmatic dependent of the previous kernel in the stream
  unsigned long long *timer;  // measurement: [0] min CTA start, [1] max CTA end (%globaltimer ns); null = off
};
namespace stc {
constexpr int kTraceN = 1024;
// trace rows: 0 softmax s_full wait begin, 1 s_full acquired, 2 scores loaded, 3 block max done,
// 4 P^T published (p_full arrive), 5 / 6 softmax item end before / after its o_free wait
// (indexed by item), 7 MMA S round committed,
// 8 MMA PV round committed, 9 K TMA issued (block), 10 V TMA issued (block), 11 / 12 MMA thread
// sees K / V landed (block)
__device__ __forceinline__ void trace(long long *tr, int row, uint32_t i) {
  if (kTesting && tr && i < (uint32_t)kTraceN) tr[row * kTraceN + i] = clock64();
}
}  // namespace stc

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// lens[b] of the item this CTA handles `k` steps ahead (0 when past the end): every role
// fetches the next item's length one item early so the load is off the critical path.
// The roles keep the raw lens[b] of their next item (item_len_raw, a bare load whose value is
// first used one item later) and derive the item's token count at use (item_len_of): clamping
// right after the load could make an item transition wait for it.  (The softmax warps still
// spend ~1000 cycles between an item's end and the next item's first wait on one-tile GQA
// items, tools/suffix_trace.py FIRST=7 -- not this load.  ncu at that shape
// (profiles/r1n_suffix_tc_c6shape_raw.csv): 3.05 warps stalled on no_instruction per issue,
// next to 3.8 on barriers -- instruction-fetch misses: 5.1 K SASS instructions for G = 8,
// every role's per-item path executed once per ~2 us.  Unresolved.)
// SPLIT (compile time): split-K over tokens.  The unsplit instantiation keeps the plain
// item = b * Hkv + j arithmetic (the general form cost ~2 % of the C3 step, measured A/B).
template <bool SPLIT>
__device__ __forceinline__ int item_len_raw(const SuffixTcParams &P, int item) {
  return item < P.n_items ? __ldg(P.lens + (SPLIT ? item / P.n_split : item) / P.Hkv) : 0;
}
template <bool SPLIT>
__device__ __forceinline__ int item_len_of(const SuffixTcParams &P, int item, int raw) {
  raw = min(max(raw, 0), P.S_cap);  // out-of-range lens[b] (a precondition violation) is clamped
  if (!SPLIT) return raw;
  const int sp = item % P.n_split;
  return max(0, min(P.split_len, raw - sp * P.split_len));
}
template <bool SPLIT>
__device__ __forceinline__ int item_len(const SuffixTcParams &P, int item) {
  return item_len_of<SPLIT>(P, item, item_len_raw<SPLIT>(P, item));
}
// (sequence, KV head, first token, output offset in elements of o / lse) of an item
struct ItemRef {
  int b, j, t_base;
  int64_t o_off, lse_off;
};
template <bool SPLIT>
__device__ __forceinline__ ItemRef item_ref(const SuffixTcParams &P, int item) {
  if (!SPLIT) return {item / P.Hkv, item % P.Hkv, 0, 0, 0};
  const int bj = item / P.n_split, sp = item - bj * P.n_split;
  return {bj / P.Hkv, bj % P.Hkv, sp * P.split_len, sp * P.o_split_stride, sp * P.lse_split_stride};
}

// Paged cache: one lane of warp 13 walks the CTA's tile sequence (the one the K / V
// producers walk) up to PR tiles ahead of them and copies each tile's block-table entries into
// ring slot (tile % PR) with cp.async, tracked by tab_full[slot] (cp.async.mbarrier.arrive).
// Measured (tools/paged_rate.py, C3 suffix on 76 SMs): block-table loads in the producer
// thread, or this loop on a second lane of the producer warp, held the paged kernel at
// 3.6-4.0 TB/s even with identity pages; on its own warp 6.4-6.6 TB/s (pages >= 16).
template <bool SPLIT>
__device__ __forceinline__ void page_table_lane(const SuffixTcParams &P, int32_t *ring, uint64_t *tab_full,
                                                uint64_t *tab_empty) {
  uint32_t k = 0;
  for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
    const int len = item_len<SPLIT>(P, item);
    const int nblk = (len + stc::BT - 1) / stc::BT;
    const ItemRef ir = item_ref<SPLIT>(P, item);
    const int32_t *bt = P.block_table + (int64_t)ir.b * P.bt_stride;
    for (int n = 0; n < nblk; ++n, ++k) {
      const int slot = k % stc::PR;
      ptx::mbar_wait(&tab_empty[slot], ((k / stc::PR) & 1) ^ 1);
      const int t0 = ir.t_base + n * stc::BT;
      const int nsub = min(stc::BT >> P.pbox_shift, (ir.t_base + len - t0 + (1 << P.pbox_shift) - 1) >> P.pbox_shift);
      const uint32_t dst = ptx::smem_u32(ring + slot * 16);
      for (int c = 0; c < nsub; ++c)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst + 4 * c),
                     "l"(bt + ((t0 + (c << P.pbox_shift)) >> P.page_shift))
                     : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(ptx::smem_u32(&tab_full[slot]))
                   : "memory");
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Walks the rounds (up to CB consecutive 128-token blocks of one item) a CTA processes, in
// order, with the ring positions the producers use: gb = first block's ring index, gr =
// round index, qi / item_no = index of the item among this CTA's non-empty items.
template <int CB, bool SPLIT>
struct RoundCursor {
  int item, len, len_next, nblk, n0, nb;
  uint32_t gb, gr, qi, item_no;
  bool valid;
  __device__ __forceinline__ void seek(const SuffixTcParams &P) {  // first round of the next non-empty item
    while (item < P.n_items) {
      len = item_len_of<SPLIT>(P, item, len_next);
      len_next = item_len_raw<SPLIT>(P, item + gridDim.x);
      nblk = (len + stc::BT - 1) / stc::BT;
      if (nblk > 0) {
        n0 = 0;
        nb = min(CB, nblk);
        valid = true;
        return;
      }
      item += gridDim.x;
    }
    valid = false;
  }
  __device__ __forceinline__ void init(const SuffixTcParams &P) {
    item = blockIdx.x;
    len_next = item_len_raw<SPLIT>(P, item);
    gb = gr = qi = item_no = 0;
    seek(P);
  }
  __device__ __forceinline__ void next(const SuffixTcParams &P) {
    gb += nb;
    ++gr;
    n0 += nb;
    if (n0 < nblk) {
      nb = min(CB, nblk - n0);
      return;
    }
    ++qi;
    ++item_no;
    item += gridDim.x;
    seek(P);
  }
};

// G = query heads per KV group (compile-time: no per-head predicates).
// CB = 128-token blocks per softmax round: the softmax warps take one block max / barrier /
// P^T write per round of up to CB blocks (thread r owns tokens r, 128 + r, ...), so the
// per-round latency chain (S MMA -> TMEM load -> cross-warp max -> exp -> P^T -> PV MMA)
// is paid once per CB blocks.  Online softmax across the rounds of an item.
template <int G, int CB, bool SPLIT, bool PAGED>
__global__ void __launch_bounds__(stc::kThreads, 1) suffix_tc_kernel(const __grid_constant__ SuffixTcParams P) {
  using namespace stc;
  constexpr int OFF_P = off_p(CB), OFF_RED = off_red(CB), OFF_BAR = off_bar(CB);
  constexpr int NSP = nsp(CB), NQS = nqs(CB);
  constexpr uint32_t TMEM_COLS = tmem_cols(CB);
  constexpr uint32_t O_COL = NSP * CB * NQ;  // O^T buffers start after the S^T round slots
  extern __shared__ uint8_t smem_raw[];
  if (P.timer && threadIdx.x == 0) atomicMin(P.timer, gtimer());
  // diagnostics (testing build): every CTA's %globaltimer at entry / setup done / exit, rows 13-15
  long long *cta_tr = (kTesting && P.trace && blockIdx.x < kTraceN) ? P.trace + 13 * kTraceN + blockIdx.x : nullptr;
  if (cta_tr && threadIdx.x == 0) cta_tr[0] = (long long)gtimer();
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *k_full = bars, *k_empty = bars + NS, *v_full = bars + 2 * NS, *v_empty = bars + 3 * NS;
  uint64_t *q_full = bars + 4 * NS, *q_empty = q_full + 4, *s_full = q_full + 8, *p_full = q_full + 12,
           *pv_done = q_full + 16, *o_free = q_full + 20, *o_full = q_full + 22, *ml_full = q_full + 24;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + N_BARS);
  int32_t *tab_ring = reinterpret_cast<int32_t *>(smem + off_tab(CB));                  // [PR][16] page ids
  uint64_t *tab_full = reinterpret_cast<uint64_t *>(smem + off_tab(CB) + PR * 16 * 4);  // [PR]
  uint64_t *tab_empty = tab_full + PR;                                                   // [PR]
  float *red_max = reinterpret_cast<float *>(smem + OFF_RED);  // [2][4][NQ]
  float *red_sum = red_max + 2 * 4 * NQ;                        // [2][4][NQ] per-warp row-sum partials
  float *item_m = red_sum + 2 * 4 * NQ;                         // [2][NQ] running max per head (log2)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int g = G;

  // zero Q^T / P^T slots once: rows >= g (padding heads) must stay 0 forever
  for (int i = threadIdx.x; i < (NQS * QTILE + NSP * CB * PTILE) / 16; i += kThreads)
    reinterpret_cast<uint4 *>(smem + OFF_Q)[i] = make_uint4(0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&P.tmK);
    ptx::prefetch_tmap(&P.tmV);
    ptx::prefetch_tmap(&P.tmQ);
    for (int i = 0; i < PR; ++i) {
      ptx::mbar_init(&tab_full[i], 1);   // the table lane's cp.async arrival (noinc)
      ptx::mbar_init(&tab_empty[i], 2);  // K and V producers
    }
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], 4);  // one elected arrival per softmax warp
      ptx::mbar_init(&pv_done[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&o_free[i], 4);   // one elected arrival per epilogue warp
      ptx::mbar_init(&o_full[i], 1);   // tcgen05.commit after the item's last PV
      ptx::mbar_init(&ml_full[i], 4);  // one elected arrival per softmax warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (cta_tr && threadIdx.x == 0) cta_tr[kTraceN] = (long long)gtimer();

  if (warp == 13) {
    // ================= paged cache: block-table entries into the page-id ring =================
    if (PAGED && ptx::elect_one())
      page_table_lane<SPLIT>(P, tab_ring, tab_full, tab_empty);
  } else if (warp == 0 || warp == 6 || warp == 7) {
    // ================= TMA producers: warp 0 K ring, warp 6 V ring, warp 7 Q slots =================
    // Separate threads so no load waits behind another kind of slot (V slots free only after
    // the PV MMA, K slots right after the score MMA, Q slots after an item's last PV).
    if (ptx::elect_one()) {
      long long *tr = blockIdx.x == 0 ? P.trace : nullptr;
      uint32_t gb = 0, qi = 0;
      int len_next = item_len_raw<SPLIT>(P, blockIdx.x);
      for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
        const ItemRef ir = item_ref<SPLIT>(P, item);
        const int b = ir.b, j = ir.j;
        const int len = item_len_of<SPLIT>(P, item, len_next);
        len_next = item_len_raw<SPLIT>(P, item + gridDim.x);
        const int nblk = (len + BT - 1) / BT;
        if (nblk == 0) continue;
        if (warp == 7) {
          const int qs = qi % NQS;
          ptx::mbar_wait(&q_empty[qs], ((qi / NQS) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&q_full[qs], 2 * 64 * g * 2);
          uint8_t *sQ = smem + OFF_Q + qs * QTILE;
          ptx::tma_load_3d(sQ, &P.tmQ, &q_full[qs], 0, j * g, b);
          ptx::tma_load_3d(sQ + QPANEL, &P.tmQ, &q_full[qs], 64, j * g, b);
          ++qi;
          continue;
        }
        for (int n = 0; n < nblk; ++n, ++gb) {
          const int st = gb % NS;
          const uint32_t ph = ((gb / NS) & 1) ^ 1;
          const int t0 = ir.t_base + n * BT;  // first token of the tile in the sequence
          const CUtensorMap *tm = warp == 0 ? &P.tmK : &P.tmV;
          uint64_t *full = warp == 0 ? &k_full[st] : &v_full[st];
          uint8_t *dst = smem + (warp == 0 ? OFF_K : OFF_V) + st * TILE;
          if constexpr (!PAGED) {
            ptx::mbar_wait(warp == 0 ? &k_empty[st] : &v_empty[st], ph);
            ptx::mbar_arrive_expect_tx(full, TILE);
            ptx::tma_load_4d(dst, tm, full, 0, j, t0, b);
            ptx::tma_load_4d(dst + PANEL, tm, full, 64, j, t0, b);
          } else {
            // Paged: BT / pbox sub-tiles of pbox tokens, each inside one page.  Sub-tiles past
            // lens[b] are not loaded (their block-table entries need not be valid); the rows
            // they leave stale are masked like every row >= lens[b] (scores -> -inf, V rows
            // zeroed by the PV warp).  Each sub-tile lands at a multiple of pbox * 128 B
            // >= 1024 B, so the 128-B swizzle pattern equals that of one whole-tile load.
            const int ts = gb % PR;
            ptx::mbar_wait(&tab_full[ts], (gb / PR) & 1);  // this tile's page ids have landed
            const int nsub = min(BT >> P.pbox_shift, (ir.t_base + len - t0 + (1 << P.pbox_shift) - 1) >> P.pbox_shift);
            ptx::mbar_wait(warp == 0 ? &k_empty[st] : &v_empty[st], ph);
            ptx::mbar_arrive_expect_tx(full, (uint32_t)nsub * (256u << P.pbox_shift));
#pragma unroll 8
            for (int c = 0; c < nsub; ++c) {
              const int pg = tab_ring[ts * 16 + c];
              const int row = (t0 + (c << P.pbox_shift)) & ((1 << P.page_shift) - 1);
              uint8_t *d = dst + (c << P.pbox_shift) * 128;
              ptx::tma_load_4d(d, tm, full, 0, j, row, pg);
              ptx::tma_load_4d(d + PANEL, tm, full, 64, j, row, pg);
            }
            ptx::mbar_arrive(&tab_empty[ts]);
          }
          trace(tr, warp == 0 ? 9 : 10, gb);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (event-driven) =================
    // Two cursors over the same flat round sequence: the S cursor issues score MMAs as soon
    // as a round's K tiles land (at most two rounds ahead of the PV cursor: two S^T slots),
    // the PV cursor issues a round's PV MMAs as soon as its P^T and V tiles are ready.
    // Neither waits behind the other, so a V slot is held only for load + softmax + PV.
    const bool leader = ptx::elect_one();
    if (kTesting && leader && (P.debug & 256)) {  // drain only: release each tile as soon as it lands
      RoundCursor<CB, SPLIT> c;
      c.init(P);
      while (c.valid) {
        if (c.n0 == 0) ptx::mbar_wait(&q_full[c.qi % NQS], (c.qi / NQS) & 1);
        for (int i = 0; i < c.nb; ++i) {
          const uint32_t gbc = c.gb + i, st = gbc % NS;
          ptx::mbar_wait(&k_full[st], (gbc / NS) & 1);
          trace(blockIdx.x == 0 ? P.trace : nullptr, 11, gbc);
          ptx::mbar_arrive(&k_empty[st]);
          ptx::mbar_wait(&v_full[st], (gbc / NS) & 1);
          trace(blockIdx.x == 0 ? P.trace : nullptr, 12, gbc);
          ptx::mbar_arrive(&v_empty[st]);
        }
        if (c.n0 + c.nb >= c.nblk) ptx::mbar_arrive(&q_empty[c.qi % NQS]);
        c.next(P);
      }
    } else if (leader) {
      // ================= score-MMA issuer (warp 1; the PV MMAs are issued by warp 12) =================
      // S(n) needs K(n) landed and S^T slot n % NSP consumed by the softmax (p_full of round
      // n - NSP).  Two issuing threads, each blocking on one barrier at a time: a score MMA
      // never waits behind a V tile and a PV MMA never waits behind a K tile.
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(BT, kMmaN<G>, false);  // A=K, B=Q^T (K-major)
      long long *tr = blockIdx.x == 0 ? P.trace : nullptr;
      RoundCursor<CB, SPLIT> sc;
      sc.init(P);
      while (sc.valid) {
        if (sc.gr >= (uint32_t)NSP) ptx::mbar_wait(&p_full[sc.gr % NSP], ((sc.gr - NSP) / NSP) & 1);
        const uint32_t qs = sc.qi % NQS;
        if (sc.n0 == 0) ptx::mbar_wait(&q_full[qs], (sc.qi / NQS) & 1);
        const uint32_t q_addr = ptx::smem_u32(smem + OFF_Q + qs * QTILE);
        for (int c = 0; c < sc.nb; ++c) {
          const uint32_t gbc = sc.gb + c, st = gbc % NS;
          ptx::mbar_wait(&k_full[st], (gbc / NS) & 1);
          trace(tr, 11, gbc);
          ptx::tc_fence_after();
          const uint32_t k_addr = ptx::smem_u32(smem + OFF_K + st * TILE);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk / 4) * PANEL + (kk % 4) * 32, qoff = (kk / 4) * QPANEL + (kk % 4) * 32;
            ptx::mma_ss(tmem + ((sc.gr % NSP) * CB + c) * NQ, ptx::smem_desc_sw128(k_addr + off, 16, 1024),
                        ptx::smem_desc_sw128(q_addr + qoff, 16, 1024), idesc_s, kk > 0);
          }
          ptx::mma_commit(&k_empty[st]);
        }
        ptx::mma_commit(&s_full[sc.gr % NSP]);
        if (sc.n0 + sc.nb >= sc.nblk) ptx::mma_commit(&q_empty[qs]);  // the item's last score MMA
        trace(tr, 7, sc.gr);
        sc.next(P);
      }
    }
  } else if (warp == 12) {
    // ================= PV-MMA issuer (one elected lane issues; the warp zeroes ragged V rows) =================
    // V rows past lens[b] in an item's last block are zeroed here, after the tile landed and
    // before the PV MMA reads it (0 * NaN would poison O).  The softmax warps cannot do it:
    // they may run up to three rounds ahead of the V ring, where a parity wait on v_full
    // could not tell the tile's phase from the one two loads earlier.
    if (!(kTesting && (P.debug & 256))) {
      const bool leader = ptx::elect_one();
      constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(HD, kMmaN<G>, false) | (1u << 15);  // A=V^T (MN-major), B=P^T
      long long *tr = (blockIdx.x == 0 && leader) ? P.trace : nullptr;
      RoundCursor<CB, SPLIT> pc;
      pc.init(P);
      while (pc.valid) {
        const uint32_t slot = pc.gr % NSP, ob = pc.item_no & 1;
        ptx::mbar_wait(&p_full[slot], (pc.gr / NSP) & 1);
        if (pc.n0 == 0) ptx::mbar_wait(&o_free[ob], ((pc.item_no >> 1) & 1) ^ 1);
        const uint32_t p_base = ptx::smem_u32(smem + OFF_P + slot * CB * PTILE);
        for (int c = 0; c < pc.nb; ++c) {
          const uint32_t gbc = pc.gb + c, st = gbc % NS;
          ptx::mbar_wait(&v_full[st], (gbc / NS) & 1);
          trace(tr, 12, gbc);
          const int valid = pc.len - (pc.n0 + c) * BT;
          if (valid < BT) {  // ragged last block: zero rows valid..127 of both 64-column panels
            uint8_t *sV = smem + OFF_V + st * TILE;
            for (int i = lane; i < (BT - valid) * 16; i += 32) {
              const int row = valid + i / 16, ch = i % 16;
              *reinterpret_cast<uint4 *>(sV + (ch / 8) * PANEL + row * 128 + (ch % 8) * 16) = make_uint4(0, 0, 0, 0);
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
          }
          if (leader) {
            ptx::tc_fence_after();
            const uint32_t v_addr = ptx::smem_u32(smem + OFF_V + st * TILE);
            const uint32_t p_addr = p_base + c * PTILE;
#pragma unroll
            for (int kk = 0; kk < BT / 16; ++kk)
              ptx::mma_ss(tmem + O_COL + ob * NQ, ptx::smem_desc_sw128(v_addr + kk * 2048, PANEL, 1024),
                          ptx::smem_desc_sw128(p_addr + (kk / 4) * PPANEL + (kk % 4) * 32, 16, 1024), idesc_pv,
                          (pc.n0 > 0 || c > 0 || kk > 0));
            ptx::mma_commit(&v_empty[st]);
          }
          __syncwarp();
        }
        if (leader) {
          ptx::mma_commit(&pv_done[slot]);
          trace(tr, 8, pc.gr);
          if (pc.n0 + pc.nb >= pc.nblk) ptx::mma_commit(&o_full[ob]);
        }
        __syncwarp();
        pc.next(P);
      }
    }
  } else if (warp < 8 && !(kTesting && (P.debug & 256))) {
    // ================= softmax (thread = token lane) =================
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const float c2 = P.scale_log2;
    uint32_t gr = 0, gb = 0, item_no = 0;
    long long *tr = (blockIdx.x == 0 && quarter == 0 && lane == 0) ? P.trace : nullptr;
    int len_next = item_len_raw<SPLIT>(P, blockIdx.x);
    for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
      const ItemRef ir = item_ref<SPLIT>(P, item);
      const int len = item_len_of<SPLIT>(P, item, len_next);
      len_next = item_len_raw<SPLIT>(P, item + gridDim.x);
      const int nblk = (len + BT - 1) / BT;
      const int64_t row0 = (int64_t)ir.b * P.Hq + (int64_t)ir.j * g;
      if (nblk == 0) {  // empty suffix (or split): (0, -inf) sentinel (fused: written by the epilogue warps)
        if (P.fc.cnt) continue;
        for (int h = 0; h < g; ++h) {
          P.o[ir.o_off + (row0 + h) * HD + r] = 0.f;
          if (r == 0) P.lse[ir.lse_off + row0 + h] = -INFINITY;
        }
        continue;
      }
      const uint32_t ob = item_no & 1;
      const uint32_t o_tmem = tmem + lane_base + O_COL + ob * NQ;
      float m[G], l[G];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        m[h] = -INFINITY;
        l[h] = 0.f;
      }
      for (int n0 = 0; n0 < nblk; n0 += CB, ++gr) {
        const int nb = min(CB, nblk - n0);
        const uint32_t buf = gr % NSP;
        trace(tr, 0, gr);
        ptx::mbar_wait(&s_full[buf], (gr / NSP) & 1);
        trace(tr, 1, gr);
        ptx::tc_fence_after();
        if (kTesting && (P.debug & 512)) {  // timing experiment only: no softmax work
          if (gr >= (uint32_t)NSP) ptx::mbar_wait(&pv_done[buf], ((gr - NSP) / NSP) & 1);
          ptx::warp_arrive(&p_full[buf]);
          gb += nb;
          continue;
        }
        uint32_t sv[CB][NQ];
#pragma unroll
        for (int c = 0; c < CB; ++c)
          if (c < nb) ptx::tmem_ld16(tmem + lane_base + (buf * CB + c) * NQ, sv[c]);
        ptx::tmem_ld_wait();
        trace(tr, 2, gr);
        float s[CB][G];
        bool tok[CB];
        float *rm = red_max + (gr & 1) * 4 * NQ;
#pragma unroll
        for (int c = 0; c < CB; ++c) tok[c] = c < nb && (n0 + c) * BT + r < len;
#pragma unroll
        for (int h = 0; h < G; ++h) {
          float x = -INFINITY;
#pragma unroll
          for (int c = 0; c < CB; ++c) {
            s[c][h] = tok[c] ? __uint_as_float(sv[c][h]) : -INFINITY;
            x = fmaxf(x, s[c][h]);
          }
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
          if (lane == 0) rm[quarter * NQ + h] = x;
        }
        named_bar_sync(1, 128);
        trace(tr, 3, gr);
        float alpha[NQ];
        bool resc = false;
#pragma unroll
        for (int h = 0; h < NQ; ++h) alpha[h] = 1.f;
#pragma unroll
        for (int h = 0; h < G; ++h) {
          const float bm = fmaxf(fmaxf(rm[h], rm[NQ + h]), fmaxf(rm[2 * NQ + h], rm[3 * NQ + h]));
          const float mnew = bm * c2;
          if (mnew > m[h] + 8.0f) {  // round-uniform decision
            const float mt = fmaxf(m[h], mnew);
            alpha[h] = fast_exp2(m[h] - mt);
            m[h] = mt;
            resc = true;
          }
        }
        float p[CB][G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
          float acc = 0.f;
#pragma unroll
          for (int c = 0; c < CB; ++c) {
            p[c][h] = tok[c] ? fast_exp2(fmaf(s[c][h], c2, -m[h])) : 0.f;
            acc += p[c][h];
          }
          l[h] = l[h] * alpha[h] + acc;
        }
        // P slot `buf` was last read by PV(gr - NSP)
        if (gr >= (uint32_t)NSP) ptx::mbar_wait(&pv_done[buf], ((gr - NSP) / NSP) & 1);
        if (resc && n0 > 0) {  // rare: O^T column h *= alpha[h] once PV(gr - 1) has landed
          ptx::mbar_wait(&pv_done[(gr - 1) % NSP], ((gr - 1) / NSP) & 1);
          ptx::tc_fence_after();
          uint32_t ov[NQ];
          ptx::tmem_ld16(o_tmem, ov);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int h = 0; h < NQ; ++h) ov[h] = __float_as_uint(__uint_as_float(ov[h]) * alpha[h]);
          ptx::tmem_st16(o_tmem, ov);
          ptx::tmem_st_wait();
        }
        const int cc = (r % 64) / 8, e = r % 8;
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          if (c >= nb) break;
          uint8_t *sp = smem + OFF_P + (buf * CB + c) * PTILE + (r / 64) * PPANEL;
#pragma unroll
          for (int h = 0; h < G; ++h)
            *reinterpret_cast<__nv_bfloat16 *>(sp + h * 128 + ((cc ^ (h % 8)) * 16) + e * 2) =
                __float2bfloat16_rn(p[c][h]);
        }
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        ptx::warp_arrive(&p_full[buf]);
        trace(tr, 4, gr);
        gb += nb;
      }
      // hand (m, row-sum partials) to the epilogue warps; slot ob was last read by the
      // epilogue of item item_no - 2
      trace(tr, 5, item_no);
      ptx::mbar_wait(&o_free[ob], ((item_no >> 1) & 1) ^ 1);
      trace(tr, 6, item_no);
      float *rs = red_sum + ob * 4 * NQ;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float x = l[h];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) rs[quarter * NQ + h] = x;
        if (r == 0) item_m[ob * NQ + h] = m[h];
      }
      ptx::warp_arrive(&ml_full[ob]);
      ++item_no;
    }
  } else if (warp >= 8 && !(kTesting && (P.debug & 256))) {
    // ================= epilogue (thread = head dim): O = O^T / l, LSE =================
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    uint32_t item_no = 0;
    __shared__ uint32_t fc_mask;  // fused Eq. 5: rows of the current item completed by this part
    // Fused Eq. 5 (fused.cuh): the 4 epilogue warps' stores of an item's part precede the
    // arrivals (one per row, warp 8); every completed row is merged by all 128 threads.
    auto fused_arrive = [&](const ItemRef &ir, int64_t row0) {
      if (fc_counting(P.fc)) __threadfence();
      named_bar_sync(2, 128);
      if (warp == 8) {
        const bool last = lane < G && fc_arrive(P.fc, row0 + lane, fc_expected(P.fc, ir.b, ir.j * G + lane));
        const uint32_t m = __ballot_sync(0xffffffffu, last);
        if (lane == 0) fc_mask = m;
      }
      named_bar_sync(2, 128);
      uint32_t m = fc_mask;
      if (m) __threadfence();
      while (m) {
        const int h = __ffs(m) - 1;
        m &= m - 1;
        fc_merge_row_dim(P.fc, row0 + h, fc_prefix_pieces(P.fc, ir.b, ir.j * G + h), r);
      }
    };
    int len_next = item_len_raw<SPLIT>(P, blockIdx.x);
    for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
      const int len = item_len_of<SPLIT>(P, item, len_next);
      len_next = item_len_raw<SPLIT>(P, item + gridDim.x);
      if (len <= 0) {
        if (P.fc.cnt) {  // fused: the empty part (0, -inf) is written and counted here
          const ItemRef ir = item_ref<SPLIT>(P, item);
          const int64_t row0 = (int64_t)ir.b * P.Hq + (int64_t)ir.j * g;
#pragma unroll
          for (int h = 0; h < G; ++h) {
            P.o[ir.o_off + (row0 + h) * HD + r] = 0.f;
            if (r == h) P.lse[ir.lse_off + row0 + h] = -INFINITY;
          }
          fused_arrive(ir, row0);
        }
        continue;
      }
      const ItemRef ir = item_ref<SPLIT>(P, item);
      const int64_t row0 = (int64_t)ir.b * P.Hq + (int64_t)ir.j * g;
      const uint32_t ob = item_no & 1, ph = (item_no >> 1) & 1;
      ptx::mbar_wait(&o_full[ob], ph);
      ptx::mbar_wait(&ml_full[ob], ph);
      ptx::tc_fence_after();
      uint32_t ov[NQ];
      ptx::tmem_ld16(tmem + lane_base + O_COL + ob * NQ, ov);
      ptx::tmem_ld_wait();
      const float *rs = red_sum + ob * 4 * NQ;
      float L[G], M[G];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        L[h] = rs[h] + rs[NQ + h] + rs[2 * NQ + h] + rs[3 * NQ + h];
        M[h] = item_m[ob * NQ + h];
      }
      ptx::tc_fence_before();
      ptx::warp_arrive(&o_free[ob]);  // O^T buffer and (m, l) slot free
      // testing build: the parity suite's "unwritten rows" mutation (must fail parity)
      const bool skip0 = kTesting && P.mutate == 2 && blockIdx.x == 0 && item_no == 0;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        if (!(skip0 && h == 0)) P.o[ir.o_off + (row0 + h) * HD + r] = __uint_as_float(ov[h]) / L[h];
        if (r == h) P.lse[ir.lse_off + row0 + h] = (M[h] + log2f(L[h])) * HYDRA_LN2;
      }
      if (P.fc.cnt) fused_arrive(ir, row0);
      ++item_no;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem);
  }
  if (P.timer && threadIdx.x == 0) atomicMax(P.timer + 1, gtimer());
  if (cta_tr && threadIdx.x == 0) cta_tr[2 * kTraceN] = (long long)gtimer();
  // Launched as a programmatic dependent of the prefix kernel (SM-partitioned schedule on one
  // stream): the grid completes only after the prefix grid has, so the combine that follows in
  // the stream sees both.  Without a programmatic prerequisite this returns at once.
  asm volatile("griddepcontrol.launch_dependents;");  // the combine may launch as the CTAs drain
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ------------------------------------------------------------------ host side
bool suffix_tc_supported(const hydra_heads *h) {
  const int g = h->num_q_heads / h->num_kv_heads;
  const bool g_ok = g == 1 || g == 2 || g == 4 || g == 8 || g == 16;
  return h->dtype == HYDRA_BF16 && h->head_dim == 128 && g_ok && tensor_maps_available();
}

template <int G, int CB, bool SPLIT, bool PAGED>
static cudaError_t launch_gcsp(const SuffixTcParams &P, int grid, cudaStream_t s) {
  constexpr int alloc = stc::alloc_bytes(CB);
  const cudaError_t attr = ensure_smem_attr(reinterpret_cast<const void *>(suffix_tc_kernel<G, CB, SPLIT, PAGED>), alloc);
  if (attr != cudaSuccess) return attr;
  if (!P.pdl) {
    suffix_tc_kernel<G, CB, SPLIT, PAGED><<<grid, stc::kThreads, alloc, s>>>(P);
    return cudaGetLastError();
  }
  // programmatic dependent launch: starts once every CTA of the preceding kernel in the stream
  // (the persistent prefix on its SM share) is resident, and fills the remaining SMs
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(stc::kThreads, 1, 1);
  cfg.dynamicSmemBytes = alloc;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, suffix_tc_kernel<G, CB, SPLIT, PAGED>, P);
}
// PAGED (compile time): the contiguous kernel carries no paging branch in its producers
template <int G, int CB, bool SPLIT>
static cudaError_t launch_gcs(const SuffixTcParams &P, int grid, cudaStream_t s) {
  return P.block_table ? launch_gcsp<G, CB, SPLIT, true>(P, grid, s) : launch_gcsp<G, CB, SPLIT, false>(P, grid, s);
}
template <int G, int CB>
static cudaError_t launch_gc(const SuffixTcParams &P, int grid, cudaStream_t s) {
  return P.n_split > 1 ? launch_gcs<G, CB, true>(P, grid, s) : launch_gcs<G, CB, false>(P, grid, s);
}
template <int G>
static cudaError_t launch_g(const SuffixTcParams &P, int cb, int grid, cudaStream_t s) {
  return cb == 1 ? launch_gc<G, 1>(P, grid, s) : launch_gc<G, 2>(P, grid, s);
}

hydra_status launch_suffix_tc(const SuffixTcArgs &a, int n_ctas, cudaStream_t s) {
  SuffixTcParams P;
  memset(&P, 0, sizeof(P));
  const int g = a.Hq / a.Hkv;
  const bool paged = a.block_table != nullptr;
  if (paged && (a.page_size < 8 || (a.page_size & (a.page_size - 1)) || a.n_pages <= 0)) return HYDRA_EUNSUPPORTED;
  {
    // contiguous: [B, S_cap, Hkv, d], one 128-token box per panel; paged: the page pools
    // [n_pages, page_size, Hkv, d] with min(page_size, 128)-token boxes
    const uint32_t pbox = paged ? (uint32_t)std::min(a.page_size, stc::BT) : (uint32_t)stc::BT;
    const uint64_t dims[4] = {(uint64_t)stc::HD, (uint64_t)a.Hkv, (uint64_t)(paged ? a.page_size : a.S_cap),
                              (uint64_t)(paged ? a.n_pages : a.B)};
    const uint64_t strides[3] = {(uint64_t)a.s_sh * 2, (uint64_t)a.s_st * 2, (uint64_t)a.s_sb * 2};
    const uint32_t box[4] = {64, 1, pbox, 1};
    if (!encode_bf16_map(&P.tmK, 4, a.k, dims, strides, box)) return HYDRA_ECUDA;
    if (!encode_bf16_map(&P.tmV, 4, a.v, dims, strides, box)) return HYDRA_ECUDA;
  }
  {
    const uint64_t dims[3] = {(uint64_t)stc::HD, (uint64_t)a.Hq, (uint64_t)a.B};
    const uint64_t strides[2] = {(uint64_t)a.q_sh * 2, (uint64_t)a.q_sb * 2};
    const uint32_t box[3] = {64, (uint32_t)g, 1};
    if (!encode_bf16_map(&P.tmQ, 3, a.q, dims, strides, box)) return HYDRA_ECUDA;
  }
  P.lens = a.lens;
  P.B = a.B;
  P.Hq = a.Hq;
  P.Hkv = a.Hkv;
  P.g = g;
  P.scale_log2 = a.scale_log2;
  P.n_split = a.n_split > 0 ? a.n_split : 1;
  P.split_len = P.n_split > 1 ? a.split_len : (int32_t)std::min<int64_t>(a.S_cap, INT32_MAX);
  P.o_split_stride = a.o_split_stride;
  P.lse_split_stride = a.lse_split_stride;
  P.n_items = a.B * a.Hkv * P.n_split;
  P.o = a.o;
  P.lse = a.lse;
  P.trace = kTesting ? reinterpret_cast<long long *>(a.trace) : nullptr;
  P.debug = kTesting ? a.debug : 0;
  P.mutate = kTesting ? a.mutate : 0;
  P.S_cap = (int32_t)std::min<int64_t>(a.S_cap, INT32_MAX);
  P.fc = a.fc;
  P.pdl = a.pdl;
  P.timer = a.timer;
  if (P.fc.cnt && P.fc.n_suf != P.n_split) return HYDRA_EINVAL;
  P.block_table = a.block_table;
  P.bt_stride = a.bt_stride;
  if (paged) {
    P.page_shift = __builtin_ctz((unsigned)a.page_size);
    P.pbox_shift = __builtin_ctz((unsigned)std::min(a.page_size, stc::BT));
  }
  if (P.n_items == 0) return HYDRA_OK;
  const int grid = n_ctas > 0 && n_ctas < P.n_items ? n_ctas : P.n_items;
  cudaError_t e = cudaErrorInvalidValue;
  switch (g) {
    case 1: e = launch_g<1>(P, a.cb, grid, s); break;
    case 2: e = launch_g<2>(P, a.cb, grid, s); break;
    case 4: e = launch_g<4>(P, a.cb, grid, s); break;
    case 8: e = launch_g<8>(P, a.cb, grid, s); break;
    case 16: e = launch_g<16>(P, 1, grid, s); break;  // CB = 2 would spill at G = 16
  }
  return e == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

}  // namespace hydra

// prefix_tc2.cu -- persistent two-tile (M = 256) tcgen05 prefix attention for sm_100a.
//
// PAPER.md §3.2: all B*g decode queries of a KV head attend to the same
// prefix K/V, so they are stacked into one matrix (rows r = b*g + i hold q[b, j*g+i])
// and prefix attention is a dense GEMM-shaped problem reading the prefix once
// (App. B `attention(batched_q, prefix_k, prefix_v)`).  Output per row:
// O = softmax(s) V (fp32, normalised) and LSE (natural log, Eq. 4) for Eq. 5.
//
// Work item = (pair of 128-row query tiles, KV head j, KV split).  Persistent CTAs walk
// the items round-robin (consecutive items share the KV range, so concurrently running
// CTAs hit the same K/V tiles in L2).  384 threads per CTA:
//   warp 0       TMA producer: K and V tiles (128 tokens x 128 dims, two 64-column
//                SWIZZLE_128B boxes each) into a 2-stage ring; runs ahead across items
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-3    idle
//   warps 4-7    softmax / correction / epilogue for query tile 0 (one row per thread)
//   warps 8-11   the same for query tile 1
// Every K/V tile in shared memory feeds both query tiles (256 rows), halving the K/V
// smem/L2 traffic per FLOP compared with one 128-row tile, and the two softmax
// warpgroups ping-pong: while one computes exp() the tensor core runs the other
// tile's MMAs.  TMEM (512 columns): S_t at [128t, 128t+128) fp32 (P_t aliases its
// first 64 columns as bf16 pairs and feeds the PV MMA from TMEM), O_t at
// [256+128t, 384+128t).  MMA issue order per block n:
//   PV0(n) S0(n+1) PV1(n) S1(n+1)       (S_t(n+1) may overwrite P_t(n): in-order pipe)
// Online softmax in the log2 domain (scale folded into one FFMA2), running max raised
// only when a row max grows by > 8 (P <= 256, rare O correction, exact final O / l).
// Epilogue: O rows go TMEM -> registers -> XOR-swizzled smem (this warp's Q rows) ->
// coalesced 128-B row stores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"
#include "fused.cuh"

namespace hydra {


namespace tc2 {
constexpr int BM = 128;  // rows per query tile (UMMA M)
constexpr int BN = 128;  // KV tokens per block
constexpr int HD = 128;  // head dim
constexpr int NS = 2;    // K/V pipeline stages
constexpr int kThreads = 384;
constexpr int PANEL = BN * 128;  // 128 rows x 128 B (one 64-column SWIZZLE_128B panel)
constexpr int TILE = 2 * PANEL;  // 128 x 128 bf16 = 32 KB
constexpr int OFF_Q = 0;         // Q0, Q1
constexpr int OFF_K = 2 * TILE;
constexpr int OFF_V = OFF_K + NS * TILE;
constexpr int OFF_BAR = OFF_V + NS * TILE;
// k_full, k_empty, v_full, v_empty [NS]; q_full, s_full, p_full, pv_done, o_free, p_half [2]
constexpr int N_BARS = 4 * NS + 12;
constexpr int BYTES = OFF_BAR + N_BARS * 8 + 16;
constexpr int ALLOC = BYTES + 1024;
constexpr uint32_t TMEM_COLS = 512;
constexpr int kTraceN = 1024;  // diagnostics: events per trace row
}  // namespace tc2

struct __align__(64) PrefixTc2Params {
  CUtensorMap tmK;
  CUtensorMap tmV;
  const __nv_bfloat16 *q;
  int64_t q_sb, q_sh;
  int32_t Hq, Hkv, g;
  float scale_log2;
  int64_t P;      // flat mode: prefix length
  int32_t B;      // flat mode: sequences
  int32_t n_pairs;  // flat mode: ceil(B*g / 256)
  const PrefixTask *tasks;  // task mode: task.tile = pair index within the group
  int32_t n_tasks;
  const int32_t *seq_list;
  int32_t n_splits;   // task mode: KV splits per task
  int32_t n_items;    // task mode: tasks * Hkv * n_splits
  int32_t nb;         // flat mode: KV blocks per item (ceil(P / 128))
  int64_t total_blocks;  // flat mode: units in the stream-K space (Hkv*nb grouped, n_pairs*Hkv*nb not)
  int32_t group;         // flat mode: CTAs per group (= n_pairs when grouped, else 1)
  int32_t bn;            // KV tokens per block (128: v3, 64: v4)
  int32_t debug;         // timing experiments only (invalid results): bit 1 no softmax math, bit 2 no K/V TMA
  long long *trace;      // diagnostics: CTA 0 event timestamps (clock64), see tools/prefix_trace.py; null = off
  int32_t mutate;        // testing build only: 1 = CTA 0 skips one 4-row store group of its epilogues
  FusedCombine fc;       // fc.cnt != null: the Eq. 5 merge of every completed row in this epilogue (fused.cuh)
  unsigned long long *timer;  // measurement: [0] min CTA start, [1] max CTA end (%globaltimer ns); null = off
  float *o, *lse;
  int64_t o_slot_stride, lse_slot_stride;
};

struct Item {
  int64_t kv_off, kv_len, n_rows, row0;
  int32_t seq_off, slot, j, blk_begin, nblk;
};

// Iterates the KV segments a persistent CTA owns.
//  flat mode, grouped stream-K: CTAs form groups of `group` members; member m of a group
//    owns query-tile pair m (rows 256m .. 256m+255) of every head, and the group walks a
//    contiguous range of the (head, 128-token KV block) space -- the space of
//    Hkv * nb units is cut into G = gridDim.x / group equal ranges.  All members of a
//    group read the same K/V tiles at about the same time, so each tile comes from DRAM
//    once and from L2 for the other members.  With group == 1 the unit space is
//    (pair, head, block) instead.  A range may start or end inside a head; every piece
//    writes its own partial slot (slot = this group - the group owning the head's first
//    block), merged later by the LSE combine.
//  task mode (tree): items = (task, head, split) dealt round-robin.
struct SegIter {
  int64_t x, end;
  int w;
};

__device__ __forceinline__ int n_groups(const PrefixTc2Params &P) { return gridDim.x / P.group; }

__device__ __forceinline__ int64_t sk_start(const PrefixTc2Params &P, int64_t c) {
  return c * P.total_blocks / n_groups(P);
}

__device__ __forceinline__ void seg_begin(const PrefixTc2Params &P, SegIter &s) {
  const int grp = blockIdx.x / P.group;
  if (grp >= n_groups(P)) {  // leftover CTAs when gridDim.x % group != 0
    s.x = s.end = 0;
  } else {
    s.x = sk_start(P, grp);
    s.end = sk_start(P, grp + 1);
  }
  s.w = blockIdx.x;
}

__device__ __forceinline__ bool seg_next(const PrefixTc2Params &P, SegIter &s, Item &it) {
  PrefixTask task;
  if (P.tasks) {
    if (s.w >= P.n_items) return false;
    const int w = s.w;
    s.w += gridDim.x;
    task = P.tasks[w % P.n_tasks];
    const int rest = w / P.n_tasks;
    const int split = rest % P.n_splits;
    it.j = rest / P.n_splits;
    it.kv_off = task.kv_off;
    it.kv_len = task.kv_len;
    it.n_rows = (int64_t)task.n_seq * P.g;
    it.row0 = (int64_t)task.tile * (2 * tc2::BM);
    it.seq_off = task.seq_off;
    it.slot = task.depth * P.n_splits + split;
    const int nblk_total = (int)((task.kv_len + P.bn - 1) / P.bn);
    const int per_split = (nblk_total + P.n_splits - 1) / P.n_splits;
    it.blk_begin = split * per_split;
    it.nblk = max(0, min(nblk_total, it.blk_begin + per_split) - it.blk_begin);
    return true;
  }
  if (s.x >= s.end) return false;
  const int64_t unit = s.x / P.nb;  // head (grouped) or (pair, head)
  const int b = (int)(s.x % P.nb);
  const int64_t room = s.end - s.x;
  const int len = (int)(P.nb - b < room ? P.nb - b : room);
  // group owning this unit's first block: largest c with sk_start(c) <= unit*nb
  const int G = n_groups(P);
  const int64_t x0 = unit * P.nb;
  int64_t c0 = x0 * G / P.total_blocks;
  while (c0 + 1 < G && sk_start(P, c0 + 1) <= x0) ++c0;
  while (c0 > 0 && sk_start(P, c0) > x0) --c0;
  const int64_t pair = P.group > 1 ? (int64_t)(blockIdx.x % P.group) : unit % P.n_pairs;
  it.j = (int)(P.group > 1 ? unit : unit / P.n_pairs);
  it.kv_off = 0;
  it.kv_len = P.P;
  it.n_rows = (int64_t)P.B * P.g;
  it.row0 = pair * (2 * tc2::BM);
  it.seq_off = 0;
  it.slot = (int)(blockIdx.x / P.group - c0);
  it.blk_begin = b;
  it.nblk = len;
  s.x += len;
  return true;
}

// Fused Eq. 5 (fused.cuh): after this warp's rows of a piece are stored, count each live row's
// arrival; the warp merges the rows this piece completed, one row at a time.
__device__ __forceinline__ void tc2_fused_arrive(const PrefixTc2Params &P, bool live, int64_t seq, int h, int lane) {
  if (P.fc.pre_done) return;  // sequential schedule: the suffix kernel counts and merges
  __threadfence();
  __syncwarp();
  const int64_t row = seq * P.Hq + h;
  int n_pre = 0;
  bool last = false;
  if (live) {
    n_pre = fc_prefix_pieces(P.fc, seq, h);
    last = fc_arrive(P.fc, row, n_pre + P.fc.n_suf);
  }
  unsigned mask = __ballot_sync(0xffffffffu, last);
  if (mask) __threadfence();
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    fc_merge_row_warp(P.fc, __shfl_sync(0xffffffffu, row, src), __shfl_sync(0xffffffffu, n_pre, src), lane);
  }
}

// kPolyEvery -- 0: all exp2 on MUFU; k: every k-th column pair on the FMA pipe.
// kSpec -- speculative softmax with the running max (variant 5, see the loop).
// kSplit -- P published in two 64-token halves (variant 6): the PV MMAs of the first half
//   run while the softmax still computes exp() of the second half.
template <int kPolyEvery, bool kSpec, bool kSplit = false>
__global__ void __launch_bounds__(tc2::kThreads, 1) prefix_tc2_kernel(const __grid_constant__ PrefixTc2Params P) {
  using namespace tc2;
  extern __shared__ uint8_t smem_raw[];
  // SM-partitioned schedule on one stream: the suffix kernel (a programmatic dependent) may start
  // as soon as every CTA of this persistent grid is resident -- it then takes the other SMs
  asm volatile("griddepcontrol.launch_dependents;");
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *k_full = bars, *k_empty = bars + NS, *v_full = bars + 2 * NS, *v_empty = bars + 3 * NS;
  uint64_t *q_full = bars + 4 * NS, *s_full = q_full + 2, *p_full = q_full + 4, *pv_done = q_full + 6,
           *o_free = q_full + 8, *p_half = q_full + 10;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + N_BARS);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // diagnostics: every CTA's globaltimer at entry / setup done / first S / last P / exit
  long long *cta_tr = (kTesting && P.trace && blockIdx.x < 256) ? P.trace + 14 * kTraceN + blockIdx.x * 8 : nullptr;
  if (cta_tr && threadIdx.x == 0) cta_tr[0] = (long long)gtimer();
  if (P.timer && threadIdx.x == 0) atomicMin(P.timer, gtimer());

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&P.tmK);
    ptx::prefetch_tmap(&P.tmV);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&q_full[t], 4);  // one elected arrival per softmax warp
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&p_full[t], 4);  // one elected arrival per softmax warp
      ptx::mbar_init(&pv_done[t], 1);
      ptx::mbar_init(&o_free[t], 4);  // one elected arrival per softmax warp
      ptx::mbar_init(&p_half[t], 4);  // one elected arrival per softmax warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (cta_tr && threadIdx.x == 0) cta_tr[1] = (long long)gtimer();

  // Register rebalancing per warpgroup (inside disjoint role branches so ptxas allocates each
  // region separately): producer / MMA / idle warps need few registers, the two softmax
  // warpgroups hold a 128-column score row each.  The launch grants 168 per thread (384 threads,
  // 64K / 384 rounded down to 8): 128 x (168 - 88) released = 256 x (208 - 168) acquired --
  // an increase not covered by the decrease would block setmaxnreg.inc forever.
  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 88;" ::: "memory");
  if (warp == 0) {
    // ================= TMA producer =================
    if (ptx::elect_one()) {
      uint32_t gb = 0;  // global block counter (stage ring position)
      SegIter si;
      seg_begin(P, si);
      Item it;
      while (seg_next(P, si, it)) {
        for (int n = 0; n < it.nblk; ++n, ++gb) {
          const int st = gb % NS;
          const uint32_t ph = (gb / NS) & 1;
          const int t0 = (int)(it.kv_off + (int64_t)(it.blk_begin + n) * BN);
          uint8_t *sK = smem + OFF_K + st * TILE;
          uint8_t *sV = smem + OFF_V + st * TILE;
          if (kTesting && (P.debug & 4) && gb >= (uint32_t)NS) {  // timing experiment only: no K/V traffic after the fill
            ptx::mbar_wait(&k_empty[st], ph ^ 1);
            ptx::mbar_arrive(&k_full[st]);
            ptx::mbar_wait(&v_empty[st], ph ^ 1);
            ptx::mbar_arrive(&v_full[st]);
            continue;
          }
          ptx::mbar_wait(&k_empty[st], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&k_full[st], TILE);
          ptx::tma_load_3d(sK, &P.tmK, &k_full[st], 0, it.j, t0);
          ptx::tma_load_3d(sK + PANEL, &P.tmK, &k_full[st], 64, it.j, t0);
          ptx::mbar_wait(&v_empty[st], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&v_full[st], TILE);
          ptx::tma_load_3d(sV, &P.tmV, &v_full[st], 0, it.j, t0);
          ptx::tma_load_3d(sV + PANEL, &P.tmV, &v_full[st], 64, it.j, t0);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (ptx::elect_one()) {
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(BM, BN, false);  // S = Q K^T (both K-major)
      constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(BM, HD, true);  // O += P V (V MN-major)
      uint32_t gb = 0, qc[2] = {0, 0}, pc[2] = {0, 0}, oc[2] = {0, 0};
      long long *tr = (kTesting && P.trace && blockIdx.x == 0) ? P.trace : nullptr;
      SegIter si;
      seg_begin(P, si);
      Item it;
      while (seg_next(P, si, it)) {
        if (it.nblk == 0) continue;
        const int ntile = (it.n_rows - it.row0 > BM) ? 2 : 1;
        auto issue_s = [&](int t, int st) {
          const uint32_t q_addr = ptx::smem_u32(smem + OFF_Q + t * TILE);
          const uint32_t k_addr = ptx::smem_u32(smem + OFF_K + st * TILE);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk / 4) * PANEL + (kk % 4) * 32;
            ptx::mma_ss(tmem + t * BN, ptx::smem_desc_sw128(q_addr + off, 16, 1024),
                        ptx::smem_desc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0);
          }
          ptx::mma_commit(&s_full[t]);
        };
        {  // prologue: S_t(0), each tile as soon as its Q is in shared memory
          const int st = gb % NS;
          ptx::mbar_wait(&k_full[st], (gb / NS) & 1);
          for (int t = 0; t < ntile; ++t) {
            ptx::mbar_wait(&q_full[t], qc[t] & 1);
            ++qc[t];
            ptx::tc_fence_after();
            issue_s(t, st);
          }
          ptx::mma_commit(&k_empty[st]);
        }
        for (int n = 0; n < it.nblk; ++n) {
          const uint32_t g0 = gb + n, g1 = g0 + 1;
          const int st = g0 % NS, st1 = g1 % NS;
          const bool more = n + 1 < it.nblk;
          ptx::mbar_wait(&v_full[st], (g0 / NS) & 1);
          const uint32_t v_addr = ptx::smem_u32(smem + OFF_V + st * TILE);
          for (int t = 0; t < ntile; ++t) {
            if (kSplit) {  // first half of P(n): tokens 0-63 (P columns 0-31)
              ptx::mbar_wait(&p_half[t], pc[t] & 1);
              if (n == 0) {
                ptx::mbar_wait(&o_free[t], (oc[t] & 1) ^ 1);
                ++oc[t];
              }
              ptx::tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < BN / 32; ++kk)
                ptx::mma_ts(tmem + 256 + t * BN, tmem + t * BN + kk * 8,
                            ptx::smem_desc_sw128(v_addr + kk * 2048, PANEL, 1024), idesc_pv, (n > 0 || kk > 0));
            }
            ptx::mbar_wait(&p_full[t], pc[t] & 1);
            ++pc[t];
            if (tr && pc[t] <= kTraceN) tr[(6 + t) * kTraceN + pc[t] - 1] = clock64();
            if (!kSplit && n == 0) {  // O_t must have been drained by the previous item's epilogue
              ptx::mbar_wait(&o_free[t], (oc[t] & 1) ^ 1);
              ++oc[t];
            }
            ptx::tc_fence_after();
#pragma unroll
            for (int kk = kSplit ? BN / 32 : 0; kk < BN / 16; ++kk)
              ptx::mma_ts(tmem + 256 + t * BN, tmem + t * BN + kk * 8,
                          ptx::smem_desc_sw128(v_addr + kk * 2048, PANEL, 1024), idesc_pv, (n > 0 || kk > 0));
            ptx::mma_commit(&pv_done[t]);
            if (more) {
              if (t == 0) {
                ptx::mbar_wait(&k_full[st1], (g1 / NS) & 1);
                ptx::tc_fence_after();
              }
              issue_s(t, st1);
            }
          }
          ptx::mma_commit(&v_empty[st]);
          if (more) ptx::mma_commit(&k_empty[st1]);
        }
        gb += it.nblk;
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    // ================= softmax / correction / epilogue =================
    const int t = (warp - 4) / 4;          // query tile of this warpgroup
    const int quarter = warp % 4;           // TMEM lane quarter
    const int r = quarter * 32 + lane;      // row within the tile
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t s_col = tmem + lane_base + t * BN;
    const uint32_t o_col = tmem + lane_base + 256 + t * BN;
    uint8_t *sQ = smem + OFF_Q + t * TILE;
    const float c2 = P.scale_log2;
    uint32_t sc = 0, pvc = 0;  // phase counters of s_full[t] / pv_done[t]
    long long *tr = (kTesting && P.trace && blockIdx.x == 0 && quarter == 0 && lane == 0) ? P.trace : nullptr;
    SegIter si;
    seg_begin(P, si);
    Item it;
    while (seg_next(P, si, it)) {
      const int64_t trow0 = it.row0 + t * BM;
      if (trow0 >= it.n_rows) continue;  // tile inactive for this item
      const int64_t rr = trow0 + r;
      const bool live = rr < it.n_rows;
      int64_t seq = 0;
      int h = 0;
      if (live) {
        seq = P.seq_list ? P.seq_list[it.seq_off + rr / P.g] : rr / P.g;
        h = it.j * P.g + (int)(rr % P.g);
      }
      float *orow = P.o + it.slot * P.o_slot_stride + (seq * P.Hq + h) * HD;
      if (it.nblk == 0) {  // empty KV range: (0, -inf) sentinel
        if (live) {
          P.lse[it.slot * P.lse_slot_stride + seq * P.Hq + h] = -INFINITY;
          for (int c = 0; c < HD / 4; ++c) reinterpret_cast<float4 *>(orow)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (P.fc.cnt) tc2_fused_arrive(P, live, seq, h, lane);
        continue;
      }
      // ---- Q row -> sQ (canonical K-major SWIZZLE_128B: 16-B chunk c of row r at c ^ (r % 8))
      {
        uint4 ch[16];
        if (live) {
          const uint4 *src = reinterpret_cast<const uint4 *>(P.q + seq * P.q_sb + (int64_t)h * P.q_sh);
#pragma unroll
          for (int c = 0; c < 16; ++c) ch[c] = __ldg(src + c);
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) ch[c] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int c = 0; c < 16; ++c)
          *reinterpret_cast<uint4 *>(sQ + (c / 8) * PANEL + r * 128 + (((c % 8) ^ (r % 8)) * 16)) = ch[c];
        ptx::fence_proxy_async_smem();
        ptx::warp_arrive(&q_full[t]);
      }
      float m2 = -INFINITY, l = 0.f;
      for (int n = 0; n < it.nblk; ++n) {
        if (tr && sc < kTraceN) tr[(3 * t + 0) * kTraceN + sc] = clock64();
        ptx::mbar_wait(&s_full[t], sc & 1);
        if (tr && sc < kTraceN) tr[(3 * t + 1) * kTraceN + sc] = clock64();
        if (cta_tr && sc == 0 && t == 0 && quarter == 0 && lane == 0) cta_tr[2] = (long long)gtimer();
        ++sc;
        ptx::tc_fence_after();
        if (kTesting && (P.debug & 2)) {  // timing experiment only: MMA pipeline without the softmax math
          if (n >= 1) {
            ptx::mbar_wait(&pv_done[t], pvc & 1);
            ++pvc;
          }
          ptx::tc_fence_before();
          ptx::warp_arrive(&p_full[t]);
          continue;
        }
        const int64_t rem = it.kv_len - (int64_t)(it.blk_begin + n) * BN;
        const uint64_t cc = ptx::pack2(c2, c2);
        uint32_t sr[4][32];
        uint64_t sacc[4];
        // exp2(s * c2 - m2) of S chunk c (32 columns) -> bf16 P chunk c (16 TMEM columns), row sums
        auto exp_chunk = [&](const uint32_t(&src)[32], int c, uint64_t nm) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float x0, x1;
            ptx::unpack2(ptx::fma2(ptx::pack2(__uint_as_float(src[2 * i]), __uint_as_float(src[2 * i + 1])), cc, nm),
                         x0, x1);
            float p0, p1;
            if (kTesting && kPolyEvery < 0) {  // timing experiment only (testing build): no exp at all (wrong results)
              p0 = x0 * 0.01f;
              p1 = x1 * 0.01f;
            } else if (kPolyEvery > 0 && (i % (kPolyEvery > 0 ? kPolyEvery : 1)) == kPolyEvery - 1) {
              ptx::exp2_poly2(x0, x1, p0, p1);  // FMA-pipe exp2 for 1/kPolyEvery of the pairs
            } else {
              p0 = fast_exp2(x0);
              p1 = fast_exp2(x1);
            }
            sacc[i % 4] = ptx::add2(sacc[i % 4], ptx::pack2(p0, p1));
            pk[i] = ptx::cvt_bf16x2(p0, p1);
          }
          ptx::tmem_st16(s_col + c * 16, pk);  // P(n) -> first 64 columns of S_t
        };
        auto mask_chunk = [&](uint32_t(&src)[32], int c) {
          if (rem < BN) {  // partial last block only
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i >= rem) src[i] = 0xff800000u;
          }
        };
        float acc[8];
        auto max_chunk = [&](const uint32_t(&src)[32], bool first) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float a = __uint_as_float(src[2 * k]), b = __uint_as_float(src[2 * k + 1]);
            acc[k] = first ? fmaxf(a, b) : ptx::fmax3(acc[k], a, b);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k)
            acc[k] = ptx::fmax3(acc[k], __uint_as_float(src[16 + 2 * k]), __uint_as_float(src[17 + 2 * k]));
        };
        bool any;
        float alpha = 1.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::tmem_ld32(s_col + c * 32, sr[c]);
        ptx::tmem_ld_wait();
        if (tr && sc <= kTraceN) tr[(10 + t) * kTraceN + sc - 1] = clock64();
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::reg_fence32(sr[c]);
#pragma unroll
        for (int k = 0; k < 4; ++k) sacc[k] = 0;
        if (kSpec && n > 0) {
          // Speculative (variant 5): P = exp2(s*c2 - m2) with the running max of the previous
          // blocks, chunk by chunk as each TMEM load lands (the four loads are in flight
          // together), the block max reduced alongside -- the row max leaves the critical
          // path.  If some row's max grew by > 8 (p could exceed 2^8) the block is redone
          // with the raised max: the same rule as the exact path.
          const uint64_t nm = ptx::pack2(-m2, -m2);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            mask_chunk(sr[c], c);
            max_chunk(sr[c], c == 0);
            exp_chunk(sr[c], c, nm);
          }
          const float mx = fmaxf(ptx::fmax3(acc[0], acc[1], acc[2]),
                                 fmaxf(ptx::fmax3(acc[3], acc[4], acc[5]), fmaxf(acc[6], acc[7])));
          const float mnew = mx * c2;
          any = __any_sync(0xffffffffu, mnew > m2 + 8.0f);
          if (any) {  // rare
            const float mt = fmaxf(m2, mnew);
            alpha = fast_exp2(m2 - mt);
            m2 = mt;
            const uint64_t nm2 = ptx::pack2(-m2, -m2);
#pragma unroll
            for (int k = 0; k < 4; ++k) sacc[k] = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) exp_chunk(sr[c], c, nm2);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            mask_chunk(sr[c], c);
            max_chunk(sr[c], c == 0);
          }
          const float mx = fmaxf(ptx::fmax3(acc[0], acc[1], acc[2]),
                                 fmaxf(ptx::fmax3(acc[3], acc[4], acc[5]), fmaxf(acc[6], acc[7])));
          const float mnew = mx * c2;
          any = __any_sync(0xffffffffu, mnew > m2 + 8.0f);
          if (any) {
            const float mt = fmaxf(m2, mnew);
            alpha = fast_exp2(m2 - mt);  // 0 on the first block
            m2 = mt;
          }
          const uint64_t nm = ptx::pack2(-m2, -m2);
          if (tr && sc <= kTraceN) {
            asm volatile("" ::"l"(nm));  // the max is done before this timestamp
            tr[(12 + t) * kTraceN + sc - 1] = clock64();
          }
          if (kSplit) {
            // first half of P, then the O correction (PV_t(n-1) landed: S_t(n) was issued after
            // it; done here so the first half's scores are dead), then the first half is
            // published so its PV MMAs overlap the exp() of the second half
            exp_chunk(sr[0], 0, nm);
            exp_chunk(sr[1], 1, nm);
            if (n >= 1) {
              ptx::mbar_wait(&pv_done[t], pvc & 1);
              ++pvc;
              ptx::tc_fence_after();
              if (any) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  uint32_t ov[32];
                  ptx::tmem_ld32(o_col + c * 32, ov);
                  ptx::tmem_ld_wait();
#pragma unroll
                  for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                  ptx::tmem_st32(o_col + c * 32, ov);
                }
              }
            }
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            ptx::warp_arrive(&p_half[t]);
            exp_chunk(sr[2], 2, nm);
            exp_chunk(sr[3], 3, nm);
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) exp_chunk(sr[c], c, nm);
          }
        }
        float s0, s1, s2, s3;
        ptx::unpack2(ptx::add2(sacc[0], sacc[1]), s0, s1);
        ptx::unpack2(ptx::add2(sacc[2], sacc[3]), s2, s3);
        l = l * alpha + ((s0 + s1) + (s2 + s3));
        if (tr && sc <= kTraceN) tr[(8 + t) * kTraceN + sc - 1] = clock64();
        if (!kSplit && n >= 1) {
          ptx::mbar_wait(&pv_done[t], pvc & 1);  // PV_t(n-1) landed in O_t
          ++pvc;
          ptx::tc_fence_after();
          if (any) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t ov[32];
              ptx::tmem_ld32(o_col + c * 32, ov);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
              ptx::tmem_st32(o_col + c * 32, ov);
            }
          }
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::warp_arrive(&p_full[t]);
        if (tr && sc <= kTraceN) tr[(3 * t + 2) * kTraceN + sc - 1] = clock64();
      }
      ptx::mbar_wait(&pv_done[t], pvc & 1);  // last PV_t
      ++pvc;
      ptx::tc_fence_after();
      // ---- epilogue: O / l, staged through this warp's 4 KB of sQ (XOR swizzle), coalesced rows
      const float inv = 1.f / l;
      uint32_t *stage = reinterpret_cast<uint32_t *>(sQ + quarter * 32 * 128);  // rows 32q..32q+31 of panel 0
      const uint64_t my_row = live ? reinterpret_cast<uint64_t>(orow) : 0ull;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(o_col + c * 32, ov);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) stage[lane * 32 + (i ^ lane)] = __float_as_uint(__uint_as_float(ov[i]) * inv);
        __syncwarp();
        // 4 rows per step, 16 B per lane: lane = 8 * (row % 4) + column group (4 floats);
        // conflict-free: (4 cg + k) ^ rw spans 32 banks over the 8 column groups x 4 rows
        const int cg = lane % 8;
#pragma unroll
        for (int rw4 = 0; rw4 < 8; ++rw4) {
          const int rw = rw4 * 4 + lane / 8;
          const uint64_t base = __shfl_sync(0xffffffffu, my_row, rw);
          float4 v;
          v.x = __uint_as_float(stage[rw * 32 + ((cg * 4 + 0) ^ rw)]);
          v.y = __uint_as_float(stage[rw * 32 + ((cg * 4 + 1) ^ rw)]);
          v.z = __uint_as_float(stage[rw * 32 + ((cg * 4 + 2) ^ rw)]);
          v.w = __uint_as_float(stage[rw * 32 + ((cg * 4 + 3) ^ rw)]);
          // testing build: the parity suite's "unwritten rows" mutation (must fail parity)
          const bool skip = kTesting && P.mutate == 1 && blockIdx.x == 0 && c == 0 && rw4 == 1;
          if (base && !skip) reinterpret_cast<float4 *>(base)[c * 8 + cg] = v;
        }
        __syncwarp();
      }
      ptx::tc_fence_before();
      ptx::warp_arrive(&o_free[t]);
      if (live) P.lse[it.slot * P.lse_slot_stride + seq * P.Hq + h] = (m2 + log2f(l)) * HYDRA_LN2;
      if (P.fc.cnt) tc2_fused_arrive(P, live, seq, h, lane);
      // the staging writes to sQ were generic-proxy; order them before the next item's Q writes+TMA reads
      ptx::fence_proxy_async_smem();
    }
  }

  if (cta_tr && warp == 4 && lane == 0) cta_tr[3] = (long long)gtimer();  // tile-0 softmax/epilogue done
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem);
  }
  if (cta_tr && threadIdx.x == 0) cta_tr[4] = (long long)gtimer();
  if (P.timer && threadIdx.x == 0) atomicMax(P.timer + 1, gtimer());
}

// ===================================================================================
// v4: 64-token KV blocks with two score buffers per query tile.
// TMEM per tile t (256 columns): S_t[0] at [256t, 256t+64), S_t[1] at [256t+64, 256t+128),
// O_t at [256t+128, 256t+256).  P_t(n) aliases the first 32 columns of S_t[n & 1].
// Because S_t(n+2) lands in the other buffer than S_t(n+1), the MMA thread issues
//   prologue: S_0(0) S_1(0) S_0(1) S_1(1);   block n: PV_0(n) S_0(n+2) PV_1(n) S_1(n+2)
// and the score MMA of the next block is always done before the softmax of the current
// block ends, so the softmax warpgroups run back to back instead of waiting a full
// PV + S round trip per block (the v3 limiter).  The commit after S_t(n+2) also covers
// PV_t(n), so the P write of block n+2 into the same buffer is ordered; the rare O
// correction of block n waits for PV_t(n-1) explicitly.
namespace tc4 {
constexpr int BM = 128;
constexpr int BN = 64;
constexpr int HD = 128;
constexpr int NS = 4;
constexpr int kThreads = 384;
constexpr int QPANEL = BM * 128;  // 16 KB
constexpr int QTILE = 2 * QPANEL;  // 32 KB
constexpr int KPANEL = BN * 128;   // 8 KB: 64 rows x 128 B
constexpr int KTILE = 2 * KPANEL;  // 16 KB
constexpr int OFF_Q = 0;
constexpr int OFF_K = 2 * QTILE;
constexpr int OFF_V = OFF_K + NS * KTILE;
constexpr int OFF_BAR = OFF_V + NS * KTILE;
// k_full, k_empty, v_full, v_empty [NS]; q_full[2]; s_full[2][2]; p_full[2][2]; pv_done[2]; o_free[2];
// o_ready[2] (one completion per item: the last PV of the item has landed)
constexpr int N_BARS = 4 * NS + 2 + 4 + 4 + 2 + 2 + 2;
constexpr int BYTES = OFF_BAR + N_BARS * 8 + 16;
constexpr int ALLOC = BYTES + 1024;
constexpr uint32_t TMEM_COLS = 512;
}  // namespace tc4

__global__ void __launch_bounds__(tc4::kThreads, 1) prefix_tc4_kernel(const __grid_constant__ PrefixTc2Params P) {
  using namespace tc4;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *k_full = bars, *k_empty = bars + NS, *v_full = bars + 2 * NS, *v_empty = bars + 3 * NS;
  uint64_t *q_full = bars + 4 * NS;      // [2]
  uint64_t *s_full = q_full + 2;         // [tile][buf]
  uint64_t *p_full = s_full + 4;         // [tile][buf]
  uint64_t *pv_done = p_full + 4;        // [tile]
  uint64_t *o_free = pv_done + 2;        // [tile]
  uint64_t *o_ready = o_free + 2;        // [tile]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + N_BARS);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&P.tmK);
    ptx::prefetch_tmap(&P.tmV);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&q_full[t], 4);  // one elected arrival per softmax warp
      ptx::mbar_init(&pv_done[t], 1);
      ptx::mbar_init(&o_free[t], 4);  // one elected arrival per softmax warp
      ptx::mbar_init(&o_ready[t], 1);
      for (int b = 0; b < 2; ++b) {
        ptx::mbar_init(&s_full[2 * t + b], 1);
        ptx::mbar_init(&p_full[2 * t + b], 4);  // one elected arrival per softmax warp
      }
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;" ::: "memory");
    if (warp == 0) {
      // ================= TMA producer =================
      if (ptx::elect_one()) {
        uint32_t gb = 0;
        SegIter si;
        seg_begin(P, si);
        Item it;
        while (seg_next(P, si, it)) {
          for (int n = 0; n < it.nblk; ++n, ++gb) {
            const int st = gb % NS;
            const uint32_t ph = (gb / NS) & 1;
            const int t0 = (int)(it.kv_off + (int64_t)(it.blk_begin + n) * BN);
            uint8_t *sK = smem + OFF_K + st * KTILE;
            uint8_t *sV = smem + OFF_V + st * KTILE;
            ptx::mbar_wait(&k_empty[st], ph ^ 1);
            ptx::mbar_arrive_expect_tx(&k_full[st], KTILE);
            ptx::tma_load_3d(sK, &P.tmK, &k_full[st], 0, it.j, t0);
            ptx::tma_load_3d(sK + KPANEL, &P.tmK, &k_full[st], 64, it.j, t0);
            ptx::mbar_wait(&v_empty[st], ph ^ 1);
            ptx::mbar_arrive_expect_tx(&v_full[st], KTILE);
            ptx::tma_load_3d(sV, &P.tmV, &v_full[st], 0, it.j, t0);
            ptx::tma_load_3d(sV + KPANEL, &P.tmV, &v_full[st], 64, it.j, t0);
          }
        }
      }
    } else if (warp == 1) {
      // ================= MMA issuer =================
      if (ptx::elect_one()) {
        constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(BM, BN, false);
        constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(BM, HD, true);
        uint32_t gb = 0, qc[2] = {0, 0}, pc[4] = {0, 0, 0, 0}, oc[2] = {0, 0};
        long long *tr = (kTesting && P.trace && blockIdx.x == 0) ? P.trace : nullptr;
        uint32_t trn[2] = {0, 0};
        SegIter si;
        seg_begin(P, si);
        Item it;
        while (seg_next(P, si, it)) {
          if (it.nblk == 0) continue;
          const int ntile = (it.n_rows - it.row0 > BM) ? 2 : 1;
          auto issue_s = [&](int t, int n) {  // S_t(n) into buffer n & 1
            const uint32_t st = (gb + n) % NS;
            const uint32_t q_addr = ptx::smem_u32(smem + OFF_Q + t * QTILE);
            const uint32_t k_addr = ptx::smem_u32(smem + OFF_K + st * KTILE);
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
              ptx::mma_ss(tmem + t * 256 + (n & 1) * BN,
                          ptx::smem_desc_sw128(q_addr + (kk / 4) * QPANEL + (kk % 4) * 32, 16, 1024),
                          ptx::smem_desc_sw128(k_addr + (kk / 4) * KPANEL + (kk % 4) * 32, 16, 1024), idesc_s,
                          kk > 0);
            ptx::mma_commit(&s_full[2 * t + (n & 1)]);
          };
          auto wait_k = [&](int n) {
            const uint32_t g0 = gb + n;
            ptx::mbar_wait(&k_full[g0 % NS], (g0 / NS) & 1);
            ptx::tc_fence_after();
          };
          for (int t = 0; t < ntile; ++t) {
            ptx::mbar_wait(&q_full[t], qc[t] & 1);
            ++qc[t];
          }
          for (int n = 0; n < 2 && n < it.nblk; ++n) {  // prologue: S_t(0), S_t(1)
            wait_k(n);
            for (int t = 0; t < ntile; ++t) issue_s(t, n);
            ptx::mma_commit(&k_empty[(gb + n) % NS]);
          }
          for (int n = 0; n < it.nblk; ++n) {
            const uint32_t g0 = gb + n;
            const int st = g0 % NS;
            const bool more = n + 2 < it.nblk;
            ptx::mbar_wait(&v_full[st], (g0 / NS) & 1);
            const uint32_t v_addr = ptx::smem_u32(smem + OFF_V + st * KTILE);
            for (int t = 0; t < ntile; ++t) {
              const int pb = 2 * t + (n & 1);
              ptx::mbar_wait(&p_full[pb], pc[pb] & 1);
              ++pc[pb];
              if (tr && trn[t] < tc2::kTraceN) tr[(6 + t) * tc2::kTraceN + trn[t]++] = clock64();
              if (n == 0) {
                ptx::mbar_wait(&o_free[t], (oc[t] & 1) ^ 1);
                ++oc[t];
              }
              ptx::tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < BN / 16; ++kk)
                ptx::mma_ts(tmem + t * 256 + 128, tmem + t * 256 + (n & 1) * BN + kk * 8,
                            ptx::smem_desc_sw128(v_addr + kk * 2048, KPANEL, 1024), idesc_pv, (n > 0 || kk > 0));
              ptx::mma_commit(&pv_done[t]);
              if (n == it.nblk - 1) ptx::mma_commit(&o_ready[t]);
              if (more) {
                if (t == 0) wait_k(n + 2);
                issue_s(t, n + 2);
              }
            }
            ptx::mma_commit(&v_empty[st]);
            if (more) ptx::mma_commit(&k_empty[(g0 + 2) % NS]);
          }
          gb += it.nblk;
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    // ================= softmax / correction / epilogue =================
    const int t = (warp - 4) / 4;
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t o_col = tmem + lane_base + t * 256 + 128;
    uint8_t *sQ = smem + OFF_Q + t * QTILE;
    const float c2 = P.scale_log2;
    uint32_t sc[2] = {0, 0}, pvn = 0, orc = 0;  // s_full phase per buffer; PV_t count; items done
    long long *tr = (kTesting && P.trace && blockIdx.x == 0 && quarter == 0 && lane == 0) ? P.trace : nullptr;
    constexpr int kTN = tc2::kTraceN;
    SegIter si;
    seg_begin(P, si);
    Item it;
    while (seg_next(P, si, it)) {
      const int64_t trow0 = it.row0 + t * BM;
      if (trow0 >= it.n_rows) continue;
      const int64_t rr = trow0 + r;
      const bool live = rr < it.n_rows;
      int64_t seq = 0;
      int h = 0;
      if (live) {
        seq = P.seq_list ? P.seq_list[it.seq_off + rr / P.g] : rr / P.g;
        h = it.j * P.g + (int)(rr % P.g);
      }
      float *orow = P.o + it.slot * P.o_slot_stride + (seq * P.Hq + h) * HD;
      if (it.nblk == 0) {
        if (live) {
          P.lse[it.slot * P.lse_slot_stride + seq * P.Hq + h] = -INFINITY;
          for (int c = 0; c < HD / 4; ++c) reinterpret_cast<float4 *>(orow)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        continue;
      }
      {
        uint4 ch[16];
        if (live) {
          const uint4 *src = reinterpret_cast<const uint4 *>(P.q + seq * P.q_sb + (int64_t)h * P.q_sh);
#pragma unroll
          for (int c = 0; c < 16; ++c) ch[c] = __ldg(src + c);
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) ch[c] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int c = 0; c < 16; ++c)
          *reinterpret_cast<uint4 *>(sQ + (c / 8) * QPANEL + r * 128 + (((c % 8) ^ (r % 8)) * 16)) = ch[c];
        ptx::fence_proxy_async_smem();
        ptx::warp_arrive(&q_full[t]);
      }
      float m2 = -INFINITY, l = 0.f;
      for (int n = 0; n < it.nblk; ++n) {
        const int b = n & 1;
        const uint32_t s_col = tmem + lane_base + t * 256 + b * BN;
        const uint32_t trk = pvn;  // block counter of this tile
        if (tr && trk < kTN) tr[(3 * t + 0) * kTN + trk] = clock64();
        ptx::mbar_wait(&s_full[2 * t + b], sc[b] & 1);
        if (tr && trk < kTN) tr[(3 * t + 1) * kTN + trk] = clock64();
        ++sc[b];
        ptx::tc_fence_after();
        uint32_t sr[2][32];
        ptx::tmem_ld32(s_col, sr[0]);
        ptx::tmem_ld32(s_col + 32, sr[1]);
        ptx::tmem_ld_wait();
        if (tr && trk < kTN) tr[(10 + t) * kTN + trk] = clock64();
        const int64_t rem = it.kv_len - (int64_t)(it.blk_begin + n) * BN;
        if (rem < BN) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i >= rem) sr[c][i] = 0xff800000u;
        }
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
        const bool any = __any_sync(0xffffffffu, mnew > m2 + 8.0f);
        float alpha = 1.f;
        if (any) {
          const float mt = fmaxf(m2, mnew);
          alpha = fast_exp2(m2 - mt);
          m2 = mt;
        }
        const uint64_t cc = ptx::pack2(c2, c2), nm = ptx::pack2(-m2, -m2);
        uint64_t sacc[4] = {0, 0, 0, 0};
        if (tr && trk < kTN) {
          asm volatile("" ::"l"(nm));
          tr[(12 + t) * kTN + trk] = clock64();
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float x0, x1;
            ptx::unpack2(ptx::fma2(ptx::pack2(__uint_as_float(sr[c][2 * i]), __uint_as_float(sr[c][2 * i + 1])), cc,
                                   nm),
                         x0, x1);
            const float p0 = fast_exp2(x0), p1 = fast_exp2(x1);
            sacc[i % 4] = ptx::add2(sacc[i % 4], ptx::pack2(p0, p1));
            pk[i] = ptx::cvt_bf16x2(p0, p1);
          }
          ptx::tmem_st16(s_col + c * 16, pk);  // P(n) -> first 32 columns of S_t[n & 1]
        }
        float s0, s1, s2, s3;
        ptx::unpack2(ptx::add2(sacc[0], sacc[1]), s0, s1);
        ptx::unpack2(ptx::add2(sacc[2], sacc[3]), s2, s3);
        l = l * alpha + ((s0 + s1) + (s2 + s3));
        if (tr && trk < kTN) tr[(8 + t) * kTN + trk] = clock64();
        if (any && n >= 1) {  // rare O correction: needs PV_t(n-1) (completion index pvn-1) landed
          ptx::mbar_wait(&pv_done[t], (pvn - 1) & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t ov[32];
            ptx::tmem_ld32(o_col + c * 32, ov);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            ptx::tmem_st32(o_col + c * 32, ov);
          }
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::warp_arrive(&p_full[2 * t + b]);
        if (tr && trk < kTN) tr[(3 * t + 2) * kTN + trk] = clock64();
        ++pvn;
      }
      // All PVs of this item landed.  (pv_done cannot be used here: up to two PVs may be in
      // flight, and a parity wait cannot tell "one phase behind" from "two phases behind".)
      ptx::mbar_wait(&o_ready[t], orc & 1);
      ++orc;
      ptx::tc_fence_after();
      const float inv = 1.f / l;
      uint32_t *stage = reinterpret_cast<uint32_t *>(sQ + quarter * 32 * 128);
      const uint64_t my_row = live ? reinterpret_cast<uint64_t>(orow) : 0ull;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(o_col + c * 32, ov);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) stage[lane * 32 + (i ^ lane)] = __float_as_uint(__uint_as_float(ov[i]) * inv);
        __syncwarp();
#pragma unroll 4
        for (int rw = 0; rw < 32; ++rw) {
          const uint64_t base = __shfl_sync(0xffffffffu, my_row, rw);
          const uint32_t v = stage[rw * 32 + (lane ^ rw)];
          if (base) reinterpret_cast<float *>(base)[c * 32 + lane] = __uint_as_float(v);
        }
        __syncwarp();
      }
      ptx::tc_fence_before();
      ptx::warp_arrive(&o_free[t]);
      if (live) P.lse[it.slot * P.lse_slot_stride + seq * P.Hq + h] = (m2 + log2f(l)) * HYDRA_LN2;
      ptx::fence_proxy_async_smem();
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc<tc4::TMEM_COLS>(tmem);
  }
}

// ------------------------------------------------------------------ host side
static bool make_kv_map2(CUtensorMap *m, const void *base, int64_t T, int Hkv, int64_t st, int64_t sh,
                         int box_rows = tc2::BN) {
  const uint64_t dims[3] = {(uint64_t)tc2::HD, (uint64_t)Hkv, (uint64_t)T};
  const uint64_t strides[2] = {(uint64_t)sh * 2, (uint64_t)st * 2};
  const uint32_t box[3] = {64, 1, (uint32_t)box_rows};
  return encode_bf16_map(m, 3, base, dims, strides, box);
}

// Flat-mode schedule: grouped stream-K when there are at least two groups' worth of CTAs.
struct Tc2Plan {
  int group, ctas;
  int64_t total;  // stream-K units
};
static Tc2Plan tc2_plan(int64_t B, int g, int Hkv, int64_t P, int n_ctas, int bn = 128) {
  const int64_t nb = (P + bn - 1) / bn;
  const int64_t n_pairs = (B * g + 255) / 256;
  Tc2Plan pl;
  pl.group = (n_pairs > 1 && 2 * n_pairs <= n_ctas) ? (int)n_pairs : 1;
  pl.total = pl.group > 1 ? (int64_t)Hkv * nb : n_pairs * Hkv * nb;
  const int64_t G = std::min<int64_t>(n_ctas / pl.group, pl.total);
  pl.ctas = (int)(std::max<int64_t>(G, 1) * pl.group);
  return pl;
}

// Flat mode: number of partial slots per row the schedule over n_ctas CTAs produces.
int prefix_tc2_slots(int64_t B, int g, int Hkv, int64_t P, int n_ctas, int bn, bool pair, int pair_cluster,
                     int pair_item_cost) {
  if (pair) return prefix_pair_slots(B, g, Hkv, P, n_ctas, pair_cluster, pair_item_cost);
  const Tc2Plan pl = tc2_plan(B, g, Hkv, P, n_ctas, bn);
  if (pl.total <= 0) return 1;
  const int64_t nb = (P + bn - 1) / bn;
  const int64_t range = pl.total / (pl.ctas / pl.group);  // >= 1
  return (int)((nb + range - 1) / range + 1);
}

int prefix_tc2_ctas(int64_t B, int g, int Hkv, int64_t P, int n_ctas, int bn, bool pair, int pair_cluster) {
  if (pair) return prefix_pair_plan(B, g, Hkv, P, n_ctas, pair_cluster).ctas;
  return tc2_plan(B, g, Hkv, P, n_ctas, bn).ctas;
}

void prefix_tc2_plan_into(FusedCombine &fc, int64_t B, int g, int Hkv, int64_t P, int n_ctas, int bn) {
  const Tc2Plan pl = tc2_plan(B, g, Hkv, P, n_ctas, bn);
  fc.sk_total = pl.total;
  fc.sk_group = pl.group;
  fc.sk_G = pl.ctas / pl.group;
  fc.sk_nb = (int32_t)((P + bn - 1) / bn);
  fc.sk_npairs = (int32_t)((B * g + 255) / 256);
  fc.n_pre_splits = 0;
}

template <int kPoly, bool kPP, bool kSplit = false>
static cudaError_t tc2_launch(const PrefixTc2Params &P, int grid, cudaStream_t s) {
  const cudaError_t attr = ensure_smem_attr(reinterpret_cast<const void *>(prefix_tc2_kernel<kPoly, kPP, kSplit>),
                                            tc2::ALLOC);
  if (attr != cudaSuccess) return attr;
  prefix_tc2_kernel<kPoly, kPP, kSplit><<<grid, tc2::kThreads, tc2::ALLOC, s>>>(P);
  return cudaGetLastError();
}

static cudaError_t tc4_attr() {
  return ensure_smem_attr(reinterpret_cast<const void *>(prefix_tc4_kernel), tc4::ALLOC);
}

hydra_status launch_prefix_tc2(const PrefixTcArgs &a, int n_ctas, cudaStream_t s) {
  if (a.variant == 9 && !a.tasks && prefix_pair_supported(a.g)) return launch_prefix_pair(a, n_ctas, s);
  const int poly = a.poly_every;
  const bool v4 = a.variant == 4;
  const int bn = v4 ? tc4::BN : tc2::BN;
  // instantiations: kPolyEvery 0 (all MUFU), 3/4/8 (1/k of the pairs on the FMA pipe),
  // -1 (timing experiment: no exp); kSpec for variant 5 (v3 + speculative softmax)
  if (!(poly == 0 || poly == 3 || poly == 4 || poly == 8 || (kTesting && poly == -1))) return HYDRA_EINVAL;
  if (v4 && tc4_attr() != cudaSuccess) return HYDRA_ECUDA;
  PrefixTc2Params P;
  memset(&P, 0, sizeof(P));
  if (a.kv_total > 0) {
    if (!make_kv_map2(&P.tmK, a.k, a.kv_total, a.Hkv, a.kv_st, a.kv_sh, bn)) return HYDRA_ECUDA;
    if (!make_kv_map2(&P.tmV, a.v, a.kv_total, a.Hkv, a.kv_st, a.kv_sh, bn)) return HYDRA_ECUDA;
  }
  P.bn = bn;
  P.debug = kTesting ? a.debug_variant : 0;
  P.trace = kTesting ? reinterpret_cast<long long *>(a.trace) : nullptr;
  P.mutate = kTesting ? a.mutate : 0;
  P.q = reinterpret_cast<const __nv_bfloat16 *>(a.q);
  P.q_sb = a.q_sb;
  P.q_sh = a.q_sh;
  P.Hq = a.Hq;
  P.Hkv = a.Hkv;
  P.g = a.g;
  P.scale_log2 = a.scale_log2;
  P.P = a.P;
  P.B = a.B;
  P.n_pairs = (int)(((int64_t)a.B * a.g + 255) / 256);
  P.tasks = a.tasks;
  P.n_tasks = a.n_tasks;
  P.seq_list = a.seq_list;
  P.n_splits = a.n_splits;
  P.n_items = a.tasks ? a.n_tasks * a.Hkv * a.n_splits : 0;
  P.nb = (int)((a.P + bn - 1) / bn);
  Tc2Plan pl{1, n_ctas, 0};
  if (!a.tasks) pl = tc2_plan(a.B, a.g, a.Hkv, a.P, n_ctas > 0 ? n_ctas : 1 << 30, bn);
  P.total_blocks = a.tasks ? 0 : pl.total;
  P.group = pl.group;
  P.o = a.o;
  P.lse = a.lse;
  P.o_slot_stride = a.o_slot_stride;
  P.lse_slot_stride = a.lse_slot_stride;
  P.fc = a.fc;
  P.timer = a.timer;
  if (P.fc.cnt) {  // fused Eq. 5: flat mode, variants 3 / 5 / 6; the plan must be this launch's
    if (a.tasks || v4 || P.fc.sk_total != pl.total || P.fc.sk_G != pl.ctas / pl.group || P.fc.sk_group != pl.group)
      return HYDRA_EINVAL;
  }
  const int64_t work = a.tasks ? P.n_items : P.total_blocks;
  if (work == 0) return HYDRA_OK;
  const int grid = a.tasks ? (int)(n_ctas > 0 && n_ctas < work ? n_ctas : work) : pl.ctas;
  if (v4) {
    prefix_tc4_kernel<<<grid, tc4::kThreads, tc4::ALLOC, s>>>(P);
    return cudaGetLastError() == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
  }
  const bool spec = a.variant == 5;
  cudaError_t e;
  if (a.variant == 6 || a.variant == 9) {  // split P publication (9: task mode / other g of the pair kernel)
    e = poly == 4 ? tc2_launch<4, false, true>(P, grid, s) : tc2_launch<0, false, true>(P, grid, s);
    return e == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
  }
  switch (poly * 2 + (spec ? 1 : 0)) {
    case 0: e = tc2_launch<0, false>(P, grid, s); break;
    case 1: e = tc2_launch<0, true>(P, grid, s); break;
    case 6: e = tc2_launch<3, false>(P, grid, s); break;
    case 7: e = tc2_launch<3, true>(P, grid, s); break;
    case 8: e = tc2_launch<4, false>(P, grid, s); break;
    case 9: e = tc2_launch<4, true>(P, grid, s); break;
    case 16: e = tc2_launch<8, false>(P, grid, s); break;
    case 17: e = tc2_launch<8, true>(P, grid, s); break;
#ifdef HYDRA_TESTING
    case -2: e = tc2_launch<-1, false>(P, grid, s); break;  // timing experiment: no exp (invalid results)
    case -1: e = tc2_launch<-1, true>(P, grid, s); break;
#endif
    default: return HYDRA_EINVAL;
  }
  return e == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

}  // namespace hydra

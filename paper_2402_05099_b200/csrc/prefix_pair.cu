// prefix_pair.cu -- persistent CTA-pair (cta_group::2) tcgen05 prefix attention for sm_100a.
//
// PAPER.md §3.2: the B*g decode queries of a KV head are stacked into one
// matrix (row r = b*g + i holds q[b, j*g+i]) and attend to the shared prefix K/V as a dense
// GEMM-shaped problem that reads the prefix once (App. B).  Output per row: the
// normalised partial O (fp32) and its natural-log LSE (Eq. 4) for the Eq. 5 combine.
//
// Why a CTA pair (measured limiter of the one-CTA two-tile kernel, prefix_tc2.cu): there each
// 128-row tile owns ONE score buffer in TMEM (2 tiles x (S 128 + O 128) = 512 columns), so a
// tile's chain S(n) -> softmax -> PV(n) -> S(n+1) is serial and the tensor pipe idles for the
// whole softmax: ~3.4-3.6 K cycles per 2 K-cycle block pair (57-60 % tensor occupancy).
// Here two CTAs on the two SMs of a TPC share every MMA (M = 256: each CTA supplies and
// receives 128 query rows; B is split along N, so each CTA stages HALF of every K/V tile),
// each CTA holds ONE query tile, and its TMEM holds two score buffers plus two output
// accumulators:
//   S[0] cols [0,128)  S[1] cols [128,256)  O_a cols [256,384)  O_b cols [384,512)
// The score MMA of block n+2 is issued right after the PV of block n, so S(n+1) is already
// in TMEM when the softmax of block n ends: the softmax runs back to back and the tensor
// pipe only waits for it when the softmax is slower than the MMAs.
// Two softmax warpgroups per CTA split every 128-token block by TOKENS: WG a takes tokens
// 0-63 (S cols 0-63 -> P_a packed in cols 0-31, accumulated in O_a), WG b tokens 64-127
// (cols 64-127 -> P_b in cols 64-95, O_b).  Each is an independent online softmax over its
// half of the prefix (own running max m and sum l); the epilogue merges the two states
// exactly (Eq. 5 with two parts).  So every SM sub-partition runs two softmax warps (one per
// WG) over 64 columns each instead of one warp over 128: half the serial chain per block.
//
// Roles per CTA (384 threads):
//   warp 0      TMA producer (both CTAs): K tokens [64*rank, +64) of each block (4-stage
//               ring); completions counted on the pair LEADER's barriers
//   warp 2      TMA producer (both CTAs): V dims [64*rank, +64) of each block (4-stage ring)
//   warp 3      TMA producer (both CTAs): the Q tile of each item (2 buffers), as early as a
//               buffer frees
//   warp 1      TMEM allocation (both CTAs, cta_group::2) and, in the leader only, the single
//               MMA-issuing thread:  S(0) S(1) | PV_a(n) PV_b(n) S(n+2) | ...  (polls its
//               barriers: try_wait's suspension cost ~500 cycles of reaction per block)
//   warps 4-7   softmax WG a (thread = query row = TMEM lane), warps 8-11 WG b
// Schedule: grouped stream-K over (head, 128-token block) as prefix_tc2.cu, with the CTA pair
// as the worker: pair p of a group takes query rows [256p, 256p+256) of every head.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace hydra {

namespace pr {
constexpr int BM = 128;     // query rows per CTA
constexpr int BN = 128;     // KV tokens per block
constexpr int HD = 128;     // head dim
constexpr int NQ = 2;       // Q buffers
constexpr int NSK = 4;      // K stages
constexpr int NSV = 4;      // V stages
// HYDRA_PAIR_SPLIT_ISSUE: the score MMAs are issued from warp 3's thread (SM sub-partition 3, next
// to the Q loads: one polling loop runs both) and the PV MMAs stay on warp 1, so the cost an
// MMA-issuing warp puts on the softmax warps of its sub-partition (~600 cycles per block,
// tools/pair_trace.py) is split between two of them.  S(n+3) then waits for PV(n) to COMPLETE
// (barrier sfree) instead of queueing behind it in one thread.  Measured SLOWER (profiles/
// r2z_pair_split_issue_ab.log: C3 1164 -> 1082, C4 1236 -> 1134, C6 1013 -> 919 TFLOP/s; parity
// green): the wait for PV(n)'s completion costs more than the shared issue slots did.  Kept as a
// compile-time option, off.
#ifndef HYDRA_PAIR_SPLIT_ISSUE
#define HYDRA_PAIR_SPLIT_ISSUE 0
#endif
constexpr bool kSplitIssue = HYDRA_PAIR_SPLIT_ISSUE != 0;
// HYDRA_PAIR_SPEC: speculative softmax -- a warpgroup computes P(n) with its own previous running max
// right after loading S(n) and checks m(n) afterwards (recomputing P only when the max moved).
// Bit-identical results; measured ~1 % SLOWER (profiles/r3e_pair_spec_softmax_ab.log: C3 1164 -> 1153,
// C4 1235 -> 1220 TFLOP/s), so the row max and the m hand-off are not what bounds the block period.
// Kept as a compile-time option, off.
#ifndef HYDRA_PAIR_SPEC
#define HYDRA_PAIR_SPEC 0
#endif
constexpr bool kSpec = HYDRA_PAIR_SPEC != 0;
constexpr int kThreads = 384;
constexpr int kLowRegs = 88;  // producer / MMA warps (softmax warps: 208; 16 K registers per sub-partition)
constexpr int QPANEL = BM * 128;      // 128 rows x 128 B
constexpr int QTILE = 2 * QPANEL;     // 32 KB
constexpr int KPANEL = 64 * 128;      // 64 tokens x 128 B
constexpr int KHALF = 2 * KPANEL;     // 16 KB: this CTA's 64 tokens x 128 dims
constexpr int VHALF = BN * 128;       // 16 KB: 128 tokens x this CTA's 64 dims
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + NQ * QTILE;
constexpr int OFF_V = OFF_K + NSK * KHALF;
constexpr int NSB = 3;                      // score buffers in TMEM
// Lazy running max: raised only when a row's block max exceeds it by more than kRaise (log2
// units), so P <= 2^32 (bf16 and the fp32 O / l accumulators have the range: over a piece of
// <= 2^20 tokens they stay finite for |v| < 2^70), and a needle-like score jump (the 'mixed' inputs:
// ~12-17 log2 units above the rest) needs no O correction at all.  8 (prefix_tc2) made a
// quarter of the blocks at C3 wait for the previous PV before publishing P.
constexpr float kRaise = 32.0f;
#ifndef HYDRA_PAIR_POLL_NS
#define HYDRA_PAIR_POLL_NS 64
#endif
constexpr int kPollSleepNs = HYDRA_PAIR_POLL_NS;
#ifndef HYDRA_PAIR_MMA_WARP
#define HYDRA_PAIR_MMA_WARP 1
#endif
constexpr int kMmaWarp = HYDRA_PAIR_MMA_WARP;  // 1 or 3 (warp 1 allocates TMEM either way)

  // MMA thread's back-off between barrier probe rounds
constexpr int O_COL = NSB * BN;             // O accumulator: TMEM columns [384, 512)
constexpr int OFF_X = OFF_V + NSV * VHALF;  // row max / sum exchange [parity][WG][128 rows]
constexpr int OFF_BAR = OFF_X + 6 * BM * 4;  // m exchange [WG][128] + epilogue (m, l) [WG][128][2]
// kf, ke [NSK]; vf, ve [NSV]; qf, qe [NQ]; sf [NSB]; pf [NSB]; ordy; ofree; xfree [NQ]; sfree [NSB]
constexpr int N_BARS = 2 * NSK + 2 * NSV + 3 * NQ + 3 * NSB + 2;
constexpr int BYTES = OFF_BAR + N_BARS * 8 + 16;
constexpr int ALLOC = BYTES + 1024;
static_assert(ALLOC <= 232448, "prefix_pair smem over the 227 KB opt-in limit");
constexpr uint32_t TMEM_COLS = 512;
// diagnostics (testing build): per block, clock64 of cluster 0's events.  Rows 0-5 WG a warp 4
// lane 0 of the leader (S wait begin, S ready, S in registers, max done, exps done, P arrived),
// 6-11 the same for WG b, 12 / 13 MMA thread saw P_a / P_b, 14 S(n+2) issued, 16-21 WG a of the
// peer CTA.
constexpr int kTraceN = 1024;
__device__ __forceinline__ void trace(long long *tr, int row, uint32_t i) {
  if (kTesting && tr && i < (uint32_t)kTraceN) tr[row * kTraceN + i] = clock64();
}
constexpr int kMaxGroups = 80;  // stream-K groups per launch (<= 74 CTA pairs on 148 SMs)
}  // namespace pr

struct __align__(64) PrefixPairParams {
  CUtensorMap tmQ;  // 4-D {128 dims, g, Hkv, B}, box {64, g, 1, 128/g}
  CUtensorMap tmK;  // 3-D {128, Hkv, P}, box {64, 1, 64}
  CUtensorMap tmV;  // 3-D {128, Hkv, P}, box {64, 1, 128}
  int32_t Hq, Hkv, g;
  float scale_log2;
  int64_t P;
  int32_t B;
  int32_t n_pairs;       // ceil(B*g / 256)
  int32_t nb;            // ceil(P / 128)
  int64_t total_blocks;  // stream-K units: Hkv*nb (grouped) or n_pairs*Hkv*nb
  int32_t group;         // pairs (workers) per group: n_pairs when grouped, else 1
  float *o, *lse;
  int64_t o_slot_stride, lse_slot_stride;
  int32_t n_slots;  // partial slots per row the caller reserved: the piece ending a (pair, head) unit
                    // marks the slots after its own empty (LSE -inf), so no separate fill runs
  int32_t mutate;  // testing build only: 3 = worker 0 skips one 4-row group of its stores
  long long *trace;  // testing build only: cluster-0 event timestamps [kTraceRows][kTraceN] (tools/pair_trace.py)
  unsigned long long *timer;  // measurement: [0] min CTA start, [1] max CTA end (%globaltimer ns); null = off
  int32_t debug;     // testing build only, timing experiments (invalid results): 4 = no K/V TMA after the ring
                     // fill, 2 = no softmax (P published as soon as S lands), 8 = no epilogue O stores
  int64_t bound[pr::kMaxGroups + 1];  // stream-K group c walks blocks [bound[c], bound[c+1]) (pair_bounds)
};

namespace pr {
struct Item {
  int64_t row0;  // first stacked row of the 256-row pair
  int32_t j, slot, blk_begin, nblk;
};

// Grouped stream-K over workers (CTA pairs), the flat-mode plan of prefix_tc2.cu: workers form
// groups of `group`; member m of a group owns pair m of every head and the group walks a
// contiguous range of the (head, block) space; a range may start / end inside a head, and
// each piece writes its own partial slot (index of this group relative to the head's first).
struct Iter {
  int64_t x, end;
};
__device__ __forceinline__ int n_workers() { return gridDim.x / 2; }
__device__ __forceinline__ int worker() { return blockIdx.x / 2; }
__device__ __forceinline__ int n_groups(const PrefixPairParams &P) { return n_workers() / P.group; }
__device__ __forceinline__ int64_t sk_start(const PrefixPairParams &P, int64_t c) { return P.bound[c]; }
__device__ __forceinline__ void it_begin(const PrefixPairParams &P, Iter &s) {
  const int grp = worker() / P.group;
  if (grp >= n_groups(P)) {
    s.x = s.end = 0;
  } else {
    s.x = sk_start(P, grp);
    s.end = sk_start(P, grp + 1);
  }
}
__device__ __forceinline__ bool it_next(const PrefixPairParams &P, Iter &s, Item &it) {
  if (s.x >= s.end) return false;
  const int64_t unit = s.x / P.nb;
  const int b = (int)(s.x % P.nb);
  const int64_t room = s.end - s.x;
  const int len = (int)(P.nb - b < room ? P.nb - b : room);
  const int G = n_groups(P);
  const int64_t x0 = unit * P.nb;
  int64_t c0 = x0 * G / P.total_blocks;
  while (c0 + 1 < G && sk_start(P, c0 + 1) <= x0) ++c0;
  while (c0 > 0 && sk_start(P, c0) > x0) --c0;
  const int64_t pair = P.group > 1 ? (int64_t)(worker() % P.group) : unit % P.n_pairs;
  it.j = (int)(P.group > 1 ? unit : unit / P.n_pairs);
  it.row0 = pair * (2 * BM);
  it.slot = (int)(worker() / P.group - c0);
  it.blk_begin = b;
  it.nblk = len;
  s.x += len;
  return true;
}

// Block cursor of the MMA thread: walks this worker's blocks in order across items.
struct Cursor {
  Iter si;
  Item it;
  int n;        // block within the item
  uint32_t qi;  // item index (Q buffer = qi % NQ)
  bool valid;
  __device__ __forceinline__ void init(const PrefixPairParams &P) {
    it_begin(P, si);
    valid = it_next(P, si, it);
    n = 0;
    qi = 0;
  }
  __device__ __forceinline__ void advance(const PrefixPairParams &P) {
    if (++n >= it.nblk) {
      valid = it_next(P, si, it);
      n = 0;
      ++qi;
    }
  }
};
}  // namespace pr

// kC: CTA pairs per cluster (1, 2 or 4).  The kC pairs of a cluster are members of one
// stream-K group (same heads and blocks, different query rows), so every K / V tile they need is
// the same: each CTA loads a 1/kC piece of its half tile and multicasts it to the CTAs with the
// same rank in their pair -- L2 -> SM traffic / kC.  (Measured with the K/V loads switched off:
// the prefix alone at the power cap ran 13 % faster at 12 % higher SM clock -- tools/pair_power.py.)
template <int kPolyEvery, int kC>
__global__ void __launch_bounds__(pr::kThreads, 1) prefix_pair_kernel(const __grid_constant__ PrefixPairParams P) {
  using namespace pr;
  extern __shared__ uint8_t smem_raw[];
  // SM-partitioned schedule on one stream: the suffix kernel (a programmatic dependent) may start
  // as soon as every CTA of this persistent grid is resident -- it then takes the other SMs
  asm volatile("griddepcontrol.launch_dependents;");
  if (P.timer && threadIdx.x == 0) atomicMin(P.timer, gtimer());
  // diagnostics (testing build): every CTA's %globaltimer at entry / setup done / exit, rows 40..
  long long *cta_tr = (kTesting && P.trace && blockIdx.x < 1024) ? P.trace + 40 * kTraceN + blockIdx.x * 4 : nullptr;
  if (cta_tr && threadIdx.x == 0) cta_tr[0] = (long long)gtimer();
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *kf = bars, *ke = kf + NSK, *vf = ke + NSK, *ve = vf + NSV, *qf = ve + NSV, *qe = qf + NQ;
  uint64_t *sf = qe + NQ, *pf = sf + NSB, *ordy = pf + NSB, *ofree = ordy + 1, *xfree = ofree + 1;
  uint64_t *sfree = xfree + NQ;  // split issue: PV(n) done, score buffer n % NSB may be overwritten
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + N_BARS);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = ptx::cluster_ctarank();
  const uint32_t rank = crank & 1;       // rank within the CTA pair (0: the pair's MMA leader)
  const uint32_t pip = crank >> 1;       // pair within the cluster
  const uint32_t lead = crank & ~1u;     // cluster rank of this pair's leader
  constexpr uint16_t kAll = (uint16_t)((1u << (2 * kC)) - 1);
  const uint16_t pair_mask = (uint16_t)(3u << (2 * pip));
  const uint16_t half_mask = (uint16_t)((kC == 1 ? 1u : kC == 2 ? 0x5u : 0x55u) << rank);  // same rank-in-pair

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&P.tmQ);
    ptx::prefetch_tmap(&P.tmK);
    ptx::prefetch_tmap(&P.tmV);
    for (int i = 0; i < NSK; ++i) {
      ptx::mbar_init(&kf[i], 1);
      ptx::mbar_init(&ke[i], kC);  // one release per pair of the cluster
    }
    for (int i = 0; i < NSV; ++i) {
      ptx::mbar_init(&vf[i], 1);
      ptx::mbar_init(&ve[i], kC);
    }
    for (int i = 0; i < NQ; ++i) {
      ptx::mbar_init(&qf[i], 1);
      ptx::mbar_init(&qe[i], 1);
      ptx::mbar_init(&xfree[i], 8);  // this CTA's 8 softmax warps: done staging the epilogue in Q buffer i
    }
    for (int i = 0; i < NSB; ++i) {
      ptx::mbar_init(&sf[i], 1);
      ptx::mbar_init(&pf[i], 8);  // the 4 warps of the block's WG x 2 CTAs (leader's copy)
      ptx::mbar_init(&sfree[i], 1);
    }
    ptx::mbar_init(ordy, 1);
    ptx::mbar_init(ofree, 16);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (cta_tr && threadIdx.x == 0) cta_tr[1] = (long long)gtimer();

  if (warp == 3) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kLowRegs) : "memory");
    // ================= Q producer (both CTAs): this CTA's 128 stacked query rows per item =================
    // Its own thread, so the next item's Q is loaded as soon as its buffer is free (the item two
    // back has finished its score MMAs and its epilogue staging), not behind the current item's
    // K loads: issued there, it landed ~3 K cycles after the current item's epilogue.
    const bool elected = ptx::elect_one();  // once, converged (elect.sync takes the full warp)
    if (kSplitIssue && rank == 0 && elected) {
      // Q producer and score-MMA issuer in one polling loop (split issue, the pair's leader)
      const uint32_t qf0 = ptx::mapa(ptx::smem_u32(qf), lead);
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(2 * BM, BN, false);
      long long *tr = (kTesting && P.trace && blockIdx.x == 0) ? P.trace : nullptr;
      uint32_t qi = 0, gs = 0;
      Iter si;
      it_begin(P, si);
      Item it;
      bool q_more = it_next(P, si, it);
      Cursor cs;
      cs.init(P);
      while (q_more || cs.valid) {
        bool progress = false;
        if (q_more) {  // the next item's Q once its buffer is free (score MMAs and epilogue staging done)
          const int qb = qi % NQ;
          const uint32_t par = ((qi / NQ) & 1) ^ 1;
          if (ptx::mbar_test_wait(&qe[qb], par) && ptx::mbar_test_wait(&xfree[qb], par)) {
            ptx::mbar_arrive_expect_tx(&qf[qb], 2 * QTILE);
            const int b0 = (int)(it.row0 / P.g);
            uint8_t *sQ = smem + OFF_Q + qb * QTILE;
            ptx::tma_load_4d_pair(sQ, &P.tmQ, qf0 + qb * 8, 0, 0, it.j, b0);
            ptx::tma_load_4d_pair(sQ + QPANEL, &P.tmQ, qf0 + qb * 8, 64, 0, it.j, b0);
            ++qi;
            q_more = it_next(P, si, it);
            progress = true;
          }
        }
        if (cs.valid) {  // S(gs): its buffer's PV(gs - NSB) done, its Q (first block) and K landed
          const int qb = cs.qi % NQ, ks = gs % NSK, sb = gs % NSB;
          if ((gs < (uint32_t)NSB || ptx::mbar_test_wait(&sfree[sb], ((gs / NSB) - 1) & 1)) &&
              (cs.n != 0 || ptx::mbar_test_wait(&qf[qb], (cs.qi / NQ) & 1)) &&
              ptx::mbar_test_wait(&kf[ks], (gs / NSK) & 1)) {
            trace(tr, 22, gs);
            ptx::tc_fence_after();
            const uint32_t qa = ptx::smem_u32(smem + OFF_Q + qb * QTILE), ka = ptx::smem_u32(smem + OFF_K + ks * KHALF);
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
              ptx::mma2_ss(tmem + sb * BN, ptx::smem_desc_sw128(qa + (kk / 4) * QPANEL + (kk % 4) * 32, 16, 1024),
                           ptx::smem_desc_sw128(ka + (kk / 4) * KPANEL + (kk % 4) * 32, 16, 1024), idesc_s, kk > 0);
            ptx::mma2_commit(&sf[sb], pair_mask);
            ptx::mma2_commit(&ke[ks], kAll);
            if (cs.n == cs.it.nblk - 1) ptx::mma2_commit(&qe[qb], pair_mask);
            trace(tr, 14, gs);
            ++gs;
            cs.advance(P);
            progress = true;
          }
        }
        if (!progress) __nanosleep(kPollSleepNs);
      }
    } else if (elected) {
      const uint32_t qf0 = ptx::mapa(ptx::smem_u32(qf), lead);
      uint32_t qi = 0;
      Iter si;
      it_begin(P, si);
      Item it;
      while (it_next(P, si, it)) {
        const int qb = qi % NQ;
        ptx::mbar_wait(&qe[qb], ((qi / NQ) & 1) ^ 1);
        ptx::mbar_wait(&xfree[qb], ((qi / NQ) & 1) ^ 1);  // and the epilogue staged there is done
        if (rank == 0) ptx::mbar_arrive_expect_tx(&qf[qb], 2 * QTILE);
        const int b0 = (int)((it.row0 + BM * rank) / P.g);
        uint8_t *sQ = smem + OFF_Q + qb * QTILE;
        ptx::tma_load_4d_pair(sQ, &P.tmQ, qf0 + qb * 8, 0, 0, it.j, b0);
        ptx::tma_load_4d_pair(sQ + QPANEL, &P.tmQ, qf0 + qb * 8, 64, 0, it.j, b0);
        if (kTesting && P.trace && blockIdx.x == 0) trace(P.trace, 36, qi);  // Q(qi) issued
        ++qi;
      }
    }
  } else if (warp == 0 || warp == 2) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kLowRegs) : "memory");
    // ================= TMA producers (both CTAs): warp 0 K, warp 2 V =================
    // (separate threads, so a K tile is issued as soon as its slot frees, independently of V)
    if (ptx::elect_one()) {
      const bool kq_role = warp == 0;
      const uint32_t kf0 = ptx::mapa(ptx::smem_u32(kf), lead), vf0 = ptx::mapa(ptx::smem_u32(vf), lead);
      uint32_t kq = 0, vq = 0;
      long long *tr = (kTesting && P.trace && blockIdx.x == 0 && kq_role) ? P.trace : nullptr;
      Iter si;
      it_begin(P, si);
      Item it;
      while (it_next(P, si, it)) {
        for (int n = 0; n < it.nblk; ++n) {
          const int t0 = (it.blk_begin + n) * BN;
          if (kTesting && (P.debug & 4) && (kq_role ? kq : vq) >= (uint32_t)NSK) {  // timing experiment only
            uint64_t *e = kq_role ? &ke[kq % NSK] : &ve[vq % NSV];
            ptx::mbar_wait(e, (((kq_role ? kq : vq) / NSK) & 1) ^ 1);
            if (rank == 0) ptx::mbar_arrive(kq_role ? &kf[kq % NSK] : &vf[vq % NSV]);
            if (kq_role)
              ++kq;
            else
              ++vq;
            continue;
          }
          if (kq_role) {
            const int ks = kq % NSK;
            ptx::mbar_wait(&ke[ks], ((kq / NSK) & 1) ^ 1);
            trace(tr, 20, kq);
            if (rank == 0) ptx::mbar_arrive_expect_tx(&kf[ks], 2 * KHALF);
            uint8_t *sK = smem + OFF_K + ks * KHALF;
            if constexpr (kC == 1) {
              ptx::tma_load_3d_pair(sK, &P.tmK, kf0 + ks * 8, 0, it.j, t0 + 64 * (int)rank);
              ptx::tma_load_3d_pair(sK + KPANEL, &P.tmK, kf0 + ks * 8, 64, it.j, t0 + 64 * (int)rank);
            } else {  // this CTA's piece of the half tile: panel pip % 2, token rows (pip / 2) * 32 (kC = 4)
              const int panel = kC == 2 ? (int)pip : (int)(pip & 1), trow = kC == 2 ? 0 : (int)(pip >> 1) * 32;
              ptx::tma_load_3d_pair_mc(sK + panel * KPANEL + trow * 128, &P.tmK, kf0 + ks * 8, 64 * panel, it.j,
                                       t0 + 64 * (int)rank + trow, half_mask);
            }
            ++kq;
          } else {
            const int vs = vq % NSV;
            ptx::mbar_wait(&ve[vs], ((vq / NSV) & 1) ^ 1);
            if (rank == 0) ptx::mbar_arrive_expect_tx(&vf[vs], 2 * VHALF);
            if constexpr (kC == 1) {
              ptx::tma_load_3d_pair(smem + OFF_V + vs * VHALF, &P.tmV, vf0 + vs * 8, 64 * (int)rank, it.j, t0);
            } else {  // token rows [pip * 128 / kC, +128 / kC) of this half's 64 dims
              const int trow = (int)pip * (BN / kC);
              ptx::tma_load_3d_pair_mc(smem + OFF_V + vs * VHALF + trow * 128, &P.tmV, vf0 + vs * 8, 64 * (int)rank,
                                       it.j, t0 + trow, half_mask);
            }
            ++vq;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kLowRegs) : "memory");
    // ================= MMA issuer (leader CTA, one thread) =================
    if (rank == 0 && ptx::elect_one()) {  // the pair's leader
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(2 * BM, BN, false);  // S = Q K^T, M = 256
      constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(2 * BM, HD, true);  // O += P V, V MN-major
      long long *tr = (kTesting && P.trace && blockIdx.x == 0) ? P.trace : nullptr;
      Cursor cs, cp;
      cs.init(P);
      cp.init(P);
      uint32_t gs = 0, gp = 0, oi = 0;
      // S(gs) = Q K(gs)^T into score buffer gs % NSB; `ready` = its Q (first block of an item) and
      // K tile were already seen landed
      auto issue_s = [&](bool ready) {
        if (!cs.valid) return;
        const int qb = cs.qi % NQ;
        const int ks = gs % NSK, sb = gs % NSB;
        if (!ready) {
          if (cs.n == 0) ptx::mbar_poll(&qf[qb], (cs.qi / NQ) & 1);
          ptx::mbar_poll(&kf[ks], (gs / NSK) & 1);
        }
        trace(tr, 21, gs);
        ptx::tc_fence_after();
        const uint32_t qa = ptx::smem_u32(smem + OFF_Q + qb * QTILE), ka = ptx::smem_u32(smem + OFF_K + ks * KHALF);
#ifndef HYDRA_PAIR_DUP_S
#define HYDRA_PAIR_DUP_S 1
#endif
#pragma unroll
        for (int rep = 0; rep < HYDRA_PAIR_DUP_S; ++rep)  // diagnostics: > 1 re-issues identical score MMAs
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::mma2_ss(tmem + sb * BN, ptx::smem_desc_sw128(qa + (kk / 4) * QPANEL + (kk % 4) * 32, 16, 1024),
                       ptx::smem_desc_sw128(ka + (kk / 4) * KPANEL + (kk % 4) * 32, 16, 1024), idesc_s, kk > 0);
        ptx::mma2_commit(&sf[sb], pair_mask);
        ptx::mma2_commit(&ke[ks], kAll);  // every CTA of the cluster: its K piece went to all pairs
        if (cs.n == cs.it.nblk - 1) ptx::mma2_commit(&qe[qb], pair_mask);
        trace(tr, 14, gs);
        ++gs;
        cs.advance(P);
      };
      if constexpr (!kSplitIssue)
        for (int i = 0; i < NSB; ++i) issue_s(false);
      // Per block: PV(gp) (both token halves into the one O), then S(gp + NSB) into the score
      // buffer PV(gp) just read.  A barrier probe costs ~150 cycles of latency
      // (tools/pair_trace.py), so every barrier this block still needs is probed together each
      // round (independent SYNCS.PHASECHK in flight at once) instead of one after another.
      while (cp.valid) {
        const int sb = gp % NSB, vs = gp % NSV;
        const uint32_t acc0 = cp.n > 0 ? 1u : 0u;
        const bool s_next = !kSplitIssue && cs.valid;
        const int qb = cs.qi % NQ, ks = gs % NSK;
        const uint32_t qpar = (cs.qi / NQ) & 1, kpar = (gs / NSK) & 1, ppar = (gp / NSB) & 1;
        bool of = cp.n != 0, v = false, a = false, k = !s_next, q = !(s_next && cs.n == 0);
        do {
          if (!of) of = ptx::mbar_test_wait(ofree, (oi & 1) ^ 1);  // previous item's epilogue done with O
          if (!v) v = ptx::mbar_test_wait(&vf[vs], (gp / NSV) & 1);
          if (!a) a = ptx::mbar_test_wait(&pf[sb], ppar);
          if (!k) k = ptx::mbar_test_wait(&kf[ks], kpar);
          if (!q) q = ptx::mbar_test_wait(&qf[qb], qpar);
          if (!(of && v && a)) __nanosleep(kPollSleepNs);  // yield issue slots to the softmax warps of this SMSP
        } while (!(of && v && a));
        if (cp.n == 0) ++oi;
        trace(tr, 12, gp);
        ptx::tc_fence_after();
        const uint32_t va = ptx::smem_u32(smem + OFF_V + vs * VHALF);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // P(gp): bf16 pairs in the first 64 columns of its score buffer
          ptx::mma2_ts(tmem + O_COL, tmem + sb * BN + kk * 8,
                       ptx::smem_desc_sw128(va + kk * 2048, 16, 1024), idesc_pv, acc0 | (kk > 0));
        trace(tr, 19, gp);
        if (cp.n == cp.it.nblk - 1) ptx::mma2_commit(ordy, pair_mask);  // the item's last PV: epilogue may read O
        if constexpr (kSplitIssue) {  // the score thread may overwrite buffer sb; the V slot is free
          ptx::mma2_commit(&sfree[sb], (uint16_t)(1u << lead));
          ptx::mma2_commit(&ve[vs], kAll);
          ++gp;
          cp.advance(P);
          continue;
        }
        ++gp;
        cp.advance(P);
        while (!(k && q)) {
          if (!k) k = ptx::mbar_test_wait(&kf[ks], kpar);
          if (!q) q = ptx::mbar_test_wait(&qf[qb], qpar);
          if (!(k && q)) __nanosleep(kPollSleepNs);
        }
        trace(tr, 22, gs);
        // S(gp - 1 + NSB) right behind the PV (it overwrites the score buffer whose P the PV read),
        // then the V slot release: one commit covering both, off the path to the next score MMA
        issue_s(true);
        ptx::mma2_commit(&ve[vs], kAll);
      }
    }
  } else if (warp >= 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    // ================= softmax / epilogue (both CTAs) =================
    // Block n of an item goes to WG (n & 1) (warps 4-7 even, 8-11 odd).  The running max is one
    // chain through the blocks: the WG of block n receives m(n-1) from the other WG (shared
    // memory + named barrier of the two warps holding the same rows), decides m(n) and passes
    // it on right after its row max, then spends the rest of the block on exp2 / P while the
    // other WG already works on block n+1.  P(n) is scaled by m(n); O is one accumulator,
    // rescaled (rarely: the max is raised only by > kRaise, log2 units) by the WG whose block
    // raised m, after PV(n-1) landed.  Each WG keeps its own l relative to the last m it used.
    const int x = (warp - 4) / 4;
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t pf0 = ptx::mapa(ptx::smem_u32(pf), lead), of0 = ptx::mapa(ptx::smem_u32(ofree), lead);
    float *xch = reinterpret_cast<float *>(smem + OFF_X);  // [2 slots][128 rows]
    const int bar_out = 1 + quarter + 4 * x, bar_in = 1 + quarter + 4 * (1 - x), bar_epi = 9 + quarter;
    long long *tr = (kTesting && P.trace && blockIdx.x < 2 && quarter == 0 && lane == 0 && (rank == 0 || x == 0))
                        ? P.trace : nullptr;
    const int tb = rank == 0 ? 6 * x : 16 - 1;  // trace row base (peer: rows 16 / 17 via +1 / +2 below)
    const float c2 = P.scale_log2;
    const uint64_t cc = ptx::pack2(c2, c2);
    const uint32_t o_col = tmem + lane_base + O_COL;
    uint32_t gs0 = 0, oi = 0;  // global index of the item's first block; items done
    Iter si;
    it_begin(P, si);
    Item it;
    while (it_next(P, si, it)) {
      const int64_t rr = it.row0 + BM * rank + r;
      const bool live = rr < (int64_t)P.B * P.g;
      const int64_t seq = live ? rr / P.g : 0;
      const int h = it.j * P.g + (int)(rr % P.g);
      float m_own = -INFINITY, l = 0.f;
      for (int n = x; n < it.nblk; n += 2) {
        const uint32_t gs = gs0 + n;
        const int sb = gs % NSB;
        if (rank == 0) trace(tr, tb + 0, gs);
        ptx::mbar_wait(&sf[sb], (gs / NSB) & 1);
        trace(tr, tb + 1, gs);
        ptx::tc_fence_after();
        if (kTesting && (P.debug & 2)) {  // timing experiment only: the MMA pipeline without the softmax
          if (n > 0) ptx::named_bar_sync(bar_in, 64);
          if (n + 1 < it.nblk) ptx::named_bar_arrive(bar_out, 64);
          ptx::tc_fence_before();
          ptx::warp_arrive_cluster(pf0 + sb * 8);
          if (rank == 0) trace(tr, tb + 5, gs);
          continue;
        }
        const uint32_t s_col = tmem + lane_base + sb * BN;
        const int64_t rem = P.P - (int64_t)(it.blk_begin + n) * BN;  // valid tokens of this block
        uint32_t sr[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::tmem_ld32(s_col + 32 * c, sr[c]);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::reg_fence32(sr[c]);
        if (rank == 0) trace(tr, tb + 2, gs);
        if (rem < BN) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i >= rem) sr[c][i] = 0xff800000u;
        }
        // exp2(s*c2 - mu) -> bf16 P in the first 64 columns of the score buffer; returns the row sum.
        // With kMax it also folds the 128 scores into 8 FMNMX3 chains (acc), interleaved with the
        // exponentials so the ALU work fills the MUFU's issue gaps.
        float acc[8];
        auto exps = [&](float mu, auto kmax) -> float {
          constexpr bool kMax = decltype(kmax)::value;
          const uint64_t nm = ptx::pack2(-mu, -mu);
          uint64_t sacc[4] = {0, 0, 0, 0};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float a0 = __uint_as_float(sr[c][2 * i]), a1 = __uint_as_float(sr[c][2 * i + 1]);
              if constexpr (kMax) {
                const int k = (c * 16 + i) % 8;
                acc[k] = (c == 0 && i < 8) ? fmaxf(a0, a1) : ptx::fmax3(acc[k], a0, a1);
              }
              float x0, x1;
              ptx::unpack2(ptx::fma2(ptx::pack2(a0, a1), cc, nm), x0, x1);
              float p0, p1;
              if (kPolyEvery > 0 && (i % (kPolyEvery > 0 ? kPolyEvery : 1)) == kPolyEvery - 1) {
                ptx::exp2_poly2(x0, x1, p0, p1);
              } else {
                p0 = fast_exp2(x0);
                p1 = fast_exp2(x1);
              }
              sacc[i % 4] = ptx::add2(sacc[i % 4], ptx::pack2(p0, p1));
              pk[i] = ptx::cvt_bf16x2(p0, p1);
            }
            ptx::tmem_st16(s_col + c * 16, pk);
          }
          float s0, s1, s2, s3;
          ptx::unpack2(ptx::add2(sacc[0], sacc[1]), s0, s1);
          ptx::unpack2(ptx::add2(sacc[2], sacc[3]), s2, s3);
          return (s0 + s1) + (s2 + s3);
        };
        // Speculative (kSpec, this WG's own previous m known): P(n) with that stale max at once,
        // the row max folded in; m(n-1) / m(n) are checked afterwards and P recomputed only if m(n)
        // differs (the max was raised in block n-1 or n: rare, kRaise) -- so the exponentials no
        // longer wait for the row max and the m hand-off between the warpgroups.
        const bool spec = kSpec && m_own != -INFINITY;
        float rs = 0.f;
        if (spec) {
          rs = exps(m_own, std::true_type{});
        } else {
          // row max of the 128 scores: 8 independent FMNMX3 chains over column pairs
          auto sv = [&](int j) { return __uint_as_float(sr[j >> 5][j & 31]); };
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] = sv(k);
#pragma unroll
          for (int j = 8; j < BN; j += 2) acc[(j / 2) % 8] = ptx::fmax3(acc[(j / 2) % 8], sv(j), sv(j + 1));
        }
        const float mnew = fmaxf(ptx::fmax3(acc[0], acc[1], acc[2]),
                                 fmaxf(ptx::fmax3(acc[3], acc[4], acc[5]), fmaxf(acc[6], acc[7]))) * c2;
        // m(n-1) from the other WG (the item's first block starts the chain at -inf)
        float m_in = -INFINITY;
        if (rank == 0 && tr) {
          asm volatile("" ::"f"(mnew));
          trace(tr, 15 + 3 * x, gs);  // row max done (rows 15 / 18, tools/pair_trace.py)
        }
        if (n > 0) {
          ptx::named_bar_sync(bar_in, 64);
          m_in = xch[(1 - x) * BM + r];
        }
        // raised only when a row's max grows by > kRaise (log2 units): P <= 2^kRaise, so the O
        // correction (which waits for PV(n-1)) is rare; exact because the epilogue divides by l.
        // The partner warps see the same m(n-1) and row max, so they take the same decision.
        const bool any = __any_sync(0xffffffffu, mnew > m_in + kRaise);
        const float m_n = any ? fmaxf(m_in, mnew) : m_in;
        if (n + 1 < it.nblk) {  // pass m(n) on
          xch[x * BM + r] = m_n;
          ptx::named_bar_arrive(bar_out, 64);
        }
        const bool redo = !spec || __any_sync(0xffffffffu, m_n != m_own);
        // this WG's l follows the last m it used
        l *= (m_own == m_n) ? 1.f : fast_exp2(m_own - m_n);
        m_own = m_n;
        if (rank == 0 && tr) trace(tr, tb + 3, gs);
        // a row whose tokens are all masked so far keeps m = -inf: its p = 2^-inf = 0
        if (redo) rs = exps(m_n == -INFINITY ? 0.f : m_n, std::false_type{});
        l += rs;
        if (rank == 0 && tr) {
          asm volatile("" ::"f"(l));
          trace(tr, tb + 4, gs);
        }
        if (any && n >= 1 && m_in != -INFINITY) {  // rare: O *= 2^(m(n-1) - m(n)) once PV(n-1) landed
          const float alpha = fast_exp2(m_in - m_n);
          ptx::mbar_wait(&ve[(gs - 1) % NSV], ((gs - 1) / NSV) & 1);  // PV(n-1) done (its V slot freed)
          ptx::tc_fence_after();
#pragma unroll 1
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
        ptx::warp_arrive_cluster(pf0 + sb * 8);
        trace(tr, tb + (rank == 0 ? 5 : 2), gs);
        if (kTesting && P.trace && blockIdx.x < 2 && lane == 0)  // every warp's arrival: rows 23-26 / 27-30 (peer)
          trace(P.trace, 23 + 4 * (int)rank + quarter, gs);
      }
      // ---- epilogue: (m, l) of both WGs -> L relative to the final m; O / L (this WG's 64 columns)
      if (rank == 0 && tr && x == 0) trace(tr, 32, oi);  // rows 32-35: item oi's epilogue (WG a, leader)
      ptx::mbar_wait(ordy, oi & 1);
      if (rank == 0 && tr && x == 0) trace(tr, 33, oi);
      ptx::tc_fence_after();
      float *xe = xch + 2 * BM;  // [WG][128 rows][2]
      xe[(x * BM + r) * 2] = m_own;
      xe[(x * BM + r) * 2 + 1] = l;
      ptx::named_bar_sync(bar_epi, 64);
      if (rank == 0 && tr && x == 0) trace(tr, 35, oi);  // (m, l) exchanged
      const float mo = xe[((1 - x) * BM + r) * 2], lo = xe[((1 - x) * BM + r) * 2 + 1];
      const float M = fmaxf(m_own, mo);
      const float L = (m_own == -INFINITY ? 0.f : l * fast_exp2(m_own - M)) + (mo == -INFINITY ? 0.f : lo * fast_exp2(mo - M));
      const float inv = 1.f / L;
      // O / L through shared memory into coalesced stores: this warp's 32 rows x 32 columns at a
      // time (XOR-swizzled, 4 KB of the item's Q buffer, free once the item's last PV landed),
      // then 4 rows x 128 B per store instruction.  Storing straight from the TMEM layout (each
      // lane 16 B of a different row, rows Hq*512 B apart) made the epilogue ~8 K cycles.
      const uint64_t my_row =
          live ? reinterpret_cast<uint64_t>(P.o + it.slot * P.o_slot_stride + (seq * P.Hq + h) * HD + 64 * x) : 0ull;
      uint32_t *stage = reinterpret_cast<uint32_t *>(smem + OFF_Q + (oi % NQ) * QTILE + (warp - 4) * 4096);
      const int cg = lane % 8;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(o_col + 64 * x + 32 * c, ov);
        ptx::tmem_ld_wait();
        if (rank == 0 && tr && x == 0 && c == 0) {
          asm volatile("" ::"r"(ov[0]), "r"(ov[31]));
          trace(tr, 31, oi);  // chunk 0 in registers
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) stage[lane * 32 + (i ^ lane)] = __float_as_uint(__uint_as_float(ov[i]) * inv);
        __syncwarp();
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
          const bool skip = kTesting && P.mutate == 3 && blockIdx.x == 0 && quarter == 0 && rw4 == 0;
          if (base && !skip && !(kTesting && (P.debug & 8))) reinterpret_cast<float4 *>(base)[c * 8 + cg] = v;
        }
        __syncwarp();
        if (rank == 0 && tr && x == 0) trace(tr, 38 + c, oi);  // chunk c stored
      }
      // the staging writes were generic-proxy: order them before the next Q load (TMA) there
      ptx::fence_proxy_async_smem();
      ptx::warp_arrive(&xfree[oi % NQ]);
      if (rank == 0 && tr && x == 0) trace(tr, 34, oi);
      ptx::tc_fence_before();
      ptx::warp_arrive_cluster(of0);
      if (x == 0 && live) {
        float *lrow = P.lse + seq * P.Hq + h;
        lrow[it.slot * P.lse_slot_stride] = (M + log2f(L)) * HYDRA_LN2;
        if (it.blk_begin + it.nblk == P.nb)  // the unit's last piece: later slots hold no piece of it
          for (int sl = it.slot + 1; sl < P.n_slots; ++sl) lrow[sl * P.lse_slot_stride] = -INFINITY;
      }
      // the exchange slots are reused by the next item's first blocks: both WGs past the reads
      ptx::named_bar_sync(bar_epi, 64);
      gs0 += it.nblk;
      ++oi;
    }
    if (cta_tr && warp == 4 && lane == 0) cta_tr[2] = (long long)gtimer();  // this CTA's softmax / epilogues done
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kLowRegs) : "memory");
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<TMEM_COLS>(tmem);
  }
  if (P.timer && threadIdx.x == 0) atomicMax(P.timer + 1, gtimer());
  if (cta_tr && threadIdx.x == 0) cta_tr[3] = (long long)gtimer();
}

// ------------------------------------------------------------------ host side
bool prefix_pair_supported(int g) { return g >= 1 && g <= 128 && 128 % g == 0; }

template <int kPoly, int kC>
static const void *pair_fn() {
  return reinterpret_cast<const void *>(prefix_pair_kernel<kPoly, kC>);
}
template <int kPoly>
static const void *pair_fn_c(int kC) {
  return kC == 4 ? pair_fn<kPoly, 4>() : kC == 2 ? pair_fn<kPoly, 2>() : pair_fn<kPoly, 1>();
}
// poly (config key pair_poly): every poly-th exponential pair on the FMA pipe (0 = all on the
// MUFU).  The release build carries 0 (default) and 4; the testing build also 2 and 3.  Measured
// (profiles/r2f_poly_ab.jsonl): 0 beats 4 by 1-2.5 % on every shape, 3 and 2 are slower still --
// this kernel's softmax is bound by its latency chain and issue, not by MUFU throughput.
static bool pair_poly_ok(int poly) { return poly == 0 || poly == 4 || (kTesting && (poly == 2 || poly == 3)); }
static const void *pair_kernel(int poly, int kC) {
#ifdef HYDRA_TESTING
  if (poly == 2) return pair_fn_c<2>(kC);
  if (poly == 3) return pair_fn_c<3>(kC);
#endif
  return poly == 4 ? pair_fn_c<4>(kC) : pair_fn_c<0>(kC);
}

// CTA pairs that can be resident at once in clusters of kC pairs (cached per device and kC).
static int max_pair_workers(int kC) {
  static int cached[64][3] = {};
  const int ci = kC == 4 ? 2 : kC == 2 ? 1 : 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 74;
  if (cached[dev][ci] > 0) return cached[dev][ci];
  const void *fn = pair_kernel(4, kC);
  int n = 0;
  if (ensure_smem_attr(fn, pr::ALLOC) == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * 148, 1, 1);
    cfg.blockDim = dim3(pr::kThreads, 1, 1);
    cfg.dynamicSmemBytes = pr::ALLOC;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2 * kC;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) n = 0;
  }
  cudaGetLastError();
  if (n <= 0) n = device_sm_count() / (2 * kC);
  cached[dev][ci] = n * kC;
  return n * kC;
}

// Pairs per cluster: the largest kC in {4, 2} that divides the group (n_pairs; the grouped
// plan) without leaving fewer workers than kC = 1 would use; config key pair_cluster forces it.
static int choose_cluster(int64_t n_pairs, int n_workers_req, int forced) {
  if (forced == 1 || n_pairs < 2) return 1;
  auto workers = [&](int kC) {
    const int w = std::min(n_workers_req, max_pair_workers(kC));
    return 2 * n_pairs <= w ? (int)(w / n_pairs * n_pairs) : 0;  // grouped plan only
  };
  const int w1 = std::max(workers(1), 1);
  for (int kC : {4, 2}) {
    if (forced > 1 && kC != forced) continue;
    if (n_pairs % kC == 0 && workers(kC) >= (forced > 1 ? 1 : w1)) return kC;
  }
  // Groups of >= 8 pairs (C4, C6: 2048 stacked rows per KV head): 2 pairs per cluster even at the
  // cost of one stream-K group -- inside a sustained step the multicast's saved L2 -> SM traffic is
  // worth more (C4 sequential 0.253-0.263 -> 0.236 ms, C6 0.088-0.090 -> 0.084-0.085 ms,
  // profiles/r3s_pair_cluster_step_ab.jsonl; same-box A/B of this rule, profiles/
  // r3v_pair_cluster_rule_ab.log: sequential C6 0.102-0.104 -> 0.098 ms, C4 0.257 -> 0.243 ms, the
  // short-suffix overlap unchanged), although alone, unthrottled, 144 CTAs without multicast are
  // ~1 % faster.
#ifndef HYDRA_PAIR_CLUSTER_LEGACY
  if (forced == 0 && n_pairs >= 8 && n_pairs % 2 == 0 && workers(2) > 0 && workers(2) >= w1 - n_pairs) return 2;
#endif
  return 1;
}

PairPlan prefix_pair_plan(int64_t B, int g, int Hkv, int64_t P, int n_ctas, int forced_cluster) {
  const int64_t nb = (P + pr::BN - 1) / pr::BN;
  const int64_t n_pairs = (B * g + 255) / 256;
  const int kC = choose_cluster(n_pairs, std::max(1, n_ctas / 2), forced_cluster);
  const int workers = std::max(1, std::min(n_ctas / 2, max_pair_workers(kC)));
  PairPlan pl;
  pl.cluster = kC;
  pl.group = (n_pairs > 1 && 2 * n_pairs <= workers) ? (int)n_pairs : 1;
  if (pl.group == 1) pl.cluster = 1;
  pl.total = pl.group > 1 ? (int64_t)Hkv * nb : n_pairs * Hkv * nb;
  const int64_t G = std::min<int64_t>(workers / pl.group, pl.total);
  pl.workers = (int)(std::max<int64_t>(G, 1) * pl.group);
  pl.ctas = 2 * pl.workers;
  return pl;
}

// Stream-K group boundaries over the flattened (unit, 128-token block) space.  Uniform: group c
// takes blocks [c * total / G, (c + 1) * total / G).  Balanced (item_cost > 0): a group also pays
// item_cost blocks for every item (piece of a unit) it touches -- the Q load, the pipeline restart
// and the epilogue of an item cost ~5 us, about 5 block periods (tools/pair_trace.py PER_CTA at C6:
// the 3 of 9 groups whose range crossed a head boundary finished 5.5 us after the others) -- and
// the boundaries equalise blocks + item_cost x items: the smallest per-group budget T for which a
// greedy walk covers every block with G groups (binary search).  Measured (profiles/r2x_balance.jsonl):
// no faster -- C6 0.098 -> 0.102 ms with cost 5 (the slow groups of the trace were not slow for
// their extra item), C3@16K overlapped 0.840 -> 0.835 -- so the default is uniform (config 0).
static void pair_bounds(const PairPlan &pl, int64_t nb, int item_cost, int64_t *bound) {
  const int64_t G = pl.workers / pl.group, total = pl.total;
  for (int64_t c = 0; c <= G; ++c) bound[c] = c * total / G;
  if (item_cost <= 0 || total < 4 * G || nb <= 0) return;
  const double t = item_cost;
  auto end_of = [&](int64_t a, double T) -> int64_t {  // furthest end of a group starting at block a
    const int64_t u = a / nb, o = a % nb;
    double R = T - t;  // the first item
    const int64_t rest = nb - o;
    if (R < (double)rest) return std::min(total, a + std::max<int64_t>(1, (int64_t)R));
    R -= (double)rest;
    int64_t e = (u + 1) * nb;
    const int64_t k = (int64_t)(R / (t + (double)nb));
    e += k * nb;
    R -= (double)k * (t + (double)nb);
    if (R > t) e += (int64_t)(R - t);
    return std::min(total, e);
  };
  auto fits = [&](double T) {
    int64_t a = 0;
    for (int64_t c = 0; c < G && a < total; ++c) a = end_of(a, T);
    return a >= total;
  };
  double lo = (double)total / G, hi = (double)total / G + t * ((double)total / nb + 2.0) + (double)nb;
  if (!fits(hi)) return;
  for (int it = 0; it < 48; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (fits(mid)) hi = mid; else lo = mid;
  }
  int64_t a = 0;
  for (int64_t c = 0; c < G; ++c) {
    bound[c] = a;
    a = c + 1 == G ? total : end_of(a, hi);
  }
  bound[G] = total;
}

// The most pieces any unit is cut into under these boundaries (units in order, two pointers).
static int pair_max_pieces(const int64_t *bound, int64_t G, int64_t total, int64_t nb) {
  int64_t most = 1, c = 0;
  for (int64_t u = 0; u < total / nb; ++u) {
    while (c + 1 < G && bound[c + 1] <= u * nb) ++c;  // group of the unit's first block
    int64_t d = c;
    while (d + 1 < G && bound[d + 1] <= u * nb + nb - 1) ++d;  // ... and of its last block
    most = std::max(most, d - c + 1);
  }
  return (int)most;
}

// Partial slots per row = the most stream-K pieces any (pair, head) unit is cut into, under the
// uniform boundaries (the fused Eq. 5 plan counts pieces with them) or the balanced ones,
// whichever is more (an extra, always-empty slot would cost the combine a full read of its O rows).
int prefix_pair_slots(int64_t B, int g, int Hkv, int64_t P, int n_ctas, int forced_cluster, int item_cost) {
  const PairPlan pl = prefix_pair_plan(B, g, Hkv, P, n_ctas, forced_cluster);
  if (pl.total <= 0) return 1;
  const int64_t nb = (P + pr::BN - 1) / pr::BN;
  const int64_t G = pl.workers / pl.group;
  if (G > pr::kMaxGroups) return 1;
  int64_t bound[pr::kMaxGroups + 1];
  pair_bounds(pl, nb, 0, bound);
  int most = pair_max_pieces(bound, G, pl.total, nb);
  if (item_cost > 0) {
    pair_bounds(pl, nb, item_cost, bound);
    most = std::max(most, pair_max_pieces(bound, G, pl.total, nb));
  }
  return most;
}

hydra_status launch_prefix_pair(const PrefixTcArgs &a, int n_ctas, cudaStream_t s) {
  const int poly = a.pair_poly;
  if (a.tasks || !prefix_pair_supported(a.g) || !pair_poly_ok(poly)) return HYDRA_EINVAL;
  const PairPlan pl = prefix_pair_plan(a.B, a.g, a.Hkv, a.P, n_ctas, a.pair_cluster);
  const void *fn = pair_kernel(poly, pl.cluster);
  if (ensure_smem_attr(fn, pr::ALLOC) != cudaSuccess) return HYDRA_ECUDA;
  PrefixPairParams P;
  memset(&P, 0, sizeof(P));
  if (a.P <= 0 || a.B <= 0) return HYDRA_OK;
  {
    const uint64_t dims[4] = {(uint64_t)pr::HD, (uint64_t)a.g, (uint64_t)a.Hkv, (uint64_t)a.B};
    const uint64_t strides[3] = {(uint64_t)a.q_sh * 2, (uint64_t)a.q_sh * 2 * a.g, (uint64_t)a.q_sb * 2};
    const uint32_t box[4] = {64, (uint32_t)a.g, 1, (uint32_t)(pr::BM / a.g)};
    if (!encode_bf16_map(&P.tmQ, 4, a.q, dims, strides, box)) return HYDRA_ECUDA;
  }
  {
    const uint64_t dims[3] = {(uint64_t)pr::HD, (uint64_t)a.Hkv, (uint64_t)a.kv_total};
    const uint64_t strides[2] = {(uint64_t)a.kv_sh * 2, (uint64_t)a.kv_st * 2};
    // multicast pieces (pl.cluster pairs share every tile): K panels of 64 tokens (32 at 4 pairs),
    // V rows of 128 / pairs tokens
    const uint32_t boxk[3] = {64, 1, pl.cluster == 4 ? 32u : 64u}, boxv[3] = {64, 1, (uint32_t)(pr::BN / pl.cluster)};
    if (!encode_bf16_map(&P.tmK, 3, a.k, dims, strides, boxk)) return HYDRA_ECUDA;
    if (!encode_bf16_map(&P.tmV, 3, a.v, dims, strides, boxv)) return HYDRA_ECUDA;
  }
  P.Hq = a.Hq;
  P.Hkv = a.Hkv;
  P.g = a.g;
  P.scale_log2 = a.scale_log2;
  P.P = a.P;
  P.B = a.B;
  P.n_pairs = (int32_t)(((int64_t)a.B * a.g + 255) / 256);
  P.nb = (int32_t)((a.P + pr::BN - 1) / pr::BN);
  P.total_blocks = pl.total;
  P.group = pl.group;
  P.o = a.o;
  P.lse = a.lse;
  P.o_slot_stride = a.o_slot_stride;
  P.lse_slot_stride = a.lse_slot_stride;
  P.n_slots = a.n_splits;
  P.mutate = kTesting ? a.mutate : 0;
  P.trace = kTesting ? reinterpret_cast<long long *>(a.trace) : nullptr;
  P.debug = kTesting ? a.debug_variant : 0;
  P.timer = a.timer;
  if (pl.total <= 0) return HYDRA_OK;
  if (pl.workers / pl.group > pr::kMaxGroups) return HYDRA_EINVAL;
  // the fused Eq. 5 plan (fused.cuh) counts pieces with the uniform boundaries
  pair_bounds(pl, P.nb, a.fc.cnt ? 0 : a.pair_item_cost, P.bound);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.ctas, 1, 1);
  cfg.blockDim = dim3(pr::kThreads, 1, 1);
  cfg.dynamicSmemBytes = pr::ALLOC;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2 * pl.cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, reinterpret_cast<void (*)(PrefixPairParams)>(const_cast<void *>(fn)), P);
  return e == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

}  // namespace hydra

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
//   warp 0      TMA producer (both CTAs): this CTA's Q tile (2 buffers), K tokens
//               [64*rank, +64) of each block (4-stage ring), V dims [64*rank, +64) of each
//               block (4-stage ring); completions counted on the LEADER's barriers
//   warp 1      TMEM allocation (both CTAs, cta_group::2) and, in the leader only, the single
//               MMA-issuing thread:  S(0) S(1) | PV_a(n) PV_b(n) S(n+2) | ...
//   warps 4-7   softmax WG a (thread = query row = TMEM lane), warps 8-11 WG b
// Schedule: grouped stream-K over (head, 128-token block) as prefix_tc2.cu, with the CTA pair
// as the worker: pair p of a group takes query rows [256p, 256p+256) of every head.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
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
constexpr int kThreads = 384;
constexpr int QPANEL = BM * 128;      // 128 rows x 128 B
constexpr int QTILE = 2 * QPANEL;     // 32 KB
constexpr int KPANEL = 64 * 128;      // 64 tokens x 128 B
constexpr int KHALF = 2 * KPANEL;     // 16 KB: this CTA's 64 tokens x 128 dims
constexpr int VHALF = BN * 128;       // 16 KB: 128 tokens x this CTA's 64 dims
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + NQ * QTILE;
constexpr int OFF_V = OFF_K + NSK * KHALF;
constexpr int OFF_X = OFF_V + NSV * VHALF;  // (m, l) exchange [item parity][WG][128 rows][2]
constexpr int OFF_BAR = OFF_X + 2 * 2 * BM * 2 * 4;
// kf, ke [NSK]; vf, ve [NSV]; qf, qe [NQ]; sf [2]; pfa [2]; pfb [2]; pvd [2]; ordy; ofree
constexpr int N_BARS = 2 * NSK + 2 * NSV + 2 * NQ + 2 + 2 + 2 + 2 + 2;
constexpr int BYTES = OFF_BAR + N_BARS * 8 + 16;
constexpr int ALLOC = BYTES + 1024;
static_assert(ALLOC <= 232448, "prefix_pair smem over the 227 KB opt-in limit");
constexpr uint32_t TMEM_COLS = 512;
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
  int32_t mutate;  // testing build only: 3 = worker 0 skips one 4-row group of its stores
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
__device__ __forceinline__ int64_t sk_start(const PrefixPairParams &P, int64_t c) {
  return c * P.total_blocks / n_groups(P);
}
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

template <int kPolyEvery>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pr::kThreads, 1)
    prefix_pair_kernel(const __grid_constant__ PrefixPairParams P) {
  using namespace pr;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *kf = bars, *ke = kf + NSK, *vf = ke + NSK, *ve = vf + NSV, *qf = ve + NSV, *qe = qf + NQ;
  uint64_t *sf = qe + NQ, *pfa = sf + 2, *pfb = pfa + 2, *pvd = pfb + 2, *ordy = pvd + 2, *ofree = ordy + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + N_BARS);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&P.tmQ);
    ptx::prefetch_tmap(&P.tmK);
    ptx::prefetch_tmap(&P.tmV);
    for (int i = 0; i < NSK; ++i) {
      ptx::mbar_init(&kf[i], 1);
      ptx::mbar_init(&ke[i], 1);
    }
    for (int i = 0; i < NSV; ++i) {
      ptx::mbar_init(&vf[i], 1);
      ptx::mbar_init(&ve[i], 1);
    }
    for (int i = 0; i < NQ; ++i) {
      ptx::mbar_init(&qf[i], 1);
      ptx::mbar_init(&qe[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&sf[i], 1);
      ptx::mbar_init(&pfa[i], 8);  // 4 warps x 2 CTAs (leader's copy)
      ptx::mbar_init(&pfb[i], 8);
      ptx::mbar_init(&pvd[i], 1);
    }
    ptx::mbar_init(ordy, 1);
    ptx::mbar_init(ofree, 16);  // 8 softmax warps x 2 CTAs (leader's copy)
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================= TMA producer (both CTAs) =================
    if (ptx::elect_one()) {
      const uint32_t kf0 = ptx::mapa(ptx::smem_u32(kf), 0), vf0 = ptx::mapa(ptx::smem_u32(vf), 0),
                     qf0 = ptx::mapa(ptx::smem_u32(qf), 0);
      uint32_t kq = 0, vq = 0, qi = 0;
      Iter si;
      it_begin(P, si);
      Item it;
      while (it_next(P, si, it)) {
        {
          const int qb = qi % NQ;
          ptx::mbar_wait(&qe[qb], ((qi / NQ) & 1) ^ 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&qf[qb], 2 * QTILE);
          const int b0 = (int)((it.row0 + BM * rank) / P.g);
          uint8_t *sQ = smem + OFF_Q + qb * QTILE;
          ptx::tma_load_4d_pair(sQ, &P.tmQ, qf0 + qb * 8, 0, 0, it.j, b0);
          ptx::tma_load_4d_pair(sQ + QPANEL, &P.tmQ, qf0 + qb * 8, 64, 0, it.j, b0);
          ++qi;
        }
        for (int n = 0; n < it.nblk; ++n) {
          const int t0 = (it.blk_begin + n) * BN;
          const int ks = kq % NSK;
          ptx::mbar_wait(&ke[ks], ((kq / NSK) & 1) ^ 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&kf[ks], 2 * KHALF);
          uint8_t *sK = smem + OFF_K + ks * KHALF;
          ptx::tma_load_3d_pair(sK, &P.tmK, kf0 + ks * 8, 0, it.j, t0 + 64 * (int)rank);
          ptx::tma_load_3d_pair(sK + KPANEL, &P.tmK, kf0 + ks * 8, 64, it.j, t0 + 64 * (int)rank);
          ++kq;
          const int vs = vq % NSV;
          ptx::mbar_wait(&ve[vs], ((vq / NSV) & 1) ^ 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&vf[vs], 2 * VHALF);
          ptx::tma_load_3d_pair(smem + OFF_V + vs * VHALF, &P.tmV, vf0 + vs * 8, 64 * (int)rank, it.j, t0);
          ++vq;
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA, one thread) =================
    if (rank == 0 && ptx::elect_one()) {
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(2 * BM, BN, false);  // S = Q K^T, M = 256
      constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(2 * BM, HD, true);  // O += P V, V MN-major
      Cursor cs, cp;
      cs.init(P);
      cp.init(P);
      uint32_t gs = 0, gp = 0, oi = 0;
      auto issue_s = [&]() {
        if (!cs.valid) return;
        const int qb = cs.qi % NQ;
        if (cs.n == 0) {
          ptx::mbar_wait(&qf[qb], (cs.qi / NQ) & 1);
          ptx::tc_fence_after();
        }
        const int ks = gs % NSK, sb = gs % 2;
        ptx::mbar_wait(&kf[ks], (gs / NSK) & 1);
        ptx::tc_fence_after();
        const uint32_t qa = ptx::smem_u32(smem + OFF_Q + qb * QTILE), ka = ptx::smem_u32(smem + OFF_K + ks * KHALF);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::mma2_ss(tmem + sb * BN, ptx::smem_desc_sw128(qa + (kk / 4) * QPANEL + (kk % 4) * 32, 16, 1024),
                       ptx::smem_desc_sw128(ka + (kk / 4) * KPANEL + (kk % 4) * 32, 16, 1024), idesc_s, kk > 0);
        ptx::mma2_commit(&sf[sb]);
        ptx::mma2_commit(&ke[ks]);
        if (cs.n == cs.it.nblk - 1) ptx::mma2_commit(&qe[qb]);
        ++gs;
        cs.advance(P);
      };
      issue_s();
      issue_s();
      while (cp.valid) {
        const int sb = gp % 2, vs = gp % NSV;
        const uint32_t acc0 = cp.n > 0 ? 1u : 0u;
        if (cp.n == 0) {  // O_a / O_b drained by the previous item's epilogue (both CTAs)
          ptx::mbar_wait_cluster(ofree, (oi & 1) ^ 1);
          ++oi;
        }
        ptx::mbar_wait(&vf[vs], (gp / NSV) & 1);
        const uint32_t va = ptx::smem_u32(smem + OFF_V + vs * VHALF);
        ptx::mbar_wait_cluster(&pfa[sb], (gp / 2) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma2_ts(tmem + 256, tmem + sb * BN + kk * 8, ptx::smem_desc_sw128(va + kk * 2048, 16, 1024), idesc_pv,
                       acc0 | (kk > 0));
        ptx::mbar_wait_cluster(&pfb[sb], (gp / 2) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma2_ts(tmem + 384, tmem + sb * BN + 64 + kk * 8, ptx::smem_desc_sw128(va + (4 + kk) * 2048, 16, 1024),
                       idesc_pv, acc0 | (kk > 0));
        ptx::mma2_commit(&ve[vs]);
        ptx::mma2_commit(&pvd[sb]);
        if (cp.n == cp.it.nblk - 1) ptx::mma2_commit(ordy);
        ++gp;
        cp.advance(P);
        issue_s();  // S(gp + 1): overwrites the score buffer whose P the PV above consumed
      }
    }
  } else if (warp >= 4) {
    // ================= softmax / epilogue (both CTAs) =================
    const int x = (warp - 4) / 4;  // 0: tokens 0-63 of each block (O_a), 1: tokens 64-127 (O_b)
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t pf0 = ptx::mapa(ptx::smem_u32(x == 0 ? pfa : pfb), 0), of0 = ptx::mapa(ptx::smem_u32(ofree), 0);
    float *xch = reinterpret_cast<float *>(smem + OFF_X);
    const float c2 = P.scale_log2;
    const uint64_t cc = ptx::pack2(c2, c2);
    uint32_t gs = 0, oi = 0;
    Iter si;
    it_begin(P, si);
    Item it;
    while (it_next(P, si, it)) {
      const int64_t rr = it.row0 + BM * rank + r;
      const bool live = rr < (int64_t)P.B * P.g;
      const int64_t seq = live ? rr / P.g : 0;
      const int h = it.j * P.g + (int)(rr % P.g);
      float m2 = -INFINITY, l = 0.f;
      for (int n = 0; n < it.nblk; ++n, ++gs) {
        const int sb = gs % 2;
        ptx::mbar_wait(&sf[sb], (gs / 2) & 1);
        ptx::tc_fence_after();
        const uint32_t s_col = tmem + lane_base + sb * BN + 64 * x;
        const int64_t rem = P.P - (int64_t)(it.blk_begin + n) * BN - 64 * x;  // valid tokens of this half
        uint32_t sr[2][32];
        ptx::tmem_ld32(s_col, sr[0]);
        ptx::tmem_ld32(s_col + 32, sr[1]);
        ptx::tmem_ld_wait();
        ptx::reg_fence32(sr[0]);
        ptx::reg_fence32(sr[1]);
        if (rem < 64) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i >= rem) sr[c][i] = 0xff800000u;
        }
        float acc[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          acc[k] = ptx::fmax3(__uint_as_float(sr[0][4 * k]), __uint_as_float(sr[0][4 * k + 1]),
                              __uint_as_float(sr[0][4 * k + 2]));
#pragma unroll
        for (int k = 0; k < 8; ++k)
          acc[k] = ptx::fmax3(acc[k], __uint_as_float(sr[0][4 * k + 3]), __uint_as_float(sr[1][4 * k]));
#pragma unroll
        for (int k = 0; k < 8; ++k)
          acc[k] = ptx::fmax3(acc[k], __uint_as_float(sr[1][4 * k + 1]), __uint_as_float(sr[1][4 * k + 2]));
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = fmaxf(acc[k], __uint_as_float(sr[1][4 * k + 3]));
        const float mx = fmaxf(ptx::fmax3(acc[0], acc[1], acc[2]),
                               fmaxf(ptx::fmax3(acc[3], acc[4], acc[5]), fmaxf(acc[6], acc[7])));
        const float mnew = mx * c2;
        // the running max is raised only when a row's max grows by > 8 (log2 units): P <= 256,
        // and the O correction below is rare; exact because the epilogue divides by l
        const bool any = __any_sync(0xffffffffu, mnew > m2 + 8.0f);
        float alpha = 1.f;
        if (any) {
          const float mt = fmaxf(m2, mnew);
          alpha = fast_exp2(m2 - mt);  // 0 while m2 is -inf
          m2 = mt;
        }
        // a half whose tokens are all masked so far keeps m2 = -inf: its p = 2^-inf = 0
        const float mu = m2 == -INFINITY ? 0.f : m2;
        const uint64_t nm = ptx::pack2(-mu, -mu);
        uint64_t sacc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float x0, x1;
            ptx::unpack2(ptx::fma2(ptx::pack2(__uint_as_float(sr[c][2 * i]), __uint_as_float(sr[c][2 * i + 1])), cc, nm),
                         x0, x1);
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
          ptx::tmem_st16(s_col + c * 16, pk);  // P(n) of this half -> its first 32 score columns
        }
        float s0, s1, s2, s3;
        ptx::unpack2(ptx::add2(sacc[0], sacc[1]), s0, s1);
        ptx::unpack2(ptx::add2(sacc[2], sacc[3]), s2, s3);
        l = l * alpha + ((s0 + s1) + (s2 + s3));
        if (any && n >= 1) {  // rare: rescale O_x once PV(n-1) has landed in it
          ptx::mbar_wait(&pvd[(gs - 1) % 2], ((gs - 1) / 2) & 1);
          ptx::tc_fence_after();
          const uint32_t o_col = tmem + lane_base + 256 + 128 * x;
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
      }
      // ---- epilogue: merge the two halves' states (Eq. 5 with two parts), O / L, LSE
      ptx::mbar_wait(ordy, oi & 1);
      ptx::tc_fence_after();
      float *xb = xch + (oi & 1) * (2 * BM * 2);
      xb[(x * BM + r) * 2] = m2;
      xb[(x * BM + r) * 2 + 1] = l;
      ptx::named_bar_sync(1, 256);
      const float mo = xb[((1 - x) * BM + r) * 2], lo = xb[((1 - x) * BM + r) * 2 + 1];
      const float M = fmaxf(m2, mo);
      const float ws = m2 == -INFINITY ? 0.f : fast_exp2(m2 - M), wo = mo == -INFINITY ? 0.f : fast_exp2(mo - M);
      const float L = l * ws + lo * wo;
      const float inv = 1.f / L;
      const float wa = (x == 0 ? ws : wo) * inv, wb = (x == 0 ? wo : ws) * inv;
      float *orow = P.o + it.slot * P.o_slot_stride + (seq * P.Hq + h) * HD + 64 * x;
      const bool skip = kTesting && P.mutate == 3 && blockIdx.x == 0 && quarter == 0 && lane < 4;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t va[32], vb[32];
        ptx::tmem_ld32(tmem + lane_base + 256 + 64 * x + 32 * c, va);
        ptx::tmem_ld32(tmem + lane_base + 384 + 64 * x + 32 * c, vb);
        ptx::tmem_ld_wait();
        if (live && !skip) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 v;
            v.x = __uint_as_float(va[4 * i]) * wa + __uint_as_float(vb[4 * i]) * wb;
            v.y = __uint_as_float(va[4 * i + 1]) * wa + __uint_as_float(vb[4 * i + 1]) * wb;
            v.z = __uint_as_float(va[4 * i + 2]) * wa + __uint_as_float(vb[4 * i + 2]) * wb;
            v.w = __uint_as_float(va[4 * i + 3]) * wa + __uint_as_float(vb[4 * i + 3]) * wb;
            reinterpret_cast<float4 *>(orow)[c * 8 + i] = v;
          }
        }
      }
      ptx::tc_fence_before();
      ptx::warp_arrive_cluster(of0);
      if (x == 0 && live) P.lse[it.slot * P.lse_slot_stride + seq * P.Hq + h] = (M + log2f(L)) * HYDRA_LN2;
      ++oi;
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<TMEM_COLS>(tmem);
  }
}

// ------------------------------------------------------------------ host side
bool prefix_pair_supported(int g) { return g >= 1 && g <= 128 && 128 % g == 0; }

// Clusters of two that can be resident at once on this device (cached per device).
static int max_pair_workers() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 74;
  if (cached[dev] > 0) return cached[dev];
  if (ensure_smem_attr(reinterpret_cast<const void *>(prefix_pair_kernel<4>), pr::ALLOC) != cudaSuccess) {
    cudaGetLastError();
    return device_sm_count() / 2;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * 148, 1, 1);
  cfg.blockDim = dim3(pr::kThreads, 1, 1);
  cfg.dynamicSmemBytes = pr::ALLOC;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void *)prefix_pair_kernel<4>, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = device_sm_count() / 2;
  }
  cached[dev] = n;
  return n;
}

PairPlan prefix_pair_plan(int64_t B, int g, int Hkv, int64_t P, int n_ctas) {
  const int workers = std::max(1, std::min(n_ctas / 2, max_pair_workers()));
  const int64_t nb = (P + pr::BN - 1) / pr::BN;
  const int64_t n_pairs = (B * g + 255) / 256;
  PairPlan pl;
  pl.group = (n_pairs > 1 && 2 * n_pairs <= workers) ? (int)n_pairs : 1;
  pl.total = pl.group > 1 ? (int64_t)Hkv * nb : n_pairs * Hkv * nb;
  const int64_t G = std::min<int64_t>(workers / pl.group, pl.total);
  pl.workers = (int)(std::max<int64_t>(G, 1) * pl.group);
  pl.ctas = 2 * pl.workers;
  return pl;
}

int prefix_pair_slots(int64_t B, int g, int Hkv, int64_t P, int n_ctas) {
  const PairPlan pl = prefix_pair_plan(B, g, Hkv, P, n_ctas);
  if (pl.total <= 0) return 1;
  const int64_t nb = (P + pr::BN - 1) / pr::BN;
  const int64_t range = pl.total / (pl.workers / pl.group);  // >= 1
  return (int)((nb + range - 1) / range + 1);
}

hydra_status launch_prefix_pair(const PrefixTcArgs &a, int n_ctas, cudaStream_t s) {
  if (a.tasks || !prefix_pair_supported(a.g) || (a.poly_every != 0 && a.poly_every != 4)) return HYDRA_EINVAL;
  const void *fn = a.poly_every == 4 ? reinterpret_cast<const void *>(prefix_pair_kernel<4>)
                                     : reinterpret_cast<const void *>(prefix_pair_kernel<0>);
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
    const uint32_t boxk[3] = {64, 1, 64}, boxv[3] = {64, 1, (uint32_t)pr::BN};
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
  const PairPlan pl = prefix_pair_plan(a.B, a.g, a.Hkv, a.P, n_ctas);
  P.total_blocks = pl.total;
  P.group = pl.group;
  P.o = a.o;
  P.lse = a.lse;
  P.o_slot_stride = a.o_slot_stride;
  P.lse_slot_stride = a.lse_slot_stride;
  P.mutate = kTesting ? a.mutate : 0;
  if (pl.total <= 0) return HYDRA_OK;
  if (a.poly_every == 4)
    prefix_pair_kernel<4><<<pl.ctas, pr::kThreads, pr::ALLOC, s>>>(P);
  else
    prefix_pair_kernel<0><<<pl.ctas, pr::kThreads, pr::ALLOC, s>>>(P);
  return cudaGetLastError() == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

}  // namespace hydra

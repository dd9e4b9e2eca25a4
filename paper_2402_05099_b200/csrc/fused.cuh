// fused.cuh -- the Eq. 5 combine fused into the epilogues of the prefix and suffix kernels.
//
// PAPER.md Eq. 5 (App. B combine_lse P:321-344): a row's output is the LSE-weighted
// merge of its partial attentions.  The paper runs it as a separate Triton kernel (P:147
// footnote); here it runs in whichever kernel epilogue writes a row's LAST partial:
//   * every writer of a partial (a prefix stream-K piece or KV split, a suffix item or split)
//     stores it, fences, and increments the row's arrival counter;
//   * the writer whose increment completes the count (prefix pieces + suffix parts, known
//     on the device from the launch plan) merges all parts of the row and writes the final
//     bf16 / f32 output and the merged LSE, then resets the counter.
// With pre_done (the sequential schedule: the suffix launch follows the prefix on one stream)
// only the suffix parts are counted, and a single suffix part merges without any atomic.
// Otherwise the prefix and suffix kernels may run in either order or concurrently (the
// SM-partitioned schedule), so there is no waiting anywhere: the merge happens exactly once per row, as
// soon as its last part exists.  The caller zeroes the counters before the launches (one
// memset node) -- this replaces the -inf slot fill and the combine launch of the unfused
// path.  Partials of other writers are read with ld.global.cg (L2, never a stale L1 line).
#pragma once
#include "common.cuh"
#include "internal.h"

namespace hydra {

// largest c in [0, G) with floor(c*T/G) <= x (the stream-K range that holds unit x)
__device__ __forceinline__ int64_t fc_group_of(int64_t x, int64_t T, int64_t G) {
  int64_t c = x * G / T;
  while (c + 1 < G && (c + 1) * T / G <= x) ++c;
  while (c > 0 && c * T / G > x) --c;
  return c;
}

// Number of prefix partial slots (0 .. n-1) written for the row of sequence b, query head h.
__device__ __forceinline__ int fc_prefix_pieces(const FusedCombine &F, int64_t b, int h) {
  if (F.sk_total == 0) return F.n_pre_splits;
  const int j = h / F.g;
  const int64_t pair = (b * F.g + h % F.g) / 256;
  const int64_t unit = F.sk_group > 1 ? j : (int64_t)j * F.sk_npairs + pair;
  const int64_t x0 = unit * F.sk_nb, x1 = x0 + F.sk_nb - 1;
  return (int)(fc_group_of(x1, F.sk_total, F.sk_G) - fc_group_of(x0, F.sk_total, F.sk_G) + 1);
}

__device__ __forceinline__ int fc_expected(const FusedCombine &F, int64_t b, int h) {
  return F.pre_done ? F.n_suf : fc_prefix_pieces(F, b, h) + F.n_suf;
}

// The counters are in use unless the prefix is known complete and the suffix has one part.
__device__ __forceinline__ bool fc_counting(const FusedCombine &F) { return !(F.pre_done && F.n_suf == 1); }

// Called by the writer of a part after its stores (and a __threadfence): counts the arrival,
// true when this arrival completes the row.
__device__ __forceinline__ bool fc_arrive(const FusedCombine &F, int64_t row, int expected) {
  if (expected == 1) return true;  // the only writer of the row's parts (pre_done, one suffix part)
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(F.cnt + row) : "memory");
  return old + 1 == expected;
}

__device__ __forceinline__ float fc_part_lse(const FusedCombine &F, int k, int n_pre, int64_t row) {
  return k < n_pre ? __ldcg(F.lse_pre + k * F.lse_slot + row) : __ldcg(F.lse_suf + (k - n_pre) * F.lse_slot + row);
}
__device__ __forceinline__ const float *fc_part_o(const FusedCombine &F, int k, int n_pre, int64_t row) {
  return k < n_pre ? F.o_pre + k * F.o_slot + row * 128 : F.o_suf + (k - n_pre) * F.o_slot + row * 128;
}

// Merge of one row by one warp: lane l owns dims 4l .. 4l+3.
__device__ __forceinline__ void fc_merge_row_warp(const FusedCombine &F, int64_t row, int n_pre, int lane) {
  const int n = n_pre + F.n_suf;
  float m = -INFINITY;
  for (int k = 0; k < n; ++k) m = fmaxf(m, fc_part_lse(F, k, n_pre, row));
  float acc[4] = {0.f, 0.f, 0.f, 0.f}, den = 0.f;
  if (m != -INFINITY) {
    for (int k = 0; k < n; ++k) {
      const float lk = fc_part_lse(F, k, n_pre, row);
      if (lk == -INFINITY) continue;  // empty part: its O is never read
      const float w = F.inject_bug ? 1.f : expf(lk - m);
      den += w;
      const float4 v = __ldcg(reinterpret_cast<const float4 *>(fc_part_o(F, k, n_pre, row)) + lane);
      acc[0] = fmaf(w, v.x, acc[0]);
      acc[1] = fmaf(w, v.y, acc[1]);
      acc[2] = fmaf(w, v.z, acc[2]);
      acc[3] = fmaf(w, v.w, acc[3]);
    }
    const float inv = 1.f / den;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] *= inv;
  }
  if (F.out_f32) {
    reinterpret_cast<float4 *>(F.out)[row * 32 + lane] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  } else {
    __nv_bfloat162 a = __floats2bfloat162_rn(acc[0], acc[1]), c = __floats2bfloat162_rn(acc[2], acc[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t *>(&a);
    u.y = *reinterpret_cast<uint32_t *>(&c);
    reinterpret_cast<uint2 *>(F.out)[row * 32 + lane] = u;
  }
  if (lane == 0) {
    if (F.lse_out) F.lse_out[row] = m == -INFINITY ? -INFINITY : m + logf(den);
    if (fc_counting(F)) F.cnt[row] = 0;  // ready for the next call (stream-ordered after this kernel)
  }
}

// Merge of one row by 128 threads, thread e owning dim e (the suffix kernels' epilogues).
__device__ __forceinline__ void fc_merge_row_dim(const FusedCombine &F, int64_t row, int n_pre, int e) {
  const int n = n_pre + F.n_suf;
  float m = -INFINITY;
  for (int k = 0; k < n; ++k) m = fmaxf(m, fc_part_lse(F, k, n_pre, row));
  float acc = 0.f, den = 0.f;
  if (m != -INFINITY) {
    for (int k = 0; k < n; ++k) {
      const float lk = fc_part_lse(F, k, n_pre, row);
      if (lk == -INFINITY) continue;
      const float w = F.inject_bug ? 1.f : expf(lk - m);
      den += w;
      acc = fmaf(w, __ldcg(fc_part_o(F, k, n_pre, row) + e), acc);
    }
    acc *= 1.f / den;
  }
  if (F.out_f32)
    reinterpret_cast<float *>(F.out)[row * 128 + e] = acc;
  else
    reinterpret_cast<__nv_bfloat16 *>(F.out)[row * 128 + e] = __float2bfloat16_rn(acc);
  if (e == 0) {
    if (F.lse_out) F.lse_out[row] = m == -INFINITY ? -INFINITY : m + logf(den);
    if (fc_counting(F)) F.cnt[row] = 0;
  }
}

}  // namespace hydra

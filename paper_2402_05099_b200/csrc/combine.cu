// combine.cu -- n-ary LSE combine (Eq. 5 P:98-105 in App. B's
// max-stabilised form P:333-344, folded over n parts; associativity S:154).
//
// For row r over the parts p (parts with lse = -inf are empty: skipped, their O never used):
//   m   = max_p lse_p[r]
//   w_p = exp(lse_p[r] - m)
//   O   = sum_p w_p * O_p[r] / sum_p w_p     -> out (bf16 RNE, f32, or f16 for packing)
//   lse = m + ln(sum_p w_p)                  (the merged LSE a recursive combine needs)
// The parts come in two groups: group A in o_dtype (f32, or f16 partials received from
// other GPUs) and an optional group B in f32 (e.g. the local suffix partial merged with the
// received prefix pieces in the same pass).  Every pointer has a part stride and a row
// stride, so the kernel reads an exchange buffer whose rows interleave O and LSE in place,
// and writes such a buffer (dist.py's packed (O f16 | LSE f32) rows).  HBM-bound: it reads
// n*(d*sizeof(O)+4) and writes d*sizeof(out)(+4) bytes per row.
#include "common.cuh"
#include "internal.h"

namespace hydra {

template <typename OT>
__device__ __forceinline__ float ld_part(const OT *p);
template <>
__device__ __forceinline__ float ld_part<float>(const float *p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ld_part<__half>(const __half *p) { return __half2float(__ldg(p)); }

template <typename OT>
__device__ __forceinline__ const void *part_o(const CombineParams &p, int q, int64_t row) {
  if (q < p.n_a) return reinterpret_cast<const OT *>(p.o_a) + q * p.o_a_part + row * p.o_a_row;
  return p.o_b + (q - p.n_a) * p.o_b_part + row * p.o_b_row;
}
__device__ __forceinline__ float part_lse(const CombineParams &p, int q, int64_t row) {
  return q < p.n_a ? __ldg(p.l_a + q * p.l_a_part + row * p.l_a_row)
                   : __ldg(p.l_b + (q - p.n_a) * p.l_b_part + row * p.l_b_row);
}
// 4 consecutive elements of part q's row (16-B aligned for f32, 8-B for f16)
template <typename OT>
__device__ __forceinline__ void ld4(const CombineParams &p, int q, int64_t row, int e, float *f) {
  if (q < p.n_a && sizeof(OT) == 2) {
    const __half *src = reinterpret_cast<const __half *>(part_o<OT>(p, q, row)) + e;
    const uint2 v = __ldg(reinterpret_cast<const uint2 *>(src));
    const __half2 a = *reinterpret_cast<const __half2 *>(&v.x);
    const __half2 b = *reinterpret_cast<const __half2 *>(&v.y);
    f[0] = __low2float(a); f[1] = __high2float(a); f[2] = __low2float(b); f[3] = __high2float(b);
  } else {
    const float *src = reinterpret_cast<const float *>(part_o<OT>(p, q, row)) + e;
    const float4 v = __ldg(reinterpret_cast<const float4 *>(src));
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
  }
}
template <typename OT>
__device__ __forceinline__ float ld1(const CombineParams &p, int q, int64_t row, int e) {
  if (q < p.n_a) return ld_part<OT>(reinterpret_cast<const OT *>(part_o<OT>(p, q, row)) + e);
  return __ldg(reinterpret_cast<const float *>(part_o<OT>(p, q, row)) + e);
}

// Output row r: dense (out + r * out_row) or scattered through the table (table_rows > 0).
template <typename OutT>
__device__ __forceinline__ OutT *out_ptr(const CombineParams &p, int64_t row) {
  if (p.table_rows > 0) {
    const int64_t t = row / p.table_rows;
    return reinterpret_cast<OutT *>(p.out_table[t]) + (row - t * p.table_rows) * p.out_row;
  }
  return reinterpret_cast<OutT *>(p.out) + row * p.out_row;
}
__device__ __forceinline__ float *lse_ptr(const CombineParams &p, int64_t row) {
  if (p.table_rows > 0) {
    if (!p.lse_out_table) return nullptr;
    const int64_t t = row / p.table_rows;
    return p.lse_out_table[t] + (row - t * p.table_rows) * p.lse_out_row;
  }
  return p.lse_out ? p.lse_out + row * p.lse_out_row : nullptr;
}

// General kernel: any number of parts, VEC floats per lane (VEC = 0: element-wise, any d).
template <typename OT, typename OutT, int VEC>
__global__ void __launch_bounds__(256) combine_kernel(const CombineParams p) {
  // as a programmatic dependent (the step's suffix kernel precedes): wait for that grid's
  // completion and memory before reading any part; a no-op for a normal launch
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t row = (int64_t)blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= p.rows) return;
  const int n = p.n_a + p.n_b;
  float m = -INFINITY;
  for (int q = 0; q < n; ++q) m = fmaxf(m, part_lse(p, q, row));
  OutT *out = out_ptr<OutT>(p, row);
  float *lse_o = lse_ptr(p, row);
  if (m == -INFINITY) {  // every part empty: sentinel (0, -inf)
    for (int e = lane; e < p.d; e += 32) out[e] = OutT(0.f);
    if (lse_o && lane == 0) *lse_o = -INFINITY;
    return;
  }
  float den = 0.f;
  if constexpr (VEC > 0) {
    float acc[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
    for (int q = 0; q < n; ++q) {
      const float lq = part_lse(p, q, row);
      if (lq == -INFINITY) continue;
      const float w = p.inject_bug ? 1.f : expf(lq - m);
      den += w;
#pragma unroll
      for (int c = 0; c < VEC / 4; ++c) {
        float f[4];
        ld4<OT>(p, q, row, (c * 32 + lane) * 4, f);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[c * 4 + i] = fmaf(w, f[i], acc[c * 4 + i]);
      }
    }
    const float inv = 1.f / den;
#pragma unroll
    for (int c = 0; c < VEC / 4; ++c) {
      const int e = (c * 32 + lane) * 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) out[e + i] = OutT(acc[c * 4 + i] * inv);
    }
  } else {
    for (int q = 0; q < n; ++q) {
      const float lq = part_lse(p, q, row);
      if (lq != -INFINITY) den += p.inject_bug ? 1.f : expf(lq - m);
    }
    const float inv = 1.f / den;
    for (int e = lane; e < p.d; e += 32) {
      float a = 0.f;
      for (int q = 0; q < n; ++q) {
        const float lq = part_lse(p, q, row);
        if (lq == -INFINITY) continue;
        const float w = p.inject_bug ? 1.f : expf(lq - m);
        a = fmaf(w, ld1<OT>(p, q, row, e), a);
      }
      out[e] = OutT(a * inv);
    }
  }
  if (lse_o && lane == 0) *lse_o = m + logf(den);
}

// d = 128, at most 8 parts: the same arithmetic with the memory latency paid twice per row
// instead of twice per part -- all LSEs loaded together, then all parts' 512-B rows together
// (16 B per lane), then the weighted sum.  The part loop of combine_kernel serialises a
// dependent LSE load and O load per part, so with 3-8 parts it ran at 30-50 % of HBM
// bandwidth (e.g. 22 us instead of ~12 at C3).
template <typename OT, typename OutT, int NP, int RPW>
__global__ void __launch_bounds__(256) combine_kernel_p8(const CombineParams p) {
  // NP: parts rounded up (2, 4 or 8); RPW rows per warp.  Every part's LSE and O loads of all
  // RPW rows are issued together, before any decision on their values (one memory round trip
  // per RPW rows).  An empty part's O slot may be unwritten workspace: it is loaded but never
  // used (skipped below, not multiplied by 0, so garbage or NaN cannot leak in).
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent: see combine_kernel
  const int64_t row0 = ((int64_t)blockIdx.x * 8 + threadIdx.x / 32) * RPW;
  const int lane = threadIdx.x % 32;
  if (row0 >= p.rows) return;
  const int n = p.n_a + p.n_b;
  float lq[RPW][NP], f[RPW][NP][4];
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int64_t row = row0 + k;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      lq[k][q] = -INFINITY;
      if (q < n && row < p.rows) {
        lq[k][q] = part_lse(p, q, row);
        ld4<OT>(p, q, row, lane * 4, f[k][q]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int64_t row = row0 + k;
    if (row >= p.rows) break;
    float m = -INFINITY;
#pragma unroll
    for (int q = 0; q < NP; ++q) m = fmaxf(m, lq[k][q]);
    OutT *out = out_ptr<OutT>(p, row);
    float *lse_o = lse_ptr(p, row);
    if (m == -INFINITY) {  // every part empty: sentinel (0, -inf)
#pragma unroll
      for (int i = 0; i < 4; ++i) out[lane * 4 + i] = OutT(0.f);
      if (lse_o && lane == 0) *lse_o = -INFINITY;
      continue;
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f}, den = 0.f;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      if (lq[k][q] == -INFINITY) continue;
      const float w = p.inject_bug ? 1.f : expf(lq[k][q] - m);
      den += w;
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = fmaf(w, f[k][q][i], acc[i]);
    }
    const float inv = 1.f / den;
#pragma unroll
    for (int i = 0; i < 4; ++i) out[lane * 4 + i] = OutT(acc[i] * inv);
    if (lse_o && lane == 0) *lse_o = m + logf(den);
  }
}

template <typename OT, typename OutT>
static cudaError_t launch_c(const CombineParams &p, cudaStream_t s) {
  const dim3 grid((unsigned)((p.rows + 7) / 8));
  const dim3 grid2((unsigned)((p.rows + 15) / 16));  // two rows per warp
  const int n = p.n_a + p.n_b;
  const bool pdl = p.pdl != 0;
  const dim3 blk(256);
  if (p.d == 128 && n <= 2) return launch_maybe_pdl(combine_kernel_p8<OT, OutT, 2, 2>, grid2, blk, 0, s, pdl, p);
  if (p.d == 128 && n <= 4) return launch_maybe_pdl(combine_kernel_p8<OT, OutT, 4, 2>, grid2, blk, 0, s, pdl, p);
  if (p.d == 128 && n <= 8) return launch_maybe_pdl(combine_kernel_p8<OT, OutT, 8, 2>, grid2, blk, 0, s, pdl, p);
  if (p.d == 128) return launch_maybe_pdl(combine_kernel<OT, OutT, 4>, grid, blk, 0, s, pdl, p);
  if (p.d == 256) return launch_maybe_pdl(combine_kernel<OT, OutT, 8>, grid, blk, 0, s, pdl, p);
  return launch_maybe_pdl(combine_kernel<OT, OutT, 0>, grid, blk, 0, s, pdl, p);
}

hydra_status launch_combine(const CombineParams &p, hydra_dtype o_dtype, hydra_dtype out_dtype,
                            cudaStream_t s) {
  if (p.rows == 0) return HYDRA_OK;
  cudaError_t e;
  if (o_dtype == HYDRA_F32 && out_dtype == HYDRA_BF16) e = launch_c<float, __nv_bfloat16>(p, s);
  else if (o_dtype == HYDRA_F32 && out_dtype == HYDRA_F32) e = launch_c<float, float>(p, s);
  else if (o_dtype == HYDRA_F16 && out_dtype == HYDRA_BF16) e = launch_c<__half, __nv_bfloat16>(p, s);
  else if (o_dtype == HYDRA_F16 && out_dtype == HYDRA_F32) e = launch_c<__half, float>(p, s);
  else if (o_dtype == HYDRA_F32 && out_dtype == HYDRA_F16) e = launch_c<float, __half>(p, s);  // exchange packing
  else return HYDRA_EUNSUPPORTED;
  return e == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

__global__ void fill_neg_inf_kernel(float *x, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = -INFINITY;
}

hydra_status launch_fill_neg_inf(float *lse, int64_t n, cudaStream_t s) {
  if (n <= 0) return HYDRA_OK;
  const int64_t nb = (n + 255) / 256;
  const int blocks = (int)(nb < 4096 ? nb : 4096);
  fill_neg_inf_kernel<<<blocks, 256, 0, s>>>(lse, n);
  return cudaGetLastError() == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

}  // namespace hydra

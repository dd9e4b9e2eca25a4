// decode.cu -- memory-bound split-K decode attention (one query per sequence).
//
// This is the suffix kernel of the paper's decomposition ("suffix attention is
// therefore computed normally, with a single query per sequence", §3.2 P:116;
// App. B) and also the SIMT fallback for the prefix in the fp32
// reference mode (the prefix then is a KV segment with batch stride 0).
//
// Work decomposition: one 128-thread CTA per (sequence b, KV head j, chunk of GQ
// query heads of that group, KV split).  Each token row of K/V (d elements) is
// read by TPR = d*sizeof(T)/16 threads with 16-byte non-caching vector loads, so a
// warp reads 32*16 = 512 contiguous-per-row bytes per instruction; the CTA's
// NG = 128/TPR row groups walk the tokens with stride NG, U tokens in flight per
// group.  Scores are reduced across the TPR lanes of a row with xor-shuffles; each
// row group keeps an online softmax state (running max m, sum l, accumulator) per
// query head in the log2 domain; the NG states are merged through shared memory at
// the end with the same rescaling (Eq. 5 math).  Positions >= lens[b] are never
// loaded (poisoned padding cannot leak in).
#include "common.cuh"
#include "internal.h"
#include "fused.cuh"

namespace hydra {

template <typename T, int D, int GQ, int U, bool kStream, bool kPaged>
__global__ void __launch_bounds__(128) decode_attn_kernel(const DecodeParams p) {
  constexpr int EPT = Vec16<T>::N;          // elements per thread per row
  constexpr int TPR = D / EPT;              // threads per token row
  constexpr int NG = 128 / TPR;             // row groups per CTA
  static_assert(TPR >= 1 && TPR <= 32 && (TPR & (TPR - 1)) == 0, "bad TPR");

  __shared__ float sm_m[NG][GQ];
  __shared__ float sm_l[NG][GQ];
  __shared__ float sm_acc[NG][GQ][D];

  const int tid = threadIdx.x;
  const int64_t cta_lin = ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  const int64_t n_cta = (int64_t)gridDim.x * gridDim.y * gridDim.z;
  if (p.timer && tid == 0 && cta_lin == 0) atomicMin(p.timer, gtimer());
  const int lane = tid % TPR;
  const int grp = tid / TPR;
  const int split = blockIdx.x;
  const int n_chunks = p.g / GQ;
  const int j = blockIdx.y / n_chunks;
  const int chunk = blockIdx.y % n_chunks;
  const int slot = blockIdx.z;
  const int b = p.seq_map ? p.seq_map[slot] : slot;
  const int h0 = j * p.g + chunk * GQ;

  // out-of-range lens[b] (a documented precondition violation) is clamped to [0, len_cap]
  const int64_t len = p.lens ? min(max((int64_t)p.lens[b], (int64_t)0), p.len_cap) : p.len_uniform;
  const int64_t t_begin = (int64_t)split * p.split_len;
  const int64_t t_end = min(len, t_begin + p.split_len);

  // query fragments, pre-scaled by scale*log2(e) so scores come out in log2 units
  float qf[GQ][EPT];
#pragma unroll
  for (int i = 0; i < GQ; ++i) {
    const T *qp = reinterpret_cast<const T *>(p.q) + (int64_t)b * p.q_sb + (int64_t)(h0 + i) * p.q_sh + lane * EPT;
    Vec16<T>::unpack(ld_v4<false>(qp), qf[i]);
#pragma unroll
    for (int e = 0; e < EPT; ++e) qf[i][e] *= p.scale_log2;
  }

  float m[GQ], l[GQ], acc[GQ][EPT];
#pragma unroll
  for (int i = 0; i < GQ; ++i) {
    m[i] = -INFINITY;
    l[i] = 0.f;
#pragma unroll
    for (int e = 0; e < EPT; ++e) acc[i][e] = 0.f;
  }

  // paged: kv_sb is the page stride and the block table gives each token's page
  const int64_t seq_off = kPaged ? 0 : (int64_t)b * p.kv_sb;
  const T *kb = reinterpret_cast<const T *>(p.k) + seq_off + (int64_t)j * p.kv_sh + lane * EPT;
  const T *vb = reinterpret_cast<const T *>(p.v) + seq_off + (int64_t)j * p.kv_sh + lane * EPT;
  const int32_t *btab = kPaged ? p.block_table + (int64_t)b * p.bt_stride : nullptr;

  // Trip count is uniform across the CTA (shuffles below need converged warps).
  for (int64_t tb = t_begin; tb < t_end; tb += (int64_t)NG * U) {
    uint4 kr[U], vr[U];
    bool valid[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = tb + grp + (int64_t)u * NG;
      valid[u] = t < t_end;
      if (valid[u]) {
        const int64_t off = kPaged ? (int64_t)__ldg(btab + (t >> p.page_shift)) * p.kv_sb +
                                         (t & ((1 << p.page_shift) - 1)) * p.kv_st
                                   : (p.kv_tok_off + t) * p.kv_st;
        kr[u] = ld_v4<kStream>(kb + off);
        vr[u] = ld_v4<kStream>(vb + off);
      } else {
        kr[u] = make_uint4(0, 0, 0, 0);
        vr[u] = make_uint4(0, 0, 0, 0);
      }
    }
    float s[U][GQ];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float kf[EPT];
      Vec16<T>::unpack(kr[u], kf);
#pragma unroll
      for (int i = 0; i < GQ; ++i) {
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < EPT; ++e) a = fmaf(qf[i][e], kf[e], a);
#pragma unroll
        for (int off = TPR / 2; off >= 1; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
        s[u][i] = valid[u] ? a : -INFINITY;
      }
    }
#pragma unroll
    for (int i = 0; i < GQ; ++i) {
      float mx = m[i];
#pragma unroll
      for (int u = 0; u < U; ++u) mx = fmaxf(mx, s[u][i]);
      if (mx == -INFINITY) continue;  // nothing valid yet (uniform across the row group)
      const float alpha = exp2f(m[i] - mx);
      float pu[U];
      float ps = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        pu[u] = exp2f(s[u][i] - mx);
        ps += pu[u];
      }
      l[i] = l[i] * alpha + ps;
#pragma unroll
      for (int e = 0; e < EPT; ++e) acc[i][e] *= alpha;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float vf[EPT];
        Vec16<T>::unpack(vr[u], vf);
#pragma unroll
        for (int e = 0; e < EPT; ++e) acc[i][e] = fmaf(pu[u], vf[e], acc[i][e]);
      }
      m[i] = mx;
    }
  }

  // ---- merge the NG row-group states (Eq. 5 rescaling in the log2 domain)
#pragma unroll
  for (int i = 0; i < GQ; ++i) {
    if (lane == 0) {
      sm_m[grp][i] = m[i];
      sm_l[grp][i] = l[i];
    }
#pragma unroll
    for (int e = 0; e < EPT; ++e) sm_acc[grp][i][lane * EPT + e] = acc[i][e];
  }
  __syncthreads();
  for (int idx = tid; idx < GQ * D; idx += 128) {
    const int i = idx / D, e = idx % D;
    float M = -INFINITY;
#pragma unroll
    for (int gi = 0; gi < NG; ++gi) M = fmaxf(M, sm_m[gi][i]);
    const int h = h0 + i;
    float *o = p.o + (int64_t)split * p.o_split_stride + ((int64_t)b * p.Hq + h) * D;
    if (M == -INFINITY) {  // empty key set: (0, -inf) sentinel
      o[e] = 0.f;
      if (e == 0) p.lse[(int64_t)split * p.lse_split_stride + (int64_t)b * p.Hq + h] = -INFINITY;
      continue;
    }
    float L = 0.f, A = 0.f;
#pragma unroll
    for (int gi = 0; gi < NG; ++gi) {
      const float w = exp2f(sm_m[gi][i] - M);
      L += sm_l[gi][i] * w;
      A += sm_acc[gi][i][e] * w;
    }
    o[e] = A / L;
    if (e == 0)
      p.lse[(int64_t)split * p.lse_split_stride + (int64_t)b * p.Hq + h] = (M + log2f(L)) * HYDRA_LN2;
  }
  if constexpr (D == 128) {
    // Fused Eq. 5 (fused.cuh): this split's part of the CTA's GQ rows is stored; count the
    // arrivals and merge the rows it completed (thread = dim).
    if (p.fc.cnt) {
      __shared__ uint32_t fc_mask;
      if (fc_counting(p.fc)) __threadfence();
      __syncthreads();
      if (tid < 32) {
        const bool last = tid < GQ && fc_arrive(p.fc, (int64_t)b * p.Hq + h0 + tid, fc_expected(p.fc, b, h0 + tid));
        const uint32_t m2 = __ballot_sync(0xffffffffu, last);
        if (tid == 0) fc_mask = m2;
      }
      __syncthreads();
      uint32_t m2 = fc_mask;
      if (m2) __threadfence();
      while (m2) {
        const int i = __ffs(m2) - 1;
        m2 &= m2 - 1;
        fc_merge_row_dim(p.fc, (int64_t)b * p.Hq + h0 + i, fc_prefix_pieces(p.fc, b, h0 + i), tid);
      }
    }
  }
  // A programmatic dependent of the prefix kernel (the suffix fills the SMs the prefix leaves free)
  // must complete only after it: the LAST CTA in launch order waits for the prefix grid, so this
  // grid cannot complete earlier, while every other CTA exits at once and frees its slot for
  // the next CTA (waiting in every CTA parked the CTAs started beside the prefix until it ended:
  // that was why this kernel measured slower as a dependent).  A no-op otherwise.
  if (p.timer && tid == 0 && cta_lin >= n_cta - 1024) atomicMax(p.timer + 1, gtimer());
  asm volatile("griddepcontrol.launch_dependents;");  // the combine may launch as the last CTAs drain
  if (cta_lin == n_cta - 1) asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename T, int D, int GQ, int U>
static cudaError_t launch_u(const DecodeParams &p, cudaStream_t s) {
  const dim3 grid(p.n_splits, p.Hkv * (p.g / GQ), p.n_seq);
  const bool pdl = p.pdl != 0;
  if (p.block_table)  // paged suffix cache
    return launch_maybe_pdl(decode_attn_kernel<T, D, GQ, U, true, true>, grid, dim3(128), 0, s, pdl, p);
  if (p.kv_sb == 0)  // shared KV (prefix in SIMT mode): let L1 keep it
    return launch_maybe_pdl(decode_attn_kernel<T, D, GQ, U, false, false>, grid, dim3(128), 0, s, pdl, p);
  return launch_maybe_pdl(decode_attn_kernel<T, D, GQ, U, true, false>, grid, dim3(128), 0, s, pdl, p);
}

template <typename T, int D, int GQ>
static cudaError_t launch_t(const DecodeParams &p, cudaStream_t s) {
  // more tokens in flight per thread only where registers allow (one query head per CTA)
  if constexpr (GQ == 1) {
    if (p.unroll >= 8) return launch_u<T, D, GQ, 8>(p, s);
  }
  return launch_u<T, D, GQ, 4>(p, s);
}

template <typename T, int D>
static cudaError_t launch_d(const DecodeParams &p, cudaStream_t s) {
  switch (p.heads_per_cta) {
    case 1: return launch_t<T, D, 1>(p, s);
    case 2: return launch_t<T, D, 2>(p, s);
    case 4: return launch_t<T, D, 4>(p, s);
    case 8: return launch_t<T, D, 8>(p, s);
  }
  return cudaErrorInvalidValue;
}

hydra_status launch_decode(const DecodeParams &p, hydra_dtype dt, int d, cudaStream_t s) {
  if (p.n_seq <= 0 || p.n_splits <= 0) return HYDRA_OK;
  if (p.fc.cnt && (d != 128 || p.fc.n_suf != p.n_splits)) return HYDRA_EINVAL;
  cudaError_t e = cudaErrorInvalidValue;
  if (dt == HYDRA_BF16) {
    switch (d) {
      case 16: e = launch_d<__nv_bfloat16, 16>(p, s); break;
      case 32: e = launch_d<__nv_bfloat16, 32>(p, s); break;
      case 64: e = launch_d<__nv_bfloat16, 64>(p, s); break;
      case 128: e = launch_d<__nv_bfloat16, 128>(p, s); break;
      case 256: e = launch_d<__nv_bfloat16, 256>(p, s); break;
      default: return HYDRA_EUNSUPPORTED;
    }
  } else if (dt == HYDRA_F32) {
    switch (d) {
      case 16: e = launch_d<float, 16>(p, s); break;
      case 32: e = launch_d<float, 32>(p, s); break;
      case 64: e = launch_d<float, 64>(p, s); break;
      case 128: e = launch_d<float, 128>(p, s); break;
      default: return HYDRA_EUNSUPPORTED;
    }
  } else {
    return HYDRA_EUNSUPPORTED;
  }
  return e == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

}  // namespace hydra

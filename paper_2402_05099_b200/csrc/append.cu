// append.cu -- decode-loop KV append: the new
// token's K/V row of every sequence is written into its suffix cache at position lens[b],
// then lens[b] is incremented -- on the device, so a decode step (attention + append) can be
// replayed from one CUDA graph with no host round trip (the paper's CUDA-graph requirement,
// P:149).  Pure data movement: 16-B vector copies, one CTA per sequence.
#include "common.cuh"
#include "internal.h"

namespace hydra {

// k_new/v_new: [B, Hkv, d] rows (strides nb, nh; d contiguous), caches [B, S_cap, Hkv, d]
// (strides s_sb, s_st, s_sh) or, with a block table, page pools [n_pages, page_size, Hkv, d]
// (s_sb = page stride; S_cap = pages per sequence * page_size).  A sequence whose
// lens[b] == S_cap is left unchanged and its lens[b] is not incremented (the caller sized the
// cache too small; documented).
__global__ void append_kv_kernel(const uint4 *__restrict__ k_new, const uint4 *__restrict__ v_new, int64_t nb,
                                 int64_t nh, uint4 *__restrict__ sk, uint4 *__restrict__ sv, int64_t s_sb,
                                 int64_t s_st, int64_t s_sh, int32_t S_cap, int32_t Hkv, int32_t d16,
                                 int32_t *__restrict__ lens, const int32_t *__restrict__ block_table,
                                 int64_t bt_stride, int32_t page_shift) {
  const int b = blockIdx.x;
  const int pos = lens[b];
  if (pos >= S_cap || pos < 0) return;  // uniform across the CTA (a full or invalid entry is left unchanged)
  // contiguous: row pos of sequence b; paged (s_sb = page stride): row pos % page_size of
  // page block_table[b][pos / page_size]
  const int64_t row0 = block_table ? (int64_t)block_table[b * bt_stride + (pos >> page_shift)] * s_sb +
                                         (int64_t)(pos & ((1 << page_shift) - 1)) * s_st
                                   : b * s_sb + (int64_t)pos * s_st;
  const int per = Hkv * d16;  // 16-B chunks per token row (all KV heads)
  for (int i = threadIdx.x; i < per; i += blockDim.x) {
    const int j = i / d16, c = i % d16;
    const int64_t src = b * nb + j * nh + c;                          // in 16-B units
    const int64_t dst = row0 + j * s_sh + c;  // in 16-B units
    sk[dst] = __ldg(k_new + src);
    sv[dst] = __ldg(v_new + src);
  }
  __syncthreads();  // every thread's reads of lens[b] precede the increment
  if (threadIdx.x == 0) lens[b] = pos + 1;
}

hydra_status launch_append_kv(const void *k_new, const void *v_new, int64_t nb, int64_t nh, void *sk, void *sv,
                              int64_t s_sb, int64_t s_st, int64_t s_sh, int64_t S_cap, int32_t Hkv, int32_t d,
                              size_t es, int64_t B, int32_t *lens, cudaStream_t s,
                              const int32_t *block_table, int64_t bt_stride, int32_t page_size) {
  // strides in elements -> 16-B units (validated 16-B aligned by the caller)
  const int64_t u = 16 / (int64_t)es;
  const int d16 = (int)(d / u);
  const int threads = (int)std::min<int64_t>(1024, std::max<int64_t>(32, ((int64_t)Hkv * d16 + 31) / 32 * 32));
  append_kv_kernel<<<(unsigned)B, threads, 0, s>>>(
      reinterpret_cast<const uint4 *>(k_new), reinterpret_cast<const uint4 *>(v_new), nb / u, nh / u,
      reinterpret_cast<uint4 *>(sk), reinterpret_cast<uint4 *>(sv), s_sb / u, s_st / u, s_sh / u, (int32_t)S_cap,
      Hkv, d16, lens, block_table, bt_stride, block_table ? __builtin_ctz((unsigned)page_size) : 0);
  return cudaGetLastError() == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

}  // namespace hydra

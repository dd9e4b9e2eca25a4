/*
 * hydra.h -- C ABI of the B200 (sm_100a) shared-prefix decode-attention library
 * (libhydra.so).  Hydragen, arXiv 2402.05099; "P:NNN" = /root/reference/PAPER.md line.
 *
 * The library computes exact softmax attention (Eq. 1) for one decode step
 * (Nq = 1) of B sequences that share a prefix, by the paper's decomposition:
 *   prefix attention with all B*g queries of a KV head stacked into one dense
 *   matrix (inter-sequence batching, §3.2) -> (O_p, LSE_p);
 *   suffix attention, one query per sequence over its own KV (§3.2)
 *   -> (O_s, LSE_s);
 *   LSE combine (Eq. 5; App. B combine_lse P:321-344) -> O.
 * Tree-shaped sharing applies the decomposition at every tree vertex (§3.3).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Pointers are DEVICE pointers unless marked "host".  The caller owns every
 *    buffer; the library never allocates on the hot path (the only owned object
 *    is hydra_tree, created and destroyed by the caller).
 *  - Strides are in ELEMENTS.  The innermost (head_dim) axis must be contiguous.
 *    Tensor layouts follow App. B with Nq = 1:
 *        q        [B, Hq, d]            element (b,h,i) at q[b*q_sb + h*q_sh + i]
 *        prefix   [P, Hkv, d]           element (t,j,i) at k[t*kv_st + j*kv_sh + i]
 *        suffix   [B, S_cap, Hkv, d]    element (b,t,j,i) at k[b*s_sb + t*s_st + j*s_sh + i]
 *        o_part   [B, Hq, d] float32 contiguous,  lse_part [B, Hq] float32 contiguous
 *        out      [B, Hq, d] contiguous in out_dtype
 *  - Query head h reads KV head floor(h / (Hq/Hkv)) (reading R3).
 *  - Softmax scale: heads.scale, or 1/sqrt(d) when 0 (Eq. 1).
 *  - LSE values are NATURAL logs of the softmax denominator over scaled scores
 *    (Eq. 4).  An empty key set (P == 0, lens[b] == 0) yields the sentinel
 *    O = 0, LSE = -inf, which every combine treats as the identity (reading R6).
 *  - Every call is asynchronous and stream-ordered on `stream` (a cudaStream_t
 *    passed as void*), never synchronises the host and never reads device data
 *    on the host, so it can be captured in a CUDA graph (the paper's requirement,
 *    P:149).  Tree attention is capturable once its tree is prepared for the head
 *    grouping (hydra_tree_prepare; an unprepared tree is prepared by the first call
 *    made outside capture, and a captured call on it fails with HYDRA_EINVAL).
 *  - Errors: host-visible arguments are validated synchronously; on a non-OK
 *    status nothing has been launched and hydra_last_error() describes why.
 *    Launch failures return HYDRA_ECUDA.  Device-resident lens values are a
 *    documented precondition (0 <= lens[b] <= S_cap): the kernels clamp an
 *    out-of-range value into [0, S_cap] (never reading past the cache), and the
 *    testing build (libhydra_test.so) also counts violations on the device
 *    (hydra_debug_lens_violations).
 *  - Thread safety: all entry points are reentrant.  hydra_last_error and the
 *    settings of hydra_set_config are thread-local: one thread's switches and
 *    measurement events never affect another thread's calls.
 *  - Precision: HYDRA_BF16 inputs use fp32 accumulation, fp32 partials and a
 *    bf16 (round-to-nearest-even) final output; HYDRA_F32 inputs run an all-fp32
 *    reference mode (SIMT kernels, accurate exp).
 *  - Kernels: BF16 with head_dim 128 runs the tcgen05/TMEM/TMA kernels (the stacked
 *    prefix GEMM of §3.2 and the tensor-core suffix GEMV).  Other head dims and F32
 *    run SIMT kernels: the suffix kernel, and for the prefix the same kernel with a
 *    batch stride of 0 (every sequence reads the one prefix copy through L2, but the
 *    queries are not stacked into a tensor-core GEMM).
 */
#ifndef HYDRA_H_
#define HYDRA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HYDRA_API __attribute__((visibility("default")))
#else
#define HYDRA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t hydra_status;
#define HYDRA_OK 0
#define HYDRA_EINVAL 1       /* null pointer / negative size / bad enum         */
#define HYDRA_ESHAPE 2       /* Hq % Hkv != 0, stride or shape mismatch, B == 0   */
#define HYDRA_EUNSUPPORTED 3 /* head_dim / dtype combination not compiled        */
#define HYDRA_ECUDA 4        /* CUDA launch or runtime failure                    */
#define HYDRA_ENCCL 5        /* reserved for the multi-GPU layer                  */
#define HYDRA_ENOMEM 6       /* workspace too small / host allocation failed      */

typedef enum {
  HYDRA_BF16 = 0,
  HYDRA_F32 = 1,
  HYDRA_F16 = 2 /* only for exchanged partial outputs (hydra_combine o_dtype) */
} hydra_dtype;

/* Attention head configuration (SPEC AttentionConfig). */
typedef struct {
  int32_t num_q_heads;  /* Hq                                  */
  int32_t num_kv_heads; /* Hkv, Hq % Hkv == 0                  */
  int32_t head_dim;     /* d: 16, 32, 64, 128 or 256           */
  float scale;          /* 0 => 1/sqrt(d)                      */
  hydra_dtype dtype;    /* dtype of q and all K/V: BF16 or F32 */
} hydra_heads;

/* Workspace queries: op codes for hydra_workspace_size. */
#define HYDRA_OP_PREFIX 0
#define HYDRA_OP_SUFFIX 1
#define HYDRA_OP_ATTN 2
#define HYDRA_OP_PARTS 3 /* n_parts caller-staged partial slots (O f32 [B,Hq,d] + LSE f32 [B,Hq] each) */

/*
 * hydra_prefix_attn -- inter-sequence batched attention over the shared prefix
 * (§3.2; App. B `attention(batched_q, prefix_k, prefix_v)` P:366-378).
 * For KV head j the B*g query rows r = b*g + i (q[b, j*g+i, :]) are stacked into
 * one matrix and attend, as one dense GEMM-shaped problem, to prefix K/V
 * [P, Hkv, d] read once.  Output: o_part[b,h,:] = SDP(q[b,h], K_p, V_p) (fp32,
 * normalised) and lse_part[b,h] = LSE(q[b,h], K_p) (Eq. 4).
 * BF16 with d == 128 runs the tcgen05/TMEM/TMA kernel; other shapes and F32 run
 * the SIMT kernel.  ws may be NULL when hydra_workspace_size(HYDRA_OP_PREFIX,...)
 * returns 0.
 */
HYDRA_API hydra_status hydra_prefix_attn(const hydra_heads *h, int64_t B,
                               const void *q, int64_t q_sb, int64_t q_sh,
                               int64_t P, const void *k, const void *v, int64_t kv_st, int64_t kv_sh,
                               float *o_part, float *lse_part,
                               void *ws, size_t ws_bytes, void *stream);

/*
 * hydra_suffix_attn -- per-sequence attention over each sequence's own suffix
 * ("computed normally, with a single query per sequence", §3.2; App. B
 * P:381-388 with the per-sequence q, reading R4).  Sequence b attends to its
 * first lens[b] suffix tokens (device int32 array [B]; positions >= lens[b] are
 * never read).  Split-K over tokens when B*Hkv is small.  Output as
 * hydra_prefix_attn.
 */
HYDRA_API hydra_status hydra_suffix_attn(const hydra_heads *h, int64_t B,
                               const void *q, int64_t q_sb, int64_t q_sh,
                               const void *k, const void *v, int64_t s_sb, int64_t s_st, int64_t s_sh,
                               int64_t S_cap, const int32_t *lens,
                               float *o_part, float *lse_part,
                               void *ws, size_t ws_bytes, void *stream);

/*
 * hydra_combine -- n-ary LSE combine (Eq. 5 P:98-105 in App. B's max-stabilised
 * form P:333-344, folded over n_parts; associativity S:154).  For each row r:
 *   m = max_p lse_p[r];  w_p = exp(lse_p[r] - m);  O[r] = sum_p w_p O_p[r] / sum_p w_p;
 *   lse_out[r] = m + ln(sum_p w_p).
 * Parts whose lse is -inf are skipped (their O is never read).  Part p row r is at
 * o_parts + p*o_part_stride + r*d (elements of o_dtype = F32 or F16) and
 * lse_parts[p*lse_part_stride + r]; strides let it read an all-gathered
 * [rank][O|LSE] buffer in place.  out_dtype BF16 or F32 (or F16 from F32 parts: packing
 * partials for a cross-GPU exchange, n_parts may be 1); lse_out may be NULL.
 * (The testing build's config key "inject_combine_bug" drops the rescaling, w_p = 1:
 * a sabotage switch the parity suite must catch.  The release build has none.)
 */
HYDRA_API hydra_status hydra_combine(int64_t rows, int32_t d, int32_t n_parts,
                           const void *o_parts, hydra_dtype o_dtype, int64_t o_part_stride,
                           const float *lse_parts, int64_t lse_part_stride,
                           void *out, hydra_dtype out_dtype, float *lse_out, void *stream);

/*
 * hydra_combine_ex -- the same Eq. 5 combine over two groups of parts with explicit row
 * strides (elements; 0 = dense rows: d for O, 1 for LSE):
 *   group A: n_parts parts in o_dtype (F32, or F16 partials received from other GPUs), part p
 *            row r at o_parts + p*o_part_stride + r*o_row_stride, LSE at
 *            lse_parts[p*lse_part_stride + r*lse_row_stride];
 *   group B: n_parts_f32 parts in F32 (may be 0), addressed the same way;
 *   out row r at out + r*out_row_stride (out_dtype), lse_out[r*lse_out_row_stride] (nullable).
 * Every row merges all n_parts + n_parts_f32 parts at once.  Row strides let one call read or
 * write a buffer whose rows interleave O and LSE -- the multi-GPU layer packs a rank's
 * (O f16 | LSE f32) rows with one call and merges the N received pieces with the local suffix
 * part with one call (paper_2402_05099_b200/dist.py).  For d = 128 / 256 the O bases and
 * strides must be 16-byte (F32) or 8-byte (F16) aligned (EINVAL).  Output rows must not
 * overlap input rows.
 */
typedef struct {
  int64_t rows;
  int32_t d;
  int32_t n_parts;
  const void *o_parts;
  hydra_dtype o_dtype;
  int64_t o_part_stride, o_row_stride;
  const float *lse_parts;
  int64_t lse_part_stride, lse_row_stride;
  int32_t n_parts_f32;
  const float *o_parts_f32;
  int64_t o_f32_part_stride, o_f32_row_stride;
  const float *lse_parts_f32;
  int64_t lse_f32_part_stride, lse_f32_row_stride;
  void *out;
  hydra_dtype out_dtype;
  int64_t out_row_stride;
  float *lse_out;
  int64_t lse_out_row_stride;
  /* Scattered output (table_rows > 0; then out / lse_out are ignored): output row r goes to
   * out_table[r / table_rows] + (r % table_rows) * out_row_stride, its LSE to
   * lse_out_table[r / table_rows][(r % table_rows) * lse_out_row_stride] (lse_out_table
   * nullable).  Device arrays of ceil(rows / table_rows) device pointers, which may point into
   * other GPUs' memory (peer-mapped / symmetric buffers): the multi-GPU layer's pack writes each
   * batch shard's rows straight into the owning GPU's receive buffer over NVLink.  The caller
   * orders those stores before the owner reads them (a cross-GPU barrier after this call). */
  void *const *out_table;
  float *const *lse_out_table;
  int64_t table_rows;
} hydra_combine_desc;
HYDRA_API hydra_status hydra_combine_ex(const hydra_combine_desc *c, void *stream);

/*
 * hydra_attn -- the whole decode-step attention of App. B `hydragen_attention`
 * (P:347-399): prefix (hydra_prefix_attn) || suffix (hydra_suffix_attn) ->
 * combine, writing out[B,Hq,d] (out_dtype) and optionally lse_out[B,Hq].
 * Everything is launched on `stream`.  s_aux non-NULL means the caller allows the prefix and
 * the suffix to run concurrently: the suffix then becomes a programmatic dependent launch of
 * the prefix on disjoint SMs -- the persistent tensor-core suffix on the SMs the prefix leaves
 * (heavy prefix), the short-suffix kernel on all but one stream-K group's SMs (short GQA
 * suffixes), or the SIMT suffix over its full grid beside a prefix on >= 32 CTAs (light MHA
 * prefix) -- whichever the planner finds faster than prefix-then-suffix (config keys
 * overlap_prefix_ctas, overlap_short, overlap_simt; hydra_get_config("last_overlap_k") /
 * "last_overlap_simt" report the choice).  Without s_aux the two run one after the other (GQA
 * tensor-core suffixes still start in the prefix's tail as its programmatic dependents).  s_aux
 * itself receives no work.  The combine follows on `stream` (a programmatic dependent of the
 * suffix, waiting for it at entry).
 * Requires ws_bytes >= hydra_workspace_size(HYDRA_OP_ATTN, h, B, P, S_cap, 0).
 */
HYDRA_API hydra_status hydra_attn(const hydra_heads *h, int64_t B,
                        const void *q, int64_t q_sb, int64_t q_sh,
                        int64_t P, const void *pk, const void *pv, int64_t kv_st, int64_t kv_sh,
                        const void *sk, const void *sv, int64_t s_sb, int64_t s_st, int64_t s_sh,
                        int64_t S_cap, const int32_t *lens,
                        void *out, hydra_dtype out_dtype, float *lse_out,
                        void *ws, size_t ws_bytes, void *stream, void *s_aux);

/*
 * hydra_append_kv -- decode-loop KV append: for every sequence b,
 * write its new token's rows k_new[b, :, :] / v_new[b, :, :] ([B, Hkv, d], strides nb / nh
 * in elements, d contiguous) into the suffix caches at position lens[b]
 * (suffix_k/v[B, S_cap, Hkv, d], strides s_sb / s_st / s_sh), then increment lens[b] -- on
 * the device, so "attend, then append" (the order of SPEC's toy model) replays
 * from one CUDA graph step after step.  Precondition: lens[b] < S_cap; a sequence whose
 * cache is full is left unchanged (no write, no increment).  Same dtype as h->dtype;
 * every pointer and stride 16-byte aligned (EINVAL otherwise).  Asynchronous on `stream`.
 */
HYDRA_API hydra_status hydra_append_kv(const hydra_heads *h, int64_t B,
                             const void *k_new, const void *v_new, int64_t nb, int64_t nh,
                             void *sk, void *sv, int64_t s_sb, int64_t s_st, int64_t s_sh, int64_t S_cap,
                             int32_t *lens, void *stream);

/*
 * Paged suffix cache ("per-step suffix KV append into a growable or
 * paged cache").  The paper keeps each sequence's suffix K/V in its own contiguous tensor
 * (App. B, suffix_k/v [B, Nq+S, Hkv, d]); a serving engine instead allocates
 * the suffixes from a pool of fixed-size pages so sequences can grow without a
 * worst-case reservation.  The attention is unchanged -- only where token t of sequence
 * b is read from (reading R14):
 *     suffix row (b, t)  ==  pool row (block_table[b * bt_stride + t / page_size], t % page_size)
 * Pools: k_pool / v_pool [n_pages, page_size, Hkv, d], element (p, r, j, i) at
 * pool[p*p_sp + r*p_st + j*p_sh + i] (same dtype as h->dtype, 16-byte aligned strides).
 * block_table: DEVICE int32 [B, bt_stride], owned by the caller; entries for the pages
 * that cover tokens 0 .. lens[b]-1 must be in [0, n_pages) (a documented precondition
 * like lens, not checked); entries past them are never read.  Pages may be shared or
 * listed in any order.  S_cap (capacity, tokens per sequence) must be
 * <= bt_stride * page_size and bounds lens[b] as in the contiguous calls.
 */
typedef struct {
  const int32_t *block_table; /* device [B, bt_stride]                             */
  int64_t bt_stride;          /* row stride of block_table (pages per sequence)    */
  int32_t page_size;          /* tokens per page: a power of two >= 8 (ESHAPE)     */
  int64_t n_pages;            /* pages in each pool, in [1, 2^31)                  */
} hydra_paging;

/* hydra_suffix_attn over a paged cache; otherwise identical (same kernels, same
 * workspace size as hydra_workspace_size(HYDRA_OP_SUFFIX, h, B, 0, S_cap, 0)). */
HYDRA_API hydra_status hydra_suffix_attn_paged(const hydra_heads *h, int64_t B,
                                     const void *q, int64_t q_sb, int64_t q_sh,
                                     const void *k_pool, const void *v_pool, int64_t p_sp, int64_t p_st, int64_t p_sh,
                                     const hydra_paging *pg, int64_t S_cap, const int32_t *lens,
                                     float *o_part, float *lse_part,
                                     void *ws, size_t ws_bytes, void *stream);

/* hydra_attn with the suffix in a paged cache (prefix stays a dense [P, Hkv, d] tensor:
 * it is read once per step by the stacked-query GEMM, §3.2).  Workspace as hydra_attn. */
HYDRA_API hydra_status hydra_attn_paged(const hydra_heads *h, int64_t B,
                              const void *q, int64_t q_sb, int64_t q_sh,
                              int64_t P, const void *pk, const void *pv, int64_t kv_st, int64_t kv_sh,
                              const void *k_pool, const void *v_pool, int64_t p_sp, int64_t p_st, int64_t p_sh,
                              const hydra_paging *pg, int64_t S_cap, const int32_t *lens,
                              void *out, hydra_dtype out_dtype, float *lse_out,
                              void *ws, size_t ws_bytes, void *stream, void *s_aux);

/* hydra_append_kv into a paged cache: sequence b's new row goes to row lens[b] % page_size
 * of page block_table[b][lens[b] / page_size] (the caller has mapped that page before the
 * call, e.g. when lens[b] % page_size == 0), then lens[b] += 1 on the device.  A sequence
 * with lens[b] >= S_cap is left unchanged. */
HYDRA_API hydra_status hydra_append_kv_paged(const hydra_heads *h, int64_t B,
                                   const void *k_new, const void *v_new, int64_t nb, int64_t nh,
                                   void *k_pool, void *v_pool, int64_t p_sp, int64_t p_st, int64_t p_sh,
                                   const hydra_paging *pg, int64_t S_cap, int32_t *lens, void *stream);

/*
 * Sharing tree (§3.3, Fig. 2; SPEC SharingTree S:182-193).
 * Host arrays: parent[n_nodes] (root = -1, exactly one root), node_off/node_len
 * [n_nodes] (node n owns tokens node_off[n] .. node_off[n]+node_len[n]-1 of the
 * pooled node K/V [T_nodes, Hkv, d]), leaf_of_seq[B] (sequence b's leaf node).
 * Validation: one root, parents in range, no cycles, node_len >= 1 for
 * every non-root node (the root may be empty), node_off >= 0, every sequence on a
 * leaf (a node without children) and every leaf used by >= 1 sequence.
 * hydra_tree_create builds the per-node query groups (ascending sequence ids of
 * every sequence whose root->leaf path passes through the node) and
 * copies them to the device (synchronous; call outside graph capture).
 * hydra_tree_prepare uploads the node-attention work list for the head grouping of `h`
 * (synchronous, outside capture; idempotent).  After it, every hydra_tree_attn /
 * hydra_tree_attn_paged call with that grouping is a pure, capturable launch sequence.
 * A tree may be prepared for several groupings.
 */
struct hydra_tree;
HYDRA_API hydra_status hydra_tree_create(const int32_t *parent, const int64_t *node_off, const int64_t *node_len,
                               int32_t n_nodes, const int32_t *leaf_of_seq, int64_t B,
                               struct hydra_tree **out);
HYDRA_API hydra_status hydra_tree_prepare(struct hydra_tree *t, const hydra_heads *h);
HYDRA_API void hydra_tree_destroy(struct hydra_tree *t);
/* Depth (number of nodes on the longest root->leaf path) and group sizes, for tooling. */
HYDRA_API int32_t hydra_tree_depth(const struct hydra_tree *t);
HYDRA_API int64_t hydra_tree_group_size(const struct hydra_tree *t, int32_t node);
HYDRA_API size_t hydra_tree_workspace_size(const hydra_heads *h, const struct hydra_tree *t, int64_t S_cap);

/*
 * hydra_tree_attn -- tree attention: for every node, the stacked queries of all
 * sequences in its group attend to the node's K/V (one grouped launch over
 * (node, KV head, query tile)); each sequence's suffix attention; then an n-ary
 * combine over the path partials and the suffix (decomposition at every vertex,
 * §3.3).  Output as hydra_attn.  Capturable once the tree is prepared for
 * this Hq/Hkv grouping (hydra_tree_prepare); an unprepared tree is prepared
 * synchronously by the first call made outside capture, and a captured call on an
 * unprepared tree returns HYDRA_EINVAL with nothing launched.
 * stream_aux: nullable second stream.  When given (and both the node attention and the
 * suffix take their persistent tensor-core kernels), the node attention runs on k SMs
 * on stream_aux while the suffix runs on the other SMs on `stream`, as in hydra_attn;
 * stream_aux is forked from and joined back into `stream` inside the call.
 */
HYDRA_API hydra_status hydra_tree_attn(const hydra_heads *h, const struct hydra_tree *t,
                             const void *q, int64_t q_sb, int64_t q_sh,
                             const void *node_k, const void *node_v, int64_t kv_st, int64_t kv_sh,
                             const void *sk, const void *sv, int64_t s_sb, int64_t s_st, int64_t s_sh,
                             int64_t S_cap, const int32_t *lens,
                             void *out, hydra_dtype out_dtype, float *lse_out,
                             void *ws, size_t ws_bytes, void *stream, void *stream_aux);

/* hydra_tree_attn with the sequences' suffixes in a paged cache (hydra_paging above); the
 * node K/V stay pooled [T_nodes, Hkv, d].  Workspace as hydra_tree_attn. */
HYDRA_API hydra_status hydra_tree_attn_paged(const hydra_heads *h, const struct hydra_tree *t,
                                   const void *q, int64_t q_sb, int64_t q_sh,
                                   const void *node_k, const void *node_v, int64_t kv_st, int64_t kv_sh,
                                   const void *k_pool, const void *v_pool, int64_t p_sp, int64_t p_st, int64_t p_sh,
                                   const hydra_paging *pg, int64_t S_cap, const int32_t *lens,
                                   void *out, hydra_dtype out_dtype, float *lse_out,
                                   void *ws, size_t ws_bytes, void *stream, void *stream_aux);

/* Bytes of device workspace the op needs for these sizes (0 if none).  n_parts is read by
 * HYDRA_OP_PARTS only: n_parts partial slots of B*Hq rows (for callers that stage their
 * own partials for hydra_combine, e.g. a cross-GPU exchange); the other ops ignore it. */
HYDRA_API size_t hydra_workspace_size(int op, const hydra_heads *h, int64_t B, int64_t P, int64_t S_cap,
                            int32_t n_parts);

/*
 * Tuning switches, per calling thread (thread-local; 0 = automatic unless stated):
 *   "prefix_impl"         1 SIMT, 2 one-tile tcgen05 kernel, 3 persistent two-tile tcgen05 kernel
 *   "prefix_variant"      persistent kernel: 9 (default: CTA-pair kernel, cta_group::2 M = 256
 *                         MMAs, three score buffers, blocks alternating between two softmax
 *                         warpgroups; flat mode with 128 % g == 0, else 6 runs), 6 (one CTA, two
 *                         128-row tiles, P published in two 64-token halves), 3 (6 without the
 *                         split), 4 (64-token blocks, double-buffered scores), 5 (3 + speculative
 *                         running-max softmax)
 *   "prefix_poly"         4 (default): every 4th exp2 pair on the FMA pipe; 0 all exp2 on MUFU; 3 / 8
 *                         (variants 3-6; variant 9 reads "pair_poly")
 *   "pair_poly"           CTA-pair kernel: 0 (default) all exp2 on MUFU; 4 every 4th pair on the FMA
 *                         pipe
 *   "pair_item_cost"      CTA-pair kernel: stream-K group boundaries balance blocks + this many
 *                         block-equivalents per item a group touches (default 0 = uniform split;
 *                         5 measured no faster: C6 0.098 -> 0.102 ms, C3@16K 0.840 -> 0.835)
 *   "pair_cluster"        CTA-pair kernel: CTA pairs per cluster that share every K/V tile by TMA
 *                         multicast (1, 2 or 4; 0 = automatic: the most that divides the stream-K
 *                         group without idling SMs)
 *   "overlap_short"       1 (default): hydra_attn's SM-partitioned schedule runs short GQA suffixes (g = 2/4/8,
 *                         S_cap <= 128, contiguous) on the short-suffix kernel, 3 CTAs per SM of the
 *                         suffix's share, and plans the split for it; 0: the persistent kernel
 *   "overlap_simt"        0 (default) automatic, 1 force, 2 never: hydra_attn's SM-partitioned schedule with
 *                         the SIMT suffix (MHA) as the prefix's programmatic dependent over its full grid,
 *                         the prefix on >= 32 persistent CTAs (taken when the prefix is light)
 *   "combine_pdl"         1 (default): hydra_attn's combine is a programmatic dependent of the suffix
 *                         kernel (waits for it at entry; -0.5 to -1 us per step); 0 a normal launch
 *   "seq_pdl"             1 (default): in the sequential schedule the tensor-core suffix is a
 *                         programmatic dependent launch of the prefix (starts in its tail); 0 off
 *   "step_timer"          measurement: device address of 4 x u64 the persistent prefix / suffix
 *                         kernels fill with their spans (%globaltimer ns: prefix start, end,
 *                         suffix start, end; preset UINT64_MAX, 0, UINT64_MAX, 0)
 *   "prefix_splits"       KV splits of the one-tile / SIMT prefix kernels
 *   "prefix_ctas"         CTAs of the persistent prefix kernel
 *   "suffix_impl"         1 SIMT split-K GEMV, 2 persistent TMA-fed tensor-core kernel, 3 the short-suffix
 *                         tensor-core kernel (g = 2/4/8, S_cap <= 256; 3 CTAs per SM; automatic for
 *                         S_cap <= 128)
 *   "suffix_splits"       KV splits of the suffix kernels (tensor-core kernel: split-K over
 *                         tokens, only when set; SIMT kernel: automatic when 0)
 *   "suffix_ctas"         CTAs of the persistent suffix kernel
 *   "suffix_cb"           tensor-core suffix: 128-token blocks per softmax round, 2 (default) or 1
 *   "suffix_unroll"       tokens in flight per row group of the SIMT suffix kernel (4 or 8)
 *   "overlap_prefix_ctas" SM split of hydra_attn with an aux stream (prefix CTAs)
 *   "prefix_stages"       K/V pipeline stages of the one-tile kernel (2 or 3)
 *   "fuse_combine"        hydra_attn's Eq. 5 merge: 0 (default) a separate combine launch; 1 in
 *                         the suffix kernel's epilogue in the sequential schedule; 2 also in the
 *                         SM-partitioned schedule (per-row arrival counters, the writer of a
 *                         row's last part merges it).  Same bits in every mode; 1 and 2 were
 *                         measured slower (profiles/r2_fuse_ab.jsonl)
 *   "ev_prefix_begin" / "ev_prefix_end" / "ev_suffix_begin" / "ev_suffix_end"
 *                         measurement: a cudaEvent_t (as an integer) that hydra_attn records
 *                         right before / after its prefix (on the prefix's stream) or suffix
 *                         launches, also inside graph capture; 0 = off
 * Testing build only (libhydra_test.so; the release library returns HYDRA_EINVAL for these):
 *   "tc_debug_variant"    timing experiments (invalid results)
 *   "prefix_trace" / "suffix_trace"  device buffer for CTA-0 timestamps (tools/)
 *   "inject_combine_bug"  1: the combine drops its rescaling (w_p = 1) -- the sabotage of S:522
 *   "mutate"              1: the persistent prefix kernel's CTA 0 skips one 4-row store group of
 *                         its epilogues; 2: the tensor-core suffix's (persistent or short) CTA 0
 *                         skips head 0's output row of its first item; 3: the CTA-pair prefix's
 *                         worker 0 skips 4 rows (unwritten rows the parity suite must catch)
 * hydra_get_config also answers "last_overlap_simt" (1 when that split ran the SIMT suffix as the
 * prefix's programmatic dependent over its full grid) and "last_overlap_k" (prefix CTAs of this thread's last hydra_attn /
 * hydra_tree_attn overlap split, 0 = sequential) and "testing_build" (1 in libhydra_test.so).
 * Returns HYDRA_EINVAL for an unknown key.
 */
HYDRA_API hydra_status hydra_set_config(const char *key, int64_t value);
HYDRA_API int64_t hydra_get_config(const char *key);

/* Testing build: number of lens[b] values outside [0, S_cap] the suffix launches have seen
 * since the last reset (synchronises the device; reset != 0 zeroes the count).  The release
 * build returns -1 (no device check; its kernels clamp). */
HYDRA_API int64_t hydra_debug_lens_violations(int32_t reset);

/* Message for the last non-OK status on this thread ("" if none). */
HYDRA_API const char *hydra_last_error(void);
HYDRA_API const char *hydra_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HYDRA_H_ */

// internal.h -- launch parameter blocks and launchers behind the C ABI (not exported).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hydra.h"

namespace hydra {

// Testing build (-DHYDRA_TESTING, libhydra_test.so): diagnostics (CTA timestamps), timing
// experiments that produce invalid results, and the parity suite's sabotage switches.  The
// release library compiles none of them: every use is guarded by this constant.
#ifdef HYDRA_TESTING
constexpr bool kTesting = true;
#else
constexpr bool kTesting = false;
#endif

// ---------------------------------------------------------------- host helpers (hostutil.cu)
bool tensor_maps_available();
// bf16 TMA tensor map, 128-B swizzle, dims innermost first; strides (bytes) of dims 1..rank-1.
bool encode_bf16_map(void *map, int rank, const void *base, const uint64_t *dims, const uint64_t *strides_bytes,
                     const uint32_t *box);
// cudaFuncAttributeMaxDynamicSharedMemorySize for `func` on the current device (cached per device).
cudaError_t ensure_smem_attr(const void *func, int bytes);
int device_sm_count();
// Testing build: count lens[b] outside [0, S_cap] on the device (no-op in release).
hydra_status launch_lens_check(const int32_t *lens, int64_t B, int64_t S_cap, cudaStream_t s);
int64_t read_lens_violations(bool reset);

// ---------------------------------------------------------------- fused Eq. 5 combine (fused.cuh)
// Per-row arrival counting: the epilogue that writes a row's last partial merges the row.
struct FusedCombine {
  int32_t *cnt;                 // [B*Hq] arrival counters (zero before the launches); null = not fused
  const float *o_pre, *lse_pre;  // prefix piece k of row r: o_pre + k*o_slot + r*128, lse_pre[k*lse_slot + r]
  const float *o_suf, *lse_suf;  // suffix part s of row r:  o_suf + s*o_slot + r*128, lse_suf[s*lse_slot + r]
  int64_t o_slot, lse_slot;
  int32_t n_suf;                // suffix parts per row (1, or the split count)
  // Prefix pieces covering a row's 256-row pair (persistent kernel, grouped stream-K plan) or
  // the fixed split count (one-tile kernel, sk_total == 0).
  int64_t sk_total;
  int32_t sk_G, sk_group, sk_nb, sk_npairs, n_pre_splits;
  int32_t g, Hq, Hkv;
  void *out;                    // [B*Hq, 128] bf16 (out_f32 = 0) or f32
  int32_t out_f32;
  float *lse_out;               // [B*Hq] merged LSE (nullable)
  int32_t inject_bug;           // testing build only: w_p = 1
  // 1: the prefix kernel completed before the suffix launch (same stream, sequential schedule):
  // the prefix neither counts nor merges, the suffix parts alone are counted (expected = n_suf),
  // and with one suffix part its writer merges at once -- no atomics, no counter reset
  int32_t pre_done;
};

// ---------------------------------------------------------------- SIMT decode kernel
// One CTA = one (sequence-slot b, KV head j, head chunk, KV split).  Used for the
// suffix (§3.2), the fp32 reference-mode prefix / tree nodes, and odd shapes.
struct DecodeParams {
  const void *q;
  int64_t q_sb, q_sh;
  const void *k, *v;
  int64_t kv_sb, kv_st, kv_sh;  // kv_sb == 0: every sequence reads the same KV (shared prefix)
  int64_t kv_tok_off;           // token offset added to every position (tree node offset)
  const int32_t *lens;          // device [n_seq]; nullptr -> len_uniform for every sequence
  int64_t len_cap;              // lens[b] is clamped to [0, len_cap] (hydra.h precondition)
  int64_t len_uniform;
  const int32_t *seq_map;       // device [n_seq] slot -> sequence id; nullptr -> identity
  int32_t n_seq, Hq, Hkv, g;
  float scale_log2;             // softmax scale * log2(e)
  int32_t n_splits;
  int64_t split_len;            // tokens per split
  int32_t heads_per_cta;        // GQ: query heads of one KV group handled per CTA
  int32_t unroll;               // tokens in flight per row group (4 or 8; 0 -> 4)
  float *o;                     // [split][B][Hq][d] partial outputs (fp32, normalised)
  float *lse;                   // [split][B][Hq] natural-log LSE
  int64_t o_split_stride, lse_split_stride;
  // Paged suffix cache (hydra_paging): when block_table != nullptr, token t of sequence b is
  // at k + block_table[b * bt_stride + (t >> page_shift)] * kv_sb + (t & page_mask) * kv_st
  // (kv_sb is then the page stride of the pool).
  const int32_t *block_table;
  int64_t bt_stride;
  int32_t page_shift;
  FusedCombine fc;  // fc.cnt != null: merge each completed row in the epilogue (d = 128, bf16 suffix only)
  int32_t pdl;      // host only: programmatic dependent of the previous kernel in the stream (its last CTA
                    // ends with griddepcontrol.wait, so its completion implies the predecessor's)
  unsigned long long *timer = nullptr;  // measurement: [0] first CTA's start, [1] max end over the last
                                        // 1024 CTAs in launch order (%globaltimer ns); null = off
};

hydra_status launch_decode(const DecodeParams &p, hydra_dtype dt, int d, cudaStream_t s);

// ---------------------------------------------------------------- combine
// Two part groups: A (o_dtype: f32 or f16) and B (f32, may be empty); strides in elements.
struct CombineParams {
  int64_t rows;
  int32_t d;
  int32_t n_a;
  const void *o_a;
  int64_t o_a_part, o_a_row;
  const float *l_a;
  int64_t l_a_part, l_a_row;
  int32_t n_b;
  const float *o_b;
  int64_t o_b_part, o_b_row;
  const float *l_b;
  int64_t l_b_part, l_b_row;
  void *out;
  int64_t out_row;
  float *lse_out;
  int64_t lse_out_row;
  // scattered output (table_rows > 0): row r goes to table [r / table_rows], row r % table_rows
  // (out_row / lse_out_row strides) -- e.g. straight into other GPUs' receive buffers
  void *const *out_table;
  float *const *lse_out_table;
  int64_t table_rows;
  int32_t inject_bug;  // testing build only: w_p = 1 (the sabotage of S:522)
  int32_t pdl;         // host only: programmatic dependent of the previous kernel (it waits for that grid at entry)
};
hydra_status launch_combine(const CombineParams &p, hydra_dtype o_dtype, hydra_dtype out_dtype,
                            cudaStream_t s);
// Fill lse[i] = -inf for i < n (marks empty partial slots).
hydra_status launch_fill_neg_inf(float *lse, int64_t n, cudaStream_t s);

// ---------------------------------------------------------------- tcgen05 prefix kernel
// A work item of the tensor-core prefix kernel: one KV segment (flat prefix or a
// tree node) and the list of sequences whose stacked queries attend to it.
struct PrefixTask {
  int64_t kv_off;    // first token of the segment in the pooled K/V
  int64_t kv_len;    // tokens in the segment
  int32_t seq_off;   // offset into the sequence list
  int32_t n_seq;     // sequences in the group
  int32_t depth;     // tree depth of the segment: its partials go to slot depth * n_splits + split
  int32_t tile;      // query tile index within the group (128 stacked rows each)
};

struct PrefixTcArgs {
  const void *q;
  int64_t q_sb, q_sh;
  const void *k, *v;      // pooled [T, Hkv, 128] bf16
  int64_t kv_st, kv_sh;
  int64_t kv_total;       // T (tokens addressable by the tensor maps)
  int32_t Hq, Hkv, g;
  float scale_log2;
  // flat mode (tasks == nullptr): one segment [0, P) for B sequences
  int64_t P;
  int32_t B;
  // task mode
  const PrefixTask *tasks;   // device
  int32_t n_tasks;
  const int32_t *seq_list;   // device
  int32_t n_splits;
  float *o, *lse;
  int64_t o_slot_stride, lse_slot_stride;
  int32_t debug_variant;
  void *trace = nullptr;  // diagnostics only (config key prefix_trace): device buffer for CTA-0 timestamps
  int32_t mutate = 0;     // testing build only: parity-suite mutation (prefix_tc2 epilogue store skip)
  FusedCombine fc{};      // fc.cnt != null: fused Eq. 5 merge in the epilogue (flat mode)
  int32_t poly_every = 0;  // v3: every k-th exp2 column pair on the FMA pipe (0 = all MUFU)
  int32_t variant = 3;     // persistent kernel: 3 (128-token blocks) or 4 (64-token, double-buffered S)
  int32_t stages;  // K/V pipeline stages: 2 (160 KB smem, leaves room for co-resident suffix CTAs) or 3
  unsigned long long *timer = nullptr;  // measurement: [0] min CTA start, [1] max CTA end (ns); persistent kernels
  int32_t pair_cluster = 0;  // CTA-pair kernel: pairs per cluster (0 = automatic)
  int32_t pair_poly = 0;     // CTA-pair kernel: every k-th exp2 pair on the FMA pipe (0 = all MUFU)
  int32_t pair_item_cost = 0;  // CTA-pair kernel: stream-K boundaries balance blocks + this x items (0 = uniform)
};
bool prefix_tc_supported(const hydra_heads *h);
hydra_status launch_prefix_tc(const PrefixTcArgs &a, cudaStream_t s);
// v3: persistent, two 128-row query tiles per CTA; flat mode is stream-K over n_ctas CTAs
// (partial slots per row = prefix_tc2_slots), task mode deals (task, head, split) items.
hydra_status launch_prefix_tc2(const PrefixTcArgs &a, int n_ctas, cudaStream_t s);
int prefix_tc2_slots(int64_t B, int g, int Hkv, int64_t P, int n_ctas, int bn, bool pair = false, int pair_cluster = 0,
                     int pair_item_cost = 0);
int prefix_tc2_ctas(int64_t B, int g, int Hkv, int64_t P, int n_ctas, int bn, bool pair = false, int pair_cluster = 0);
// The flat-mode stream-K plan of launch_prefix_tc2 over n_ctas CTAs, as the fused combine
// needs it (which partial slots hold a row's pieces): fills fc.sk_*.
void prefix_tc2_plan_into(FusedCombine &fc, int64_t B, int g, int Hkv, int64_t P, int n_ctas, int bn);
// CTA-pair (cta_group::2) persistent prefix kernel, flat mode, 128 % g == 0 (prefix_pair.cu):
// same grouped stream-K plan as launch_prefix_tc2 with a CTA pair as the worker.
struct PairPlan {
  int group, workers, ctas;
  int cluster;  // CTA pairs per cluster (1, 2, 4): they share every K/V tile by TMA multicast
  int64_t total;
};
bool prefix_pair_supported(int g);
// forced_cluster: 0 = automatic, 1 / 2 / 4 = pairs per cluster (config key pair_cluster)
PairPlan prefix_pair_plan(int64_t B, int g, int Hkv, int64_t P, int n_ctas, int forced_cluster = 0);
int prefix_pair_slots(int64_t B, int g, int Hkv, int64_t P, int n_ctas, int forced_cluster = 0, int item_cost = 0);
hydra_status launch_prefix_pair(const PrefixTcArgs &a, int n_ctas, cudaStream_t s);
// Persistent tensor-core suffix kernel (bf16, d = 128, g <= 16), TMA-fed.
struct SuffixTcArgs {
  const void *q;
  int64_t q_sb, q_sh;
  const void *k, *v;
  int64_t s_sb, s_st, s_sh, S_cap;
  const int32_t *lens;
  int32_t B, Hq, Hkv;
  float scale_log2;
  float *o, *lse;  // [B, Hq, 128], [B, Hq]
  int32_t cb;      // 128-token blocks per softmax round (1 or 2)
  void *trace;     // diagnostics (suffix_trace config key); null = off
  int32_t debug;   // tc_debug_variant (timing experiments only, testing build)
  int32_t mutate;  // testing build only: 2 = CTA 0's epilogue skips head 0's store of its first item
  // paged cache (block_table != nullptr): k/v are page pools [n_pages, page_size, Hkv, 128]
  // with s_sb = page stride; S_cap = bt_stride * page_size
  const int32_t *block_table;
  int64_t bt_stride, n_pages;
  int32_t page_size;
  // split-K over tokens (0 / 1 = none): split sp of a sequence covers tokens
  // [sp * split_len, (sp + 1) * split_len) (split_len a multiple of 128) and writes its
  // (O, LSE) partial at o + sp * o_split_stride, lse + sp * lse_split_stride
  int32_t n_split, split_len;
  int64_t o_split_stride, lse_split_stride;
  FusedCombine fc;  // fc.cnt != null: fused Eq. 5 merge in the epilogue
  int32_t pdl = 0;  // 1: programmatic dependent of the previous kernel in the stream (SM-partitioned schedule)
  unsigned long long *timer = nullptr;  // measurement: [0] min CTA start, [1] max CTA end (ns)
};
bool suffix_tc_supported(const hydra_heads *h);
hydra_status launch_suffix_tc(const SuffixTcArgs &a, int n_ctas, cudaStream_t s);
// short grouped-query suffixes (S_cap <= 256, g in {2, 4, 8, 16}, contiguous, unsplit, unfused):
// three small CTAs per SM (suffix_short.cu); n_ctas 0 = 3 x SMs
bool suffix_short_supported(int g, int64_t S_cap);
hydra_status launch_suffix_short(const SuffixTcArgs &a, int n_ctas, cudaStream_t s);
hydra_status launch_append_kv(const void *k_new, const void *v_new, int64_t nb, int64_t nh, void *sk, void *sv,
                              int64_t s_sb, int64_t s_st, int64_t s_sh, int64_t S_cap, int32_t Hkv, int32_t d,
                              size_t es, int64_t B, int32_t *lens, cudaStream_t s,
                              const int32_t *block_table = nullptr, int64_t bt_stride = 0, int32_t page_size = 0);

}  // namespace hydra

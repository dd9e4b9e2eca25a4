// capi.cu -- the exported C ABI of libhydra.so (declared in include/hydra.h).
//
// Host-side argument validation, work decomposition (KV splits), workspace layout
// and stream orchestration of the prefix / suffix / combine kernels.  No device
// allocation and no host<->device synchronisation on any hot-path entry point.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

using namespace hydra;

// ------------------------------------------------------------------ errors / config
static thread_local std::string g_last_error;

static hydra_status fail(hydra_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

static hydra_status cuda_fail(const char *what) {
  cudaError_t e = cudaGetLastError();
  return fail(HYDRA_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Settings of the calling thread (hydra_set_config).  Thread-local, so calls made by
// different threads never see each other's switches or measurement events (hydra.h:
// "reentrant"); a thread that never calls hydra_set_config runs the automatic choices.
struct Config {
  int64_t prefix_impl = 0, prefix_splits = 0, prefix_ctas = 0, prefix_stages = 3, prefix_poly = 4, prefix_variant = 9;
  int64_t suffix_impl = 0, suffix_splits = 0, suffix_ctas = 0, suffix_unroll = 4, suffix_cb = 2;
  int64_t overlap_prefix_ctas = 0;
  // measurement: device pointer to 4 x u64 that hydra_attn's persistent prefix / tensor-core suffix
  // kernels fill with [prefix min CTA start, prefix max CTA end, suffix start, suffix end]
  // (%globaltimer ns, atomicMin / atomicMax: the caller presets UINT64_MAX, 0, UINT64_MAX, 0)
  int64_t step_timer = 0;
  // 1: the sequential schedule launches the suffix as a programmatic dependent of the prefix
  int64_t seq_pdl = 1;
  int64_t combine_pdl = 1;  // -0.5 to -1 us per step (C6 / C4 / C2, profiles/r3p_combine_pdl_ab.jsonl)
  int64_t overlap_short = 1;  // SM-partitioned schedule: the short-suffix kernel on the suffix's SM share  // hydra_attn's combine as a programmatic dependent of the suffix kernel
  int64_t overlap_simt = 0;  // 0 auto, 1 force, 2 never: the SIMT-dependent overlap schedule (overlap_prefix_ctas)
  // CTA-pair prefix kernel: pairs per cluster sharing K/V tiles by multicast (0 auto, 1, 2, 4)
  int64_t pair_cluster = 0;
  int64_t pair_poly = 0;  // all exponentials on the MUFU: measured faster than 4 on the pair kernel (issue/latency-bound)
  int64_t pair_item_cost = 0;  // stream-K group boundaries balance blocks + this x items (0 = uniform; measured no gain)
  // Eq. 5 merged in the kernel epilogues (fused.cuh): 1 in the sequential schedule only (the
  // suffix merges each row after the prefix kernel), 2 also in the SM-partitioned schedule
  // (arrival counters), 0 never: a separate combine launch (default).  Measured
  // (tools/fuse_ab.py, profiles/r2_fuse_ab.jsonl): the epilogue merges serialise a memory
  // round trip per row behind each item -- C3@16K 0.93 (1) / 3.93 (2) vs 0.96 ms overlapped,
  // 1.12 vs 1.06 sequential; C4 0.82 vs 0.30 ms; C6 0.28 vs 0.12 ms.
  int64_t fuse_combine = 0;
  // Measurement: cudaEvent_t handles hydra_attn / hydra_attn_paged record around the prefix (on
  // its stream) and the suffix launches, so a benchmark can time each kernel within the step
  // (also inside a captured graph); 0 = off.  [0] prefix begin, [1] prefix end, [2] suffix
  // begin, [3] suffix end.
  int64_t step_ev[4] = {0, 0, 0, 0};
  // testing build only (libhydra_test.so): timing experiments, diagnostics, sabotage
  int64_t tc_debug = 0, prefix_trace = 0, suffix_trace = 0, inject_combine_bug = 0, mutate = 0;
  int64_t last_overlap_k = 0;  // read-only: prefix CTAs of this thread's last overlap split (0 = sequential)
  int64_t last_overlap_simt = 0;  // read-only: 1 when that split ran the SIMT suffix as the prefix's dependent
};
static thread_local Config g_cfg;
static const char *kStepEvKeys[4] = {"ev_prefix_begin", "ev_prefix_end", "ev_suffix_begin", "ev_suffix_end"};

static void record_step_ev(int i, cudaStream_t s) {
  const int64_t e = g_cfg.step_ev[i];
  // External: under stream capture the record becomes an observable event-record node (an
  // internal record would only be a capture dependency and could not be timed)
  if (!e) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  cudaEvent_t ev = reinterpret_cast<cudaEvent_t>((intptr_t)e);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
  else
    cudaEventRecord(ev, s);
  (void)cudaGetLastError();  // a failed measurement record must not surface as a launch error
}

namespace {
struct Key {
  const char *name;
  int64_t Config::*field;
  bool testing_only;
};
const Key kKeys[] = {
    {"prefix_impl", &Config::prefix_impl, false},         {"prefix_splits", &Config::prefix_splits, false},
    {"prefix_ctas", &Config::prefix_ctas, false},         {"prefix_stages", &Config::prefix_stages, false},
    {"prefix_poly", &Config::prefix_poly, false},         {"prefix_variant", &Config::prefix_variant, false},
    {"suffix_impl", &Config::suffix_impl, false},         {"suffix_splits", &Config::suffix_splits, false},
    {"suffix_ctas", &Config::suffix_ctas, false},         {"suffix_unroll", &Config::suffix_unroll, false},
    {"suffix_cb", &Config::suffix_cb, false},             {"overlap_prefix_ctas", &Config::overlap_prefix_ctas, false},
    {"step_timer", &Config::step_timer, false},          {"seq_pdl", &Config::seq_pdl, false},
    {"overlap_simt", &Config::overlap_simt, false},
    {"combine_pdl", &Config::combine_pdl, false},
    {"overlap_short", &Config::overlap_short, false},
    {"pair_cluster", &Config::pair_cluster, false},
    {"pair_poly", &Config::pair_poly, false},
    {"pair_item_cost", &Config::pair_item_cost, false},
    {"fuse_combine", &Config::fuse_combine, false},
    {"tc_debug_variant", &Config::tc_debug, true},        {"prefix_trace", &Config::prefix_trace, true},
    {"suffix_trace", &Config::suffix_trace, true},        {"inject_combine_bug", &Config::inject_combine_bug, true},
    {"mutate", &Config::mutate, true},
};
}  // namespace

extern "C" hydra_status hydra_set_config(const char *key, int64_t value) {
  if (!key) return fail(HYDRA_EINVAL, "null key");
  for (int i = 0; i < 4; ++i)
    if (!strcmp(key, kStepEvKeys[i])) {
      g_cfg.step_ev[i] = value;
      return HYDRA_OK;
    }
  for (const Key &k : kKeys) {
    if (strcmp(key, k.name)) continue;
    if (k.testing_only && !kTesting)
      return fail(HYDRA_EINVAL, "config key '%s' exists only in the testing build (libhydra_test.so)", key);
    int64_t v = value;
    if (!strcmp(key, "prefix_poly")) v = (v == 0 || v == 3 || v == 4 || v == 8 || (kTesting && (v == -1 || v == 2))) ? v : 4;
    if (!strcmp(key, "pair_cluster")) v = (v == 1 || v == 2 || v == 4) ? v : 0;
    if (!strcmp(key, "pair_poly")) v = (v == 4 || (kTesting && (v == 2 || v == 3))) ? v : 0;
    if (!strcmp(key, "pair_item_cost")) v = std::max<int64_t>(0, std::min<int64_t>(v, 64));
    if (!strcmp(key, "prefix_variant")) v = (v == 3 || v == 4 || v == 5 || v == 6) ? v : 9;
    if (!strcmp(key, "prefix_stages")) v = (v == 2 ? 2 : 3);
    if (!strcmp(key, "suffix_cb")) v = (v == 1 ? 1 : 2);
    if (!strcmp(key, "suffix_unroll")) v = (v >= 8 ? 8 : v >= 4 ? 4 : 2);
    g_cfg.*(k.field) = v;
    return HYDRA_OK;
  }
  return fail(HYDRA_EINVAL, "unknown config key '%s'", key);
}

extern "C" int64_t hydra_get_config(const char *key) {
  if (!key) return -1;
  if (!strcmp(key, "last_overlap_k")) return g_cfg.last_overlap_k;
  if (!strcmp(key, "last_overlap_simt")) return g_cfg.last_overlap_simt;
  if (!strcmp(key, "testing_build")) return kTesting ? 1 : 0;
  // resident CTAs of the CTA-pair kernel in clusters of 1 / 2 / 4 pairs (2 x pairs, 1024 x 4 groups)
  if (!strcmp(key, "pair_max_ctas")) return prefix_pair_plan(1024, 1, 1, 1 << 20, 1 << 20, 1).ctas;
  if (!strcmp(key, "pair_max_ctas_c2")) return prefix_pair_plan(1024, 1, 1, 1 << 20, 1 << 20, 2).ctas;
  if (!strcmp(key, "pair_max_ctas_c4")) return prefix_pair_plan(1024, 1, 1, 1 << 20, 1 << 20, 4).ctas;
  for (int i = 0; i < 4; ++i)
    if (!strcmp(key, kStepEvKeys[i])) return g_cfg.step_ev[i];
  for (const Key &k : kKeys)
    if (!strcmp(key, k.name)) return (k.testing_only && !kTesting) ? -1 : g_cfg.*(k.field);
  return -1;
}

extern "C" const char *hydra_last_error(void) { return g_last_error.c_str(); }
extern "C" const char *hydra_version(void) {
  return kTesting ? "hydra-b200 0.2.0 (sm_100a, testing build)" : "hydra-b200 0.2.0 (sm_100a)";
}
extern "C" int64_t hydra_debug_lens_violations(int32_t reset) { return read_lens_violations(reset != 0); }

static bool inject_combine_bug() { return kTesting && g_cfg.inject_combine_bug != 0; }

// ------------------------------------------------------------------ validation helpers
static size_t elem_size(hydra_dtype d) { return d == HYDRA_F32 ? 4 : 2; }

static hydra_status check_heads(const hydra_heads *h) {
  if (!h) return fail(HYDRA_EINVAL, "heads is NULL");
  if (h->num_q_heads <= 0 || h->num_kv_heads <= 0)
    return fail(HYDRA_ESHAPE, "head counts must be positive (Hq=%d, Hkv=%d)", h->num_q_heads, h->num_kv_heads);
  if (h->num_q_heads % h->num_kv_heads)
    return fail(HYDRA_ESHAPE, "Hq %% Hkv != 0 (Hq=%d, Hkv=%d)", h->num_q_heads, h->num_kv_heads);
  if (h->dtype != HYDRA_BF16 && h->dtype != HYDRA_F32) return fail(HYDRA_EUNSUPPORTED, "dtype must be BF16 or F32");
  const int d = h->head_dim;
  const bool ok = (d == 16 || d == 32 || d == 64 || d == 128) || (d == 256 && h->dtype == HYDRA_BF16);
  if (!ok) return fail(HYDRA_EUNSUPPORTED, "head_dim %d unsupported for this dtype", d);
  if (!(h->scale >= 0.f) || std::isinf(h->scale)) return fail(HYDRA_EINVAL, "scale must be finite and >= 0");
  return HYDRA_OK;
}

static float scale_of(const hydra_heads *h) { return h->scale > 0.f ? h->scale : 1.0f / sqrtf((float)h->head_dim); }

// 16-byte vector loads need 16-B aligned rows: base and every stride a multiple of 16 B.
static bool aligned16(const void *p, size_t es, std::initializer_list<int64_t> strides) {
  if (reinterpret_cast<uintptr_t>(p) % 16) return false;
  for (int64_t s : strides)
    if ((s * (int64_t)es) % 16) return false;
  return true;
}

static int heads_per_cta(int g) {
  for (int c : {8, 4, 2, 1})
    if (g % c == 0) return c;
  return 1;
}

// ------------------------------------------------------------------ work decomposition
// Suffix kernel choice: the persistent tensor-core kernel (one item per (sequence, KV
// head), TMA-fed) when there are enough items to keep every CTA busy; otherwise the SIMT
// split-K kernel, which can split one sequence's tokens across CTAs.
// On the full chip the SIMT kernel streams slightly faster (7.2 vs 7.0 TB/s at C3), so
// `auto` uses the tensor-core kernel only for the SM-partitioned (overlapped) schedule,
// where its low instruction count per byte lets a subset of SMs carry the suffix.
// With GQA (g >= 2) the tensor-core kernel is also the faster one on the full chip: it reads
// each K/V row once for all g heads of the group (N = 16 MMA), where the SIMT kernel holds g
// query heads and accumulators in registers (2 CTAs/SM at g = 8).  Measured on B200
// (tools/suffix_shapes.py, L2 flushed): g = 8, B = 256, S = 128: 28 vs 66-117 us; g = 4,
// B = 512: 67 vs 96 us; g = 16: 108 vs 357-410 us; MHA (g = 1): 0.83 vs 0.79 ms at C3.
// The short-suffix kernel where it is chosen automatically: one-block items (S_cap <= 128).  With
// two-block items the persistent kernel's 2-block rounds measured faster on some shapes (tools/
// suffix_span.py, profiles/r4a_suffix_short_vs_tc.jsonl: 64 x 8 kv heads x 256 tokens 13.1 vs
// 16.5 us, 128 x 8 x 256 21.7 vs 24.6 us) while one-block items favour the short kernel (1024 x 8 x
// 64: 64.6 vs 89.0 us; 2048 x 4 x 128: 88.7 vs 102.5 us).  suffix_impl 3 forces it up to 256.
static bool short_auto(int g, int64_t S_cap) { return suffix_short_supported(g, S_cap) && S_cap <= 128; }

static bool use_suffix_tc(const hydra_heads *h, int64_t B, int64_t S_cap, bool overlap = false) {
  if (g_cfg.suffix_impl == 1 || S_cap <= 0 || !suffix_tc_supported(h)) return false;
  if (g_cfg.suffix_impl == 2 || g_cfg.suffix_impl == 3) return true;
  const int64_t items = B * h->num_kv_heads, sms = device_sm_count();
  if (overlap) return items >= 2 * sms;
  // (also with fewer items than SMs: 64-128 items of 1-8K-token suffixes, 62-64 us against
  // 106-210 us for the SIMT kernel's best split)
  return h->num_q_heads / h->num_kv_heads >= 2;
}

// Tensor-core suffix time model (us) on n SMs: HBM streaming at R_S bytes/us per SM (capped
// by BW), or the per-item floor -- pipeline fill plus a per-item cost that grows with the
// tiles and the heads of an item (tools/suffix_shapes.py: g = 8 one-tile items ~2.5 us at
// 7 items per CTA; the floor stays below the streaming term for C3's MHA two-tile items, so
// C3's split is the streaming model's).
static double suffix_tc_us(const hydra_heads *h, int64_t B, int64_t S_cap, int n, double R_S, double BW) {
  const int g = h->num_q_heads / h->num_kv_heads;
  const int64_t items = B * h->num_kv_heads;
  const double bytes = (double)items * S_cap * h->head_dim * 4.0;
  const double per_item = 0.45 * (double)((S_cap + 127) / 128) + 0.25 * g;
  return std::max(bytes / std::min(n * R_S, BW), 10.0 + (double)((items + n - 1) / n) * per_item);
}

// KV splits of the suffix kernel: enough CTAs to keep every SM streaming
// (~16 resident 128-thread CTAs per SM), never fewer than 32 tokens per split.
static int suffix_splits(const hydra_heads *h, int64_t B, int64_t S_cap, bool overlap = false) {
  if (use_suffix_tc(h, B, S_cap, overlap)) {
    // Tensor-core kernel: split-K over tokens only on request (config key suffix_splits).
    // Measured (tools/suffix_shapes.py): an automatic split that fills the last wave (512
    // items on 148 SMs, 2048-token suffixes -> 2 splits) was 11 % slower (114 vs 103 us;
    // 64 x 8 heads x 1024 tokens: 68 vs 60 us) -- the kernel streams ~40 GB/s per SM there,
    // so the extra items' fill / epilogue and the partial combine cost more than the tail.
    if (overlap) return 1;
    if (g_cfg.suffix_splits > 0) return (int)std::min<int64_t>(g_cfg.suffix_splits, std::max<int64_t>(1, (S_cap + 127) / 128));
    // Very few items (< SMs / 4, e.g. 4 sequences x 8 KV heads): split into one wave of
    // items x splits <= SMs (32 items x 16K tokens: 64.5 us with 4 splits, 74 with 5 = two
    // waves, 91 unsplit); at 64+ items the split measured slower.
    const int64_t items = B * h->num_kv_heads, sms = device_sm_count();
    if (items * 4 >= sms) return 1;
    return (int)std::max<int64_t>(1, std::min<int64_t>({sms / items, S_cap / 512, 16}));  // one wave
  }
  if (g_cfg.suffix_splits > 0) return (int)std::min<int64_t>(g_cfg.suffix_splits, std::max<int64_t>(1, S_cap));
  if (S_cap <= 0) return 1;
  const int g = h->num_q_heads / h->num_kv_heads;
  const int64_t items = B * h->num_kv_heads * (g / heads_per_cta(g));
  // ~6 resident 128-thread CTAs per SM and >= 256 tokens per split (tools/suffix_shapes.py:
  // MHA 2-16 sequences x 32-40 heads x 0.5-16K tokens; 16 per SM and 32-token splits were
  // 10-18 % slower through the extra partials and the combine)
  const int64_t target = (int64_t)device_sm_count() * 6;
  int64_t s = (target + items - 1) / items;
  s = std::min<int64_t>(s, std::max<int64_t>(1, S_cap / 256));
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, 64));
}

// Prefix kernel choice: the persistent two-tile tcgen05 kernel (v3) by default; the
// one-tile tcgen05 kernel (v1) or the SIMT kernel on request / for unsupported shapes.
enum PrefixKind { PK_SIMT = 1, PK_TC1 = 2, PK_TC2 = 3 };
static int prefix_ctas() { return g_cfg.prefix_ctas > 0 ? (int)g_cfg.prefix_ctas : device_sm_count(); }
static int prefix_bn() { return g_cfg.prefix_variant == 4 ? 64 : 128; }  // KV tokens per persistent-kernel block
// flat mode of the persistent prefix kernel on CTA pairs (variant 9, prefix_pair.cu)
static bool pair_mode(int g) { return g_cfg.prefix_variant == 9 && prefix_pair_supported(g); }
// B/P-dependent choice (rows = stacked query rows per KV head, P = KV tokens per row):
// the persistent kernel amortises its per-segment Q load / epilogue only when every CTA
// owns enough 128-token blocks; small problems run the one-tile kernel (more parallelism).
// ctas: the persistent kernel's CTA count (0 = all SMs, or the prefix_ctas override).
static PrefixKind prefix_kind(const hydra_heads *h, int64_t rows = -1, int64_t P = -1, int ctas = 0) {
  if (g_cfg.prefix_impl == 1 || !prefix_tc_supported(h)) return PK_SIMT;
  if (g_cfg.prefix_impl == 2) return PK_TC1;
  if (g_cfg.prefix_impl == 3 || rows < 0) return PK_TC2;
  // Persistent kernel when each CTA owns enough 256-row x 128-token blocks to amortise its
  // pipeline fill: 24 on an SM share (the overlap split needs the persistent kernel), 40 on
  // the full chip (tools/prefix_shapes.py: C6 at 34 blocks per CTA, one-tile kernel 104 us vs
  // 108 us; C4 at 110 blocks, persistent 266 vs 312 us).
  // The CTA-pair kernel (one worker = 2 CTAs) keeps its pipeline full at fewer blocks: from 16
  // per worker (tools/prefix_ab.py: C6, 67 per worker, 0.084 ms vs 0.097 one-tile; C2, 7 per
  // worker, 0.031 vs 0.024 one-tile).
  const int64_t blocks = ((rows + 255) / 256) * h->num_kv_heads * ((P + 127) / 128);
  const int64_t n = ctas > 0 ? ctas : prefix_ctas();
  if (pair_mode((int)(h->num_q_heads / h->num_kv_heads))) return blocks >= 8 * n ? PK_TC2 : PK_TC1;
  return blocks >= (ctas > 0 ? 24 : 40) * n ? PK_TC2 : PK_TC1;
}
static bool use_tc(const hydra_heads *h) { return prefix_kind(h) != PK_SIMT; }

// Splits of the tensor-core prefix kernel: minimise (waves x blocks per CTA) plus the
// HBM cost of writing/reading the extra fp32 partials, in units of one KV block.
static int prefix_splits_tc(int64_t tiles, int64_t P) {
  if (g_cfg.prefix_splits > 0) return (int)g_cfg.prefix_splits;
  const int64_t nblk = (P + 127) / 128;
  if (nblk <= 1) return 1;
  const int64_t sms = device_sm_count();
  double best = 1e300;
  int best_s = 1;
  for (int s = 1; s <= std::min<int64_t>(nblk, 32); ++s) {
    const double waves = std::ceil((double)tiles * s / sms);
    const double per = std::ceil((double)nblk / s);
    // one block ~ 0.6 us per wave; one extra split moves tiles*128 rows*1 KB (~0.16 us/tile/148)
    const double cost = waves * per * 0.6 + (s - 1) * tiles * 128.0 * 1032.0 / 6.5e3 / 1e3;
    if (cost < best - 1e-9) {
      best = cost;
      best_s = s;
    }
  }
  return best_s;
}

static int prefix_splits_simt(const hydra_heads *h, int64_t B, int64_t P) {
  if (g_cfg.prefix_splits > 0) return (int)g_cfg.prefix_splits;
  if (P <= 0) return 1;
  const int g = h->num_q_heads / h->num_kv_heads;
  const int64_t items = B * h->num_kv_heads * (g / heads_per_cta(g));
  const int64_t target = (int64_t)device_sm_count() * 16;
  int64_t s = (target + items - 1) / items;
  s = std::min<int64_t>(s, std::max<int64_t>(1, P / 64));
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, 64));
}

// Number of partial (O, LSE) slots per row the prefix kernel writes.
static int prefix_splits(const hydra_heads *h, int64_t B, int64_t P, int tc2_ctas = 0) {
  if (P <= 0) return 1;
  const int g = h->num_q_heads / h->num_kv_heads;
  switch (prefix_kind(h, B * g, P, tc2_ctas)) {
    case PK_TC2:
      return prefix_tc2_slots(B, g, h->num_kv_heads, P, tc2_ctas > 0 ? tc2_ctas : prefix_ctas(), prefix_bn(),
                              pair_mode(g), (int)g_cfg.pair_cluster, (int)g_cfg.pair_item_cost);
    case PK_TC1:
      return prefix_splits_tc(((B * g + 127) / 128) * h->num_kv_heads, P);
    default:
      return prefix_splits_simt(h, B, P);
  }
}

// SM split for running the persistent prefix (tensor-bound) and suffix (HBM-bound)
// kernels concurrently.  k prefix CTAs balance the two finish times:
//   t_prefix(k) = pair_blocks / (k * R_P),  t_suffix(k) = kv_bytes / min((SMs-k) * R_S, BW)
// with per-SM rates measured on B200 at C3@16K, each kernel alone on its SM share
// (tools/overlap_var.py, tools/overlap_sweep.py): R_P = 256-row x 128-token blocks per us
// per SM (0.46 at 48-64 SMs), R_S = suffix bytes per us per SM (100 KB/us at 64 SMs for
// the two-issuer tensor-core suffix, 7.0 TB/s at 80-92 SMs), BW = HBM read ceiling.
// Candidates are multiples of the prefix plan's group size so no SM is left idle; on ties
// (suffix-bound) the smallest k wins.  Measured at C3@16K: k = 56-60 best (0.86 ms).
// 0 = no overlap.
static int overlap_prefix_ctas(const hydra_heads *h, int64_t B, int64_t P, int64_t S_cap, bool *simt = nullptr,
                               bool paged = false) {
  if (simt) *simt = false;
  if (P <= 0 || S_cap <= 0) return 0;
  const int g = h->num_q_heads / h->num_kv_heads;
  // SIMT-dependent overlap: where the sequential schedule's suffix is the SIMT kernel (MHA) and
  // the prefix is light, the prefix runs on a few persistent CTAs (>= 32, the plan's nearest
  // valid count) and the SIMT suffix is its programmatic dependent with its full grid: its CTAs
  // stream on every other SM from the start and spread to all SMs as the prefix ends (only its
  // last CTA waits for the prefix grid, decode.cu).  Taken when the prefix on those CTAs
  // (model rate R_P below) needs at most 0.6x the suffix's full-chip streaming time.  Measured
  // (tools/config_ab.py, profiles/r2s_simt.jsonl): C2 0.104 -> 0.092 ms, C3@1K 0.804 -> 0.788;
  // C3@16K keeps the tensor-core split (prefix too heavy: 0.96 ms this way vs 0.91-0.95).
  if (g_cfg.overlap_simt != 2 && simt && !use_suffix_tc(h, B, S_cap, false) && prefix_kind(h, B * g, P, 8) == PK_TC2) {
    const int sms = device_sm_count();
    int k = 0;
    const int k0 = g_cfg.overlap_prefix_ctas > 0 ? (int)g_cfg.overlap_prefix_ctas : 32;
    for (int c = k0; c <= sms / 2 && !k; ++c)
      if (prefix_kind(h, B * g, P, c) == PK_TC2 &&
          prefix_tc2_ctas(B, g, h->num_kv_heads, P, c, prefix_bn(), pair_mode(g), (int)g_cfg.pair_cluster) == c)
        k = c;
    if (k > 0) {
      const double R_P = pair_mode(g) ? 0.42 : 0.38, BW = 7.0e6;
      const double pair_blocks = (double)((B * g + 255) / 256) * h->num_kv_heads * ((P + 127) / 128);
      const double bytes = (double)B * h->num_kv_heads * S_cap * h->head_dim * 4.0;
      if (g_cfg.overlap_simt == 1 || pair_blocks / (k * R_P) <= 0.6 * bytes / BW) {
        *simt = true;
        return k;
      }
    }
  }
  if (!use_suffix_tc(h, B, S_cap, true)) return 0;
  if (prefix_kind(h, B * g, P, 8) != PK_TC2) return 0;  // not even 8 persistent CTAs' worth of blocks
  const int sms = device_sm_count();
  if (g_cfg.overlap_prefix_ctas > 0) return (int)std::min<int64_t>(g_cfg.overlap_prefix_ctas, sms - 1);
  // R_P derated from 0.46 (full clock) for the ~1.45-1.7 GHz the 1 kW cap holds the SMs at in a
  // sustained overlapped step: the tensor-bound prefix slows with the clock, the HBM-bound
  // suffix does not (tools/power_profile.py, tools/overlap_sustained.py)
  // (CTA-pair kernel: 0.49 alone at full clock on 144 SMs, 0.43 in the power-capped step at k = 72)
  const double R_P = pair_mode(g) ? 0.42 : 0.38, R_S = 1.0e5, BW = 7.0e6;
  const int64_t pairs = (B * g + 255) / 256;
  const double pair_blocks = (double)pairs * h->num_kv_heads * ((P + 127) / 128);
  int best_k = 0;
  double best = 1e300;
  for (int k = 8; k <= sms - 8; ++k) {
    if (prefix_kind(h, B * g, P, k) != PK_TC2) break;  // too few blocks per CTA beyond this k
    if (prefix_tc2_ctas(B, g, h->num_kv_heads, P, k, prefix_bn(), pair_mode(g), (int)g_cfg.pair_cluster) != k)
      continue;  // plan would idle SMs
    const double t = std::max(pair_blocks / (k * R_P), suffix_tc_us(h, B, S_cap, sms - k, R_S, BW));
    if (t < best) {
      best = t;
      best_k = k;
    }
  }
  // Short GQA suffixes (suffix_short_kernel, three CTAs per SM) on the suffix's SM share
  // (overlap_short, default on): the tensor-bound prefix keeps all but one stream-K group's worth of
  // SMs and the short kernel streams the suffix beside it at ~50 GB/s per SM.  Model: t(k) =
  // max(prefix on k, suffix on SMs - k), against the sequential prefix + suffix (+ ~8 us of tail).
  // Measured (tools/config_ab.py, profiles/r3j_ovshort.jsonl): C6 0.098 -> 0.090 ms, C4 0.259 ->
  // 0.243 ms at k = 128 (8 of 9 groups).
  if (g_cfg.overlap_short && !paged && g_cfg.suffix_impl == 0 && g_cfg.overlap_prefix_ctas == 0 &&
      short_auto(g, S_cap)) {
    const double R_P = pair_mode(g) ? 0.42 : 0.38, R_SH = 5.0e4, BW = 7.0e6;
    const double bytes = (double)B * h->num_kv_heads * S_cap * h->head_dim * 4.0;
    int bk = 0;
    double bt = 1e300;
    for (int k = 8; k <= sms - 8; ++k) {
      if (prefix_kind(h, B * g, P, k) != PK_TC2) break;
      if (prefix_tc2_ctas(B, g, h->num_kv_heads, P, k, prefix_bn(), pair_mode(g), (int)g_cfg.pair_cluster) != k) continue;
      const double t = std::max(pair_blocks / (k * R_P), bytes / std::min((sms - k) * R_SH, BW));
      if (t < bt) {
        bt = t;
        bk = k;
      }
    }
    const int kf = prefix_tc2_ctas(B, g, h->num_kv_heads, P, sms, prefix_bn(), pair_mode(g), (int)g_cfg.pair_cluster);
    const double t_seq = pair_blocks / (kf * R_P) + bytes / BW + 8.0;
    return bk > 0 && bt < t_seq ? bk : 0;
  }
  // GQA: the sequential schedule runs the tensor-core suffix on every SM, which the split
  // starves of SMs when the suffix is short (C6: 146 us on 12 SMs against 29 us on 148).
  // Overlap only when the model says it is clearly (> 10 %) faster than prefix-then-suffix.
  // (MHA keeps the split: there the measured overlap wins at every shard size.)
  if (use_suffix_tc(h, B, S_cap, false)) {
    const double t_seq = pair_blocks / (sms * R_P) + suffix_tc_us(h, B, S_cap, sms, R_S, BW);
    if (best * 1.1 >= t_seq) return 0;
  }
  return best_k;
}

// fused Eq. 5 arrival counters (int32 per row), after the partial slots in the workspace
static size_t counter_bytes(int64_t rows) { return ((size_t)rows * sizeof(int32_t) + 255) / 256 * 256; }

static size_t part_bytes(const hydra_heads *h, int64_t B) {
  return (size_t)B * h->num_q_heads * ((size_t)h->head_dim + 1) * sizeof(float);
}

// ------------------------------------------------------------------ launch helpers
struct PartsView {  // n slots of [B,Hq,d] f32 followed by n slots of [B,Hq] f32
  float *o;
  float *lse;
  int64_t o_stride, lse_stride;
};

static PartsView parts_in_ws(void *ws, const hydra_heads *h, int64_t B, int n) {
  PartsView v;
  v.o_stride = B * h->num_q_heads * (int64_t)h->head_dim;
  v.lse_stride = B * h->num_q_heads;
  v.o = reinterpret_cast<float *>(ws);
  v.lse = v.o + v.o_stride * n;
  return v;
}

static hydra_status run_prefix(const hydra_heads *h, int64_t B, const void *q, int64_t q_sb, int64_t q_sh,
                               int64_t P, const void *k, const void *v, int64_t kv_st, int64_t kv_sh, int splits,
                               const PartsView &dst, cudaStream_t s, int tc2_ctas = 0,
                               const FusedCombine *fc = nullptr) {
  const int g = h->num_q_heads / h->num_kv_heads;
  const float sl2 = scale_of(h) * 1.4426950408889634f;
  const PrefixKind kind = prefix_kind(h, B * g, P, tc2_ctas);
  if (kind != PK_SIMT) {
    PrefixTcArgs a{};
    a.q = q;
    a.q_sb = q_sb;
    a.q_sh = q_sh;
    a.k = k;
    a.v = v;
    a.kv_st = kv_st;
    a.kv_sh = kv_sh;
    a.kv_total = P;
    a.Hq = h->num_q_heads;
    a.Hkv = h->num_kv_heads;
    a.g = g;
    a.scale_log2 = sl2;
    a.P = P;
    a.B = (int32_t)B;
    a.n_splits = splits;
    a.o = dst.o;
    a.lse = dst.lse;
    a.o_slot_stride = dst.o_stride;
    a.lse_slot_stride = dst.lse_stride;
    a.debug_variant = (int32_t)g_cfg.tc_debug;
    a.trace = reinterpret_cast<void *>((intptr_t)g_cfg.prefix_trace);
    a.stages = (int32_t)g_cfg.prefix_stages;
    a.poly_every = (int32_t)g_cfg.prefix_poly;
    a.variant = (int32_t)g_cfg.prefix_variant;
    a.mutate = (int32_t)g_cfg.mutate;
    if (fc) a.fc = *fc;
    a.timer = reinterpret_cast<unsigned long long *>((intptr_t)g_cfg.step_timer);
    a.pair_cluster = (int32_t)g_cfg.pair_cluster;
    a.pair_poly = (int32_t)g_cfg.pair_poly;
    a.pair_item_cost = (int32_t)g_cfg.pair_item_cost;
    hydra_status st;
    if (kind == PK_TC2) {
      // stream-K pieces leave some slots of a row unwritten: mark every slot empty first (the
      // fused merge knows which slots hold a row's pieces and needs no fill)
      // (the CTA-pair kernel marks them itself: the piece that ends a unit fills the later slots)
      if (!fc && splits > 1 && !(pair_mode(g) && !a.tasks) &&
          launch_fill_neg_inf(dst.lse, dst.lse_stride * splits, s) != HYDRA_OK)
        return cuda_fail("fill");
      st = launch_prefix_tc2(a, tc2_ctas > 0 ? tc2_ctas : prefix_ctas(), s);
    } else {
      st = launch_prefix_tc(a, s);
    }
    return st == HYDRA_OK ? st : cuda_fail("prefix tcgen05 launch");
  }
  DecodeParams p{};
  p.q = q;
  p.q_sb = q_sb;
  p.q_sh = q_sh;
  p.k = k;
  p.v = v;
  p.kv_sb = 0;
  p.kv_st = kv_st;
  p.kv_sh = kv_sh;
  p.lens = nullptr;
  p.len_uniform = P;
  p.n_seq = (int32_t)B;
  p.Hq = h->num_q_heads;
  p.Hkv = h->num_kv_heads;
  p.g = g;
  p.scale_log2 = sl2;
  p.n_splits = splits;
  p.split_len = (P + splits - 1) / splits;
  p.heads_per_cta = heads_per_cta(g);
  p.o = dst.o;
  p.lse = dst.lse;
  p.o_split_stride = dst.o_stride;
  p.lse_split_stride = dst.lse_stride;
  hydra_status st = launch_decode(p, h->dtype, h->head_dim, s);
  return st == HYDRA_OK ? st : (st == HYDRA_ECUDA ? cuda_fail("prefix SIMT launch") : fail(st, "prefix SIMT"));
}

static hydra_status run_suffix(const hydra_heads *h, int64_t B, const void *q, int64_t q_sb, int64_t q_sh,
                               const void *k, const void *v, int64_t s_sb, int64_t s_st, int64_t s_sh,
                               int64_t S_cap, const int32_t *lens, int splits, const PartsView &dst,
                               cudaStream_t s, int tc_ctas = 0, const hydra_paging *pg = nullptr,
                               const FusedCombine *fc = nullptr, bool pdl = false) {
  const int g = h->num_q_heads / h->num_kv_heads;
  // (the testing build's lens check is a kernel of its own: it would sit between the prefix
  // and a programmatic-dependent suffix, so it is skipped there)
  if (kTesting && !pdl && launch_lens_check(lens, B, S_cap, s) != HYDRA_OK) return cuda_fail("lens check");
  if (use_suffix_tc(h, B, S_cap, tc_ctas > 0)) {
    SuffixTcArgs a{};
    a.q = q;
    a.q_sb = q_sb;
    a.q_sh = q_sh;
    a.k = k;
    a.v = v;
    a.s_sb = s_sb;
    a.s_st = s_st;
    a.s_sh = s_sh;
    a.S_cap = S_cap;
    a.lens = lens;
    a.B = (int32_t)B;
    a.Hq = h->num_q_heads;
    a.Hkv = h->num_kv_heads;
    a.scale_log2 = scale_of(h) * 1.4426950408889634f;
    a.o = dst.o;
    a.lse = dst.lse;
    a.cb = (int32_t)g_cfg.suffix_cb;
    a.trace = reinterpret_cast<void *>((intptr_t)g_cfg.suffix_trace);
    a.debug = (int32_t)g_cfg.tc_debug;
    a.mutate = (int32_t)g_cfg.mutate;
    if (fc) a.fc = *fc;
    a.pdl = pdl ? 1 : 0;
    if (g_cfg.step_timer) a.timer = reinterpret_cast<unsigned long long *>((intptr_t)g_cfg.step_timer) + 2;
    a.n_split = splits;
    a.split_len = (int32_t)(((S_cap + splits - 1) / splits + 127) / 128 * 128);
    a.o_split_stride = dst.o_stride;
    a.lse_split_stride = dst.lse_stride;
    if (pg) {
      a.block_table = pg->block_table;
      a.bt_stride = pg->bt_stride;
      a.n_pages = pg->n_pages;
      a.page_size = pg->page_size;
    }
    // Short grouped-query suffixes (<= 2 blocks): the three-CTAs-per-SM kernel, on the full chip
    // (auto) or on request (suffix_impl 3).  Measured alone (tools/suffix_span.py, kernel span):
    // C6's g = 8 128-token suffixes 18.4 -> 13.3 us, C4's g = 4 46.5 -> 42.2 us.
    const bool short_ok = !pg && !fc && splits <= 1 && suffix_short_supported(g, S_cap);
    if (short_ok && tc_ctas == 0 &&
        (g_cfg.suffix_impl == 3 || (g_cfg.suffix_impl == 0 && g_cfg.suffix_ctas == 0 && short_auto(g, S_cap)))) {
      hydra_status st = launch_suffix_short(a, (int)g_cfg.suffix_ctas, s);
      return st == HYDRA_OK ? st : cuda_fail("suffix (short) tcgen05 launch");
    }
    // SM-partitioned schedule with short GQA suffixes (overlap_short): three short-kernel CTAs per
    // SM of the suffix's share, a programmatic dependent of the prefix
    if (short_ok && tc_ctas > 0 && g_cfg.overlap_short && g_cfg.suffix_impl == 0 && short_auto(g, S_cap)) {
      hydra_status st = launch_suffix_short(a, 3 * tc_ctas, s);
      return st == HYDRA_OK ? st : cuda_fail("suffix (short) tcgen05 launch");
    }
    const int ctas = tc_ctas > 0 ? tc_ctas : (g_cfg.suffix_ctas > 0 ? (int)g_cfg.suffix_ctas : device_sm_count());
    hydra_status st = launch_suffix_tc(a, ctas, s);
    return st == HYDRA_OK ? st : cuda_fail("suffix tcgen05 launch");
  }
  DecodeParams p{};
  p.q = q;
  p.q_sb = q_sb;
  p.q_sh = q_sh;
  p.k = k;
  p.v = v;
  p.kv_sb = s_sb;
  p.kv_st = s_st;
  p.kv_sh = s_sh;
  p.lens = lens;
  p.len_cap = S_cap;
  p.len_uniform = 0;
  p.n_seq = (int32_t)B;
  p.Hq = h->num_q_heads;
  p.Hkv = h->num_kv_heads;
  p.g = g;
  p.scale_log2 = scale_of(h) * 1.4426950408889634f;
  p.n_splits = splits;
  p.split_len = (S_cap + splits - 1) / splits;
  p.heads_per_cta = heads_per_cta(g);
  p.unroll = (int32_t)g_cfg.suffix_unroll;
  p.o = dst.o;
  p.lse = dst.lse;
  p.o_split_stride = dst.o_stride;
  p.lse_split_stride = dst.lse_stride;
  if (fc) p.fc = *fc;
  if (pg) {
    p.block_table = pg->block_table;
    p.bt_stride = pg->bt_stride;
    p.page_shift = __builtin_ctz((unsigned)pg->page_size);
  }
  p.pdl = pdl ? 1 : 0;
  if (g_cfg.step_timer) p.timer = reinterpret_cast<unsigned long long *>((intptr_t)g_cfg.step_timer) + 2;
  hydra_status st = launch_decode(p, h->dtype, h->head_dim, s);
  return st == HYDRA_OK ? st : (st == HYDRA_ECUDA ? cuda_fail("suffix launch") : fail(st, "suffix"));
}

static hydra_status run_combine(int64_t rows, int d, int n, const PartsView &src, void *out, hydra_dtype out_dtype,
                                float *lse_out, cudaStream_t s, bool pdl = false) {
  CombineParams c{};
  c.rows = rows;
  c.d = d;
  c.n_a = n;
  c.o_a = src.o;
  c.o_a_part = src.o_stride;
  c.o_a_row = d;
  c.l_a = src.lse;
  c.l_a_part = src.lse_stride;
  c.l_a_row = 1;
  c.out = out;
  c.out_row = d;
  c.lse_out = lse_out;
  c.lse_out_row = 1;
  c.inject_bug = inject_combine_bug() ? 1 : 0;
  c.pdl = pdl ? 1 : 0;
  hydra_status st = launch_combine(c, HYDRA_F32, out_dtype, s);
  return st == HYDRA_OK ? st : cuda_fail("combine launch");
}

// ------------------------------------------------------------------ workspace
extern "C" size_t hydra_workspace_size(int op, const hydra_heads *h, int64_t B, int64_t P, int64_t S_cap,
                                       int32_t n_parts) {
  if (check_heads(h) != HYDRA_OK || B <= 0) return 0;
  const size_t pb = part_bytes(h, B);
  switch (op) {
    case HYDRA_OP_PARTS:  // caller-staged partials for hydra_combine: n_parts x (O f32 [B,Hq,d] + LSE f32 [B,Hq])
      return n_parts > 0 ? pb * (size_t)n_parts : 0;
    case HYDRA_OP_PREFIX: {
      const int s = prefix_splits(h, B, P);
      return s > 1 ? pb * s : 0;
    }
    case HYDRA_OP_SUFFIX: {
      const int s = suffix_splits(h, B, S_cap);
      return s > 1 ? pb * s : 0;
    }
    case HYDRA_OP_ATTN: {  // enough for both the sequential and the SM-partitioned schedules (+ fused counters)
      bool simt = false;
      const int k = overlap_prefix_ctas(h, B, P, S_cap), k2 = overlap_prefix_ctas(h, B, P, S_cap, &simt);
      const int np = std::max({prefix_splits(h, B, P), k > 0 ? prefix_splits(h, B, P, k) : 1,
                               k2 > 0 ? prefix_splits(h, B, P, k2) : 1});
      return pb * (size_t)(np + std::max(suffix_splits(h, B, S_cap), suffix_splits(h, B, S_cap, k > 0))) +
             counter_bytes(B * h->num_q_heads);
    }
  }
  return 0;
}

// ------------------------------------------------------------------ prefix / suffix / combine
extern "C" hydra_status hydra_prefix_attn(const hydra_heads *h, int64_t B, const void *q, int64_t q_sb,
                                          int64_t q_sh, int64_t P, const void *k, const void *v, int64_t kv_st,
                                          int64_t kv_sh, float *o_part, float *lse_part, void *ws,
                                          size_t ws_bytes, void *stream) {
  hydra_status st = check_heads(h);
  if (st) return st;
  if (B <= 0) return fail(HYDRA_ESHAPE, "B must be > 0 (S:291)");
  if (P < 0) return fail(HYDRA_ESHAPE, "P must be >= 0");
  if (!q || !o_part || !lse_part || (P > 0 && (!k || !v))) return fail(HYDRA_EINVAL, "null pointer argument");
  const size_t es = elem_size(h->dtype);
  if (!aligned16(q, es, {q_sb, q_sh}) || (P > 0 && (!aligned16(k, es, {kv_st, kv_sh}) || !aligned16(v, es, {}))))
    return fail(HYDRA_EINVAL, "q/k/v base pointers and strides must be 16-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int d = h->head_dim;
  PartsView out{o_part, lse_part, B * h->num_q_heads * (int64_t)d, B * h->num_q_heads};
  if (P == 0) {  // empty prefix: sentinel (reading R6)
    if (cudaMemsetAsync(o_part, 0, sizeof(float) * B * h->num_q_heads * d, s) != cudaSuccess)
      return cuda_fail("memset");
    st = launch_fill_neg_inf(lse_part, B * h->num_q_heads, s);
    return st ? cuda_fail("fill") : HYDRA_OK;
  }
  const int splits = prefix_splits(h, B, P);
  if (splits == 1) return run_prefix(h, B, q, q_sb, q_sh, P, k, v, kv_st, kv_sh, 1, out, s);
  const size_t need = part_bytes(h, B) * splits;
  if (!ws || ws_bytes < need) return fail(HYDRA_ENOMEM, "workspace too small: need %zu bytes", need);
  PartsView parts = parts_in_ws(ws, h, B, splits);
  st = run_prefix(h, B, q, q_sb, q_sh, P, k, v, kv_st, kv_sh, splits, parts, s);
  if (st) return st;
  return run_combine(B * h->num_q_heads, d, splits, parts, o_part, HYDRA_F32, lse_part, s);
}

// Paging descriptor checks shared by the *_paged entry points (hydra.h, hydra_paging).
static hydra_status check_paging(const hydra_paging *pg, int64_t S_cap) {
  if (!pg || !pg->block_table) return fail(HYDRA_EINVAL, "null paging descriptor / block table");
  if (pg->page_size < 8 || (pg->page_size & (pg->page_size - 1)))
    return fail(HYDRA_ESHAPE, "page_size must be a power of two >= 8 (got %d)", pg->page_size);
  if (pg->n_pages <= 0 || pg->n_pages > INT32_MAX) return fail(HYDRA_ESHAPE, "n_pages must be in [1, 2^31)");
  if (pg->bt_stride <= 0 || S_cap > pg->bt_stride * (int64_t)pg->page_size)
    return fail(HYDRA_ESHAPE, "S_cap (%lld) exceeds bt_stride * page_size", (long long)S_cap);
  return HYDRA_OK;
}

static hydra_status suffix_impl(const hydra_heads *h, int64_t B, const void *q, int64_t q_sb, int64_t q_sh,
                                const void *k, const void *v, int64_t s_sb, int64_t s_st, int64_t s_sh,
                                int64_t S_cap, const int32_t *lens, float *o_part, float *lse_part, void *ws,
                                size_t ws_bytes, void *stream, const hydra_paging *pg) {
  hydra_status st = check_heads(h);
  if (st) return st;
  if (B <= 0) return fail(HYDRA_ESHAPE, "B must be > 0 (S:291)");
  if (S_cap < 0) return fail(HYDRA_ESHAPE, "S_cap must be >= 0");
  if (!q || !o_part || !lse_part || (S_cap > 0 && (!k || !v || !lens)))
    return fail(HYDRA_EINVAL, "null pointer argument");
  const size_t es = elem_size(h->dtype);
  if (!aligned16(q, es, {q_sb, q_sh}) || (S_cap > 0 && (!aligned16(k, es, {s_sb, s_st, s_sh}) || !aligned16(v, es, {}))))
    return fail(HYDRA_EINVAL, "q/k/v base pointers and strides must be 16-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int d = h->head_dim;
  PartsView out{o_part, lse_part, B * h->num_q_heads * (int64_t)d, B * h->num_q_heads};
  if (S_cap == 0) {
    if (cudaMemsetAsync(o_part, 0, sizeof(float) * B * h->num_q_heads * d, s) != cudaSuccess)
      return cuda_fail("memset");
    st = launch_fill_neg_inf(lse_part, B * h->num_q_heads, s);
    return st ? cuda_fail("fill") : HYDRA_OK;
  }
  const int splits = suffix_splits(h, B, S_cap);
  if (splits == 1) return run_suffix(h, B, q, q_sb, q_sh, k, v, s_sb, s_st, s_sh, S_cap, lens, 1, out, s, 0, pg);
  const size_t need = part_bytes(h, B) * splits;
  if (!ws || ws_bytes < need) return fail(HYDRA_ENOMEM, "workspace too small: need %zu bytes", need);
  PartsView parts = parts_in_ws(ws, h, B, splits);
  st = run_suffix(h, B, q, q_sb, q_sh, k, v, s_sb, s_st, s_sh, S_cap, lens, splits, parts, s, 0, pg);
  if (st) return st;
  return run_combine(B * h->num_q_heads, d, splits, parts, o_part, HYDRA_F32, lse_part, s);
}

extern "C" hydra_status hydra_suffix_attn(const hydra_heads *h, int64_t B, const void *q, int64_t q_sb,
                                          int64_t q_sh, const void *k, const void *v, int64_t s_sb, int64_t s_st,
                                          int64_t s_sh, int64_t S_cap, const int32_t *lens, float *o_part,
                                          float *lse_part, void *ws, size_t ws_bytes, void *stream) {
  return suffix_impl(h, B, q, q_sb, q_sh, k, v, s_sb, s_st, s_sh, S_cap, lens, o_part, lse_part, ws, ws_bytes,
                     stream, nullptr);
}

extern "C" hydra_status hydra_suffix_attn_paged(const hydra_heads *h, int64_t B, const void *q, int64_t q_sb,
                                                int64_t q_sh, const void *k_pool, const void *v_pool, int64_t p_sp,
                                                int64_t p_st, int64_t p_sh, const hydra_paging *pg, int64_t S_cap,
                                                const int32_t *lens, float *o_part, float *lse_part, void *ws,
                                                size_t ws_bytes, void *stream) {
  if (S_cap > 0) {
    hydra_status st = check_paging(pg, S_cap);
    if (st) return st;
  }
  return suffix_impl(h, B, q, q_sb, q_sh, k_pool, v_pool, p_sp, p_st, p_sh, S_cap, lens, o_part, lse_part, ws,
                     ws_bytes, stream, S_cap > 0 ? pg : nullptr);
}

extern "C" hydra_status hydra_combine_ex(const hydra_combine_desc *c, void *stream) {
  if (!c) return fail(HYDRA_EINVAL, "combine descriptor is NULL");
  const int64_t d = c->d;
  if (c->rows < 0 || d <= 0 || c->n_parts < 0 || c->n_parts_f32 < 0 || c->n_parts + c->n_parts_f32 <= 0)
    return fail(HYDRA_ESHAPE, "rows >= 0, d > 0 and at least one part required");
  const bool scatter = c->table_rows > 0;
  if ((c->n_parts > 0 && (!c->o_parts || !c->lse_parts)) ||
      (c->n_parts_f32 > 0 && (!c->o_parts_f32 || !c->lse_parts_f32)) || (scatter ? !c->out_table : !c->out))
    return fail(HYDRA_EINVAL, "null pointer argument");
  if (c->table_rows < 0) return fail(HYDRA_ESHAPE, "table_rows must be >= 0");
  if (c->n_parts > 0 && c->o_dtype != HYDRA_F32 && c->o_dtype != HYDRA_F16)
    return fail(HYDRA_EUNSUPPORTED, "o_dtype must be F32 or F16");
  const hydra_dtype od = c->n_parts > 0 ? c->o_dtype : HYDRA_F32;
  if (c->out_dtype != HYDRA_F32 && c->out_dtype != HYDRA_BF16 && !(c->out_dtype == HYDRA_F16 && od == HYDRA_F32))
    return fail(HYDRA_EUNSUPPORTED, "out_dtype must be F32 or BF16 (F16 only from F32 parts)");
  const int64_t o_row = c->o_row_stride ? c->o_row_stride : d, of_row = c->o_f32_row_stride ? c->o_f32_row_stride : d;
  const int64_t l_row = c->lse_row_stride ? c->lse_row_stride : 1;
  const int64_t lf_row = c->lse_f32_row_stride ? c->lse_f32_row_stride : 1;
  const int64_t out_row = c->out_row_stride ? c->out_row_stride : d, lo_row = c->lse_out_row_stride ? c->lse_out_row_stride : 1;
  if (o_row < d || of_row < d || out_row < d || l_row < 1 || lf_row < 1 || lo_row < 1 || c->o_part_stride < 0 ||
      c->lse_part_stride < 0 || c->o_f32_part_stride < 0 || c->lse_f32_part_stride < 0)
    return fail(HYDRA_ESHAPE, "row strides must cover a row (O >= d, LSE >= 1) and part strides be >= 0");
  if (d == 128 || d == 256) {  // vector loads: 16 B of f32 or 8 B of f16 per lane
    const int64_t a = od == HYDRA_F16 ? 8 : 16, es = od == HYDRA_F16 ? 2 : 4;
    if (c->n_parts > 0 && (reinterpret_cast<uintptr_t>(c->o_parts) % a || (c->o_part_stride * es) % a ||
                           (o_row * es) % a))
      return fail(HYDRA_EINVAL, "o_parts and its strides must be %d-byte aligned", (int)a);
    if (c->n_parts_f32 > 0 && (reinterpret_cast<uintptr_t>(c->o_parts_f32) % 16 || (c->o_f32_part_stride * 4) % 16 ||
                               (of_row * 4) % 16))
      return fail(HYDRA_EINVAL, "o_parts_f32 and its strides must be 16-byte aligned");
  }
  CombineParams p{};
  p.rows = c->rows;
  p.d = (int32_t)d;
  p.n_a = c->n_parts;
  p.o_a = c->o_parts;
  p.o_a_part = c->o_part_stride;
  p.o_a_row = o_row;
  p.l_a = c->lse_parts;
  p.l_a_part = c->lse_part_stride;
  p.l_a_row = l_row;
  p.n_b = c->n_parts_f32;
  p.o_b = c->o_parts_f32;
  p.o_b_part = c->o_f32_part_stride;
  p.o_b_row = of_row;
  p.l_b = c->lse_parts_f32;
  p.l_b_part = c->lse_f32_part_stride;
  p.l_b_row = lf_row;
  p.out = c->out;
  p.out_row = out_row;
  p.lse_out = c->lse_out;
  p.lse_out_row = lo_row;
  if (scatter) {
    p.out_table = c->out_table;
    p.lse_out_table = c->lse_out_table;
    p.table_rows = c->table_rows;
  }
  p.inject_bug = inject_combine_bug() ? 1 : 0;
  hydra_status st = launch_combine(p, od, c->out_dtype, reinterpret_cast<cudaStream_t>(stream));
  return st == HYDRA_OK ? st : cuda_fail("combine launch");
}

extern "C" hydra_status hydra_combine(int64_t rows, int32_t d, int32_t n_parts, const void *o_parts,
                                      hydra_dtype o_dtype, int64_t o_part_stride, const float *lse_parts,
                                      int64_t lse_part_stride, void *out, hydra_dtype out_dtype, float *lse_out,
                                      void *stream) {
  if (rows < 0 || d <= 0 || n_parts <= 0) return fail(HYDRA_ESHAPE, "rows >= 0, d > 0, n_parts > 0 required");
  if (n_parts > 1 && (o_part_stride < rows * d || lse_part_stride < rows))
    return fail(HYDRA_ESHAPE, "part strides overlap the rows of a part");
  hydra_combine_desc c{};
  c.rows = rows;
  c.d = d;
  c.n_parts = n_parts;
  c.o_parts = o_parts;
  c.o_dtype = o_dtype;
  c.o_part_stride = o_part_stride;
  c.lse_parts = lse_parts;
  c.lse_part_stride = lse_part_stride;
  c.out = out;
  c.out_dtype = out_dtype;
  c.lse_out = lse_out;
  return hydra_combine_ex(&c, stream);
}

// ------------------------------------------------------------------ composite
// The fused Eq. 5 path (fused.cuh) of hydra_attn: bf16, d = 128, both parts present, a prefix
// kernel with a device-known piece layout (the persistent kernel's stream-K plan, variants
// 3 / 5 / 6, or the one-tile kernel's fixed splits), and either suffix kernel.
static bool attn_fused(const hydra_heads *h, int64_t B, int64_t P, int64_t S_cap, int k_over) {
  if (!g_cfg.fuse_combine || (k_over > 0 && g_cfg.fuse_combine < 2) || h->dtype != HYDRA_BF16 || h->head_dim != 128 || P <= 0 || S_cap <= 0) return false;
  const PrefixKind k = prefix_kind(h, B * (h->num_q_heads / h->num_kv_heads), P, k_over);
  return (k == PK_TC2 && g_cfg.prefix_variant != 4 && !pair_mode(h->num_q_heads / h->num_kv_heads)) || k == PK_TC1;
}

// ------------------------------------------------------------------ composite
namespace {
struct StreamEvents {
  cudaEvent_t fork = nullptr, join = nullptr;
  StreamEvents() {
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
  }
};
thread_local StreamEvents *tl_events = nullptr;
StreamEvents &events() {
  if (!tl_events) tl_events = new StreamEvents();
  return *tl_events;
}
}  // namespace

static hydra_status attn_impl(const hydra_heads *h, int64_t B, const void *q, int64_t q_sb, int64_t q_sh,
                              int64_t P, const void *pk, const void *pv, int64_t kv_st, int64_t kv_sh,
                              const void *sk, const void *sv, int64_t s_sb, int64_t s_st, int64_t s_sh,
                              int64_t S_cap, const int32_t *lens, void *out, hydra_dtype out_dtype,
                              float *lse_out, void *ws, size_t ws_bytes, void *stream, void *s_aux,
                              const hydra_paging *pg) {
  hydra_status st = check_heads(h);
  if (st) return st;
  if (B <= 0) return fail(HYDRA_ESHAPE, "B must be > 0 (S:291)");
  if (P < 0 || S_cap < 0) return fail(HYDRA_ESHAPE, "P and S_cap must be >= 0");
  if (!q || !out || (P > 0 && (!pk || !pv)) || (S_cap > 0 && (!sk || !sv || !lens)))
    return fail(HYDRA_EINVAL, "null pointer argument");
  if (out_dtype != HYDRA_BF16 && out_dtype != HYDRA_F32) return fail(HYDRA_EUNSUPPORTED, "out_dtype must be BF16 or F32");
  const size_t es = elem_size(h->dtype);
  if (!aligned16(q, es, {q_sb, q_sh}) || (P > 0 && (!aligned16(pk, es, {kv_st, kv_sh}) || !aligned16(pv, es, {}))) ||
      (S_cap > 0 && (!aligned16(sk, es, {s_sb, s_st, s_sh}) || !aligned16(sv, es, {}))))
    return fail(HYDRA_EINVAL, "q/k/v base pointers and strides must be 16-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // With a second stream given (the caller allows concurrency) and both persistent tensor-core
  // kernels, run them concurrently on disjoint SM sets: k prefix CTAs + (SMs - k) suffix CTAs,
  // one CTA per SM each.  Both go on `stream`: the suffix is a programmatic dependent launch
  // that starts once every prefix CTA (CTA pairs of a cluster need both SMs of a TPC) is
  // resident, so the prefix always gets its SM share first; the suffix grid completes only
  // after the prefix grid (griddepcontrol.wait), so everything after it in the stream sees
  // both.  (Two streams let the suffix grab SMs first and split TPCs: measured 0.96-1.35 ms
  // depending on k at C3@16K, tools/overlap_sustained.py.)  Without an SM split (k = 0) two
  // full grids would only contend: run sequentially.
  bool ov_simt = false;  // SM-partitioned with the SIMT suffix as the prefix's dependent (full grid)
  const int k_over = s_aux ? overlap_prefix_ctas(h, B, P, S_cap, &ov_simt, pg != nullptr) : 0;
  cudaStream_t sa = s;
  g_cfg.last_overlap_k = k_over;
  g_cfg.last_overlap_simt = ov_simt ? 1 : 0;
  const int sms = device_sm_count();
  const int g = h->num_q_heads / h->num_kv_heads;
  const int np = prefix_splits(h, B, P, k_over), ns = suffix_splits(h, B, S_cap, k_over > 0 && !ov_simt);
  const bool fused = !ov_simt && attn_fused(h, B, P, S_cap, k_over);  // (the SIMT dependent never fuses)
  const int64_t rows = B * h->num_q_heads;
  const size_t need = part_bytes(h, B) * (np + ns) + (fused ? counter_bytes(rows) : 0);
  if (!ws || ws_bytes < need) return fail(HYDRA_ENOMEM, "workspace too small: need %zu bytes", need);
  PartsView all = parts_in_ws(ws, h, B, np + ns);
  PartsView pre = all, suf = all;
  suf.o = all.o + all.o_stride * np;
  suf.lse = all.lse + all.lse_stride * np;

  // Fused Eq. 5 (fused.cuh): the prefix and suffix epilogues count every row's parts and the
  // writer of its last part merges it into `out`; the counters (after the partial slots in the
  // workspace) are zeroed here, before the fork -- no slot fill, no combine launch.
  FusedCombine fc{};
  if (fused) {
    fc.cnt = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(ws) + part_bytes(h, B) * (np + ns));
    fc.o_pre = pre.o;
    fc.lse_pre = pre.lse;
    fc.o_suf = suf.o;
    fc.lse_suf = suf.lse;
    fc.o_slot = all.o_stride;
    fc.lse_slot = all.lse_stride;
    fc.n_suf = ns;
    fc.g = g;
    fc.Hq = h->num_q_heads;
    fc.Hkv = h->num_kv_heads;
    fc.out = out;
    fc.out_f32 = out_dtype == HYDRA_F32;
    fc.lse_out = lse_out;
    fc.inject_bug = inject_combine_bug() ? 1 : 0;
    fc.pre_done = k_over == 0 ? 1 : 0;  // sequential: the suffix launch follows the prefix kernel
    if (prefix_kind(h, B * g, P, k_over) == PK_TC2)
      prefix_tc2_plan_into(fc, B, g, h->num_kv_heads, P, k_over > 0 ? k_over : prefix_ctas(), prefix_bn());
    else
      fc.n_pre_splits = np;
    if (!(fc.pre_done && ns == 1) && cudaMemsetAsync(fc.cnt, 0, sizeof(int32_t) * rows, s) != cudaSuccess)
      return cuda_fail("counter reset");
  }

  // Programmatic dependent launch of the suffix: in the SM-partitioned schedule it takes the SMs
  // the prefix leaves; in the sequential one the tensor-core suffix starts on the SMs the
  // prefix's last CTAs free (the prefix's tail: C6 0.104 -> 0.098 ms).  Not for the SIMT suffix
  // (C3 sequential 1.02 -> 1.24 ms measured), not with the fused merge (the suffix reads the
  // prefix partials), not with caller events between the kernels (they serialise them).
  const bool pdl = P > 0 && S_cap > 0 &&
                   (k_over > 0 || (!fused && g_cfg.seq_pdl && !g_cfg.step_ev[1] && !g_cfg.step_ev[2] &&
                                   use_suffix_tc(h, B, S_cap, false)));
  // (the testing build's lens check is a kernel of its own: with pdl it runs before the prefix)
  if (kTesting && pdl && launch_lens_check(lens, B, S_cap, s) != HYDRA_OK) return cuda_fail("lens check");
  if (P > 0) {
    // (no event between the prefix and a programmatic-dependent suffix: it would serialise them)
    record_step_ev(0, sa);
    st = run_prefix(h, B, q, q_sb, q_sh, P, pk, pv, kv_st, kv_sh, np, pre, sa, k_over, fused ? &fc : nullptr);
    if (!pdl) record_step_ev(1, sa);
  } else {
    st = launch_fill_neg_inf(pre.lse, rows, sa);
    if (st) st = cuda_fail("fill");
  }
  if (st) return st;
  if (S_cap > 0) {
    // the suffix takes every SM the prefix plan leaves free (the plan may round k down)
    const int k_eff = k_over > 0 ? prefix_tc2_ctas(B, g, h->num_kv_heads, P, k_over, prefix_bn(), pair_mode(g),
                                                   (int)g_cfg.pair_cluster)
                                 : 0;
    if (!pdl) record_step_ev(2, s);
    st = run_suffix(h, B, q, q_sb, q_sh, sk, sv, s_sb, s_st, s_sh, S_cap, lens, ns, suf, s,
                    k_over > 0 && !ov_simt ? std::max(1, sms - k_eff) : 0, pg, fused ? &fc : nullptr, pdl);
    record_step_ev(3, s);
  } else {
    st = launch_fill_neg_inf(suf.lse, rows, s);
    if (st) st = cuda_fail("fill");
  }
  if (st) return st;
  if (fused) return HYDRA_OK;  // merged in the epilogues
  // (not behind a caller event: an event node between the kernels would serialise them anyway)
  return run_combine(rows, h->head_dim, np + ns, all, out, out_dtype, lse_out, s,
                     g_cfg.combine_pdl && !g_cfg.step_ev[3]);
}

extern "C" hydra_status hydra_attn(const hydra_heads *h, int64_t B, const void *q, int64_t q_sb, int64_t q_sh,
                                   int64_t P, const void *pk, const void *pv, int64_t kv_st, int64_t kv_sh,
                                   const void *sk, const void *sv, int64_t s_sb, int64_t s_st, int64_t s_sh,
                                   int64_t S_cap, const int32_t *lens, void *out, hydra_dtype out_dtype,
                                   float *lse_out, void *ws, size_t ws_bytes, void *stream, void *s_aux) {
  return attn_impl(h, B, q, q_sb, q_sh, P, pk, pv, kv_st, kv_sh, sk, sv, s_sb, s_st, s_sh, S_cap, lens, out,
                   out_dtype, lse_out, ws, ws_bytes, stream, s_aux, nullptr);
}

extern "C" hydra_status hydra_attn_paged(const hydra_heads *h, int64_t B, const void *q, int64_t q_sb,
                                         int64_t q_sh, int64_t P, const void *pk, const void *pv, int64_t kv_st,
                                         int64_t kv_sh, const void *k_pool, const void *v_pool, int64_t p_sp,
                                         int64_t p_st, int64_t p_sh, const hydra_paging *pg, int64_t S_cap,
                                         const int32_t *lens, void *out, hydra_dtype out_dtype, float *lse_out,
                                         void *ws, size_t ws_bytes, void *stream, void *s_aux) {
  if (S_cap > 0) {
    hydra_status st = check_paging(pg, S_cap);
    if (st) return st;
  }
  return attn_impl(h, B, q, q_sb, q_sh, P, pk, pv, kv_st, kv_sh, k_pool, v_pool, p_sp, p_st, p_sh, S_cap, lens,
                   out, out_dtype, lse_out, ws, ws_bytes, stream, s_aux, S_cap > 0 ? pg : nullptr);
}

// ------------------------------------------------------------------ decode-loop KV append
static hydra_status append_impl(const hydra_heads *h, int64_t B, const void *k_new, const void *v_new, int64_t nb,
                                int64_t nh, void *sk, void *sv, int64_t s_sb, int64_t s_st, int64_t s_sh,
                                int64_t S_cap, int32_t *lens, void *stream, const hydra_paging *pg) {
  hydra_status st = check_heads(h);
  if (st) return st;
  if (B <= 0) return fail(HYDRA_ESHAPE, "B must be > 0");
  if (S_cap <= 0) return fail(HYDRA_ESHAPE, "S_cap must be > 0");
  if (!k_new || !v_new || !sk || !sv || !lens) return fail(HYDRA_EINVAL, "null pointer argument");
  const size_t es = elem_size(h->dtype);
  if (!aligned16(k_new, es, {nb, nh}) || !aligned16(v_new, es, {}) || !aligned16(sk, es, {s_sb, s_st, s_sh}) ||
      !aligned16(sv, es, {}))
    return fail(HYDRA_EINVAL, "k/v pointers and strides must be 16-byte aligned");
  if (pg) {
    st = check_paging(pg, S_cap);
    if (st) return st;
  }
  st = launch_append_kv(k_new, v_new, nb, nh, sk, sv, s_sb, s_st, s_sh, S_cap, h->num_kv_heads, h->head_dim, es, B,
                        lens, reinterpret_cast<cudaStream_t>(stream), pg ? pg->block_table : nullptr,
                        pg ? pg->bt_stride : 0, pg ? pg->page_size : 0);
  return st == HYDRA_OK ? st : cuda_fail("append_kv launch");
}

extern "C" hydra_status hydra_append_kv(const hydra_heads *h, int64_t B, const void *k_new, const void *v_new,
                                        int64_t nb, int64_t nh, void *sk, void *sv, int64_t s_sb, int64_t s_st,
                                        int64_t s_sh, int64_t S_cap, int32_t *lens, void *stream) {
  return append_impl(h, B, k_new, v_new, nb, nh, sk, sv, s_sb, s_st, s_sh, S_cap, lens, stream, nullptr);
}

extern "C" hydra_status hydra_append_kv_paged(const hydra_heads *h, int64_t B, const void *k_new, const void *v_new,
                                              int64_t nb, int64_t nh, void *k_pool, void *v_pool, int64_t p_sp,
                                              int64_t p_st, int64_t p_sh, const hydra_paging *pg, int64_t S_cap,
                                              int32_t *lens, void *stream) {
  if (!pg) return fail(HYDRA_EINVAL, "null paging descriptor");
  return append_impl(h, B, k_new, v_new, nb, nh, k_pool, v_pool, p_sp, p_st, p_sh, S_cap, lens, stream, pg);
}

// ------------------------------------------------------------------ sharing tree
struct hydra_tree {
  int32_t n_nodes = 0;
  int64_t B = 0;
  std::vector<int32_t> parent, depth, leaf_of_seq;
  std::vector<int64_t> node_off, node_len;
  std::vector<int32_t> grp_off, grp_seq;  // CSR: sequences of node n = grp_seq[grp_off[n]..grp_off[n+1])
  int32_t max_depth = 0;                  // nodes on the longest root->leaf path
  int32_t *d_grp_seq = nullptr;           // device copy of grp_seq
  // Work lists of the tensor-core node attention, built by hydra_tree_prepare (off the hot
  // path) per query-group size g: [0] 128-row tiles (one-tile kernel), [1] 256-row tile
  // pairs (persistent kernel).  A task stores its node's depth, not a slot, so the lists do
  // not depend on the KV split count.
  struct Lists {
    PrefixTask *d[2] = {nullptr, nullptr};
    int n[2] = {0, 0};
  };
  mutable std::mutex mu;
  std::map<int, Lists> work;  // g -> lists
};

extern "C" hydra_status hydra_tree_create(const int32_t *parent, const int64_t *node_off, const int64_t *node_len,
                                          int32_t n_nodes, const int32_t *leaf_of_seq, int64_t B,
                                          struct hydra_tree **out) {
  if (!out) return fail(HYDRA_EINVAL, "out is NULL");
  *out = nullptr;
  if (!parent || !node_off || !node_len || !leaf_of_seq) return fail(HYDRA_EINVAL, "null host array");
  if (n_nodes <= 0) return fail(HYDRA_ESHAPE, "tree needs at least one node");
  if (B <= 0) return fail(HYDRA_ESHAPE, "B must be > 0");
  int root = -1;
  for (int n = 0; n < n_nodes; ++n) {
    if (parent[n] == -1) {
      if (root >= 0) return fail(HYDRA_ESHAPE, "multiple roots (nodes %d and %d)", root, n);
      root = n;
    } else if (parent[n] < 0 || parent[n] >= n_nodes || parent[n] == n) {
      return fail(HYDRA_ESHAPE, "node %d has invalid parent %d", n, parent[n]);
    }
    if (node_off[n] < 0 || node_len[n] < 0) return fail(HYDRA_ESHAPE, "node %d has negative offset/length", n);
  }
  if (root < 0) return fail(HYDRA_ESHAPE, "no root (parent == -1)");
  auto t = new hydra_tree();
  t->n_nodes = n_nodes;
  t->B = B;
  t->parent.assign(parent, parent + n_nodes);
  t->node_off.assign(node_off, node_off + n_nodes);
  t->node_len.assign(node_len, node_len + n_nodes);
  t->leaf_of_seq.assign(leaf_of_seq, leaf_of_seq + B);
  t->depth.assign(n_nodes, -1);
  for (int n = 0; n < n_nodes; ++n) {  // depth by walking to the root; detects cycles
    int d = 0, x = n;
    while (x != root) {
      x = t->parent[x];
      if (++d > n_nodes) {
        delete t;
        return fail(HYDRA_ESHAPE, "cycle through node %d", n);
      }
    }
    t->depth[n] = d;
    if (n != root && t->node_len[n] < 1) {
      delete t;
      return fail(HYDRA_ESHAPE, "non-root node %d is empty (only the root may be empty, S:186)", n);
    }
  }
  std::vector<int> n_children(n_nodes, 0), n_users(n_nodes, 0);
  for (int n = 0; n < n_nodes; ++n)
    if (n != root) n_children[t->parent[n]]++;
  for (int64_t b = 0; b < B; ++b) {
    const int lf = leaf_of_seq[b];
    if (lf < 0 || lf >= n_nodes) {
      delete t;
      return fail(HYDRA_ESHAPE, "sequence %lld assigned to invalid node %d", (long long)b, lf);
    }
    if (n_children[lf]) {
      delete t;
      return fail(HYDRA_ESHAPE, "sequence %lld assigned to non-leaf node %d", (long long)b, lf);
    }
    n_users[lf]++;
  }
  for (int n = 0; n < n_nodes; ++n)
    if (!n_children[n] && !n_users[n]) {
      delete t;
      return fail(HYDRA_ESHAPE, "leaf node %d has no sequences (S:191)", n);
    }
  // CSR groups: ascending sequence ids of every sequence whose path passes through n
  std::vector<std::vector<int32_t>> groups(n_nodes);
  for (int64_t b = 0; b < B; ++b)
    for (int x = leaf_of_seq[b];; x = t->parent[x]) {
      groups[x].push_back((int32_t)b);
      if (x == root) break;
    }
  t->grp_off.assign(n_nodes + 1, 0);
  for (int n = 0; n < n_nodes; ++n) t->grp_off[n + 1] = t->grp_off[n] + (int32_t)groups[n].size();
  for (int n = 0; n < n_nodes; ++n) t->grp_seq.insert(t->grp_seq.end(), groups[n].begin(), groups[n].end());
  for (int n = 0; n < n_nodes; ++n) t->max_depth = std::max(t->max_depth, t->depth[n] + 1);
  if (cudaMalloc(&t->d_grp_seq, sizeof(int32_t) * std::max<size_t>(1, t->grp_seq.size())) != cudaSuccess ||
      cudaMemcpy(t->d_grp_seq, t->grp_seq.data(), sizeof(int32_t) * t->grp_seq.size(), cudaMemcpyHostToDevice) !=
          cudaSuccess) {
    cudaFree(t->d_grp_seq);
    delete t;
    return cuda_fail("tree device upload");
  }
  *out = t;
  return HYDRA_OK;
}

extern "C" void hydra_tree_destroy(struct hydra_tree *t) {
  if (!t) return;
  for (auto &kv : t->work)
    for (int k = 0; k < 2; ++k) cudaFree(kv.second.d[k]);
  cudaFree(t->d_grp_seq);
  delete t;
}

extern "C" int32_t hydra_tree_depth(const struct hydra_tree *t) { return t ? t->max_depth : -1; }

extern "C" int64_t hydra_tree_group_size(const struct hydra_tree *t, int32_t node) {
  if (!t || node < 0 || node >= t->n_nodes) return -1;
  return t->grp_off[node + 1] - t->grp_off[node];
}

// Builds and uploads the node-attention work lists for query groups of g rows per
// sequence (synchronous; the only device allocation of the tree path).
static hydra_status tree_prepare_g(const hydra_tree *t, int g) {
  std::lock_guard<std::mutex> lock(t->mu);
  if (t->work.count(g)) return HYDRA_OK;
  hydra_tree::Lists L;
  for (int k = 0; k < 2; ++k) {
    const int rows_per_task = k ? 256 : 128;
    std::vector<PrefixTask> tasks;
    for (int n = 0; n < t->n_nodes; ++n) {
      if (t->node_len[n] <= 0) continue;
      const int32_t ns_ = t->grp_off[n + 1] - t->grp_off[n];
      const int tiles = (int)(((int64_t)ns_ * g + rows_per_task - 1) / rows_per_task);
      for (int tl = 0; tl < tiles; ++tl)
        tasks.push_back(PrefixTask{t->node_off[n], t->node_len[n], t->grp_off[n], ns_, t->depth[n], tl});
    }
    L.n[k] = (int)tasks.size();
    if (tasks.empty()) continue;
    if (cudaMalloc(&L.d[k], sizeof(PrefixTask) * tasks.size()) != cudaSuccess ||
        cudaMemcpy(L.d[k], tasks.data(), sizeof(PrefixTask) * tasks.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
      hydra_status st = cuda_fail("tree work-list upload");
      cudaFree(L.d[0]);
      cudaFree(L.d[1]);
      return st;
    }
  }
  const_cast<hydra_tree *>(t)->work.emplace(g, L);
  return HYDRA_OK;
}

extern "C" hydra_status hydra_tree_prepare(struct hydra_tree *t, const hydra_heads *h) {
  if (!t) return fail(HYDRA_EINVAL, "tree is NULL");
  hydra_status st = check_heads(h);
  if (st) return st;
  return tree_prepare_g(t, h->num_q_heads / h->num_kv_heads);
}

static int tree_prefix_splits(const hydra_heads *h, const hydra_tree *t) {
  if (g_cfg.prefix_splits > 0) return (int)g_cfg.prefix_splits;
  if (!use_tc(h)) {
    int64_t maxlen = 0;
    for (auto L : t->node_len) maxlen = std::max(maxlen, L);
    return prefix_splits_simt(h, t->B, maxlen);
  }
  // total query tiles (v3: tile pairs) over all non-empty nodes; the longest node sets the work
  const int g = h->num_q_heads / h->num_kv_heads;
  const int rows_per = prefix_kind(h) == PK_TC2 ? 256 : 128;
  int64_t tiles = 0, maxlen = 0;
  for (int n = 0; n < t->n_nodes; ++n) {
    if (t->node_len[n] <= 0) continue;
    tiles += ((int64_t)(t->grp_off[n + 1] - t->grp_off[n]) * g + rows_per - 1) / rows_per;
    maxlen = std::max(maxlen, t->node_len[n]);
  }
  return prefix_splits_tc(tiles * h->num_kv_heads, maxlen);
}

// SM split for the tree: node attention (persistent tcgen05 kernel in task mode) on k SMs
// || tensor-core suffix on the rest.  Work units are
// 256-row x 128-token blocks; a node group whose last tile pair holds <= 128 rows runs one
// M=128 tile for it (half a unit).  Items are dealt whole, so a 10 % imbalance is allowed for.
static int tree_overlap_ctas(const hydra_heads *h, const struct hydra_tree *t, int64_t S_cap) {
  if (S_cap <= 0 || !use_suffix_tc(h, t->B, S_cap, true) || prefix_kind(h) != PK_TC2) return 0;
  const int sms = device_sm_count();
  if (g_cfg.overlap_prefix_ctas > 0) return (int)std::min<int64_t>(g_cfg.overlap_prefix_ctas, sms - 1);
  const int g = h->num_q_heads / h->num_kv_heads;
  double units = 0.0;
  for (int n = 0; n < t->n_nodes; ++n) {
    if (t->node_len[n] <= 0) continue;
    const int64_t r = (int64_t)(t->grp_off[n + 1] - t->grp_off[n]) * g;
    const double pairs = (double)(r / 256) + (r % 256 == 0 ? 0.0 : (r % 256 <= 128 ? 0.5 : 1.0));
    units += pairs * h->num_kv_heads * (double)((t->node_len[n] + 127) / 128);
  }
  // R_P measured for the task-mode kernel on C5 (tools/tree_overlap_sweep.py: 0.26-0.28 units
  // per us per SM on 15-64 SMs, below the flat kernel's 0.46: half-filled branch tiles,
  // per-item prologue/epilogue); the node side is kept at <= 1/2.3 of the suffix time
  // (interference and the power-capped clock slow it further when both run).  Measured at
  // C5 (tools/tree_overlap_sweep.py): 1.344 / 1.312 / 1.322 / 1.379 ms at k = 32 / 48 / 64 /
  // 80 vs 1.372 ms sequential; this picks k = 48.
  const double R_P = 0.27, R_S = 1.0e5, BW = 7.0e6;
  const double kv_bytes = (double)t->B * h->num_kv_heads * S_cap * h->head_dim * 4.0;
  int best_k = 0;
  double best = 1e300;
  for (int k = 4; k <= sms - 8; ++k) {
    const double tt = std::max(2.3 * 1.1 * units / (k * R_P), kv_bytes / std::min((sms - k) * R_S, BW));
    if (tt < best) {
      best = tt;
      best_k = k;
    }
  }
  return best_k;
}

extern "C" size_t hydra_tree_workspace_size(const hydra_heads *h, const struct hydra_tree *t, int64_t S_cap) {
  if (!t || check_heads(h) != HYDRA_OK) return 0;
  return part_bytes(h, t->B) * (size_t)(t->max_depth * tree_prefix_splits(h, t) + suffix_splits(h, t->B, S_cap));
}

static hydra_status tree_impl(const hydra_heads *h, const struct hydra_tree *t, const void *q, int64_t q_sb,
                              int64_t q_sh, const void *node_k, const void *node_v, int64_t kv_st, int64_t kv_sh,
                              const void *sk, const void *sv, int64_t s_sb, int64_t s_st, int64_t s_sh,
                              int64_t S_cap, const int32_t *lens, void *out, hydra_dtype out_dtype, float *lse_out,
                              void *ws, size_t ws_bytes, void *stream, void *stream_aux, const hydra_paging *pg) {
  hydra_status st = check_heads(h);
  if (st) return st;
  if (!t) return fail(HYDRA_EINVAL, "tree is NULL");
  const int64_t B = t->B;
  int64_t T = 0;
  for (int n = 0; n < t->n_nodes; ++n) T = std::max(T, t->node_off[n] + t->node_len[n]);
  if (!q || !out || (T > 0 && (!node_k || !node_v)) || (S_cap > 0 && (!sk || !sv || !lens)))
    return fail(HYDRA_EINVAL, "null pointer argument");
  if (out_dtype != HYDRA_BF16 && out_dtype != HYDRA_F32) return fail(HYDRA_EUNSUPPORTED, "out_dtype must be BF16 or F32");
  const size_t es = elem_size(h->dtype);
  if (!aligned16(q, es, {q_sb, q_sh}) || (T > 0 && (!aligned16(node_k, es, {kv_st, kv_sh}) || !aligned16(node_v, es, {}))) ||
      (S_cap > 0 && (!aligned16(sk, es, {s_sb, s_st, s_sh}) || !aligned16(sv, es, {}))))
    return fail(HYDRA_EINVAL, "q/k/v base pointers and strides must be 16-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaStream_t sa = stream_aux ? reinterpret_cast<cudaStream_t>(stream_aux) : s;
  const int k_over = (sa != s && T > 0) ? tree_overlap_ctas(h, t, S_cap) : 0;
  if (k_over == 0) sa = s;
  g_cfg.last_overlap_k = k_over;
  const int sms = device_sm_count();
  const int np = tree_prefix_splits(h, t);
  const int ns = suffix_splits(h, B, S_cap, k_over > 0);
  const int n_parts = t->max_depth * np + ns;
  const size_t need = part_bytes(h, B) * n_parts;
  if (!ws || ws_bytes < need) return fail(HYDRA_ENOMEM, "workspace too small: need %zu bytes", need);
  const int g = h->num_q_heads / h->num_kv_heads;
  const int64_t rows = B * h->num_q_heads;
  PartsView all = parts_in_ws(ws, h, B, n_parts);
  const PrefixKind kind = prefix_kind(h);
  // the node-attention work list (looked up before anything is launched)
  PrefixTask *d_tasks = nullptr;
  int n_tasks = 0;
  if (kind != PK_SIMT && T > 0) {
    std::unique_lock<std::mutex> lock(t->mu);
    auto it = t->work.find(g);
    if (it == t->work.end()) {
      lock.unlock();
      // Not prepared for this head grouping: build the lists now unless the stream is being
      // captured (an upload cannot be part of a graph) -- hydra_tree_prepare avoids this.
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(s, &cs);
      if (cs != cudaStreamCaptureStatusNone)
        return fail(HYDRA_EINVAL, "tree not prepared for Hq/Hkv = %d: call hydra_tree_prepare before capture", g);
      st = tree_prepare_g(t, g);
      if (st) return st;
      lock.lock();
      it = t->work.find(g);
    }
    const int k = kind == PK_TC2 ? 1 : 0;
    d_tasks = it->second.d[k];
    n_tasks = it->second.n[k];
  }
  // Sequences whose path is shorter than max_depth leave slots empty: mark all node slots -inf.
  st = launch_fill_neg_inf(all.lse, all.lse_stride * (int64_t)(t->max_depth * np), s);
  if (st) return cuda_fail("fill");
  if (sa != s) {
    if (cudaEventRecord(events().fork, s) != cudaSuccess || cudaStreamWaitEvent(sa, events().fork, 0) != cudaSuccess)
      return cuda_fail("fork");
  }
  const float sl2 = scale_of(h) * 1.4426950408889634f;

  if (kind != PK_SIMT && T > 0) {
    if (n_tasks > 0) {
      PrefixTcArgs a{};
      a.q = q;
      a.q_sb = q_sb;
      a.q_sh = q_sh;
      a.k = node_k;
      a.v = node_v;
      a.kv_st = kv_st;
      a.kv_sh = kv_sh;
      a.kv_total = T;
      a.Hq = h->num_q_heads;
      a.Hkv = h->num_kv_heads;
      a.g = g;
      a.scale_log2 = sl2;
      a.tasks = d_tasks;
      a.n_tasks = n_tasks;
      a.seq_list = t->d_grp_seq;
      a.n_splits = np;
      a.o = all.o;
      a.lse = all.lse;
      a.o_slot_stride = all.o_stride;
      a.lse_slot_stride = all.lse_stride;
      a.debug_variant = (int32_t)g_cfg.tc_debug;
      a.trace = reinterpret_cast<void *>((intptr_t)g_cfg.prefix_trace);
      a.stages = (int32_t)g_cfg.prefix_stages;
      a.poly_every = (int32_t)g_cfg.prefix_poly;
      a.variant = (int32_t)g_cfg.prefix_variant;
      a.mutate = (int32_t)g_cfg.mutate;
      // the work list holds 256-row tile pairs for v3 and 128-row tiles for v1
      st = kind == PK_TC2 ? launch_prefix_tc2(a, k_over > 0 ? k_over : prefix_ctas(), sa) : launch_prefix_tc(a, sa);
      if (st) return cuda_fail("tree prefix tcgen05 launch");
    }
  } else {
    for (int n = 0; n < t->n_nodes; ++n) {
      if (t->node_len[n] <= 0) continue;
      DecodeParams p{};
      p.q = q;
      p.q_sb = q_sb;
      p.q_sh = q_sh;
      p.k = node_k;
      p.v = node_v;
      p.kv_sb = 0;
      p.kv_st = kv_st;
      p.kv_sh = kv_sh;
      p.kv_tok_off = t->node_off[n];
      p.lens = nullptr;
      p.len_uniform = t->node_len[n];
      p.seq_map = t->d_grp_seq + t->grp_off[n];
      p.n_seq = t->grp_off[n + 1] - t->grp_off[n];
      p.Hq = h->num_q_heads;
      p.Hkv = h->num_kv_heads;
      p.g = g;
      p.scale_log2 = sl2;
      p.n_splits = np;
      p.split_len = (t->node_len[n] + np - 1) / np;
      p.heads_per_cta = heads_per_cta(g);
      p.o = all.o + all.o_stride * (int64_t)(t->depth[n] * np);
      p.lse = all.lse + all.lse_stride * (int64_t)(t->depth[n] * np);
      p.o_split_stride = all.o_stride;
      p.lse_split_stride = all.lse_stride;
      st = launch_decode(p, h->dtype, h->head_dim, sa);
      if (st) return st == HYDRA_ECUDA ? cuda_fail("tree node SIMT launch") : fail(st, "tree node SIMT");
    }
  }
  PartsView suf = all;
  suf.o = all.o + all.o_stride * (int64_t)(t->max_depth * np);
  suf.lse = all.lse + all.lse_stride * (int64_t)(t->max_depth * np);
  if (S_cap > 0) {
    st = run_suffix(h, B, q, q_sb, q_sh, sk, sv, s_sb, s_st, s_sh, S_cap, lens, ns, suf, s,
                    k_over > 0 ? std::max(1, sms - k_over) : 0, pg);
    if (st) return st;
  } else {
    st = launch_fill_neg_inf(suf.lse, rows, s);
    if (st) return cuda_fail("fill");
  }
  if (sa != s) {
    if (cudaEventRecord(events().join, sa) != cudaSuccess || cudaStreamWaitEvent(s, events().join, 0) != cudaSuccess)
      return cuda_fail("join");
  }
  return run_combine(rows, h->head_dim, n_parts, all, out, out_dtype, lse_out, s);
}

extern "C" hydra_status hydra_tree_attn(const hydra_heads *h, const struct hydra_tree *t, const void *q, int64_t q_sb,
                                        int64_t q_sh, const void *node_k, const void *node_v, int64_t kv_st,
                                        int64_t kv_sh, const void *sk, const void *sv, int64_t s_sb, int64_t s_st,
                                        int64_t s_sh, int64_t S_cap, const int32_t *lens, void *out,
                                        hydra_dtype out_dtype, float *lse_out, void *ws, size_t ws_bytes,
                                        void *stream, void *stream_aux) {
  return tree_impl(h, t, q, q_sb, q_sh, node_k, node_v, kv_st, kv_sh, sk, sv, s_sb, s_st, s_sh, S_cap, lens, out,
                   out_dtype, lse_out, ws, ws_bytes, stream, stream_aux, nullptr);
}

extern "C" hydra_status hydra_tree_attn_paged(const hydra_heads *h, const struct hydra_tree *t, const void *q,
                                              int64_t q_sb, int64_t q_sh, const void *node_k, const void *node_v,
                                              int64_t kv_st, int64_t kv_sh, const void *k_pool, const void *v_pool,
                                              int64_t p_sp, int64_t p_st, int64_t p_sh, const hydra_paging *pg,
                                              int64_t S_cap, const int32_t *lens, void *out, hydra_dtype out_dtype,
                                              float *lse_out, void *ws, size_t ws_bytes, void *stream,
                                              void *stream_aux) {
  if (S_cap > 0) {
    hydra_status st = check_paging(pg, S_cap);
    if (st) return st;
  }
  return tree_impl(h, t, q, q_sb, q_sh, node_k, node_v, kv_st, kv_sh, k_pool, v_pool, p_sp, p_st, p_sh, S_cap, lens,
                   out, out_dtype, lse_out, ws, ws_bytes, stream, stream_aux, S_cap > 0 ? pg : nullptr);
}

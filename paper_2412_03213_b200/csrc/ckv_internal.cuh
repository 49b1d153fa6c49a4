// ckv_internal.cuh — launch wrappers shared between the kernel files and the
// C-ABI (ckv_capi.cu).  Internal; not part of the installed interface.
#pragma once
#include "ckv_common.cuh"

struct ckv_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint64_t launches = 0;
  // pinned host scratch for small control read-backs
  int32_t* h_flags = nullptr;
  size_t h_flags_cap = 0;
  // grow-only device scratch slots reused across calls on this context
  // (cudaMalloc / cudaFree of ~0.5 GB per k-means call cost milliseconds and
  // device-wide synchronisation)
  // slots: 1-21 k-means, 22 relayout, 23 page, 24-26 attend, 27-28 metrics,
  // 29 prefill init rows, 30-33 decode batch, 34 select, 35-36 cache, 37 misc
  static constexpr int kScratchSlots = 48;
  void* scratch[kScratchSlots];  // zeroed in ckv_ctx_create
  size_t scratch_cap[kScratchSlots];
  // a second context on the same device (own non-blocking stream and
  // scratch), created on first use: kmeans_run runs half of the units there
  // from a second host thread, so one half's latency-bound update / fix-up /
  // index kernels overlap the other half's tensor-core assignment
  ckv_ctx* aux = nullptr;
};

namespace ckvb {

// CKV_TRACE_HOST=1: host-side timestamps of the phases of a long call
// (prefill) on stderr, relative to the last trace_begin on this thread; no
// extra synchronisation, so the traced run is the untraced run
bool trace_on();
void trace_begin(const char* what);
void trace_mark(const char* what, long arg = -1);

int launch_index(cudaStream_t st, uint32_t n_units, const int32_t* labels, uint32_t n_pos,
                 uint32_t p_cap, uint32_t c_cap, const uint32_t* n_clusters,
                 uint32_t c_uniform, uint32_t* sizes, uint32_t* starts, uint32_t* sorted_ids,
                 const int32_t* prev_labels, int32_t* changed, const int32_t* active,
                 int32_t* any_empty, uint8_t* dirty = nullptr);

// k-means driver (ckv_kmeans.cu); keys may be strided per unit
struct KMeansArgs {
  uint32_t n_units, n, C, max_iters;
  uint64_t key_stride;      // elements between units' keys
  uint32_t c_stride;        // centroid rows between units
  uint32_t label_stride;    // labels between units
  uint32_t flags;
  const uint16_t* keys;
  const uint32_t* init_rows;  // device [n_units*C]
  float* centroids;
  int32_t* labels;
};
int kmeans_run(ckv_ctx* ctx, const KMeansArgs& a, ckv_kmeans_info* info_host,
               double* objective_host, uint32_t* repair_host);

// single kernels of the k-means pass, for the sequence-sharded driver
// (ckv_kmshard.cu); defined in ckv_kmeans.cu / ckv_assign_tc.cu
// the tensor-core key operands in assign_tc's scratch (assign_tc_keyprep)
struct TcKeyPrep {
  float* knorm;    // [unit][n] |k| + |k - h(k)|, rounded up (band scale)
  uint16_t* k16;   // [unit][n_pad][128] h(k), fp16 bits
  uint32_t n_pad;
  uint32_t* kerr;  // [unit] max_k |k - h(k)| as float bits (zero before the scan)
};
int launch_scan_keys(cudaStream_t st, const uint16_t* keys, uint64_t key_stride, uint32_t n,
                     uint32_t n_units, int32_t* flags, const TcKeyPrep* prep);
int launch_assign(cudaStream_t st, bool use_tc, const uint16_t* keys, uint64_t key_stride,
                  uint32_t n, uint32_t C, uint32_t c_pad, uint32_t n_units,
                  const uint16_t* dirs16, const float* deps, const float* dirs, int32_t* labels,
                  uint32_t label_stride, const int32_t* active, void* tc_scratch,
                  size_t tc_bytes, uint64_t* launches);
int launch_objective(cudaStream_t st, const uint16_t* keys, uint64_t key_stride, uint32_t n,
                     uint32_t n_units, uint32_t c_stride, uint32_t c_pad, const int32_t* labels,
                     uint32_t label_stride, const float* cents, const double* cnorm, double* obj,
                     const int32_t* active);
size_t assign_tc_scratch_bytes(uint32_t n_units, uint32_t n, uint32_t C);
// cluster_decode_batch's k-means in one launch (rows <= 512, C <= 32)
bool kmeans_small_supported(uint32_t rows, uint32_t C);
int launch_kmeans_small(cudaStream_t st, const uint16_t* keys, uint64_t key_stride,
                        uint32_t n_units, uint32_t rows, uint32_t C, uint32_t max_iters,
                        const uint32_t* init_rows, float* cents, uint32_t c_cap,
                        int32_t* labels, uint32_t label_stride, uint32_t* n_clusters,
                        uint32_t* iters, int32_t* status);
TcKeyPrep assign_tc_keyprep(void* scratch, uint32_t n_units, uint32_t n);
bool assign_tc_supported(uint32_t n, uint32_t C);
// moved-cluster reduced assignment (ckv_assign_tc.cu), passes t >= 2
bool mcr_enabled();
int assign_mcr(ckv_ctx* ctx, const uint16_t* keys, uint64_t key_stride, uint32_t n, uint32_t C,
               uint32_t c_pad, uint32_t n_units, uint32_t c_stride, const uint16_t* dirs16,
               const float* deps, const float* dirs, const int32_t* prev, int32_t* cur,
               uint32_t label_stride, const int32_t* active, const uint8_t* moved,
               const uint32_t* sorted, void* tc_scratch, size_t tc_bytes);

}  // namespace ckvb

namespace ckvb {
// internal ckv_select_desc flag: take the fused (smem-only) selection kernel
// whatever the unit count (the session's concurrent slices: the unfused path
// shares one scratch buffer)
constexpr uint32_t CKV_SEL_FORCE_FUSED = 0x80000000u;
// the session's selection may stream the centroids / sizes / starts before
// its grid dependency wait: no kernel since the previous selection wrote them
// (the step's previous kernel is the append or an attention)
constexpr uint32_t CKV_SEL_EARLY = 0x40000000u;
struct CacheDev {
  uint32_t n_slots, c_cap, retention, d, words;
  uint32_t* bits;                // [n_slots][retention][words]
  uint32_t* ring;                // [n_slots][2] = head, len
  unsigned long long* counters;  // [n_slots][4]
};
// Per-q-head hand-off from the selection to the attention of one step, so
// the attention need not wait for the whole selection grid: the selection
// publishes ready[h] = *epoch + 1 (release) once head h's runs and token
// count are stored, the attention polls it (acquire) per work item.  epoch
// is a device counter the step's last kernel (k_append_kv) advances, so the
// protocol holds under graph replay.  published: set by launch_select when
// the path it took publishes (the fused kernel); the attention uses the flags
// only then.
struct StepSync {
  uint32_t* ready = nullptr;         // [n_q]
  uint32_t* epoch = nullptr;         // [1]
  // the attention's work counter for this launch (items handed out in
  // selection order, so no CTA holds an item whose head is still being
  // selected while published heads wait); zeroed by the step's last kernel
  uint32_t* work = nullptr;
  bool published = false;
  // the step's K/V append (harness.hpp:318-320), folded into the fused
  // selection: each unit's leader CTA copies its new row (k, v: this slice's
  // first unit; possibly mapped host memory) to K/V row pos, which no kernel
  // of this step reads (the recency range ends at pos).  Set `appended` when
  // the launch took it; otherwise k_append_kv copies the row.
  const uint16_t* app_k = nullptr;
  const uint16_t* app_v = nullptr;
  uint16_t* K = nullptr;
  uint16_t* V = nullptr;
  uint32_t app_pos = 0, p_cap = 0;
  bool appended = false;
};
// the fused selection's append operand (a null k skips it)
struct SelAppend {
  const uint16_t* k;
  const uint16_t* v;
  uint16_t* K;
  uint16_t* V;
  uint32_t pos, p_cap;
};
// fp16 copy of a centroid block for the fused selection's approximate
// scores: c16[u][c] = RN_fp16(mu_c) and cerr[u][c] >= |mu_c - c16[u][c]|_2
// (components saturate at +-65504 and the bound grows with them; +inf when
// it is not finite)
struct SelC16 {
  const uint16_t* c16;
  const float* cerr;
};
// rows [0, n_clusters[u]) of every unit, or (tail > 0) only the last tail of them
int launch_cents_f16(cudaStream_t st, const float* cents, const uint32_t* n_clusters,
                     uint32_t n_units, uint32_t c_cap, uint16_t* c16, float* cerr,
                     uint32_t tail = 0);
int launch_select(cudaStream_t st, const ckv_select_desc& desc, const float* q,
                  const float* cents, const uint32_t* n_clusters, const uint32_t* sizes,
                  const uint32_t* starts, const uint32_t* sorted_ids, uint32_t* token_ids,
                  uint32_t* rows, const ckv_runs& runs, uint32_t row_base, uint32_t* n_tokens,
                  uint32_t* n_taken, uint32_t* trimmed, uint32_t* ranked, double* scores,
                  const CacheDev& cache, void* scratch, float* q_copy = nullptr,
                  StepSync* sync = nullptr, const SelC16* c16 = nullptr);
size_t select_scratch_bytes(uint32_t n_q, uint32_t c_cap);
int launch_score_approx(cudaStream_t st, uint32_t G, uint32_t n_units, const float* q,
                        const float* cents, const uint32_t* counts, uint32_t c_cap,
                        uint32_t c_pad, float* aval, float* aerr);
int launch_cache_lookup(cudaStream_t st, const CacheDev& cache, uint32_t slot,
                        const uint32_t* sel, uint32_t n_sel, const uint32_t* sizes,
                        uint32_t* hit, uint32_t* miss, uint32_t* counts);
int launch_cache_invalidate(cudaStream_t st, const CacheDev& cache, uint32_t slot,
                            const uint32_t* retired, uint32_t n);
int launch_attend(cudaStream_t st, const ckv_attend_desc& desc, const float* q,
                  const uint16_t* K, const uint16_t* V, const uint32_t* rows,
                  const ckv_runs& runs, const uint32_t* n_tokens, float* out, float* weights,
                  float* logits_ws, float* part, uint32_t* tickets, float* lse = nullptr,
                  const StepSync* sync = nullptr);
size_t attend_part_floats(uint32_t n_q, uint32_t max_tokens);
// the current device's persisting-L2 limit (cached; ckv_capi.cu)
size_t l2_persist_limit();
int ctx_scratch(ckv_ctx* ctx, int slot, size_t bytes, bool zero_new, void** out);
int attend_scratch(ckv_ctx* ctx, const ckv_attend_desc& d, bool weights, float** part,
                   uint32_t** tickets, float** lw);
uint64_t host_mix_seed(uint64_t seed, uint64_t a, uint64_t b);
// cudaFuncSetAttribute(fn, MaxDynamicSharedMemorySize, bytes) (plus the
// max-shared carveout when asked) once per (kernel, device, bytes); safe to
// call from several host threads and for contexts on different devices
cudaError_t smem_optin(const void* fn, int bytes, bool max_carveout = false);
void host_init_rows(uint32_t n, uint32_t C, uint64_t seed, uint32_t* rows);
}  // namespace ckvb

namespace ckvb {
// the physical two-tier cluster cache (ckv_tier.cu)
constexpr uint32_t TIER_PAGE_ROWS = 16;
struct TierArgs {
  uint32_t n_units_total, p_cap, c_cap, np, group, retention, sink;
  const uint32_t* n_clusters;
  const uint32_t* sizes;
  const uint32_t* starts;
  const uint16_t* back_K;  // backing tier: [unit][p_cap][128] (device store or mapped host mirror)
  const uint16_t* back_V;
  int32_t* cpage;          // [unit][c_cap] first pool page of a resident cluster, -1 if absent
  uint32_t* last;          // [unit][c_cap] last step the unit selected the cluster
  int32_t* next;           // [unit][np] page chain
  int32_t* free_stack;     // [unit][np]
  int32_t* n_free;         // [unit]
  unsigned long long* stats;  // [unit][4]: rows fetched, clusters fetched, clusters selected, evictions
  int32_t* status;         // pool exhausted -> 1
};
int launch_tier_init(cudaStream_t st, const TierArgs& a, uint32_t n_units);
int launch_tier_fetch(cudaStream_t st, const TierArgs& a, uint32_t u0, uint32_t n_units,
                      uint32_t step, const ckv_runs& runs, const ckv_runs& out,
                      const uint32_t* ranked, const uint32_t* n_taken, uint16_t* K,
                      uint16_t* V);
}  // namespace ckvb

struct ckv_cache {
  ckv_ctx* ctx;
  ckvb::CacheDev dev;
};

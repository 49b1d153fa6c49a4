/*
 * ckv_cuda.h — C-ABI of the B200-native ClusterKV hot path (libckv_b200.so).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * Device pointers are raw CUDA device addresses on the context's device.
 * Every entry point returns CKV_OK (0) or a CKV_E* status and never throws;
 * ckv_last_error() returns the message for the calling thread.
 *
 * Each entry point replaces one reference function from
 * /root/reference/proj/include/clusterkv/*.hpp, cited per declaration.
 * The reference-signature C++ drop-in (include/clusterkv_b200/clusterkv.hpp)
 * and the Python mirror (paper_2412_03213_b200/api.py) both sit on this ABI.
 *
 * Layout conventions:
 *   "unit"     = one (batch, layer, kv-head) k-means / KV problem
 *   "q head"   = one query; q head h reads kv unit h / group (GQA)
 *   keys, values: bf16 (uint16 bit patterns), row-major [unit][p_cap][d]
 *   centroids:   f32 [unit][c_cap][d]  (raw means, never renormalised)
 *   labels:      i32 [unit][p_cap]     (-1 = sink / not yet clustered)
 *   index:       sizes u32 [unit][c_cap], starts u32 [unit][c_cap+1],
 *                sorted_ids u32 [unit][p_cap]
 *   d must be 128 (Llama-3 head dim; the only shape the kernels specialise).
 */
#ifndef CKV_CUDA_H
#define CKV_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKV_OK 0
#define CKV_EINVAL 1   /* maps to ckv::ValidationError (same predicates)   */
#define CKV_ECUDA 2    /* CUDA runtime / launch failure                    */
#define CKV_ENOMEM 3   /* device allocation failure                        */
#define CKV_ENCCL 4    /* collective failure (sequence-sharded paths)      */

#define CKV_HEAD_DIM 128

typedef struct ckv_ctx ckv_ctx;
typedef struct ckv_cache ckv_cache;
typedef struct ckv_session ckv_session;

/* ------------------------------------------------------------------ */
/* context                                                             */
/* ------------------------------------------------------------------ */
/* stream: the cudaStream_t to launch on; NULL = the legacy default stream.
 * A context is single-threaded; use one context per host thread
 * (the reference calls the hot path concurrently per head,
 * harness.hpp:362-378). */
int ckv_ctx_create(int device, void* stream, ckv_ctx** out);
int ckv_ctx_destroy(ckv_ctx* ctx);
int ckv_ctx_sync(ckv_ctx* ctx);
void* ckv_ctx_stream(ckv_ctx* ctx);
const char* ckv_last_error(void);
/* number of hot-path kernels this context has launched (bench evidence) */
uint64_t ckv_ctx_launch_count(ckv_ctx* ctx);

/* device memory helpers (the C++ shim uses these; no torch) */
int ckv_malloc(ckv_ctx* ctx, void** ptr, size_t bytes);
int ckv_free(ckv_ctx* ctx, void* ptr);
int ckv_memcpy_h2d(ckv_ctx* ctx, void* dst, const void* src, size_t bytes);
int ckv_memcpy_d2h(ckv_ctx* ctx, void* dst, const void* src, size_t bytes);
int ckv_memset(ckv_ctx* ctx, void* dst, int value, size_t bytes);
/* f32 -> bf16 (RNE) on device; also reports whether every value was
 * bf16-representable (exact) in *all_exact_host (may be NULL). */
int ckv_f32_to_bf16(ckv_ctx* ctx, const float* src, uint16_t* dst, size_t n,
                    int* all_exact_host);

/* ------------------------------------------------------------------ */
/* k-means (clustering.hpp:157-263, 265-332)                           */
/* ------------------------------------------------------------------ */
/* Host-side init sampling, bit-identical to kmeans_cosine's partial
 * Fisher-Yates over std::mt19937_64(seed) (clustering.hpp:186-193). */
int ckv_kmeans_init_rows(uint32_t n, uint32_t C, uint64_t seed, uint32_t* rows_out);
uint64_t ckv_mix_seed(uint64_t seed, uint64_t a, uint64_t b); /* common.hpp:108-113 */

typedef struct {
  uint32_t n_units;      /* independent problems                          */
  uint32_t n;            /* keys per unit                                 */
  uint32_t C;            /* clusters per unit (1 <= C <= n)               */
  uint32_t max_iters;    /* ClusterConfig::max_iters                      */
  uint64_t key_stride;   /* elements between consecutive units' keys      */
  uint32_t c_stride;     /* centroid rows between units (>= C)            */
  uint32_t label_stride; /* labels between units (>= n)                   */
  uint32_t flags;        /* CKV_KM_* below                                */
} ckv_kmeans_desc;

#define CKV_KM_OBJECTIVE 1u   /* fill objective_history (diagnostic)        */
#define CKV_KM_EXACT_ONLY 2u  /* force the CUDA-core exact assignment path  */
#define CKV_KM_NO_VALIDATE 4u /* skip the finite / non-degenerate check     */

typedef struct {
  uint32_t iterations_used;  /* ClusterModel::iterations_used            */
  int32_t converged;         /* ClusterModel::converged                  */
  uint32_t n_repair;         /* entries in repair_iterations             */
  uint32_t n_objective;      /* entries in objective_history             */
} ckv_kmeans_info;

/* Batched kmeans_cosine (clustering.hpp:160-263), cosine metric.
 * keys: device bf16; init_rows: device u32 [n_units*C] (from
 * ckv_kmeans_init_rows or the caller's init_rows); outputs on device.
 * info_host: host array [n_units]; objective_host: host f64
 * [n_units*(max_iters+1)] or NULL; repair_host: host u32
 * [n_units*(max_iters+1)] or NULL.  Replaces kmeans_cosine.
 * A call of >= 16 units (here and in ckv_cluster_prefill) runs its two
 * halves concurrently: the second on an internal context of ctx's device
 * (own stream and scratch, created on first use, freed by ckv_ctx_destroy)
 * from an internal host thread; the call returns after both, with ctx's
 * stream ordered after the second half's work.  Results are those of the
 * one-stream run (units are independent).  CKV_KM_OVERLAP=0 disables it. */
int ckv_kmeans(ckv_ctx* ctx, const ckv_kmeans_desc* desc, const uint16_t* keys,
               const uint32_t* init_rows, float* centroids, int32_t* labels,
               ckv_kmeans_info* info_host, double* objective_host, uint32_t* repair_host);

/* Batched cluster_prefill (clustering.hpp:278-305): units share L; rows
 * [0,sink) get label -1, rows [sink,L) are clustered into C0 =
 * prefill_cluster_count(L) clusters with seed seeds_host[u].
 * keys [unit][p_cap][128], labels [unit][p_cap], centroids [unit][c_cap][128]. */
typedef struct {
  uint32_t n_units, L, p_cap, c_cap;
  uint32_t c0_divisor, sink_tokens, max_iters, c0_override;
  uint32_t flags;  /* CKV_KM_* */
} ckv_prefill_desc;
uint32_t ckv_prefill_cluster_count(uint32_t L, uint32_t c0_divisor, uint32_t sink_tokens,
                                   uint32_t c0_override);   /* clustering.hpp:267-274 */
int ckv_cluster_prefill(ckv_ctx* ctx, const ckv_prefill_desc* desc, const uint16_t* keys,
                        const uint64_t* seeds_host, float* centroids, int32_t* labels,
                        uint32_t* n_clusters /* device [n_units] */,
                        ckv_kmeans_info* info_host, double* objective_host,
                        uint32_t* repair_host);

/* Batched cluster_decode_batch (clustering.hpp:310-332): each unit's rows
 * [pos0, pos0+rows) of keys are clustered in isolation into
 * C+ = min(c_plus, rows) clusters, seed mix_seed(seeds_host[u], 0xdecade,
 * pos0); centroids appended at n_clusters[u], labels written with the
 * fresh ids, n_clusters[u] += C+.  Device-resident, no host round trip
 * except the init sampling. */
typedef struct {
  uint32_t n_units, pos0, rows, p_cap, c_cap, c_plus, max_iters;
} ckv_decode_cluster_desc;
int ckv_cluster_decode_batch(ckv_ctx* ctx, const ckv_decode_cluster_desc* desc,
                             const uint16_t* keys, const uint64_t* seeds_host,
                             float* centroids, int32_t* labels, uint32_t* n_clusters,
                             uint32_t* iterations_host /* [n_units] or NULL */);

/* ------------------------------------------------------------------ */
/* sequence-sharded k-means                     */
/* ------------------------------------------------------------------ */
/* kmeans_cosine (clustering.hpp:160-263) of one very long head whose N keys
 * are split into contiguous position shards, one per rank.  Each rank holds
 * its shard's keys; the caller runs the reference's loop and supplies the
 * collectives between these per-shard steps (paper_2412_03213_b200/
 * sharded.py: NCCL over NVLink in production, gloo in the CPU tests):
 *
 *   validate            -> allreduce MAX stat[:,1:3]
 *   init(rows, row_lo)  -> allreduce SUM sums; update(from_init = 1)
 *   pass 0:  assign(0) -> allreduce SUM counts; repair; finish(0)
 *   pass t:  partial_sums -> allreduce SUM sums; update(0);
 *            assign(t) -> allreduce SUM counts; repair;
 *            finish(t) -> allreduce MAX stat[:,0] (changed), SUM objective
 *   repair (clustering.hpp:128-153), per unit with an empty cluster, per
 *            empty id ascending: largest = first argmax of the global
 *            counts; farthest(unit, largest) on every rank -> all-gather
 *            (distance, global row) -> max distance, lowest row wins ->
 *            move() on the owner; counts updated identically everywhere.
 *
 * f64 sums of bf16 keys are exact in any order, so the
 * all-reduced sums, hence the centroids, labels and iteration counts, are
 * bit-identical to the single-process reference for any shard count.  All
 * units of one call advance in lock step; set_active freezes the
 * converged ones. */
typedef struct ckv_kmshard ckv_kmshard;
typedef struct {
  uint32_t n_units;     /* heads clustered together                        */
  uint32_t n_local;     /* keys of this shard per unit (>= 1)              */
  uint32_t C;           /* clusters per unit (1 <= C <= global N)          */
  uint32_t flags;       /* CKV_KM_EXACT_ONLY                               */
  uint64_t key_stride;  /* elements between consecutive units' keys        */
} ckv_kmshard_desc;

/* Collective buffers, device memory owned by the caller (the collectives
 * run on them in place). */
typedef struct {
  double* sums;       /* [n_units][C][128] partial member sums  (SUM)      */
  int32_t* counts;    /* [n_units][C] member counts              (SUM)      */
  int32_t* stat;      /* [n_units][4]: changed, non-finite, non-zero row, 0 (MAX) */
  double* objective;  /* [n_units] objective partial             (SUM)      */
} ckv_kmshard_bufs;

int ckv_kmshard_create(ckv_ctx* ctx, const ckv_kmshard_desc* desc, const uint16_t* keys,
                       const ckv_kmshard_bufs* bufs, ckv_kmshard** out);
int ckv_kmshard_destroy(ckv_kmshard* sh);
/* kmeans_cosine's input checks (clustering.hpp:166-172), this shard's part */
int ckv_kmshard_validate(ckv_kmshard* sh);
/* sums[u][c] = key row init_rows_host[u*C + c] (global row ids) if this
 * shard [row_lo, row_lo + n_local) owns it, else 0 (clustering.hpp:195-198) */
int ckv_kmshard_init(ckv_kmshard* sh, const uint32_t* init_rows_host, uint64_t row_lo);
int ckv_kmshard_set_active(ckv_kmshard* sh, const int32_t* active_host);
/* centroids = float(sums / counts) (/ 1 when from_init), then the next
 * assignment's directions (clustering.hpp:205-218, 79-83) */
int ckv_kmshard_update(ckv_kmshard* sh, int from_init);
/* assignment pass `pass` of the local keys; local member counts -> counts */
int ckv_kmshard_assign(ckv_kmshard* sh, uint32_t pass);
/* after the counts all-reduce: any_empty_host[u] = some cluster has 0 members */
int ckv_kmshard_empty(ckv_kmshard* sh, int32_t* any_empty_host);
/* the local member of `cluster` farthest from its centroid (first maximum);
 * *row_host = -1 when no local member beats distance -1 */
int ckv_kmshard_farthest(ckv_kmshard* sh, uint32_t unit, uint32_t cluster, double* dist_host,
                         int64_t* row_host);
int ckv_kmshard_move(ckv_kmshard* sh, uint32_t unit, uint32_t local_row, uint32_t cluster);
/* local index of the (repaired) labels, changed-vs-previous -> stat[u][0]
 * (pass > 0), objective partial (want_objective) */
int ckv_kmshard_finish(ckv_kmshard* sh, uint32_t pass, int want_objective);
/* f64 member sums of the current labels -> sums */
int ckv_kmshard_partial_sums(ckv_kmshard* sh);
/* final model: centroids [n_units][C][128] (replicated), this shard's
 * labels [n_units][n_local] from pass iters_host[u]; device pointers */
int ckv_kmshard_result(ckv_kmshard* sh, const uint32_t* iters_host, float* centroids,
                       int32_t* labels);

/* Communicators of the sequence-sharded paths (ckv_comm.cu).
 *   NCCL:  one rank per GPU (process or thread); rank 0 makes an id with
 *          ckv_comm_nccl_id and the caller hands it to every rank, which
 *          calls ckv_comm_create_nccl (ncclCommInitRank).  The collectives
 *          run in place on device buffers on the context's stream.  libnccl
 *          is loaded at run time; CKV_ENCCL when it is missing or fails.
 *   LOCAL: the ranks are threads of one process sharing a ckv_local_group
 *          (collectives staged through host memory): several ranks on one
 *          GPU, e.g. tests (NCCL refuses duplicate devices).
 * Every rank of a communicator must make the same sequence of calls. */
typedef struct ckv_comm ckv_comm;
typedef struct ckv_local_group ckv_local_group;
#define CKV_NCCL_ID_BYTES 128
#define CKV_DT_I32 0
#define CKV_DT_F64 1
#define CKV_OP_SUM 0
#define CKV_OP_MAX 1
int ckv_comm_nccl_id(unsigned char* id_out /* CKV_NCCL_ID_BYTES */);
int ckv_comm_create_nccl(ckv_ctx* ctx, int world, int rank, const unsigned char* id,
                         ckv_comm** out);
int ckv_local_group_create(int world, ckv_local_group** out);
int ckv_local_group_destroy(ckv_local_group* g);
int ckv_comm_create_local(ckv_ctx* ctx, ckv_local_group* g, int rank, ckv_comm** out);
int ckv_comm_destroy(ckv_comm* c);
int ckv_comm_world(const ckv_comm* c, int* world, int* rank);
/* in place, device buffer of `count` CKV_DT_* elements, CKV_OP_SUM / MAX */
int ckv_comm_allreduce(ckv_comm* c, void* dev, size_t count, int dtype, int op);
/* recv [world][bytes] <- every rank's send [bytes]; device buffers */
int ckv_comm_allgather(ckv_comm* c, const void* send, void* recv, size_t bytes);

/* kmeans_cosine (clustering.hpp:160-263) of n_units heads whose n_total keys
 * are position-sharded over the communicator's ranks: this rank holds rows
 * [row_lo, row_lo + desc->n_local) of every unit at `keys` (device bf16,
 * unit stride desc->key_stride).  The whole reference loop runs here, the
 * per-shard steps above with the collectives between them (sharded.py is
 * the same protocol over torch.distributed).  seeds_host [n_units] (the
 * reference's init_rows draw) or init_rows_host [n_units*C] (global rows).
 * Outputs on the device: centroids [n_units][C][128], identical on every
 * rank; labels [n_units][n_local] of this shard.  Bit-identical to the
 * single-process kmeans_cosine for any shard count. */
int ckv_kmeans_sharded(ckv_comm* comm, const ckv_kmshard_desc* desc, const uint16_t* keys,
                       uint64_t n_total, uint64_t row_lo, const uint64_t* seeds_host,
                       const uint32_t* init_rows_host, uint32_t max_iters, float* centroids,
                       int32_t* labels, ckv_kmeans_info* info_host);

/* ------------------------------------------------------------------ */
/* index (selection.hpp:16-48)                                         */
/* ------------------------------------------------------------------ */
/* Stable counting sort of labels[unit][0:n_pos] into the ClusterIndex
 * layout.  n_clusters: device [n_units].  Replaces build_index. */
int ckv_build_index(ckv_ctx* ctx, uint32_t n_units, uint32_t n_pos, uint32_t p_cap,
                    uint32_t c_cap, const int32_t* labels, const uint32_t* n_clusters,
                    uint32_t* sizes, uint32_t* starts, uint32_t* sorted_ids);

/* ------------------------------------------------------------------ */
/* selection + cache (selection.hpp:50-111, cache.hpp:25-93)           */
/* ------------------------------------------------------------------ */
typedef struct {
  uint32_t n_q;        /* q heads                                        */
  uint32_t group;      /* q heads per kv unit                            */
  uint32_t budget;     /* B                                              */
  uint32_t sink_count; /* ids 0..sink_count-1 appended after clusters    */
  uint32_t p_cap, c_cap;
  uint32_t sel_cap;    /* token-id slots per q head                      */
  uint32_t rec_begin;  /* recency positions [rec_begin, rec_end)         */
  uint32_t rec_end;    /*   appended after the sinks (harness.hpp:246)   */
  uint32_t flags;      /* CKV_SEL_* below                                */
  uint32_t row_base;   /* cluster-major store: sorted entry j is row
                          row_base + j (= the sink count); see `rows`    */
} ckv_select_desc;

#define CKV_SEL_FULL_RANK 1u  /* write ranked_clusters for every cluster   */
#define CKV_SEL_SCORES 2u     /* write the f64 scores (score_clusters)     */
#define CKV_SEL_L2_PERSIST 4u /* read the centroids through a persisting L2
                                 window (needs cudaLimitPersistingL2CacheSize
                                 > 0; the session sets it)                  */

/* I_T as runs of consecutive KV-store rows (the cluster-major store makes
 * every taken cluster one run; sinks and the recency window are one run
 * each): run r covers I_T entries [off[r], off[r+1]) at store rows
 * row[r] + (e - off[r]).  Device arrays, per q head. */
typedef struct {
  uint32_t* row;     /* [n_q][run_cap]                                      */
  uint32_t* off;     /* [n_q][run_cap + 1]                                  */
  uint32_t* count;   /* [n_q] number of runs                                */
  uint32_t run_cap;  /* >= c_cap + 2                                        */
} ckv_runs;

/* score_clusters + select_tokens (+ the fused cache) for n_q queries, two
 * launches.  q: device f32 [n_q][128].  Outputs (device, each optional
 * unless noted):
 *   token_ids [n_q][sel_cap]: I_T positions (selection.hpp:91-109);
 *   rows [n_q][sel_cap]: the same entries as cluster-major store rows
 *     (row_base + index position for cluster tokens, the position for
 *     sinks / recency);
 *   runs: I_T as store-row runs (see ckv_runs) — what ckv_attend consumes;
 *   n_tokens, n_taken, trimmed [n_q] (required);
 *   ranked [n_q][c_cap] (required): every cluster for CKV_SEL_FULL_RANK,
 *     otherwise the taken prefix;
 *   scores [n_q][c_cap] f64 (score_clusters) when CKV_SEL_SCORES.
 * cache: NULL, or a cache with n_q slots — each q head's taken clusters go
 * through ClusterCache::lookup_and_update (cache.hpp:38-57), fused. */
int ckv_select(ckv_ctx* ctx, const ckv_select_desc* desc, const float* q,
               const float* centroids, const uint32_t* n_clusters, const uint32_t* sizes,
               const uint32_t* starts, const uint32_t* sorted_ids, uint32_t* token_ids,
               uint32_t* rows, const ckv_runs* runs, uint32_t* n_tokens, uint32_t* n_taken,
               uint32_t* trimmed, uint32_t* ranked, double* scores, ckv_cache* cache);

/* ClusterCache with n_slots independent caches of retention R over at
 * most c_cap cluster ids (bitmap ring).  cache.hpp:25-36. */
int ckv_cache_create(ckv_ctx* ctx, uint32_t n_slots, uint32_t c_cap, uint32_t retention,
                     uint32_t d, ckv_cache** out);
int ckv_cache_destroy(ckv_cache* cache);
/* counters_host: [n_slots][4] = requested, hit, tokens, bytes (cache.hpp:12-17) */
int ckv_cache_counters(ckv_cache* cache, uint64_t* counters_host);
/* Standalone lookup_and_update for one slot (cache.hpp:38-57):
 * selected/sizes device; hit_ids/miss_ids device [n_sel];
 * counts_host[2] = n_hit, n_miss. */
int ckv_cache_lookup(ckv_ctx* ctx, ckv_cache* cache, uint32_t slot, const uint32_t* selected,
                     uint32_t n_sel, const uint32_t* sizes, uint32_t* hit_ids,
                     uint32_t* miss_ids, uint32_t* counts_host);
/* invalidate_on_recluster (cache.hpp:67-76); retired: host ids */
int ckv_cache_invalidate(ckv_ctx* ctx, ckv_cache* cache, uint32_t slot,
                         const uint32_t* retired_host, uint32_t n_retired);

/* ------------------------------------------------------------------ */
/* sparse decode attention (attention.hpp:16-69)                       */
/* ------------------------------------------------------------------ */
typedef struct {
  uint32_t n_q, group, p_cap, sel_cap;
  uint32_t max_tokens;  /* upper bound of n_tokens[] (sizes the split grid) */
} ckv_attend_desc;

/* approx_attention for n_q queries: softmax(q K[I]^T / sqrt(d)) V[I] over
 * I_T given either as per-entry store rows (rows [n_q][sel_cap]: positions
 * for a position-ordered store) or as runs (ckv_select's ckv_runs for the
 * cluster-major store; pass rows = NULL), entries 0..n_tokens[h]-1.
 * Split-K flash-decode with an LSE merge.  K, V: device bf16
 * [unit][p_cap][128].  out: device f32 [n_q][128].  weights: device f32
 * [n_q][sel_cap] in I order, or NULL.  An empty selection is CKV_EINVAL
 * (attention.hpp:66-67), checked on a host copy of n_tokens only when
 * weights != NULL (parity mode). */
int ckv_attend(ckv_ctx* ctx, const ckv_attend_desc* desc, const float* q, const uint16_t* K,
               const uint16_t* V, const uint32_t* rows, const ckv_runs* runs,
               const uint32_t* n_tokens, float* out, float* weights);

/* Cluster-major relayout of a position-ordered KV store:
 * dst row r = src row r for r < sink or r >= labeled_end, and src row
 * sorted_ids[u][r - sink] for sink <= r < labeled_end (sorted_ids from
 * ckv_build_index over the store's labels).  K2 == K and V2 == V re-lay in
 * place through a bounded (<= 1 GiB) staging buffer, chunk of units by
 * chunk, so a store filling most of HBM is never held twice. */
int ckv_relayout_kv(ckv_ctx* ctx, uint32_t n_units, uint32_t p_cap, const uint16_t* K,
                    const uint16_t* V, uint16_t* K2, uint16_t* V2, const uint32_t* sorted_ids,
                    uint32_t sink, uint32_t labeled_end, uint32_t n_rows);

/* ------------------------------------------------------------------ */
/* sequence-sharded decode step                 */
/* ------------------------------------------------------------------ */
/* Each rank holds a contiguous position shard of every unit's keys, stored
 * cluster-major by its LOCAL index (rows [0, sink_rows) sinks on the rank
 * that owns them, then the local clustered rows in local index order, then
 * the recency rows on the rank that owns them), plus the replicated
 * centroids and global cluster sizes.  One step:
 *   ckv_score_range     this rank's centroid slice [c_lo, c_lo + slice) ->
 *                       scores [n_q][slice] f64 (score_clusters,
 *                       selection.hpp:51-57, bit-exact)
 *   (all-gather)        -> scores [world][n_q][slice]
 *   ckv_select_scored   the global ranking / budget / trim of select_tokens
 *                       (selection.hpp:74-111) and this rank's share of I_T
 *                       as runs of the local store
 *   ckv_attend_partial  approx_attention over the local share, returning the
 *                       locally normalised output and its log2-sum-exp2
 *   (all-gather)        -> outs [world][n_q][128], lses [world][n_q]
 *   ckv_attend_merge    the global softmax (attention.hpp:20-50) by an LSE
 *                       merge; the local weights become global weights. */
typedef struct {
  uint32_t n_q, group, budget;
  uint32_t C;          /* clusters per unit (<= 4096)                        */
  uint32_t c_cap;      /* stride of sizes / prefix / ranked rows              */
  uint32_t slice;      /* gathered scores: cluster c at rank c / slice,       */
  uint32_t world;      /*   offset c % slice of [world][n_q][slice]           */
  uint32_t n_local;    /* local clustered rows per unit (lsorted stride)      */
  uint32_t sel_cap;    /* token-id slots per q head                           */
  uint32_t row_base;   /* store row of local index entry 0                    */
  uint32_t sink_rows;  /* sinks held here: rows [0, sink_rows) = positions 0..*/
  uint32_t rec_row;    /* recency held here: rows [rec_row, rec_row + n_rec)  */
  uint32_t rec_pos;    /*   = positions [rec_pos, rec_pos + n_rec)            */
  uint32_t n_rec;
  uint32_t pos_base;   /* global position of local clustered row 0            */
  uint32_t flags;      /* CKV_SEL_FULL_RANK                                   */
} ckv_shard_select_desc;

/* q: f32 [n_units*group][128]; centroids f32 [n_units][c_cap][128];
 * group in {1, 2, 4, 8}. */
int ckv_score_range(ckv_ctx* ctx, uint32_t n_units, uint32_t group, const float* q,
                    const float* centroids, uint32_t c_cap, uint32_t C, uint32_t c_lo,
                    uint32_t slice, double* scores);
/* scores [world][n_q][slice]; gsize = global sizes [unit][c_cap]; lsize,
 * lstart [unit][c_cap(+1)], lsorted [unit][n_local] = the local index;
 * prefix [unit][c_cap] = members of each cluster on lower-ranked shards.
 * Outputs per q head: runs (run_cap >= C + 2), n_tokens = local I_T size,
 * n_taken / trimmed (global, as SelectionResult), ranked [n_q][c_cap],
 * token_ids [n_q][sel_cap] (optional, reference positions). */
int ckv_select_scored(ckv_ctx* ctx, const ckv_shard_select_desc* desc, const double* scores,
                      const uint32_t* gsize, const uint32_t* lsize, const uint32_t* lstart,
                      const uint32_t* prefix, const uint32_t* lsorted, const ckv_runs* runs,
                      uint32_t* token_ids, uint32_t* n_tokens, uint32_t* n_taken,
                      uint32_t* trimmed, uint32_t* ranked);
/* The decode step's default scoring: approximate f32 scores of this rank's
 * centroid slice with rigorous bounds (|a - s| <= 2^-14 |q| |mu|, s the
 * dot_f64 score): out f32 [2][n_q][slice] (a, then the bound), all-gathered
 * into [world][2][n_q][slice] for ckv_select_approx, which re-scores exactly
 * (from the replicated centroids) only the clusters that can reach the
 * budget cut — the same ranking, trim and shares as ckv_select_scored. */
int ckv_score_range_approx(ckv_ctx* ctx, uint32_t n_units, uint32_t group, const float* q,
                           const float* centroids, uint32_t c_cap, uint32_t C, uint32_t c_lo,
                           uint32_t slice, float* out);
int ckv_select_approx(ckv_ctx* ctx, const ckv_shard_select_desc* desc, const float* ascores,
                      const float* q, const float* centroids, const uint32_t* gsize,
                      const uint32_t* lsize, const uint32_t* lstart, const uint32_t* prefix,
                      const uint32_t* lsorted, const ckv_runs* runs, uint32_t* token_ids,
                      uint32_t* n_tokens, uint32_t* n_taken, uint32_t* trimmed,
                      uint32_t* ranked);
/* ckv_attend over runs, returning out = the locally normalised output and
 * lse [n_q] = log2 sum 2^(logit * log2 e) of the local logits (-inf and
 * out = 0 for a q head with no local tokens).  weights optional (local). */
int ckv_attend_partial(ckv_ctx* ctx, const ckv_attend_desc* desc, const float* q,
                       const uint16_t* K, const uint16_t* V, const ckv_runs* runs,
                       const uint32_t* n_tokens, float* out, float* lse, float* weights);
/* outs [world][n_q][128], lses [world][n_q] -> out [n_q][128]; weights
 * (optional, this rank's [n_q][sel_cap] local weights) rescaled in place. */
int ckv_attend_merge(ckv_ctx* ctx, uint32_t n_q, uint32_t world, uint32_t rank,
                     const float* outs, const float* lses, float* out, float* weights,
                     const uint32_t* n_tokens, uint32_t sel_cap);

/* ------------------------------------------------------------------ */
/* page-select baseline (selection.hpp:136-194)      */
/* ------------------------------------------------------------------ */
/* The Quest-style comparison point: consecutive pages of page_size tokens of
 * a POSITION-ordered KV store, scored through per-channel representatives. */
typedef struct {
  uint32_t n_q, group;
  uint32_t n;          /* tokens per unit                                    */
  uint32_t page_size;
  uint32_t budget;     /* B: n_sel = min(n_pages, B / page_size) pages       */
  uint32_t pages_cap;  /* representative rows per unit                        */
  uint32_t sel_cap;    /* token-id slots per q head (>= n_sel * page_size)    */
  uint32_t maxmin;     /* 0 = PageRepr::Max, 1 = PageRepr::MaxMin             */
} ckv_page_desc;

/* per (unit, page) elementwise max (and min, when rep_min != NULL) of the
 * page's keys; keys bf16 [unit][p_cap][128], reps f32 [unit][pages_cap][128] */
int ckv_page_reps(ckv_ctx* ctx, uint32_t n_units, uint32_t n, uint32_t p_cap, uint32_t page_size,
                  uint32_t pages_cap, const uint16_t* keys, float* rep_max, float* rep_min);
/* page_select for n_q queries (q f32 [n_q][128]): the selected pages' tokens
 * as runs of the position-ordered store (ascending ids; adjacent pages merge;
 * run_cap > n_sel), n_tokens [n_q], token_ids [n_q][sel_cap] optional. */
int ckv_page_select(ckv_ctx* ctx, const ckv_page_desc* desc, const float* q, const float* rep_max,
                    const float* rep_min, const ckv_runs* runs, uint32_t* token_ids,
                    uint32_t* n_tokens);

/* ------------------------------------------------------------------ */
/* quality metrics (harness.hpp:228-310)             */
/* ------------------------------------------------------------------ */
/* exact_topb (selection.hpp:115-132) for n_q queries over a POSITION-ordered
 * store (keys bf16 [unit][p_cap][128], q head h reads unit h / group): the
 * min(B, n) positions with the largest dot_f64(q, k), ties to the lower
 * position, ascending, in ids [n_q][ids_cap].  n <= 49152. */
int ckv_exact_topb(ckv_ctx* ctx, uint32_t n_q, uint32_t group, uint32_t n, uint32_t p_cap,
                   const float* q, const uint16_t* keys, uint32_t budget, uint32_t* ids,
                   uint32_t ids_cap);
/* recall_rate (attention.hpp:70-93) per q head: |sel ∩ truth| / n_truth;
 * truth [n_q][truth_cap] ascending (ckv_exact_topb's order), the n_sel[h]
 * selected ids distinct; recall f64 [n_q]. */
int ckv_recall(ckv_ctx* ctx, uint32_t n_q, const uint32_t* sel, uint32_t sel_cap,
               const uint32_t* n_sel, const uint32_t* truth, uint32_t truth_cap, uint32_t n_truth,
               double* recall);
/* output_error (attention.hpp:101-131) per q head: l2_rel, cos_sim (f64). */
int ckv_output_error(ckv_ctx* ctx, uint32_t n_q, const float* approx, const float* exact,
                     double* l2_rel, double* cos_sim);
/* one run [0, n) per q head: ckv_attend over it is full_attention
 * (attention.hpp:53-60) on a position-ordered store. */
int ckv_full_runs(ckv_ctx* ctx, uint32_t n_q, uint32_t n, const ckv_runs* runs,
                  uint32_t* n_tokens);

/* ------------------------------------------------------------------ */
/* session: the batched serving path (simulate_head's ClusterKV branch, */
/* harness.hpp:155-346, minus the metric oracles), device-resident.     */
/* ------------------------------------------------------------------ */
typedef struct {
  uint32_t n_units;        /* batch * layers * kv heads                 */
  uint32_t group;          /* q heads per kv unit                       */
  uint32_t prompt_len;     /* L                                         */
  uint32_t max_decode;     /* T capacity                                */
  uint32_t budget;         /* B                                         */
  uint32_t retention;      /* cache R (0 = no cache)                    */
  uint32_t c0_divisor, c_plus, decode_batch, sink_tokens, max_iters;
  uint64_t cluster_seed;   /* ClusterConfig::seed; per-unit seed =
                              mix_seed(cluster_seed, layer, head) with
                              unit = layer * kv_heads + head             */
  uint32_t kv_heads;       /* for the per-unit seed derivation          */
  uint32_t flags;          /* CKV_KM_* for the prefill k-means, plus    */
                           /* CKV_SESSION_TOKEN_IDS                     */
  uint32_t async_delay;    /* 0: decode batches are clustered and join  */
                           /* the model at the step that completes them */
                           /* (synchronous).  d > 0: the harness's      */
                           /* async_clustering (harness.hpp:236-243,    */
                           /* 327-329): the batch's k-means runs on a   */
                           /* side stream and joins d steps later; its  */
                           /* rows stay in the recency window until     */
                           /* then.  Needs d < decode_batch <= 512,     */
                           /* c_plus <= 32.                             */
  uint32_t c0_override;    /* ClusterConfig::c0_override (0 = the rule) */
} ckv_session_desc;

/* Also materialise each step's I_T as reference token positions
 * (ckv_session_state's token_ids); the attention itself consumes the run
 * list, so this is only needed for introspection / parity checks. */
#define CKV_SESSION_TOKEN_IDS 0x100u
/* Keep the centroids L2-resident across steps: sets aside persisting L2
 * (cudaLimitPersistingL2CacheSize, device-wide, restored at destroy) and
 * selects with CKV_SEL_L2_PERSIST. */
#define CKV_SESSION_L2_PERSIST 0x200u
/* Physical two-tier cluster cache (cache.hpp:25-93; ckv_tier.cu): each step
 * the selected clusters missing from a per-unit page pool in HBM are copied
 * into it from the backing tier and the attention reads the pool pages.
 * TIERED: the backing tier is the session's HBM store; TIER_HOST: a
 * host-pinned mirror of it (misses are PCIe reads, the offload setting).
 * Residency: clusters the unit selected in the last `retention` steps. */
#define CKV_SESSION_TIERED 0x800u
#define CKV_SESSION_TIER_HOST 0x1000u

int ckv_session_create(ckv_ctx* ctx, const ckv_session_desc* desc, ckv_session** out);
int ckv_session_destroy(ckv_session* s);
/* Device pointers of the session's KV store (bf16 [unit][p_cap][128]),
 * so callers can fill the prompt KV in place.  The store is position-
 * ordered until ckv_session_prefill, which relays it cluster-major (rows
 * [0,sink) sinks, [sink, labeled_end) tokens in index order, then the
 * unclustered recency positions) into NEW buffers: query the pointers
 * again after prefill. */
int ckv_session_kv(ckv_session* s, uint16_t** K, uint16_t** V, uint32_t* p_cap);
/* Upload prompt KV from HOST bf16 [unit][L][128]. */
int ckv_session_load_prompt(ckv_session* s, const uint16_t* K_host, const uint16_t* V_host);
/* cluster_prefill + build_index for every unit (harness.hpp:209-210).
 * info_host [n_units] or NULL. */
int ckv_session_prefill(ckv_session* s, ckv_kmeans_info* info_host);
/* One decode step for every q head (harness.hpp:218-339):
 *   select (budget, sinks, recency window [labeled_end, n_ctx)) + cache,
 *   approx attention, append (k_t, v_t), decode-batch clustering every m.
 * q: f32 [n_q][128]; k_new, v_new: bf16 [n_units][128]; out: f32 [n_q][128].
 * on_device != 0: all four are device pointers; otherwise host pointers:
 * page-locked (cudaHostAlloc / pinned) buffers are read and written by the
 * kernels in place over PCIe (zero-copy: the selection reads q and leaves a
 * device copy for the attention, the attention writes out, the append reads
 * k/v); pageable buffers are staged by copies on the session stream.  Both
 * give the device path's results bit for bit; the call returns after out is
 * complete. */
int ckv_session_step(ckv_session* s, const float* q, const uint16_t* k_new,
                     const uint16_t* v_new, float* out, int on_device);
/* Select + attend only (no append/cluster), device pointers, for timing
 * the steady-state hot path.  Equivalent to the first half of step. */
int ckv_session_attend_only(ckv_session* s, const float* q_dev, float* out_dev);
/* Layer mode: each step's select + attend runs one launch pair per slice of
 * layer_units consecutive units (a model layer's kv heads), slices in order —
 * the dependency order of a decoder, where layer l+1's queries come from
 * layer l's output.  0 (default): one pair for all units (the reference
 * harness's independent (layer, head) fan-out).  layer_units must divide
 * n_units. */
int ckv_session_set_layer_units(ckv_session* s, uint32_t layer_units);
/* k-means iterations (ClusterModel::invocation_iterations' last entry,
 * clustering.hpp:330) of every unit's most recent decode batch; waits for
 * that batch's k-means and reports its input errors. */
int ckv_session_batch_iterations(ckv_session* s, uint32_t* iterations_host);
/* Tiered sessions: out[5] = rows fetched, clusters fetched, clusters
 * selected (per unit, summed), evictions, pool rows per unit. */
int ckv_session_tier_stats(ckv_session* s, uint64_t* out);
/* Introspection for tests / bench. */
typedef struct {
  uint32_t n_ctx, labeled_end, steps;
  uint32_t max_clusters;
  uint64_t launches;
} ckv_session_stats;
int ckv_session_stats_get(ckv_session* s, ckv_session_stats* st);
/* device pointers of the model/index/selection state */
int ckv_session_state(ckv_session* s, float** centroids, int32_t** labels,
                      uint32_t** n_clusters, uint32_t** sizes, uint32_t** starts,
                      uint32_t** sorted_ids, uint32_t** token_ids, uint32_t** n_tokens,
                      uint32_t* c_cap, uint32_t* sel_cap);
ckv_cache* ckv_session_cache(ckv_session* s);

#ifdef __cplusplus
}
#endif
#endif

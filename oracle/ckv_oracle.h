/*
 * ckv_oracle.h — CPU restatement of the ClusterKV reference hot path, in C.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.  The product library (libckv_b200.so) never
 * links or calls it.
 *
 * Every function restates one reference function from
 * /root/reference/proj/include/clusterkv/*.hpp (cited per function in
 * ckv_oracle.c).  Parity of this restatement is pinned by
 *   (1) the SPEC known-answer vectors, and
 *   (2) differential fixtures produced by the reference itself, compiled
 *       unmodified from /root/reference (oracle/_ref, oracle/make_golden.py),
 *       committed under tests/golden/.
 *
 * Numerics mirror the reference exactly: f32 storage, sequential f64
 * accumulation (common.hpp:86-90), IEEE sqrt/div, float() rounding.
 * Build with -O2 -ffp-contract=off, never -ffast-math.
 */
#ifndef CKV_ORACLE_H
#define CKV_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = 1 };
enum { ORC_METRIC_COSINE = 0, ORC_METRIC_L2 = 1, ORC_METRIC_IP = 2 };

/* last validation message (thread-local) */
const char* orc_last_error(void);

/* ---- RNG (common.hpp:100-138) ---------------------------------------- */
typedef struct { uint64_t mt[312]; uint32_t idx; } orc_mt64;
void     orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_mix_seed(uint64_t seed, uint64_t a, uint64_t b);
double   orc_gaussian(orc_mt64* g);

/* ---- numerics (common.hpp:86-147, clustering.hpp:59-65) -------------- */
double orc_dot_f64(const float* a, const float* b, uint32_t n);
double orc_normalize(float* v, uint32_t n);
double orc_cosine_distance(const float* a, const float* b, uint32_t n);

/* ---- k-means (clustering.hpp:157-263) --------------------------------- */
typedef struct {
  uint32_t n_clusters;
  uint32_t iterations_used;
  int32_t  converged;
  uint32_t n_objective;   /* entries written to objective_history */
  uint32_t n_repair;      /* entries written to repair_iterations  */
} orc_kmeans_info;

/* centroids_out: C*d; labels_out: n; obj_hist: >= max_iters+1;
 * repair_iters: >= max_iters+1.  init_rows may be NULL (seeded sampling). */
int orc_kmeans(const float* keys, uint32_t n, uint32_t d, uint32_t C,
               uint64_t seed, uint32_t max_iters, int metric,
               const uint32_t* init_rows, uint32_t n_init_rows,
               float* centroids_out, int32_t* labels_out,
               double* obj_hist, uint32_t* repair_iters,
               orc_kmeans_info* info);

/* AssignScorer::assign of n keys against C raw centroids (clustering.hpp:70-115) */
void orc_assign(const float* keys, uint32_t n, uint32_t d, int metric, const float* cents,
                uint32_t C, int32_t* out);

/* init rows exactly as kmeans_cosine samples them (clustering.hpp:186-193) */
void orc_kmeans_init_rows(uint32_t n, uint32_t C, uint64_t seed, uint32_t* rows_out);

typedef struct {
  uint32_t c0_divisor, c_plus, decode_batch, sink_tokens, max_iters;
  uint64_t seed;
  uint32_t c0_override;
  int32_t  metric;
} orc_cluster_config;

void     orc_cluster_config_default(orc_cluster_config* c);
int      orc_cluster_config_validate(const orc_cluster_config* c);
uint32_t orc_prefill_cluster_count(uint32_t prompt_len, const orc_cluster_config* c);

/* labels_out: L (sinks -1); centroids_out: C0*d */
int orc_cluster_prefill(const float* keys, uint32_t L, uint32_t d,
                        const orc_cluster_config* cfg,
                        float* centroids_out, int32_t* labels_out,
                        double* obj_hist, uint32_t* repair_iters,
                        orc_kmeans_info* info, uint32_t* sink_count_out);

/* Appends to (centroids, labels) in place: centroids must have room for
 * (*n_clusters + min(c_plus, rows)) * d floats, labels for *n_positions + rows.
 * Mirrors clustering.hpp:310-332. */
int orc_cluster_decode_batch(float* centroids, uint32_t* n_clusters,
                             int32_t* labels, uint32_t* n_positions,
                             const float* new_keys, uint32_t rows, uint32_t d,
                             const orc_cluster_config* cfg,
                             uint32_t* iterations_out, int32_t* converged_out);

/* ---- index + selection (selection.hpp:16-111) ------------------------- */
void orc_build_index(const int32_t* labels, uint32_t n_pos, uint32_t C,
                     uint32_t* sizes, uint32_t* starts /*C+1*/, uint32_t* sorted_ids);

void orc_score_clusters(const float* q, const float* centroids, uint32_t C,
                        uint32_t d, double* scores);

/* token_ids needs room for min(labeled,budget) + sink_count + n_recency.
 * Returns the number of token ids written. */
uint32_t orc_select_tokens(const float* q, const float* centroids, uint32_t C,
                           uint32_t d, const uint32_t* sizes,
                           const uint32_t* starts, const uint32_t* sorted_ids,
                           uint32_t sink_count, uint32_t budget,
                           const uint32_t* recency, uint32_t n_recency,
                           uint32_t* ranked_out, uint32_t* n_taken_out,
                           uint32_t* trimmed_out, uint32_t* token_ids_out);

/* selection.hpp:136-194 (maxmin = PageRepr::MaxMin); ids_out needs
 * min(n_pages, budget/page_size) * page_size slots; returns the count or
 * (uint32_t)-1 on a ValidationError */
uint32_t orc_page_select(const float* q, const float* keys, uint32_t n, uint32_t d,
                         uint32_t budget, uint32_t page_size, int maxmin, uint32_t* ids_out);

void orc_exact_topb(const float* q, const float* keys, uint32_t n, uint32_t d,
                    uint32_t budget, uint32_t* ids_out /* min(budget,n) */);

/* ---- attention (attention.hpp:16-69) ---------------------------------- */
int orc_attention_over(const float* q, const float* K, const float* V,
                       uint32_t d, const uint32_t* rows, uint32_t n_rows,
                       float* out, float* weights /* nullable */);

/* ---- cluster cache (cache.hpp:25-93) ---------------------------------- */
typedef struct orc_cache orc_cache;
orc_cache* orc_cache_new(uint32_t retention, uint32_t d);
void       orc_cache_free(orc_cache* c);
/* hit/miss arrays need room for n_sel each */
void orc_cache_lookup_and_update(orc_cache* c, const uint32_t* selected, uint32_t n_sel,
                                 const uint32_t* sizes, uint32_t* hit_ids, uint32_t* n_hit,
                                 uint32_t* miss_ids, uint32_t* n_miss);
void orc_cache_counters(const orc_cache* c, uint64_t out[4]);
void orc_cache_invalidate(orc_cache* c, const uint32_t* retired, uint32_t n_retired);

/* ---- synthetic generator (trace.hpp:87-198), input generation only ---- */
typedef struct {
  uint32_t n_centers;
  float center_spread, intra_spread, query_drift;
  uint64_t seed;
  uint32_t prompt_len, decode_len, d, n_layers, n_heads;
} orc_synth_spec;

void orc_synth_spec_default(orc_synth_spec* s);
/* buffers: keys/values L*d, queries/dkeys/dvalues T*d */
void orc_generate_head(const orc_synth_spec* s, uint64_t sub_seed,
                       float* prompt_keys, float* prompt_values,
                       float* decode_queries, float* decode_keys, float* decode_values);
/* all (layer, head) traces, multithreaded; strides: head-major blocks */
void orc_generate_synthetic(const orc_synth_spec* s, uint32_t n_threads,
                            float* prompt_keys, float* prompt_values,
                            float* decode_queries, float* decode_keys, float* decode_values);

/* ---- CPU-baseline helpers (bench.py --impl reference / cpu_baseline) -- */
/* One decode step (select + approx attention) for n_units q heads,
 * fanned out over n_threads like run_simulation (harness.hpp:362-378). */
double orc_wall_ms(void);

#ifdef __cplusplus
}
#endif
#endif

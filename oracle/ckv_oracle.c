/*
 * ckv_oracle.c — plain-C restatement of the ClusterKV reference hot path.
 * TEST INFRASTRUCTURE ONLY (see ckv_oracle.h).  Never linked by the product.
 *
 * Reference: /root/reference/proj/include/clusterkv/{common,clustering,
 * selection,attention,cache,trace}.hpp.  File:line anchors per function.
 */
#define _GNU_SOURCE
#include "ckv_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

static __thread char g_err[256];
static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return ORC_EINVAL;
}
const char* orc_last_error(void) { return g_err; }

/* ===================================================================== */
/* RNG: std::mt19937_64 (bit-specified by the C++ standard) and the       */
/* hand-built distributions of common.hpp:100-138.                        */
/* ===================================================================== */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ull
#define MT_LOWER 0x000000007FFFFFFFull

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (uint32_t i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + i;
  g->idx = MT_N;
}

static void mt64_twist(orc_mt64* g) {
  for (uint32_t i = 0; i < MT_N; ++i) {
    uint64_t y = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t v = g->mt[(i + MT_M) % MT_N] ^ (y >> 1);
    if (y & 1ull) v ^= 0xB5026F5AA96619E9ull;
    g->mt[i] = v;
  }
  g->idx = 0;
}

uint64_t orc_mt64_next(orc_mt64* g) {
  if (g->idx >= MT_N) mt64_twist(g);
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}

/* common.hpp:100-105 */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* common.hpp:108-113 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t a, uint64_t b) {
  uint64_t h = orc_splitmix64(seed);
  h = orc_splitmix64(h ^ (a + 0x9e3779b97f4a7c15ull));
  return orc_splitmix64(h ^ (b + 0xbf58476d1ce4e5b9ull));
}

/* common.hpp:119-121 */
static double uniform01(orc_mt64* g) { return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53; }
/* common.hpp:124-126 */
static uint64_t uniform_below(orc_mt64* g, uint64_t n) { return orc_mt64_next(g) % n; }

/* common.hpp:130-138: Box-Muller, no cached second variate */
double orc_gaussian(orc_mt64* g) {
  double u1 = uniform01(g);
  while (u1 <= 0.0) u1 = uniform01(g);
  double u2 = uniform01(g);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

/* ===================================================================== */
/* numerics                                                               */
/* ===================================================================== */

/* common.hpp:86-90 — strictly sequential f64 accumulation */
double orc_dot_f64(const float* a, const float* b, uint32_t n) {
  double acc = 0.0;
  for (uint32_t i = 0; i < n; ++i) acc += (double)a[i] * (double)b[i];
  return acc;
}

/* common.hpp:141-147 */
double orc_normalize(float* v, uint32_t n) {
  double nrm = sqrt(orc_dot_f64(v, v, n));
  if (nrm > 0.0)
    for (uint32_t i = 0; i < n; ++i) v[i] = (float)((double)v[i] / nrm);
  return nrm;
}

/* clustering.hpp:59-65 */
double orc_cosine_distance(const float* a, const float* b, uint32_t n) {
  double na = sqrt(orc_dot_f64(a, a, n));
  double nb = sqrt(orc_dot_f64(b, b, n));
  if (na < 1e-12 || nb < 1e-12) return 1.0;
  double dist = 1.0 - orc_dot_f64(a, b, n) / (na * nb);
  return dist < 0.0 ? 0.0 : (dist > 2.0 ? 2.0 : dist);
}

/* ===================================================================== */
/* k-means (clustering.hpp:70-263)                                        */
/* ===================================================================== */

typedef struct {
  int metric;
  const float* cents;   /* C x d raw centroids */
  float* dirs;          /* cosine: normalized copy (clustering.hpp:76-81) */
  double* norms2;       /* l2: |mu|^2 (clustering.hpp:82-85) */
  uint32_t C, d;
} scorer_t;

static void scorer_init(scorer_t* s, int metric, const float* cents, uint32_t C, uint32_t d) {
  s->metric = metric; s->cents = cents; s->C = C; s->d = d;
  s->dirs = NULL; s->norms2 = NULL;
  if (metric == ORC_METRIC_COSINE) {
    s->dirs = (float*)malloc(sizeof(float) * (size_t)C * d);
    memcpy(s->dirs, cents, sizeof(float) * (size_t)C * d);
    for (uint32_t c = 0; c < C; ++c) orc_normalize(s->dirs + (size_t)c * d, d);
  } else if (metric == ORC_METRIC_L2) {
    s->norms2 = (double*)malloc(sizeof(double) * C);
    for (uint32_t c = 0; c < C; ++c)
      s->norms2[c] = orc_dot_f64(cents + (size_t)c * d, cents + (size_t)c * d, d);
  }
}
static void scorer_free(scorer_t* s) { free(s->dirs); free(s->norms2); }

/* clustering.hpp:88-101 */
static double scorer_score(const scorer_t* s, const float* key, uint32_t c) {
  const size_t off = (size_t)c * s->d;
  if (s->metric == ORC_METRIC_COSINE) return orc_dot_f64(key, s->dirs + off, s->d);
  if (s->metric == ORC_METRIC_L2)
    return orc_dot_f64(key, s->cents + off, s->d) - 0.5 * s->norms2[c];
  return orc_dot_f64(key, s->cents + off, s->d);
}

/* clustering.hpp:104-115: strict '>' so ties keep the lowest id */
static uint32_t scorer_assign(const scorer_t* s, const float* key) {
  uint32_t best = 0;
  double best_score = -INFINITY;
  for (uint32_t c = 0; c < s->C; ++c) {
    double v = scorer_score(s, key, c);
    if (v > best_score) { best_score = v; best = c; }
  }
  return best;
}

/* clustering.hpp:118-124 */
static double objective(const float* keys, uint32_t n, uint32_t d, const int32_t* labels,
                        const float* cents) {
  double obj = 0.0;
  for (uint32_t i = 0; i < n; ++i)
    obj += orc_cosine_distance(keys + (size_t)i * d, cents + (size_t)labels[i] * d, d);
  return obj;
}

/* clustering.hpp:128-153 */
static uint32_t repair_empty(const float* keys, uint32_t n, uint32_t d, int32_t* labels,
                             const float* cents, uint32_t C, uint32_t* counts) {
  uint32_t repairs = 0;
  for (uint32_t c = 0; c < C; ++c) {
    if (counts[c] > 0) continue;
    uint32_t largest = 0;                         /* first maximum */
    for (uint32_t k = 1; k < C; ++k)
      if (counts[k] > counts[largest]) largest = k;
    if (counts[largest] <= 1) continue;
    double worst = -1.0;
    uint32_t victim = 0;
    for (uint32_t i = 0; i < n; ++i) {
      if ((uint32_t)labels[i] != largest) continue;
      double dist = orc_cosine_distance(keys + (size_t)i * d, cents + (size_t)largest * d, d);
      if (dist > worst) { worst = dist; victim = i; }
    }
    labels[victim] = (int32_t)c;
    counts[largest]--;
    counts[c]++;
    repairs++;
  }
  return repairs;
}

/* clustering.hpp:186-193: partial Fisher-Yates over mt19937_64(seed) */
void orc_kmeans_init_rows(uint32_t n, uint32_t C, uint64_t seed, uint32_t* rows_out) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  uint32_t* pool = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint32_t i = 0; i < n; ++i) pool[i] = i;
  for (uint32_t c = 0; c < C; ++c) {
    uint32_t j = c + (uint32_t)uniform_below(&g, n - c);
    uint32_t t = pool[c]; pool[c] = pool[j]; pool[j] = t;
  }
  memcpy(rows_out, pool, sizeof(uint32_t) * C);
  free(pool);
}

/* Cosine assignment of keys [i0, i1) with four centroids' dot_f64 chains
 * interleaved.  Each chain is still the sequential f64 sum of
 * common.hpp:86-90 (no contraction: -ffp-contract=off), and the candidates
 * are compared in ascending id with strict '>', so the result equals
 * scorer_assign bit for bit; the interleave only hides the add latency so
 * the checker finishes the headline shapes (32k / 128k keys) in seconds. */
static void assign_cosine_range(const scorer_t* s, const float* keys, uint32_t i0, uint32_t i1,
                                int32_t* out) {
  const uint32_t C = s->C, d = s->d;
  double* kd = (double*)malloc(sizeof(double) * d);
  for (uint32_t i = i0; i < i1; ++i) {
    const float* key = keys + (size_t)i * d;
    for (uint32_t j = 0; j < d; ++j) kd[j] = (double)key[j];
    uint32_t best = 0;
    double best_score = -INFINITY;
    uint32_t c = 0;
    for (; c + 4 <= C; c += 4) {
      const float* d0 = s->dirs + (size_t)c * d;
      const float* d1 = d0 + d;
      const float* d2 = d1 + d;
      const float* d3 = d2 + d;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      for (uint32_t j = 0; j < d; ++j) {
        a0 += kd[j] * (double)d0[j];
        a1 += kd[j] * (double)d1[j];
        a2 += kd[j] * (double)d2[j];
        a3 += kd[j] * (double)d3[j];
      }
      if (a0 > best_score) { best_score = a0; best = c; }
      if (a1 > best_score) { best_score = a1; best = c + 1; }
      if (a2 > best_score) { best_score = a2; best = c + 2; }
      if (a3 > best_score) { best_score = a3; best = c + 3; }
    }
    for (; c < C; ++c) {
      double v = orc_dot_f64(key, s->dirs + (size_t)c * d, d);
      if (v > best_score) { best_score = v; best = c; }
    }
    out[i] = (int32_t)best;
  }
  free(kd);
}

typedef struct {
  const scorer_t* s;
  const float* keys;
  uint32_t i0, i1;
  int32_t* out;
} assign_job_t;

static void* assign_job(void* p) {
  const assign_job_t* j = (const assign_job_t*)p;
  assign_cosine_range(j->s, j->keys, j->i0, j->i1, j->out);
  return NULL;
}

/* host threads for the checker's large assignments: ORC_THREADS, else all
 * online cores */
static uint32_t oracle_threads(void) {
  const char* e = getenv("ORC_THREADS");
  long n = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  if (n < 1) n = 1;
  if (n > 256) n = 256;
  return (uint32_t)n;
}

static void assign_all(const float* keys, uint32_t n, uint32_t d, int metric,
                       const float* cents, uint32_t C, int32_t* out) {
  scorer_t s;
  scorer_init(&s, metric, cents, C, d);
  if (metric != ORC_METRIC_COSINE) {
    for (uint32_t i = 0; i < n; ++i) out[i] = (int32_t)scorer_assign(&s, keys + (size_t)i * d);
    scorer_free(&s);
    return;
  }
  uint32_t nt = oracle_threads();
  if ((uint64_t)n * C < (1ull << 21) || nt == 1 || n < 2 * nt) {
    assign_cosine_range(&s, keys, 0, n, out);
  } else {
    pthread_t th[256];
    assign_job_t jobs[256];
    for (uint32_t t = 0; t < nt; ++t) {
      jobs[t] = (assign_job_t){&s, keys, (uint32_t)((uint64_t)n * t / nt),
                               (uint32_t)((uint64_t)n * (t + 1) / nt), out};
      pthread_create(&th[t], NULL, assign_job, &jobs[t]);
    }
    for (uint32_t t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  }
  scorer_free(&s);
}

/* AssignScorer::assign over a key block (clustering.hpp:70-115): the CPU
 * side of the sequence-sharded k-means tests, where each rank assigns only
 * its own shard's keys against the replicated centroids. */
void orc_assign(const float* keys, uint32_t n, uint32_t d, int metric, const float* cents,
                uint32_t C, int32_t* out) {
  assign_all(keys, n, d, metric, cents, C, out);
}

static void count_members(const int32_t* labels, uint32_t n, uint32_t C, uint32_t* counts) {
  memset(counts, 0, sizeof(uint32_t) * C);
  for (uint32_t i = 0; i < n; ++i) counts[(uint32_t)labels[i]]++;
}

/* clustering.hpp:205-218: f64 sums in token order, float(sum / count) */
static void update_centroids(const float* keys, uint32_t n, uint32_t d, const int32_t* labels,
                             const uint32_t* counts, uint32_t C, float* cents, double* sums) {
  memset(sums, 0, sizeof(double) * (size_t)C * d);
  for (uint32_t i = 0; i < n; ++i) {
    double* acc = sums + (size_t)labels[i] * d;
    const float* row = keys + (size_t)i * d;
    for (uint32_t j = 0; j < d; ++j) acc[j] += (double)row[j];
  }
  for (uint32_t c = 0; c < C; ++c)
    for (uint32_t j = 0; j < d; ++j)
      cents[(size_t)c * d + j] = (float)(sums[(size_t)c * d + j] / (double)counts[c]);
}

/* clustering.hpp:160-263 */
int orc_kmeans(const float* keys, uint32_t n, uint32_t d, uint32_t C, uint64_t seed,
               uint32_t max_iters, int metric, const uint32_t* init_rows, uint32_t n_init_rows,
               float* cents, int32_t* labels_out, double* obj_hist, uint32_t* repair_iters,
               orc_kmeans_info* info) {
  if (C < 1 || C > n) return fail("kmeans: need 1 <= C <= N");
  for (size_t i = 0; i < (size_t)n * d; ++i)
    if (!isfinite(keys[i])) return fail("kmeans: keys must be finite");
  int any_nonzero = 0;
  for (uint32_t i = 0; i < n && !any_nonzero; ++i)
    any_nonzero = sqrt(orc_dot_f64(keys + (size_t)i * d, keys + (size_t)i * d, d)) >= 1e-12;
  if (!any_nonzero) return fail("kmeans: degenerate input, all keys zero-norm");

  uint32_t* chosen = (uint32_t*)malloc(sizeof(uint32_t) * C);
  if (init_rows) {
    if (n_init_rows != C) { free(chosen); return fail("kmeans: init_rows size must equal C"); }
    memcpy(chosen, init_rows, sizeof(uint32_t) * C);
  } else {
    orc_kmeans_init_rows(n, C, seed, chosen);
  }
  for (uint32_t c = 0; c < C; ++c)
    memcpy(cents + (size_t)c * d, keys + (size_t)chosen[c] * d, sizeof(float) * d);
  free(chosen);

  int32_t* labels = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * n);
  uint32_t* counts = (uint32_t*)malloc(sizeof(uint32_t) * C);
  uint32_t* next_counts = (uint32_t*)malloc(sizeof(uint32_t) * C);
  double* sums = (double*)malloc(sizeof(double) * (size_t)C * d);
  uint32_t n_obj = 0, n_rep = 0;

  assign_all(keys, n, d, metric, cents, C, labels);
  count_members(labels, n, C, counts);
  if (repair_empty(keys, n, d, labels, cents, C, counts) > 0) repair_iters[n_rep++] = 0;
  obj_hist[n_obj++] = objective(keys, n, d, labels, cents);

  uint32_t iter = 0;
  int converged = 0;
  while (iter < max_iters) {
    update_centroids(keys, n, d, labels, counts, C, cents, sums);
    assign_all(keys, n, d, metric, cents, C, next);
    count_members(next, n, C, next_counts);
    uint32_t repairs = repair_empty(keys, n, d, next, cents, C, next_counts);
    ++iter;
    if (repairs > 0) repair_iters[n_rep++] = iter;
    obj_hist[n_obj++] = objective(keys, n, d, next, cents);
    if (memcmp(next, labels, sizeof(int32_t) * n) == 0) { converged = 1; break; }
    int32_t* t = labels; labels = next; next = t;
    uint32_t* tc = counts; counts = next_counts; next_counts = tc;
  }
  memcpy(labels_out, labels, sizeof(int32_t) * n);
  info->n_clusters = C;
  info->iterations_used = iter;
  info->converged = converged;
  info->n_objective = n_obj;
  info->n_repair = n_rep;
  free(labels); free(next); free(counts); free(next_counts); free(sums);
  return ORC_OK;
}

/* clustering.hpp:20-36 */
void orc_cluster_config_default(orc_cluster_config* c) {
  c->c0_divisor = 80; c->c_plus = 4; c->decode_batch = 320; c->sink_tokens = 16;
  c->max_iters = 50; c->seed = 0; c->c0_override = 0; c->metric = ORC_METRIC_COSINE;
}
int orc_cluster_config_validate(const orc_cluster_config* c) {
  if (c->c0_divisor < 1) return fail("ClusterConfig: c0_divisor must be >= 1");
  if (c->c_plus < 1) return fail("ClusterConfig: c_plus must be >= 1");
  if (c->decode_batch < 1) return fail("ClusterConfig: decode_batch must be >= 1");
  if (c->max_iters < 1) return fail("ClusterConfig: max_iters must be >= 1");
  return ORC_OK;
}

/* clustering.hpp:267-274 */
uint32_t orc_prefill_cluster_count(uint32_t L, const orc_cluster_config* c) {
  if (L <= c->sink_tokens) return 0;
  uint32_t n = L - c->sink_tokens;
  uint32_t c0 = c->c0_override ? c->c0_override
                               : (uint32_t)llround((double)n / (double)c->c0_divisor);
  if (c0 < 1) c0 = 1;
  if (c0 > n) c0 = n;
  return c0;
}

/* clustering.hpp:278-305 */
int orc_cluster_prefill(const float* keys, uint32_t L, uint32_t d, const orc_cluster_config* cfg,
                        float* cents, int32_t* labels_out, double* obj_hist,
                        uint32_t* repair_iters, orc_kmeans_info* info, uint32_t* sink_out) {
  int rc = orc_cluster_config_validate(cfg);
  if (rc) return rc;
  if (L <= cfg->sink_tokens) {
    for (uint32_t i = 0; i < L; ++i) labels_out[i] = -1;
    memset(info, 0, sizeof *info);
    info->converged = 1;
    *sink_out = L;
    return ORC_OK;
  }
  const uint32_t sink = cfg->sink_tokens, n = L - sink;
  uint32_t c0 = orc_prefill_cluster_count(L, cfg);
  for (uint32_t i = 0; i < sink; ++i) labels_out[i] = -1;
  rc = orc_kmeans(keys + (size_t)sink * d, n, d, c0, cfg->seed, cfg->max_iters, cfg->metric,
                  NULL, 0, cents, labels_out + sink, obj_hist, repair_iters, info);
  *sink_out = sink;
  return rc;
}

/* clustering.hpp:310-332 */
int orc_cluster_decode_batch(float* cents, uint32_t* n_clusters, int32_t* labels,
                             uint32_t* n_positions, const float* new_keys, uint32_t rows,
                             uint32_t d, const orc_cluster_config* cfg, uint32_t* iters_out,
                             int32_t* converged_out) {
  if (rows == 0) return ORC_OK;
  int rc = orc_cluster_config_validate(cfg);
  if (rc) return rc;
  uint32_t c = cfg->c_plus < rows ? cfg->c_plus : rows;
  uint64_t bseed = orc_mix_seed(cfg->seed, 0xdecadeull, *n_positions);
  double* oh = (double*)malloc(sizeof(double) * (cfg->max_iters + 1));
  uint32_t* ri = (uint32_t*)malloc(sizeof(uint32_t) * (cfg->max_iters + 1));
  int32_t* sub = (int32_t*)malloc(sizeof(int32_t) * rows);
  orc_kmeans_info info;
  uint32_t base = *n_clusters;
  rc = orc_kmeans(new_keys, rows, d, c, bseed, cfg->max_iters, cfg->metric, NULL, 0,
                  cents + (size_t)base * d, sub, oh, ri, &info);
  if (rc == ORC_OK) {
    for (uint32_t i = 0; i < rows; ++i) labels[*n_positions + i] = sub[i] + (int32_t)base;
    *n_positions += rows;
    *n_clusters += c;
    if (iters_out) *iters_out = info.iterations_used;
    if (converged_out) *converged_out = info.converged;
  }
  free(oh); free(ri); free(sub);
  return rc;
}

/* ===================================================================== */
/* index + selection                                                      */
/* ===================================================================== */

/* selection.hpp:29-48: stable counting sort of the labels */
void orc_build_index(const int32_t* labels, uint32_t n_pos, uint32_t C, uint32_t* sizes,
                     uint32_t* starts, uint32_t* sorted_ids) {
  memset(sizes, 0, sizeof(uint32_t) * C);
  for (uint32_t p = 0; p < n_pos; ++p)
    if (labels[p] >= 0) sizes[labels[p]]++;
  starts[0] = 0;
  for (uint32_t c = 0; c < C; ++c) starts[c + 1] = starts[c] + sizes[c];
  uint32_t* cursor = (uint32_t*)malloc(sizeof(uint32_t) * (C ? C : 1));
  memcpy(cursor, starts, sizeof(uint32_t) * C);
  for (uint32_t p = 0; p < n_pos; ++p)
    if (labels[p] >= 0) sorted_ids[cursor[labels[p]]++] = p;
  free(cursor);
}

/* selection.hpp:51-57 */
void orc_score_clusters(const float* q, const float* cents, uint32_t C, uint32_t d,
                        double* scores) {
  for (uint32_t c = 0; c < C; ++c) scores[c] = orc_dot_f64(q, cents + (size_t)c * d, d);
}

static const double* g_sort_scores;
/* selection.hpp:83-87: score descending, id ascending (a strict total order) */
static int rank_cmp(const void* pa, const void* pb) {
  uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  double sa = g_sort_scores[a], sb = g_sort_scores[b];
  if (sa != sb) return sa > sb ? -1 : 1;
  return a < b ? -1 : (a > b);
}

/* selection.hpp:74-111 */
uint32_t orc_select_tokens(const float* q, const float* cents, uint32_t C, uint32_t d,
                           const uint32_t* sizes, const uint32_t* starts,
                           const uint32_t* sorted_ids, uint32_t sink_count, uint32_t budget,
                           const uint32_t* recency, uint32_t n_recency, uint32_t* ranked,
                           uint32_t* n_taken_out, uint32_t* trimmed_out, uint32_t* out) {
  double* scores = (double*)malloc(sizeof(double) * (C ? C : 1));
  orc_score_clusters(q, cents, C, d, scores);
  for (uint32_t c = 0; c < C; ++c) ranked[c] = c;
  g_sort_scores = scores;   /* oracle is called single-threaded per process */
  qsort(ranked, C, sizeof(uint32_t), rank_cmp);
  uint32_t n = 0, cum = 0, taken = 0, trimmed = 0;
  for (uint32_t r = 0; r < C; ++r) {
    if (cum >= budget) break;
    uint32_t c = ranked[r], sz = sizes[c], rem = budget - cum;
    const uint32_t* slice = sorted_ids + starts[c];
    if (sz <= rem) {
      memcpy(out + n, slice, sizeof(uint32_t) * sz);
      n += sz; cum += sz;
    } else {
      memcpy(out + n, slice, sizeof(uint32_t) * rem);
      n += rem; trimmed = sz - rem; cum = budget;
    }
    taken++;
  }
  for (uint32_t s = 0; s < sink_count; ++s) out[n++] = s;
  for (uint32_t i = 0; i < n_recency; ++i) out[n++] = recency[i];
  *n_taken_out = taken;
  *trimmed_out = trimmed;
  free(scores);
  return n;
}

static const double* g_topb_scores;
static int topb_cmp(const void* pa, const void* pb) {
  uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  double sa = g_topb_scores[a], sb = g_topb_scores[b];
  if (sa != sb) return sa > sb ? -1 : 1;
  return a < b ? -1 : (a > b);
}
static int u32_cmp(const void* pa, const void* pb) {
  uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  return a < b ? -1 : (a > b);
}

/* selection.hpp:115-132 (the recall oracle; not on the hot path) */
/* selection.hpp:136-194 page_select: consecutive pages scored through a
 * per-channel representative (elementwise max; MaxMin: sum_j max(q*max, q*min)
 * in f64, sequential), top n_sel = min(n_pages, budget / page_size) pages by
 * (score desc, id asc), their ids ascending.  Returns the id count, or
 * (uint32_t)-1 for page_size < 1 (ValidationError). */
static const double* g_page_scores;
static int page_cmp(const void* pa, const void* pb) {
  uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  if (g_page_scores[a] != g_page_scores[b]) return g_page_scores[a] > g_page_scores[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}
uint32_t orc_page_select(const float* q, const float* keys, uint32_t n, uint32_t d,
                         uint32_t budget, uint32_t page_size, int maxmin, uint32_t* ids_out) {
  if (page_size < 1) { fail("page_select: page_size must be >= 1"); return (uint32_t)-1; }
  const uint32_t n_pages = (n + page_size - 1) / page_size;
  uint32_t n_sel = budget / page_size;
  if (n_sel > n_pages) n_sel = n_pages;
  double* sc = (double*)malloc(sizeof(double) * (n_pages ? n_pages : 1));
  uint32_t* pages = (uint32_t*)malloc(sizeof(uint32_t) * (n_pages ? n_pages : 1));
  float* mx = (float*)malloc(sizeof(float) * d);
  float* mn = (float*)malloc(sizeof(float) * d);
  for (uint32_t p = 0; p < n_pages; ++p) {
    const uint32_t b = p * page_size, e = b + page_size < n ? b + page_size : n;
    memcpy(mx, keys + (size_t)b * d, sizeof(float) * d);
    memcpy(mn, keys + (size_t)b * d, sizeof(float) * d);
    for (uint32_t i = b + 1; i < e; ++i)
      for (uint32_t j = 0; j < d; ++j) {
        const float v = keys[(size_t)i * d + j];
        if (v > mx[j]) mx[j] = v;   /* std::max(a, b): b only if a < b */
        if (v < mn[j]) mn[j] = v;
      }
    if (!maxmin) {
      sc[p] = orc_dot_f64(q, mx, d);
    } else {
      double s = 0.0;
      for (uint32_t j = 0; j < d; ++j) {
        const double a = (double)q[j] * (double)mx[j], c = (double)q[j] * (double)mn[j];
        s += a < c ? c : a;       /* std::max(a, c) */
      }
      sc[p] = s;
    }
    pages[p] = p;
  }
  g_page_scores = sc;
  qsort(pages, n_pages, sizeof(uint32_t), page_cmp);
  /* the selected pages' ids, ascending: sort the n_sel page ids, expand */
  qsort(pages, n_sel, sizeof(uint32_t), u32_cmp);
  uint32_t k = 0;
  for (uint32_t t = 0; t < n_sel; ++t) {
    const uint32_t b = pages[t] * page_size, e = b + page_size < n ? b + page_size : n;
    for (uint32_t i = b; i < e; ++i) ids_out[k++] = i;
  }
  free(sc); free(pages); free(mx); free(mn);
  return k;
}

void orc_exact_topb(const float* q, const float* keys, uint32_t n, uint32_t d, uint32_t budget,
                    uint32_t* ids_out) {
  double* s = (double*)malloc(sizeof(double) * n);
  uint32_t* ids = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint32_t i = 0; i < n; ++i) { s[i] = orc_dot_f64(q, keys + (size_t)i * d, d); ids[i] = i; }
  g_topb_scores = s;
  qsort(ids, n, sizeof(uint32_t), topb_cmp);
  uint32_t take = budget < n ? budget : n;
  qsort(ids, take, sizeof(uint32_t), u32_cmp);
  memcpy(ids_out, ids, sizeof(uint32_t) * take);
  free(s); free(ids);
}

/* ===================================================================== */
/* attention (attention.hpp:20-69)                                         */
/* ===================================================================== */
int orc_attention_over(const float* q, const float* K, const float* V, uint32_t d,
                       const uint32_t* rows, uint32_t n_rows, float* out, float* weights) {
  if (n_rows == 0) return fail("approx_attention: empty selection");
  const double scale = 1.0 / sqrt((double)d);
  double* logit = (double*)malloc(sizeof(double) * n_rows);
  double mx = -INFINITY;
  for (uint32_t i = 0; i < n_rows; ++i) {
    logit[i] = orc_dot_f64(q, K + (size_t)rows[i] * d, d) * scale;
    if (logit[i] > mx) mx = logit[i];
  }
  double sum = 0.0;
  for (uint32_t i = 0; i < n_rows; ++i) { logit[i] = exp(logit[i] - mx); sum += logit[i]; }
  double* acc = (double*)calloc(d, sizeof(double));
  for (uint32_t i = 0; i < n_rows; ++i) {
    double w = logit[i] / sum;
    if (weights) weights[i] = (float)w;
    const float* v = V + (size_t)rows[i] * d;
    for (uint32_t j = 0; j < d; ++j) acc[j] += w * (double)v[j];
  }
  for (uint32_t j = 0; j < d; ++j) out[j] = (float)acc[j];
  free(logit); free(acc);
  return ORC_OK;
}

/* ===================================================================== */
/* cluster cache (cache.hpp:25-93): ring of the last R selected sets       */
/* ===================================================================== */
struct orc_cache {
  uint32_t R, d;
  uint32_t** ring; uint32_t* ring_n; uint32_t ring_len, ring_head;
  uint64_t requested, hit, tokens, bytes;
};

orc_cache* orc_cache_new(uint32_t R, uint32_t d) {
  if (R < 1) { fail("ClusterCache: retention must be >= 1"); return NULL; }
  orc_cache* c = (orc_cache*)calloc(1, sizeof *c);
  c->R = R; c->d = d;
  c->ring = (uint32_t**)calloc(R, sizeof(uint32_t*));
  c->ring_n = (uint32_t*)calloc(R, sizeof(uint32_t));
  return c;
}
void orc_cache_free(orc_cache* c) {
  if (!c) return;
  for (uint32_t i = 0; i < c->R; ++i) free(c->ring[i]);
  free(c->ring); free(c->ring_n); free(c);
}
/* resident = union of ring sets (cache.hpp:83-86) */
static int resident(const orc_cache* c, uint32_t id) {
  for (uint32_t k = 0; k < c->ring_len; ++k) {
    uint32_t slot = (c->ring_head + k) % c->R;
    for (uint32_t i = 0; i < c->ring_n[slot]; ++i)
      if (c->ring[slot][i] == id) return 1;
  }
  return 0;
}
/* cache.hpp:38-57 */
void orc_cache_lookup_and_update(orc_cache* c, const uint32_t* sel, uint32_t n_sel,
                                 const uint32_t* sizes, uint32_t* hit_ids, uint32_t* n_hit,
                                 uint32_t* miss_ids, uint32_t* n_miss) {
  uint32_t nh = 0, nm = 0;
  for (uint32_t i = 0; i < n_sel; ++i) {
    if (resident(c, sel[i])) hit_ids[nh++] = sel[i]; else miss_ids[nm++] = sel[i];
  }
  c->requested += n_sel;
  c->hit += nh;
  for (uint32_t i = 0; i < nm; ++i) c->tokens += sizes[miss_ids[i]];
  c->bytes = c->tokens * 2ull * c->d * sizeof(float);
  /* ring push_back, pop_front when over R */
  uint32_t slot;
  if (c->ring_len < c->R) {
    slot = (c->ring_head + c->ring_len) % c->R;
    c->ring_len++;
  } else {
    slot = c->ring_head;                 /* oldest is dropped */
    c->ring_head = (c->ring_head + 1) % c->R;
  }
  free(c->ring[slot]);
  c->ring[slot] = (uint32_t*)malloc(sizeof(uint32_t) * (n_sel ? n_sel : 1));
  memcpy(c->ring[slot], sel, sizeof(uint32_t) * n_sel);
  c->ring_n[slot] = n_sel;
  *n_hit = nh; *n_miss = nm;
}
void orc_cache_counters(const orc_cache* c, uint64_t out[4]) {
  out[0] = c->requested; out[1] = c->hit; out[2] = c->tokens; out[3] = c->bytes;
}
/* cache.hpp:67-76 */
void orc_cache_invalidate(orc_cache* c, const uint32_t* retired, uint32_t n_retired) {
  for (uint32_t s = 0; s < c->R; ++s) {
    uint32_t w = 0;
    for (uint32_t i = 0; i < c->ring_n[s]; ++i) {
      int dead = 0;
      for (uint32_t r = 0; r < n_retired && !dead; ++r) dead = c->ring[s][i] == retired[r];
      if (!dead) c->ring[s][w++] = c->ring[s][i];
    }
    c->ring_n[s] = w;
  }
}

/* ===================================================================== */
/* synthetic generator (trace.hpp:87-225) — builds test/bench inputs       */
/* ===================================================================== */
void orc_synth_spec_default(orc_synth_spec* s) {
  s->n_centers = 8; s->center_spread = 1.0f; s->intra_spread = 0.15f; s->query_drift = 0.15f;
  s->seed = 0; s->prompt_len = 4096; s->decode_len = 256; s->d = 128; s->n_layers = 2;
  s->n_heads = 4;
}

static void fill_gaussian(orc_mt64* g, float* out, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) out[i] = (float)orc_gaussian(g);
}
/* trace.hpp:126-132 */
static void spread_direction(orc_mt64* g, const float* base, float spread, float* out,
                             uint32_t d) {
  for (uint32_t i = 0; i < d; ++i) out[i] = base[i] + spread * (float)orc_gaussian(g);
  orc_normalize(out, d);
}

/* trace.hpp:134-198 */
void orc_generate_head(const orc_synth_spec* s, uint64_t sub_seed, float* pk, float* pv,
                       float* dq, float* dk, float* dv) {
  orc_mt64 g;
  orc_mt64_seed(&g, sub_seed);
  const uint32_t d = s->d, L = s->prompt_len, T = s->decode_len, nc = s->n_centers;
  float* base = (float*)malloc(sizeof(float) * d);
  float* centers = (float*)malloc(sizeof(float) * (size_t)nc * d);
  float* u = (float*)malloc(sizeof(float) * d);
  fill_gaussian(&g, base, d);
  orc_normalize(base, d);
  for (uint32_t c = 0; c < nc; ++c) spread_direction(&g, base, s->center_spread, centers + (size_t)c * d, d);
  for (uint32_t i = 0; i < L; ++i) {
    uint32_t c = (uint32_t)uniform_below(&g, nc);
    spread_direction(&g, centers + (size_t)c * d, s->intra_spread, pk + (size_t)i * d, d);
  }
  for (uint32_t i = 0; i < L; ++i) fill_gaussian(&g, pv + (size_t)i * d, d);

  const float q_scale = 2.0f * sqrtf((float)d);
  memcpy(u, centers + (size_t)uniform_below(&g, nc) * d, sizeof(float) * d);
  uint32_t denom = 2 * nc > 1 ? 2 * nc : 1;
  uint32_t retarget = T / denom > 1 ? T / denom : 1;
  uint32_t target = 0;
  for (uint32_t t = 0; t < T; ++t) {
    if (t % retarget == 0) target = (uint32_t)uniform_below(&g, nc);
    if (s->query_drift > 0.0f) {
      const float* ct = centers + (size_t)target * d;
      for (uint32_t i = 0; i < d; ++i) {
        float pull = s->query_drift * (ct[i] - u[i]);
        float noise = 0.25f * s->query_drift * (float)orc_gaussian(&g);
        u[i] += pull + noise;
      }
      orc_normalize(u, d);
    }
    for (uint32_t i = 0; i < d; ++i) dq[(size_t)t * d + i] = q_scale * u[i];
  }
  for (uint32_t i = 0; i < T; ++i) {
    uint32_t c = (uint32_t)uniform_below(&g, nc);
    spread_direction(&g, centers + (size_t)c * d, s->intra_spread, dk + (size_t)i * d, d);
  }
  for (uint32_t i = 0; i < T; ++i) fill_gaussian(&g, dv + (size_t)i * d, d);
  free(base); free(centers); free(u);
}

typedef struct {
  const orc_synth_spec* s;
  float *pk, *pv, *dq, *dk, *dv;
  uint32_t next, units;
  pthread_mutex_t mu;
} gen_job;

static void* gen_worker(void* arg) {
  gen_job* j = (gen_job*)arg;
  const size_t Ld = (size_t)j->s->prompt_len * j->s->d, Td = (size_t)j->s->decode_len * j->s->d;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    uint32_t u = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (u >= j->units) return NULL;
    uint32_t layer = u / j->s->n_heads, head = u % j->s->n_heads;
    orc_generate_head(j->s, orc_mix_seed(j->s->seed, layer, head), j->pk + u * Ld,
                      j->pv + u * Ld, j->dq + u * Td, j->dk + u * Td, j->dv + u * Td);
  }
}

/* trace.hpp:202-225, fanned out over threads (units are independent) */
void orc_generate_synthetic(const orc_synth_spec* s, uint32_t n_threads, float* pk, float* pv,
                            float* dq, float* dk, float* dv) {
  gen_job j = {s, pk, pv, dq, dk, dv, 0, s->n_layers * s->n_heads, PTHREAD_MUTEX_INITIALIZER};
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
  for (uint32_t t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, gen_worker, &j);
  for (uint32_t t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  free(th);
}

double orc_wall_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

// ref_capi.cpp — C-ABI wrapper around the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile from the sources where
// they lie (/root/reference/proj/include), with the namespace renamed
// (-Dckv=ckv_ref) and <numeric> force-included
// (attention.hpp:58 uses std::iota without it).  Output goes only to
// oracle/_ref/libckv_ref.so (git-ignored; it travels to the GPU box).
//
// Uses: (1) pin the C restatement (oracle/ckv_oracle.c) differentially and
// generate tests/golden fixtures; (2) the CPU baseline ("kind": "reference")
// in bench.py, timed through the reference's own hot-path functions.
#include <cstring>
#include <future>
#include <thread>
#include <vector>

#include "clusterkv/attention.hpp"
#include "clusterkv/cache.hpp"
#include "clusterkv/clustering.hpp"
#include "clusterkv/selection.hpp"
#include "clusterkv/trace.hpp"
#include "clusterkv/harness.hpp"

namespace R = ckv_ref;

namespace {
thread_local std::string g_err;

R::Matrix as_matrix(const float* p, uint32_t rows, uint32_t cols) {
  R::Matrix m(rows, cols);
  std::memcpy(m.data.data(), p, sizeof(float) * size_t(rows) * cols);
  return m;
}

void export_model(const R::ClusterModel& m, float* cents, int32_t* labels, double* obj,
                  uint32_t* reps, uint32_t* info) {
  if (cents) std::memcpy(cents, m.centroids.data.data(), sizeof(float) * m.centroids.data.size());
  if (labels) std::memcpy(labels, m.labels.data(), sizeof(int32_t) * m.labels.size());
  if (obj) std::memcpy(obj, m.objective_history.data(), sizeof(double) * m.objective_history.size());
  if (reps) std::memcpy(reps, m.repair_iterations.data(), sizeof(uint32_t) * m.repair_iterations.size());
  // info: n_clusters, iterations_used, converged, n_objective, n_repair, sink_count
  info[0] = m.n_clusters;
  info[1] = m.iterations_used;
  info[2] = m.converged ? 1u : 0u;
  info[3] = uint32_t(m.objective_history.size());
  info[4] = uint32_t(m.repair_iterations.size());
  info[5] = m.sink_count;
}

R::ClusterConfig make_cfg(const uint32_t* c, uint64_t seed) {
  R::ClusterConfig cfg;
  cfg.c0_divisor = c[0];
  cfg.c_plus = c[1];
  cfg.decode_batch = c[2];
  cfg.sink_tokens = c[3];
  cfg.max_iters = c[4];
  cfg.c0_override = c[5];
  cfg.metric = R::AssignMetric(c[6]);
  cfg.seed = seed;
  return cfg;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix_seed(uint64_t s, uint64_t a, uint64_t b) { return R::mix_seed(s, a, b); }

void ref_generate_head(uint32_t n_centers, float center_spread, float intra_spread,
                       float query_drift, uint32_t L, uint32_t T, uint32_t d,
                       uint64_t sub_seed, float* pk, float* pv, float* dq, float* dk,
                       float* dv) {
  R::SynthSpec s;
  s.n_centers = n_centers;
  s.center_spread = center_spread;
  s.intra_spread = intra_spread;
  s.query_drift = query_drift;
  s.prompt_len = L;
  s.decode_len = T;
  s.d = d;
  R::HeadTrace tr = R::detail::generate_head(s, sub_seed, nullptr, nullptr);
  std::memcpy(pk, tr.prompt_keys.data.data(), sizeof(float) * size_t(L) * d);
  std::memcpy(pv, tr.prompt_values.data.data(), sizeof(float) * size_t(L) * d);
  std::memcpy(dq, tr.decode_queries.data.data(), sizeof(float) * size_t(T) * d);
  std::memcpy(dk, tr.decode_keys.data.data(), sizeof(float) * size_t(T) * d);
  std::memcpy(dv, tr.decode_values.data.data(), sizeof(float) * size_t(T) * d);
}

// generate_synthetic + write_trace (trace.hpp:200-225, 268-303): the
// reference's own CKVT file, for the trace reader/writer golden fixtures.
// Returns 0, or 1 with ref_last_error() set.
int ref_write_synthetic_trace(const char* path, uint32_t n_centers, uint64_t seed, uint32_t L,
                              uint32_t T, uint32_t d, uint32_t n_layers, uint32_t n_heads) {
  try {
    R::SynthSpec s;
    s.n_centers = n_centers;
    s.seed = seed;
    s.prompt_len = L;
    s.decode_len = T;
    s.d = d;
    s.n_layers = n_layers;
    s.n_heads = n_heads;
    R::write_trace(R::generate_synthetic(s), path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// read_trace (trace.hpp:305-367) and return its error class / ParseError code:
// 0 ok, 1 + code for ParseError, 100 IoError, 200 ValidationError
int ref_read_trace_status(const char* path) {
  try {
    R::read_trace(path);
    return 0;
  } catch (const R::ParseError& e) {
    g_err = e.what();
    return 1 + int(e.code());
  } catch (const R::IoError& e) {
    g_err = e.what();
    return 100;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 200;
  }
}

// info[6] as export_model
int ref_kmeans(const float* keys, uint32_t n, uint32_t d, uint32_t C, uint64_t seed,
               uint32_t max_iters, int metric, const uint32_t* init_rows, uint32_t n_init,
               float* cents, int32_t* labels, double* obj, uint32_t* reps, uint32_t* info) {
  try {
    R::Matrix k = as_matrix(keys, n, d);
    std::span<const uint32_t> ir;
    if (init_rows) ir = std::span<const uint32_t>(init_rows, n_init);
    R::ClusterModel m = R::kmeans_cosine(k, C, seed, max_iters, R::AssignMetric(metric), ir);
    export_model(m, cents, labels, obj, reps, info);
    return 0;
  } catch (const R::ValidationError& e) {
    g_err = e.what();
    return 1;
  }
}

uint32_t ref_prefill_cluster_count(uint32_t L, const uint32_t* c) {
  return R::prefill_cluster_count(L, make_cfg(c, 0));
}

int ref_cluster_prefill(const float* keys, uint32_t L, uint32_t d, const uint32_t* c,
                        uint64_t seed, float* cents, int32_t* labels, double* obj,
                        uint32_t* reps, uint32_t* info) {
  try {
    R::ClusterModel m = R::cluster_prefill(as_matrix(keys, L, d), make_cfg(c, seed));
    export_model(m, cents, labels, obj, reps, info);
    return 0;
  } catch (const R::ValidationError& e) {
    g_err = e.what();
    return 1;
  }
}

// In/out: centroids [(n_clusters + c_plus) * d], labels [n_positions + rows].
int ref_cluster_decode_batch(float* cents, uint32_t* n_clusters, int32_t* labels,
                             uint32_t* n_positions, const float* new_keys, uint32_t rows,
                             uint32_t d, const uint32_t* c, uint64_t seed, uint32_t* iters) {
  try {
    R::ClusterModel m;
    m.n_clusters = *n_clusters;
    m.centroids = as_matrix(cents, *n_clusters, d);
    m.labels.assign(labels, labels + *n_positions);
    m.converged = true;
    R::cluster_decode_batch(m, as_matrix(new_keys, rows, d), make_cfg(c, seed));
    std::memcpy(cents, m.centroids.data.data(), sizeof(float) * m.centroids.data.size());
    std::memcpy(labels, m.labels.data(), sizeof(int32_t) * m.labels.size());
    *n_clusters = m.n_clusters;
    *n_positions = uint32_t(m.labels.size());
    if (iters) *iters = m.invocation_iterations.empty() ? 0 : m.invocation_iterations.back();
    return 0;
  } catch (const R::ValidationError& e) {
    g_err = e.what();
    return 1;
  }
}

void ref_build_index(const int32_t* labels, uint32_t n_pos, uint32_t C, uint32_t* sizes,
                     uint32_t* starts, uint32_t* sorted) {
  R::ClusterModel m;
  m.n_clusters = C;
  m.labels.assign(labels, labels + n_pos);
  R::ClusterIndex ix = R::build_index(m);
  std::memcpy(sizes, ix.sizes.data(), sizeof(uint32_t) * ix.sizes.size());
  std::memcpy(starts, ix.cluster_start.data(), sizeof(uint32_t) * ix.cluster_start.size());
  std::memcpy(sorted, ix.sorted_token_ids.data(), sizeof(uint32_t) * ix.sorted_token_ids.size());
}

void ref_score_clusters(const float* q, const float* cents, uint32_t C, uint32_t d, double* out) {
  R::ClusterModel m;
  m.n_clusters = C;
  m.centroids = as_matrix(cents, C, d);
  auto s = R::score_clusters(std::span<const float>(q, d), m);
  std::memcpy(out, s.data(), sizeof(double) * C);
}

// Builds the index internally from labels (the reference's own build_index),
// then selects.  Returns |I_T|.
uint32_t ref_select_tokens(const float* q, const float* cents, uint32_t C, uint32_t d,
                           const int32_t* labels, uint32_t n_pos, uint32_t sink_count,
                           uint32_t budget, const uint32_t* recency, uint32_t n_rec,
                           uint32_t* ranked, uint32_t* n_taken, uint32_t* trimmed,
                           uint32_t* token_ids) {
  R::ClusterModel m;
  m.n_clusters = C;
  m.centroids = as_matrix(cents, C, d);
  m.labels.assign(labels, labels + n_pos);
  m.sink_count = sink_count;
  R::ClusterIndex ix = R::build_index(m);
  R::SelectionResult r = R::select_tokens(std::span<const float>(q, d), m, ix, budget,
                                          std::span<const uint32_t>(recency, n_rec));
  std::memcpy(ranked, r.ranked_clusters.data(), sizeof(uint32_t) * C);
  *n_taken = r.n_clusters_taken;
  *trimmed = r.trimmed_from_last;
  std::memcpy(token_ids, r.token_ids.data(), sizeof(uint32_t) * r.token_ids.size());
  return uint32_t(r.token_ids.size());
}

// page_select (selection.hpp:141-194); returns the id count, -1 on error
int64_t ref_page_select(const float* q, const float* keys, uint32_t n, uint32_t d,
                        uint32_t budget, uint32_t page_size, int maxmin, uint32_t* ids_out) {
  try {
    auto ids = R::page_select(std::span<const float>(q, d), as_matrix(keys, n, d), budget,
                              page_size, maxmin ? R::PageRepr::MaxMin : R::PageRepr::Max);
    std::memcpy(ids_out, ids.data(), sizeof(uint32_t) * ids.size());
    return int64_t(ids.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_approx_attention(const float* q, const float* K, const float* V, uint32_t n_ctx,
                         uint32_t d, const uint32_t* rows, uint32_t n_rows, float* out,
                         float* weights) {
  try {
    R::Matrix k = as_matrix(K, n_ctx, d), v = as_matrix(V, n_ctx, d);
    R::AttentionOutput o = R::approx_attention(std::span<const float>(q, d), k, v,
                                               std::span<const uint32_t>(rows, n_rows));
    std::memcpy(out, o.out.data(), sizeof(float) * d);
    if (weights) std::memcpy(weights, o.weights.data(), sizeof(float) * n_rows);
    return 0;
  } catch (const R::ValidationError& e) {
    g_err = e.what();
    return 1;
  }
}

void* ref_cache_new(uint32_t retention, uint32_t d) { return new R::ClusterCache(retention, d); }
void ref_cache_free(void* c) { delete static_cast<R::ClusterCache*>(c); }
void ref_cache_lookup_and_update(void* c, const uint32_t* sel, uint32_t n_sel,
                                 const uint32_t* sizes, uint32_t n_sizes, uint32_t* hit,
                                 uint32_t* n_hit, uint32_t* miss, uint32_t* n_miss) {
  auto r = static_cast<R::ClusterCache*>(c)->lookup_and_update(
      std::span<const uint32_t>(sel, n_sel), std::span<const uint32_t>(sizes, n_sizes));
  std::memcpy(hit, r.hit_ids.data(), sizeof(uint32_t) * r.hit_ids.size());
  std::memcpy(miss, r.miss_ids.data(), sizeof(uint32_t) * r.miss_ids.size());
  *n_hit = uint32_t(r.hit_ids.size());
  *n_miss = uint32_t(r.miss_ids.size());
}
void ref_cache_invalidate(void* c, const uint32_t* retired, uint32_t n) {
  static_cast<R::ClusterCache*>(c)->invalidate_on_recluster(
      std::span<const uint32_t>(retired, n), std::span<const uint32_t>());
}
void ref_cache_counters(void* c, uint64_t* out) {
  const auto& k = static_cast<R::ClusterCache*>(c)->counters();
  out[0] = k.clusters_requested;
  out[1] = k.clusters_hit;
  out[2] = k.tokens_transferred;
  out[3] = k.bytes_transferred;
}

// ---------------------------------------------------------------------------
// CPU baseline legs: the reference's own hot-path functions, fanned out over
// host threads exactly like run_simulation (harness.hpp:362-378).
// ---------------------------------------------------------------------------

// One decode step over `units` q heads.  Per unit u: q = qs[u], its kv model
// is kv_of[u] (centroids/labels of that kv head), K/V of that kv head.
// Each worker does select_tokens + approx_attention, like simulate_head's
// ClusterKV branch (harness.hpp:246-296) minus the metric oracles.
struct DecodeJob {
  const float* qs;
  const uint32_t* kv_of;
  const float* const* cents;
  const uint32_t* n_clusters;
  const int32_t* const* labels;
  const float* const* K;
  const float* const* V;
  uint32_t n_ctx, labeled_end, d, budget, sink;
};

double ref_decode_step_cpu(const float* qs, const uint32_t* kv_of, uint32_t units,
                           const float* const* cents, const uint32_t* n_clusters,
                           const int32_t* const* labels, const float* const* K,
                           const float* const* V, uint32_t n_kv, uint32_t n_ctx,
                           uint32_t labeled_end, uint32_t d, uint32_t budget,
                           uint32_t sink, uint32_t n_threads, float* out) {
  // Models and indices are built once, outside the timed region (the harness
  // rebuilds the index only after (re)clustering, harness.hpp:210, 333).
  std::vector<R::ClusterModel> models(n_kv);
  std::vector<R::ClusterIndex> idx(n_kv);
  std::vector<R::Matrix> Km(n_kv), Vm(n_kv);
  for (uint32_t g = 0; g < n_kv; ++g) {
    models[g].n_clusters = n_clusters[g];
    models[g].centroids = as_matrix(cents[g], n_clusters[g], d);
    models[g].labels.assign(labels[g], labels[g] + n_ctx);
    models[g].sink_count = sink;
    idx[g] = R::build_index(models[g]);
    Km[g] = as_matrix(K[g], n_ctx, d);
    Vm[g] = as_matrix(V[g], n_ctx, d);
  }
  std::vector<uint32_t> recency;
  for (uint32_t p = labeled_end; p < n_ctx; ++p) recency.push_back(p);

  auto t0 = std::chrono::steady_clock::now();
  std::atomic<uint32_t> next{0};
  auto worker = [&]() {
    for (;;) {
      uint32_t u = next.fetch_add(1);
      if (u >= units) return;
      uint32_t g = kv_of[u];
      std::span<const float> q(qs + size_t(u) * d, d);
      R::SelectionResult sel = R::select_tokens(q, models[g], idx[g], budget, recency);
      R::AttentionOutput o = R::approx_attention(q, Km[g], Vm[g], sel.token_ids);
      std::memcpy(out + size_t(u) * d, o.out.data(), sizeof(float) * d);
    }
  };
  unsigned nw = std::max(1u, std::min(n_threads, units));
  std::vector<std::future<void>> fs;
  for (unsigned w = 0; w + 1 < nw; ++w) fs.push_back(std::async(std::launch::async, worker));
  worker();
  for (auto& f : fs) f.get();
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(t1 - t0).count();
}

// Prefill k-means over `units` heads in parallel; returns wall ms and the
// total assignment passes (iterations_used + 1 per head) in *passes.
double ref_prefill_cpu(const float* const* keys, uint32_t units, uint32_t L, uint32_t d,
                       const uint64_t* seeds, uint32_t max_iters, uint32_t n_threads,
                       uint64_t* passes) {
  std::atomic<uint32_t> next{0};
  std::atomic<uint64_t> p{0};
  auto t0 = std::chrono::steady_clock::now();
  auto worker = [&]() {
    for (;;) {
      uint32_t u = next.fetch_add(1);
      if (u >= units) return;
      R::ClusterConfig cfg;
      cfg.seed = seeds[u];
      cfg.max_iters = max_iters;
      R::ClusterModel m = R::cluster_prefill(as_matrix(keys[u], L, d), cfg);
      p += m.iterations_used + 1;
    }
  };
  unsigned nw = std::max(1u, std::min(n_threads, units));
  std::vector<std::future<void>> fs;
  for (unsigned w = 0; w + 1 < nw; ++w) fs.push_back(std::async(std::launch::async, worker));
  worker();
  for (auto& f : fs) f.get();
  auto t1 = std::chrono::steady_clock::now();
  *passes = p.load();
  return std::chrono::duration<double, std::milli>(t1 - t0).count();
}

unsigned ref_hardware_concurrency() { return std::max(1u, std::thread::hardware_concurrency()); }

// The reference harness itself (run_simulation, harness.hpp:362-410, over
// simulate_head, :155-346) on generate_synthetic(spec) with every matrix
// rounded to bf16 (RNE; the GPU store is bf16): the oracle of
// the GPU decode-loop quality driver (paper_2412_03213_b200/quality.py).
// ClusterKV policy.  rows_f [n_rows][3] = recall, l2_rel, cos_sim; rows_u
// [n_rows][6] = step, layer, head, clusters_hit, clusters_requested,
// tokens_transferred; summ_f [4] = mean recall, l2_rel, cos_sim, hit_rate;
// summ_u [2] = tokens, bytes transferred; hist [hist_cap] k-means iteration
// histogram.  Returns the row count, or -1 with ref_last_error().
static float bf16_rne(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = uint32_t((uint64_t(u) + (((u >> 16) & 1u) + 0x7fffu)) >> 16) << 16;
  std::memcpy(&x, &u, 4);
  return x;
}

long ref_run_simulation_synth(uint32_t n_centers, uint64_t seed, uint32_t L, uint32_t T,
                              uint32_t n_layers, uint32_t n_heads, uint32_t budget,
                              uint32_t retention, uint32_t decode_batch, uint32_t c0_divisor,
                              int async_clustering, uint32_t async_delay, int recency_window,
                              double* rows_f, uint64_t* rows_u, double* summ_f, uint64_t* summ_u,
                              uint32_t* hist, uint32_t hist_cap) {
  try {
    R::SynthSpec s;
    s.n_centers = n_centers;
    s.seed = seed;
    s.prompt_len = L;
    s.decode_len = T;
    s.d = 128;
    s.n_layers = n_layers;
    s.n_heads = n_heads;
    R::TraceBundle b = R::generate_synthetic(s);
    for (auto& tr : b.traces)
      for (R::Matrix* m : {&tr.prompt_keys, &tr.prompt_values, &tr.decode_queries,
                           &tr.decode_keys, &tr.decode_values})
        for (float& x : m->data) x = bf16_rne(x);
    R::PolicyConfig cfg;
    cfg.policy = R::Policy::ClusterKV;
    cfg.budget = budget;
    cfg.retention = retention;
    cfg.cluster.decode_batch = decode_batch;
    cfg.cluster.c0_divisor = c0_divisor;
    cfg.async_clustering = async_clustering != 0;
    cfg.async_delay = async_delay;
    cfg.recency_window = recency_window != 0;
    R::RunReport rep = R::run_simulation(b, cfg);
    for (size_t i = 0; i < rep.rows.size(); ++i) {
      const auto& r = rep.rows[i];
      rows_f[3 * i] = r.recall;
      rows_f[3 * i + 1] = r.l2_rel;
      rows_f[3 * i + 2] = r.cos_sim;
      rows_u[6 * i] = r.step;
      rows_u[6 * i + 1] = r.layer;
      rows_u[6 * i + 2] = r.head;
      rows_u[6 * i + 3] = r.clusters_hit;
      rows_u[6 * i + 4] = r.clusters_requested;
      rows_u[6 * i + 5] = r.tokens_transferred;
    }
    summ_f[0] = rep.summary.mean_recall;
    summ_f[1] = rep.summary.mean_l2_rel;
    summ_f[2] = rep.summary.mean_cos_sim;
    summ_f[3] = rep.summary.hit_rate;
    summ_u[0] = rep.summary.tokens_transferred;
    summ_u[1] = rep.summary.bytes_transferred;
    for (uint32_t i = 0; i < hist_cap; ++i) hist[i] = 0;
    for (const auto& [it, n] : rep.summary.iteration_histogram)
      if (it < hist_cap) hist[it] = n;
    return long(rep.rows.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"

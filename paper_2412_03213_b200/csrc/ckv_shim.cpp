// ckv_shim.cpp — the reference-signature C++ API (include/clusterkv_b200/
// clusterkv.hpp) implemented on the C-ABI (include/ckv_cuda.h).  Host-side
// marshalling only: every computation runs in the sm_100a kernels.  One
// ckv_ctx per host thread (the reference calls these concurrently per head,
// harness.hpp:362-378), on the CUDA device named by $CKV_DEVICE (default 0).
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ckv_cuda.h"
#include "clusterkv_b200/clusterkv.hpp"

namespace ckv {
namespace {

constexpr uint32_t kD = CKV_HEAD_DIM;

[[noreturn]] void raise(int rc) {
  const std::string msg = ckv_last_error();
  if (rc == CKV_EINVAL) throw ValidationError(msg);
  throw Error("ckv_b200: " + msg);
}
void check(int rc) {
  if (rc != CKV_OK) raise(rc);
}

ckv_ctx* ctx() {
  thread_local struct Holder {
    ckv_ctx* c = nullptr;
    ~Holder() {
      if (c) ckv_ctx_destroy(c);
    }
  } h;
  if (!h.c) {
    const char* dev = std::getenv("CKV_DEVICE");
    check(ckv_ctx_create(dev ? std::atoi(dev) : 0, nullptr, &h.c));
  }
  return h.c;
}

struct Dev {  // owning device buffer
  void* p = nullptr;
  explicit Dev(size_t bytes) { check(ckv_malloc(ctx(), &p, bytes ? bytes : 16)); }
  ~Dev() { ckv_free(ctx(), p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};
template <typename T>
void put(const Dev& d, const T* src, size_t n) {
  if (n) check(ckv_memcpy_h2d(ctx(), d.p, src, n * sizeof(T)));
}
template <typename T>
void get(T* dst, const Dev& d, size_t n) {
  if (n) check(ckv_memcpy_d2h(ctx(), dst, d.p, n * sizeof(T)));
}

void require_d128(const Matrix& m, const char* what) {
  if (m.cols != kD) throw ValidationError(std::string(what) + ": the B200 kernels specialise d = 128");
}

// f32 -> bf16 bits; the B200 KV store is bf16
std::vector<uint16_t> to_bf16(const Matrix& m, const char* what) {
  std::vector<uint16_t> out(m.data.size());
  for (size_t i = 0; i < m.data.size(); ++i) {
    uint32_t u;
    std::memcpy(&u, &m.data[i], 4);
    if ((u & 0xffffu) != 0 && std::isfinite(m.data[i]))
      throw ValidationError(std::string(what) +
                            ": values must be bf16-representable (the B200 KV store is bf16)");
    out[i] = uint16_t(u >> 16);
  }
  return out;
}

}  // namespace

// ---------------------------------------------------------------------------
// clustering.hpp:160-263
ClusterModel kmeans_cosine(const Matrix& keys, uint32_t n_clusters, uint64_t seed,
                           uint32_t max_iters, AssignMetric metric,
                           std::span<const uint32_t> init_rows) {
  const uint32_t n = keys.rows;
  if (n_clusters < 1 || n_clusters > n) throw ValidationError("kmeans: need 1 <= C <= N");
  if (!is_finite(keys)) throw ValidationError("kmeans: keys must be finite");
  bool any_nonzero = false;
  for (uint32_t i = 0; i < n && !any_nonzero; ++i) any_nonzero = norm_f64(keys.row(i)) >= 1e-12;
  if (!any_nonzero) throw ValidationError("kmeans: degenerate input, all keys zero-norm");
  require_d128(keys, "kmeans");
  if (metric != AssignMetric::Cosine)
    throw ValidationError("kmeans: the B200 path implements the cosine metric only");
  std::vector<uint32_t> rows(n_clusters);
  if (!init_rows.empty()) {
    if (init_rows.size() != n_clusters) throw ValidationError("kmeans: init_rows size must equal C");
    for (uint32_t r : init_rows)
      if (r >= n) throw ValidationError("kmeans: init_rows out of range");
    std::copy(init_rows.begin(), init_rows.end(), rows.begin());
  } else {
    check(ckv_kmeans_init_rows(n, n_clusters, seed, rows.data()));
  }
  const std::vector<uint16_t> kb = to_bf16(keys, "kmeans");
  Dev dk(kb.size() * 2), dr(rows.size() * 4), dc(size_t(n_clusters) * kD * 4), dl(size_t(n) * 4);
  put(dk, kb.data(), kb.size());
  put(dr, rows.data(), rows.size());
  ckv_kmeans_desc desc{1, n, n_clusters, max_iters, uint64_t(n) * kD, n_clusters, n,
                       CKV_KM_OBJECTIVE | CKV_KM_NO_VALIDATE};
  ckv_kmeans_info info{};
  std::vector<double> obj(max_iters + 1);
  std::vector<uint32_t> rep(max_iters + 1);
  check(ckv_kmeans(ctx(), &desc, dk.as<uint16_t>(), dr.as<uint32_t>(), dc.as<float>(),
                   dl.as<int32_t>(), &info, obj.data(), rep.data()));
  ClusterModel m;
  m.n_clusters = n_clusters;
  m.centroids = Matrix(n_clusters, kD);
  m.labels.resize(n);
  get(m.centroids.data.data(), dc, m.centroids.data.size());
  get(m.labels.data(), dl, n);
  m.converged = info.converged != 0;
  m.iterations_used = info.iterations_used;
  m.objective_history.assign(obj.begin(), obj.begin() + info.n_objective);
  m.repair_iterations.assign(rep.begin(), rep.begin() + info.n_repair);
  m.invocation_iterations.push_back(info.iterations_used);
  return m;
}

// clustering.hpp:267-274
uint32_t prefill_cluster_count(uint32_t prompt_len, const ClusterConfig& cfg) {
  return ckv_prefill_cluster_count(prompt_len, cfg.c0_divisor, cfg.sink_tokens, cfg.c0_override);
}

// clustering.hpp:278-305
ClusterModel cluster_prefill(const Matrix& keys, const ClusterConfig& cfg) {
  cfg.validate();
  const uint32_t L = keys.rows;
  if (L <= cfg.sink_tokens) {
    ClusterModel m;
    m.sink_count = L;
    m.labels.assign(L, -1);
    m.converged = true;
    m.centroids = Matrix(0, keys.cols);
    return m;
  }
  const uint32_t sink = cfg.sink_tokens;
  Matrix clusterable(L - sink, keys.cols);
  std::copy(keys.data.begin() + size_t(sink) * keys.cols, keys.data.end(),
            clusterable.data.begin());
  ClusterModel m = kmeans_cosine(clusterable, prefill_cluster_count(L, cfg), cfg.seed,
                                 cfg.max_iters, cfg.metric);
  m.sink_count = sink;
  std::vector<int32_t> labels(L, -1);
  std::copy(m.labels.begin(), m.labels.end(), labels.begin() + sink);
  m.labels = std::move(labels);
  return m;
}

// clustering.hpp:310-332
void cluster_decode_batch(ClusterModel& model, const Matrix& new_keys, const ClusterConfig& cfg) {
  if (new_keys.rows == 0) return;
  cfg.validate();
  const uint32_t c = std::min(cfg.c_plus, new_keys.rows);
  const uint64_t bseed = mix_seed(cfg.seed, 0xdecadeull, model.n_positions());
  ClusterModel sub = kmeans_cosine(new_keys, c, bseed, cfg.max_iters, cfg.metric);
  const uint32_t base = model.n_clusters;
  Matrix merged(base + c, new_keys.cols);
  std::copy(model.centroids.data.begin(), model.centroids.data.end(), merged.data.begin());
  std::copy(sub.centroids.data.begin(), sub.centroids.data.end(),
            merged.data.begin() + size_t(base) * new_keys.cols);
  model.centroids = std::move(merged);
  model.n_clusters += c;
  for (int32_t l : sub.labels) model.labels.push_back(l + int32_t(base));
  model.iterations_used += sub.iterations_used;
  model.converged = model.converged && sub.converged;
  model.objective_history = std::move(sub.objective_history);
  model.invocation_iterations.push_back(sub.iterations_used);
}

// ---------------------------------------------------------------------------
// selection.hpp:29-48
ClusterIndex build_index(const ClusterModel& model) {
  const uint32_t C = model.n_clusters, P = model.n_positions();
  const uint32_t cc = std::max(C, 1u), pp = std::max(P, 1u);
  Dev dl(size_t(pp) * 4), dn(4), ds(size_t(cc) * 4), dst(size_t(cc + 1) * 4),
      dsrt(size_t(pp) * 4);
  put(dl, model.labels.data(), P);
  put(dn, &C, 1);
  check(ckv_build_index(ctx(), 1, P, pp, cc, dl.as<int32_t>(), dn.as<uint32_t>(),
                        ds.as<uint32_t>(), dst.as<uint32_t>(), dsrt.as<uint32_t>()));
  ClusterIndex ix;
  ix.sizes.resize(C);
  ix.cluster_start.resize(C + 1);
  get(ix.sizes.data(), ds, C);
  get(ix.cluster_start.data(), dst, C + 1);
  ix.sorted_token_ids.resize(ix.cluster_start[C]);
  get(ix.sorted_token_ids.data(), dsrt, ix.sorted_token_ids.size());
  return ix;
}

namespace {
SelectionResult run_select(std::span<const float> q, const ClusterModel& model,
                           const ClusterIndex& index, uint32_t budget,
                           std::vector<double>* scores) {
  if (q.size() != kD) throw ValidationError("select: the B200 kernels specialise d = 128");
  const uint32_t C = model.n_clusters;
  const uint32_t cc = std::max(C, 1u);
  const uint32_t pp = std::max<uint32_t>(index.labeled_total(), 1u);
  const uint32_t sel_cap = std::min(index.labeled_total(), budget) + model.sink_count + 1;
  Dev dq(kD * 4), dc(size_t(cc) * kD * 4), dn(4), ds(size_t(cc) * 4), dst(size_t(cc + 1) * 4),
      dsrt(size_t(pp) * 4), dtok(size_t(sel_cap) * 4), dnt(4), dtk(4), dtr(4),
      drk(size_t(cc) * 4), dsc(size_t(cc) * 8);
  put(dq, q.data(), kD);
  put(dc, model.centroids.data.data(), size_t(C) * kD);
  put(dn, &C, 1);
  put(ds, index.sizes.data(), C);
  put(dst, index.cluster_start.data(), C + 1);
  put(dsrt, index.sorted_token_ids.data(), index.labeled_total());
  ckv_select_desc d{};
  d.n_q = 1;
  d.group = 1;
  d.budget = budget;
  d.sink_count = model.sink_count;
  d.p_cap = pp;
  d.c_cap = cc;
  d.sel_cap = sel_cap;
  d.flags = CKV_SEL_FULL_RANK | (scores ? CKV_SEL_SCORES : 0u);
  check(ckv_select(ctx(), &d, dq.as<float>(), dc.as<float>(), dn.as<uint32_t>(),
                   ds.as<uint32_t>(), dst.as<uint32_t>(), dsrt.as<uint32_t>(),
                   dtok.as<uint32_t>(), nullptr, nullptr, dnt.as<uint32_t>(), dtk.as<uint32_t>(),
                   dtr.as<uint32_t>(), drk.as<uint32_t>(), scores ? dsc.as<double>() : nullptr,
                   nullptr));
  SelectionResult r;
  r.budget = budget;
  uint32_t nt = 0;
  get(&nt, dnt, 1);
  get(&r.n_clusters_taken, dtk, 1);
  get(&r.trimmed_from_last, dtr, 1);
  r.ranked_clusters.resize(C);
  get(r.ranked_clusters.data(), drk, C);
  r.token_ids.resize(nt);
  get(r.token_ids.data(), dtok, nt);
  if (scores) {
    scores->resize(C);
    get(scores->data(), dsc, C);
  }
  return r;
}
}  // namespace

// selection.hpp:51-57
std::vector<double> score_clusters(std::span<const float> q, const ClusterModel& model) {
  ClusterIndex empty;
  empty.sizes.assign(model.n_clusters, 0);
  empty.cluster_start.assign(model.n_clusters + 1, 0);
  std::vector<double> s;
  run_select(q, model, empty, 1, &s);
  return s;
}

// selection.hpp:74-111 (the recency span is appended verbatim after the sinks)
SelectionResult select_tokens(std::span<const float> q, const ClusterModel& model,
                              const ClusterIndex& index, uint32_t budget,
                              std::span<const uint32_t> recency) {
  SelectionResult r = run_select(q, model, index, budget, nullptr);
  r.token_ids.insert(r.token_ids.end(), recency.begin(), recency.end());
  return r;
}

// ---------------------------------------------------------------------------
// selection.hpp:141-194
std::vector<uint32_t> page_select(std::span<const float> q, const Matrix& keys, uint32_t budget,
                                  uint32_t page_size, PageRepr repr) {
  if (page_size < 1) throw ValidationError("page_select: page_size must be >= 1");
  require_d128(keys, "page_select");
  if (q.size() != kD) throw ValidationError("page_select: the B200 kernels specialise d = 128");
  const uint32_t n = keys.rows, n_pages = (n + page_size - 1) / page_size;
  const uint32_t n_sel = std::min(n_pages, budget / page_size);
  if (n_sel == 0) return {};
  const std::vector<uint16_t> kb = to_bf16(keys, "page_select keys");
  const bool mm = repr == PageRepr::MaxMin;
  Dev dk(kb.size() * 2), dq(kD * 4), dmax(size_t(n_pages) * kD * 4),
      dmin(mm ? size_t(n_pages) * kD * 4 : 16), drow(size_t(n_sel + 1) * 4),
      doff(size_t(n_sel + 2) * 4), dcnt(4), dids(size_t(n_sel) * page_size * 4), dnt(4);
  put(dk, kb.data(), kb.size());
  put(dq, q.data(), kD);
  check(ckv_page_reps(ctx(), 1, n, n, page_size, n_pages, dk.as<uint16_t>(), dmax.as<float>(),
                      mm ? dmin.as<float>() : nullptr));
  ckv_runs runs{drow.as<uint32_t>(), doff.as<uint32_t>(), dcnt.as<uint32_t>(), n_sel + 1};
  ckv_page_desc d{1, 1, n, page_size, budget, n_pages, n_sel * page_size, mm ? 1u : 0u};
  check(ckv_page_select(ctx(), &d, dq.as<float>(), dmax.as<float>(),
                        mm ? dmin.as<float>() : nullptr, &runs, dids.as<uint32_t>(),
                        dnt.as<uint32_t>()));
  uint32_t k = 0;
  get(&k, dnt, 1);
  std::vector<uint32_t> ids(k);
  get(ids.data(), dids, k);
  return ids;
}

// ---------------------------------------------------------------------------
// attention.hpp:63-69
AttentionOutput approx_attention(std::span<const float> q, const Matrix& keys,
                                 const Matrix& values, std::span<const uint32_t> selected) {
  if (selected.empty()) throw ValidationError("approx_attention: empty selection");
  require_d128(keys, "approx_attention");
  if (q.size() != kD) throw ValidationError("approx_attention: the B200 kernels specialise d = 128");
  for (uint32_t r : selected)
    if (r >= keys.rows) throw ValidationError("approx_attention: selected id out of range");
  const std::vector<uint16_t> kb = to_bf16(keys, "approx_attention keys");
  const std::vector<uint16_t> vb = to_bf16(values, "approx_attention values");
  const uint32_t n = uint32_t(selected.size());
  Dev dq(kD * 4), dk(kb.size() * 2), dv(vb.size() * 2), dr(size_t(n) * 4), dn(4), dout(kD * 4),
      dw(size_t(n) * 4);
  put(dq, q.data(), kD);
  put(dk, kb.data(), kb.size());
  put(dv, vb.data(), vb.size());
  put(dr, selected.data(), n);
  put(dn, &n, 1);
  ckv_attend_desc d{1, 1, keys.rows, n, n};
  check(ckv_attend(ctx(), &d, dq.as<float>(), dk.as<uint16_t>(), dv.as<uint16_t>(),
                   dr.as<uint32_t>(), nullptr, dn.as<uint32_t>(), dout.as<float>(),
                   dw.as<float>()));
  AttentionOutput o;
  o.out.resize(kD);
  o.weights.resize(n);
  get(o.out.data(), dout, kD);
  get(o.weights.data(), dw, n);
  return o;
}

// ---------------------------------------------------------------------------
// cache.hpp:25-93 — counters and the resident sets live on the GPU (bitmap
// ring, the same structure the fused decode path updates); the host keeps a
// mirror of the ring only to answer resident().
namespace {
constexpr uint32_t kCacheIds = 1u << 20;  // cluster-id capacity of the bitmaps
}

ClusterCache::ClusterCache(uint32_t retention, uint32_t head_dim)
    : retention_(retention), d_(head_dim) {
  if (retention < 1) throw ValidationError("ClusterCache: retention must be >= 1");
  ckv_cache* c = nullptr;
  check(ckv_cache_create(ctx(), 1, kCacheIds, retention, head_dim, &c));
  handle_ = c;
}

ClusterCache::~ClusterCache() { ckv_cache_destroy(static_cast<ckv_cache*>(handle_)); }

ClusterCache::LookupResult ClusterCache::lookup_and_update(std::span<const uint32_t> selected,
                                                           std::span<const uint32_t> sizes) {
  for (uint32_t id : selected)
    if (id >= kCacheIds) throw ValidationError("ClusterCache: cluster id beyond 2^20");
  const uint32_t n = uint32_t(selected.size());
  Dev ds(size_t(std::max(n, 1u)) * 4), dz(std::max<size_t>(sizes.size(), 1) * 4),
      dh(size_t(std::max(n, 1u)) * 4), dm(size_t(std::max(n, 1u)) * 4);
  put(ds, selected.data(), n);
  put(dz, sizes.data(), sizes.size());
  uint32_t counts[2] = {0, 0};
  check(ckv_cache_lookup(ctx(), static_cast<ckv_cache*>(handle_), 0, ds.as<uint32_t>(), n,
                         dz.as<uint32_t>(), dh.as<uint32_t>(), dm.as<uint32_t>(), counts));
  LookupResult r;
  r.hit_ids.resize(counts[0]);
  r.miss_ids.resize(counts[1]);
  get(r.hit_ids.data(), dh, counts[0]);
  get(r.miss_ids.data(), dm, counts[1]);
  ring_.emplace_back(selected.begin(), selected.end());
  if (ring_.size() > retention_) ring_.erase(ring_.begin());
  resident_.clear();
  for (const auto& s : ring_) resident_.insert(s.begin(), s.end());
  return r;
}

const CacheCounters& ClusterCache::counters() const {
  uint64_t c[4];
  check(ckv_cache_counters(static_cast<ckv_cache*>(handle_), c));
  counters_ = {c[0], c[1], c[2], c[3]};
  return counters_;
}

double ClusterCache::hit_rate() const {
  const CacheCounters& c = counters();
  if (c.clusters_requested == 0) throw ValidationError("ClusterCache: hit_rate with zero requests");
  return double(c.clusters_hit) / double(c.clusters_requested);
}

void ClusterCache::invalidate_on_recluster(std::span<const uint32_t> retired,
                                           std::span<const uint32_t> fresh) {
  (void)fresh;
  if (retired.empty()) return;
  std::vector<uint32_t> r;
  for (uint32_t id : retired)
    if (id < kCacheIds) r.push_back(id);
  check(ckv_cache_invalidate(ctx(), static_cast<ckv_cache*>(handle_), 0, r.data(),
                             uint32_t(r.size())));
  const std::set<uint32_t> dead(retired.begin(), retired.end());
  for (auto& s : ring_) std::erase_if(s, [&](uint32_t id) { return dead.count(id) > 0; });
  resident_.clear();
  for (const auto& s : ring_) resident_.insert(s.begin(), s.end());
}

}  // namespace ckv

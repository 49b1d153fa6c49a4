// clusterkv_b200/clusterkv.hpp — drop-in replacement for the hot-path API of
// the reference's proj/include/clusterkv/{common,clustering,selection,
// attention,cache}.hpp, running on B200 (sm_100a) through libckv_b200.so.
//
// Same namespace, type names, field layouts, signatures, defaults and
// ValidationError predicates as the reference (file:line per declaration), so
// a caller switches by changing the include path and linking
// -lckv_b200.  Differences, all documented in DESIGN.md:
//   * keys / values must be bf16-representable f32 (the B200 KV store is
//     bf16); anything else throws ValidationError.
//   * d must be 128; AssignMetric::Cosine only (L2 / InnerProduct are
//     reference ablations) — others throw ValidationError.
//   * approx_attention is computed in f32 (reference: f64), within the
//     tolerance of tests/test_gpu_attend.py.
// Every integer output (labels, iteration counts, selections, index, cache
// counters) and every centroid bit equals the reference's.
#pragma once

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdint>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace ckv {

// ---- errors (common.hpp:21-55) ----------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ValidationError : public Error {
 public:
  using Error::Error;
};
class IoError : public Error {
 public:
  using Error::Error;
};
class ParseError : public Error {
 public:
  enum class Code { BadMagic, BadVersion, Truncated, DimOverflow, BadMetadata, TrailingData };
  ParseError(Code code, const std::string& what) : Error(what), code_(code) {}
  Code code() const { return code_; }

 private:
  Code code_;
};

// ---- dense row-major f32 matrix (common.hpp:61-77) -----------------------------
struct Matrix {
  uint32_t rows = 0;
  uint32_t cols = 0;
  std::vector<float> data;

  Matrix() = default;
  Matrix(uint32_t r, uint32_t c) : rows(r), cols(c), data(size_t(r) * c, 0.0f) {}
  std::span<const float> row(uint32_t i) const { return {data.data() + size_t(i) * cols, cols}; }
  std::span<float> row(uint32_t i) { return {data.data() + size_t(i) * cols, cols}; }
  bool operator==(const Matrix&) const = default;
};

// ---- host numerics helpers (common.hpp:79-147) ---------------------------------
inline bool is_finite(const Matrix& m) {
  for (float v : m.data)
    if (!std::isfinite(v)) return false;
  return true;
}
inline double dot_f64(std::span<const float> a, std::span<const float> b) {
  double acc = 0.0;
  for (size_t i = 0; i < a.size(); ++i) acc += double(a[i]) * double(b[i]);
  return acc;
}
inline double norm_f64(std::span<const float> a) { return std::sqrt(dot_f64(a, a)); }
inline double normalize(std::span<float> v) {
  const double n = norm_f64(v);
  if (n > 0.0)
    for (float& x : v) x = float(double(x) / n);
  return n;
}
constexpr uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
constexpr uint64_t mix_seed(uint64_t seed, uint64_t a, uint64_t b = 0) {
  return splitmix64(splitmix64(splitmix64(seed) ^ (a + 0x9e3779b97f4a7c15ull)) ^
                    (b + 0xbf58476d1ce4e5b9ull));
}

// ---- clustering types (clustering.hpp:18-65) -----------------------------------
enum class AssignMetric { Cosine, L2, InnerProduct };

struct ClusterConfig {
  uint32_t c0_divisor = 80;
  uint32_t c_plus = 4;
  uint32_t decode_batch = 320;
  uint32_t sink_tokens = 16;
  uint32_t max_iters = 50;
  uint64_t seed = 0;
  uint32_t c0_override = 0;
  AssignMetric metric = AssignMetric::Cosine;

  void validate() const {
    if (c0_divisor < 1) throw ValidationError("ClusterConfig: c0_divisor must be >= 1");
    if (c_plus < 1) throw ValidationError("ClusterConfig: c_plus must be >= 1");
    if (decode_batch < 1) throw ValidationError("ClusterConfig: decode_batch must be >= 1");
    if (max_iters < 1) throw ValidationError("ClusterConfig: max_iters must be >= 1");
  }
};

struct ClusterModel {
  uint32_t n_clusters = 0;
  Matrix centroids;
  std::vector<int32_t> labels;
  uint32_t sink_count = 0;
  bool converged = false;
  uint32_t iterations_used = 0;
  std::vector<double> objective_history;
  std::vector<uint32_t> repair_iterations;
  std::vector<uint32_t> invocation_iterations;
  uint32_t n_positions() const { return uint32_t(labels.size()); }
};

inline double cosine_distance(std::span<const float> a, std::span<const float> b) {
  const double na = norm_f64(a), nb = norm_f64(b);
  if (na < 1e-12 || nb < 1e-12) return 1.0;
  return std::clamp(1.0 - dot_f64(a, b) / (na * nb), 0.0, 2.0);
}

// B200 implementations (libckv_b200.so)
ClusterModel kmeans_cosine(const Matrix& keys, uint32_t n_clusters, uint64_t seed,
                           uint32_t max_iters = 50, AssignMetric metric = AssignMetric::Cosine,
                           std::span<const uint32_t> init_rows = {});    // clustering.hpp:160
uint32_t prefill_cluster_count(uint32_t prompt_len, const ClusterConfig& cfg);  // :267
ClusterModel cluster_prefill(const Matrix& keys, const ClusterConfig& cfg);     // :278
void cluster_decode_batch(ClusterModel& model, const Matrix& new_keys,
                          const ClusterConfig& cfg);                            // :310

// ---- selection (selection.hpp:16-111) -------------------------------------------
struct ClusterIndex {
  std::vector<uint32_t> sizes;
  std::vector<uint32_t> sorted_token_ids;
  std::vector<uint32_t> cluster_start;
  uint32_t labeled_total() const { return uint32_t(sorted_token_ids.size()); }
  std::span<const uint32_t> cluster_slice(uint32_t c) const {
    return {sorted_token_ids.data() + cluster_start[c], sizes[c]};
  }
};

struct SelectionResult {
  std::vector<uint32_t> ranked_clusters;
  uint32_t n_clusters_taken = 0;
  std::vector<uint32_t> token_ids;
  uint32_t trimmed_from_last = 0;
  uint32_t budget = 0;
  std::span<const uint32_t> taken_clusters() const {
    return {ranked_clusters.data(), n_clusters_taken};
  }
};

ClusterIndex build_index(const ClusterModel& model);                       // selection.hpp:29
std::vector<double> score_clusters(std::span<const float> q,
                                   const ClusterModel& model);             // :51
SelectionResult select_tokens(std::span<const float> q, const ClusterModel& model,
                              const ClusterIndex& index, uint32_t budget,
                              std::span<const uint32_t> recency = {});     // :74

// ---- attention (attention.hpp:11-69) --------------------------------------------
struct AttentionOutput {
  std::vector<float> out;
  std::vector<float> weights;
};
// selection.hpp:136-194 — the page-based baseline (Quest-style)
enum class PageRepr {
  Max,     // elementwise max over member keys
  MaxMin,  // score = sum_ch max(q*max_k, q*min_k)
};
std::vector<uint32_t> page_select(std::span<const float> q, const Matrix& keys, uint32_t budget,
                                  uint32_t page_size, PageRepr repr = PageRepr::Max);

AttentionOutput approx_attention(std::span<const float> q, const Matrix& keys,
                                 const Matrix& values,
                                 std::span<const uint32_t> selected);      // attention.hpp:63

// ---- cluster cache (cache.hpp:12-93), state on the GPU --------------------------
struct CacheCounters {
  uint64_t clusters_requested = 0;
  uint64_t clusters_hit = 0;
  uint64_t tokens_transferred = 0;
  uint64_t bytes_transferred = 0;
};

class ClusterCache {
 public:
  ClusterCache(uint32_t retention, uint32_t head_dim);
  ~ClusterCache();
  ClusterCache(const ClusterCache&) = delete;
  ClusterCache& operator=(const ClusterCache&) = delete;

  struct LookupResult {
    std::vector<uint32_t> hit_ids;
    std::vector<uint32_t> miss_ids;
  };
  LookupResult lookup_and_update(std::span<const uint32_t> selected,
                                 std::span<const uint32_t> sizes);          // cache.hpp:38
  double hit_rate() const;                                                  // :59
  void invalidate_on_recluster(std::span<const uint32_t> retired,
                               std::span<const uint32_t> fresh);           // :67
  const CacheCounters& counters() const;
  const std::set<uint32_t>& resident() const { return resident_; }
  uint32_t retention() const { return retention_; }

 private:
  void* handle_ = nullptr;  // ckv_cache*
  uint32_t retention_, d_;
  mutable CacheCounters counters_;
  std::set<uint32_t> resident_;  // host mirror of the union of the last R sets
  std::vector<std::vector<uint32_t>> ring_;
};

}  // namespace ckv

// shim_parity.cpp — the reference-signature C++ drop-in
// (include/clusterkv_b200/clusterkv.hpp, running on the B200 kernels) against
// the CPU oracle (oracle/ckv_oracle.c).  Built and run by
// tests/test_gpu_shim.py; exit status 0 = every check passed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "ckv_oracle.h"
#include "clusterkv_b200/clusterkv.hpp"

static int g_fail = 0;
#define CHECK(cond, ...)                          \
  do {                                            \
    if (!(cond)) {                                \
      std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      std::fprintf(stderr, __VA_ARGS__);          \
      std::fprintf(stderr, "\n");                 \
      ++g_fail;                                   \
    }                                             \
  } while (0)

static float bf16_round(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  const uint32_t r = ((u >> 16) & 1u) + 0x7fffu;
  u = ((u + r) >> 16) << 16;
  std::memcpy(&x, &u, 4);
  return x;
}

static ckv::Matrix to_matrix(const std::vector<float>& v, uint32_t rows, uint32_t cols) {
  ckv::Matrix m(rows, cols);
  for (size_t i = 0; i < v.size(); ++i) m.data[i] = bf16_round(v[i]);
  return m;
}

int main() {
  const uint32_t d = 128, L = 2048 + 16, T = 40;
  orc_synth_spec spec;
  orc_synth_spec_default(&spec);
  spec.prompt_len = L;
  spec.decode_len = T;
  std::vector<float> pk(size_t(L) * d), pv(size_t(L) * d), dq(size_t(T) * d),
      dk(size_t(T) * d), dv(size_t(T) * d);
  orc_generate_head(&spec, orc_mix_seed(7, 0, 3), pk.data(), pv.data(), dq.data(), dk.data(),
                    dv.data());
  const ckv::Matrix K = to_matrix(pk, L, d), V = to_matrix(pv, L, d), Q = to_matrix(dq, T, d);
  const ckv::Matrix DK = to_matrix(dk, T, d);

  // ---- cluster_prefill (clustering.hpp:278) ----
  ckv::ClusterConfig cfg;
  cfg.seed = ckv::mix_seed(0, 0, 3);
  cfg.decode_batch = 20;
  const ckv::ClusterModel g = ckv::cluster_prefill(K, cfg);
  orc_cluster_config oc;
  orc_cluster_config_default(&oc);
  oc.seed = cfg.seed;
  const uint32_t C0 = orc_prefill_cluster_count(L, &oc);
  std::vector<float> oc_cent(size_t(C0 + 64) * d);
  std::vector<int32_t> oc_lab(L + T);
  std::vector<double> oh(oc.max_iters + 2);
  std::vector<uint32_t> orep(oc.max_iters + 2);
  orc_kmeans_info oi;
  uint32_t osink = 0;
  CHECK(orc_cluster_prefill(K.data.data(), L, d, &oc, oc_cent.data(), oc_lab.data(), oh.data(),
                            orep.data(), &oi, &osink) == 0, "oracle prefill");
  CHECK(g.n_clusters == C0 && g.sink_count == osink, "C0 %u vs %u", g.n_clusters, C0);
  CHECK(g.iterations_used == oi.iterations_used && g.converged == bool(oi.converged),
        "iterations %u vs %u", g.iterations_used, oi.iterations_used);
  CHECK(std::equal(g.labels.begin(), g.labels.end(), oc_lab.begin()), "prefill labels differ");
  CHECK(std::memcmp(g.centroids.data.data(), oc_cent.data(), size_t(C0) * d * 4) == 0,
        "prefill centroids differ");
  CHECK(g.objective_history.size() == oi.n_objective, "objective length");
  for (size_t i = 0; i < g.objective_history.size(); ++i)
    CHECK(std::fabs(g.objective_history[i] - oh[i]) <= 1e-9 * std::max(1.0, std::fabs(oh[i])),
          "objective[%zu] %.17g vs %.17g", i, g.objective_history[i], oh[i]);

  // ---- build_index (selection.hpp:29) ----
  const ckv::ClusterIndex ix = ckv::build_index(g);
  std::vector<uint32_t> os(C0), ost(C0 + 1), osrt(L);
  orc_build_index(oc_lab.data(), L, C0, os.data(), ost.data(), osrt.data());
  CHECK(ix.sizes == std::vector<uint32_t>(os.begin(), os.end()), "index sizes");
  CHECK(ix.cluster_start == ost, "index starts");
  CHECK(std::equal(ix.sorted_token_ids.begin(), ix.sorted_token_ids.end(), osrt.begin()),
        "sorted ids");

  // ---- select_tokens + approx_attention (selection.hpp:74, attention.hpp:63) ----
  std::vector<uint32_t> rec = {L, L + 1, L + 2};
  for (uint32_t t = 0; t < T; t += 7) {
    std::span<const float> q = Q.row(t);
    for (uint32_t B : {64u, 512u, 5000u}) {
      const ckv::SelectionResult r = ckv::select_tokens(q, g, ix, B, rec);
      std::vector<uint32_t> rk(C0), tok(L + 8);
      uint32_t nt = 0, tr = 0;
      const uint32_t n = orc_select_tokens(q.data(), oc_cent.data(), C0, d, os.data(), ost.data(),
                                           osrt.data(), osink, B, rec.data(), 3, rk.data(), &nt,
                                           &tr, tok.data());
      CHECK(r.ranked_clusters == rk, "ranking differs t=%u B=%u", t, B);
      CHECK(r.n_clusters_taken == nt && r.trimmed_from_last == tr, "taken/trim t=%u B=%u", t, B);
      CHECK(r.token_ids.size() == n && std::equal(r.token_ids.begin(), r.token_ids.end(), tok.begin()),
            "token ids differ t=%u B=%u", t, B);
      const std::vector<double> sc = ckv::score_clusters(q, g);
      std::vector<double> osc(C0);
      orc_score_clusters(q.data(), oc_cent.data(), C0, d, osc.data());
      CHECK(std::memcmp(sc.data(), osc.data(), C0 * 8) == 0, "scores differ");
      std::vector<uint32_t> rows(r.token_ids.begin(), r.token_ids.end());
      rows.erase(std::remove_if(rows.begin(), rows.end(), [&](uint32_t x) { return x >= L; }),
                 rows.end());
      const ckv::AttentionOutput a = ckv::approx_attention(q, K, V, rows);
      std::vector<float> oo(d), ow(rows.size());
      orc_attention_over(q.data(), K.data.data(), V.data.data(), d, rows.data(),
                         uint32_t(rows.size()), oo.data(), ow.data());
      double vmax = 0, err = 0, werr = 0;
      for (float x : V.data) vmax = std::max(vmax, double(std::fabs(x)));
      for (uint32_t j = 0; j < d; ++j) err = std::max(err, double(std::fabs(a.out[j] - oo[j])));
      for (size_t j = 0; j < rows.size(); ++j)  // |dw| <= 1e-6 + 2e-5 w
        werr = std::max(werr, double(std::fabs(a.weights[j] - ow[j])) - 2e-5 * ow[j]);
      CHECK(err <= 2e-5 * vmax, "attention max|dout| %.3g", err);
      CHECK(werr <= 1e-6, "attention weight error %.3g over bound", werr);
    }
  }

  // ---- cluster_decode_batch (clustering.hpp:310) ----
  ckv::ClusterModel g2 = g;
  ckv::Matrix batch(20, d);
  std::copy(DK.data.begin(), DK.data.begin() + 20 * d, batch.data.begin());
  ckv::cluster_decode_batch(g2, batch, cfg);
  uint32_t onc = C0, onp = L, oit = 0;
  int32_t oconv = 0;
  oc.decode_batch = 20;
  CHECK(orc_cluster_decode_batch(oc_cent.data(), &onc, oc_lab.data(), &onp, batch.data.data(), 20,
                                 d, &oc, &oit, &oconv) == 0, "oracle decode batch");
  CHECK(g2.n_clusters == onc && g2.n_positions() == onp, "decode batch sizes");
  CHECK(std::equal(g2.labels.begin(), g2.labels.end(), oc_lab.begin()), "decode labels");
  CHECK(std::memcmp(g2.centroids.data.data(), oc_cent.data(), size_t(onc) * d * 4) == 0,
        "decode centroids");
  CHECK(g2.invocation_iterations.back() == oit, "decode iterations");

  // ---- ClusterCache (cache.hpp:25-93) ----
  for (uint32_t R : {1u, 2u}) {
    ckv::ClusterCache cache(R, d);
    orc_cache* occ = orc_cache_new(R, d);
    for (uint32_t t = 0; t < T; ++t) {
      const ckv::SelectionResult r = ckv::select_tokens(Q.row(t), g, ix, 256);
      std::vector<uint32_t> sel(r.taken_clusters().begin(), r.taken_clusters().end());
      std::sort(sel.begin(), sel.end());
      const auto lr = cache.lookup_and_update(sel, ix.sizes);
      std::vector<uint32_t> hit(sel.size() + 1), miss(sel.size() + 1);
      uint32_t nh = 0, nm = 0;
      orc_cache_lookup_and_update(occ, sel.data(), uint32_t(sel.size()), ix.sizes.data(),
                                  hit.data(), &nh, miss.data(), &nm);
      CHECK(lr.hit_ids == std::vector<uint32_t>(hit.begin(), hit.begin() + nh), "cache hits R=%u", R);
      CHECK(lr.miss_ids == std::vector<uint32_t>(miss.begin(), miss.begin() + nm), "cache misses");
    }
    uint64_t oc4[4];
    orc_cache_counters(occ, oc4);
    const ckv::CacheCounters& c = cache.counters();
    CHECK(c.clusters_requested == oc4[0] && c.clusters_hit == oc4[1] &&
          c.tokens_transferred == oc4[2] && c.bytes_transferred == oc4[3], "cache counters R=%u", R);
    orc_cache_free(occ);
  }

  // ---- page_select (selection.hpp:141-194), both representatives ----
  for (int mm = 0; mm < 2; ++mm) {
    for (uint32_t t = 0; t < 3; ++t) {
      const auto got = ckv::page_select(Q.row(t), K, 512, 16,
                                        mm ? ckv::PageRepr::MaxMin : ckv::PageRepr::Max);
      std::vector<uint32_t> exp(512);
      const uint32_t k = orc_page_select(Q.row(t).data(), K.data.data(), L, d, 512, 16, mm,
                                         exp.data());
      exp.resize(k);
      CHECK(got == exp, "page_select repr %d step %u", mm, t);
    }
  }

  // ---- ValidationError predicates (clustering.hpp:166-172, attention.hpp:66) ----
  auto throws = [](auto&& f) {
    try {
      f();
    } catch (const ckv::ValidationError&) {
      return true;
    }
    return false;
  };
  CHECK(throws([&] { ckv::kmeans_cosine(K, L + 1, 0); }), "C > N must throw");
  CHECK(throws([&] { ckv::kmeans_cosine(K, 0, 0); }), "C = 0 must throw");
  CHECK(throws([&] { ckv::approx_attention(Q.row(0), K, V, {}); }), "empty selection must throw");
  CHECK(throws([&] { ckv::page_select(Q.row(0), K, 64, 0); }), "page_size 0 must throw");
  CHECK(throws([&] { ckv::kmeans_cosine(ckv::Matrix(32, d), 4, 0); }), "all-zero keys must throw");
  CHECK(throws([&] {
          ckv::ClusterCache c(0, d);
          (void)c;
        }), "retention 0 must throw");

  if (g_fail) {
    std::fprintf(stderr, "%d checks failed\n", g_fail);
    return 1;
  }
  std::printf("shim parity OK: C0=%u iters=%u\n", C0, g.iterations_used);
  return 0;
}

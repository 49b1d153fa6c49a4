// C++ host of the sequence-sharded k-means through the C-ABI only (no
// PyTorch, no Python): ckv_kmeans_sharded over world 1 (NCCL) and worlds 2-3
// (LOCAL: the ranks are std::threads sharing GPU 0, each with its own
// context), checked bit for bit against the C oracle's kmeans_cosine
// (clustering.hpp:160-263).  Run by tests/test_gpu_sharded_native.py.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ckv_cuda.h"
#include "ckv_oracle.h"

static int failures = 0;
#define CHECK(cond, ...)                                         \
  do {                                                           \
    if (!(cond)) {                                               \
      ++failures;                                                \
      std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      std::fprintf(stderr, __VA_ARGS__);                         \
      std::fprintf(stderr, "\n");                                \
    }                                                            \
  } while (0)

static uint16_t f32_to_bf16(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}
static float bf16_to_f32(uint16_t b) {
  const uint32_t u = uint32_t(b) << 16;
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

struct RankOut {
  std::vector<int32_t> labels;
  std::vector<float> cents;
  std::vector<ckv_kmeans_info> info;
  int rc = 0;
  std::string err;
};

// keys [U][n][128] bf16 bits; rank r holds rows [lo, hi)
static void run_rank(int world, int r, const std::vector<uint16_t>& kb, uint32_t U, uint32_t n,
                     uint32_t C, const std::vector<uint64_t>& seeds, ckv_local_group* group,
                     const unsigned char* nccl_id, RankOut* out) {
  const uint64_t lo = uint64_t(n) * r / world, hi = uint64_t(n) * (r + 1) / world;
  const uint32_t nl = uint32_t(hi - lo);
  ckv_ctx* ctx = nullptr;
  ckv_comm* comm = nullptr;
  void *dk = nullptr, *dc = nullptr, *dl = nullptr;
  auto fail = [&](int rc) { out->rc = rc; out->err = ckv_last_error(); };
  int rc = ckv_ctx_create(0, nullptr, &ctx);
  if (rc) return fail(rc);
  rc = group ? ckv_comm_create_local(ctx, group, r, &comm)
             : ckv_comm_create_nccl(ctx, world, r, nccl_id, &comm);
  if (rc) return fail(rc);
  std::vector<uint16_t> mine(size_t(U) * nl * 128);
  for (uint32_t u = 0; u < U; ++u)
    std::memcpy(&mine[size_t(u) * nl * 128], &kb[(size_t(u) * n + lo) * 128], size_t(nl) * 256);
  if ((rc = ckv_malloc(ctx, &dk, mine.size() * 2)) || (rc = ckv_malloc(ctx, &dc, size_t(U) * C * 512)) ||
      (rc = ckv_malloc(ctx, &dl, size_t(U) * nl * 4)) ||
      (rc = ckv_memcpy_h2d(ctx, dk, mine.data(), mine.size() * 2)))
    return fail(rc);
  ckv_kmshard_desc d{U, nl, C, 0u, uint64_t(nl) * 128};
  out->info.resize(U);
  rc = ckv_kmeans_sharded(comm, &d, static_cast<const uint16_t*>(dk), n, lo, seeds.data(), nullptr,
                          50, static_cast<float*>(dc), static_cast<int32_t*>(dl), out->info.data());
  if (rc) return fail(rc);
  out->labels.resize(size_t(U) * nl);
  out->cents.resize(size_t(U) * C * 128);
  ckv_memcpy_d2h(ctx, out->labels.data(), dl, out->labels.size() * 4);
  ckv_memcpy_d2h(ctx, out->cents.data(), dc, out->cents.size() * 4);
  ckv_comm_destroy(comm);
  ckv_free(ctx, dk);
  ckv_free(ctx, dc);
  ckv_free(ctx, dl);
  ckv_ctx_destroy(ctx);
}

int main() {
  const uint32_t U = 2, n = 4000, C = 40, d = 128;
  // clustered synthetic keys (20 directions + noise), bf16-representable
  orc_mt64 g;
  orc_mt64_seed(&g, 12345);
  std::vector<float> centers(20 * d);
  for (auto& x : centers) x = float(orc_gaussian(&g));
  std::vector<float> keys(size_t(U) * n * d);
  std::vector<uint16_t> kb(keys.size());
  for (uint32_t u = 0; u < U; ++u)
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t c = uint32_t(orc_mt64_next(&g) % 20);
      for (uint32_t j = 0; j < d; ++j) {
        const size_t e = (size_t(u) * n + i) * d + j;
        kb[e] = f32_to_bf16(centers[c * d + j] + 0.35f * float(orc_gaussian(&g)));
        keys[e] = bf16_to_f32(kb[e]);
      }
    }
  std::vector<uint64_t> seeds(U);
  for (uint32_t u = 0; u < U; ++u) seeds[u] = orc_mix_seed(0, 7, u);
  // the oracle, per unit
  std::vector<std::vector<float>> oc(U, std::vector<float>(size_t(C) * d));
  std::vector<std::vector<int32_t>> ol(U, std::vector<int32_t>(n));
  std::vector<orc_kmeans_info> oi(U);
  for (uint32_t u = 0; u < U; ++u) {
    std::vector<double> oh(60);
    std::vector<uint32_t> orp(60);
    CHECK(orc_kmeans(&keys[size_t(u) * n * d], n, d, C, seeds[u], 50, 0, nullptr, 0, oc[u].data(),
                     ol[u].data(), oh.data(), orp.data(), &oi[u]) == 0, "oracle kmeans");
  }
  for (int world : {1, 2, 3}) {
    const bool nccl = world == 1;
    unsigned char id[CKV_NCCL_ID_BYTES] = {0};
    ckv_local_group* group = nullptr;
    if (nccl) {
      if (ckv_comm_nccl_id(id) != 0) { CHECK(false, "nccl id: %s", ckv_last_error()); continue; }
    } else {
      ckv_local_group_create(world, &group);
    }
    std::vector<RankOut> out(world);
    std::vector<std::thread> th;
    for (int r = 0; r < world; ++r)
      th.emplace_back(run_rank, world, r, std::cref(kb), U, n, C, std::cref(seeds), group, id, &out[r]);
    for (auto& t : th) t.join();
    if (group) ckv_local_group_destroy(group);
    bool ok = true;
    for (int r = 0; r < world; ++r)
      if (out[r].rc) { CHECK(false, "world %d rank %d: rc %d %s", world, r, out[r].rc, out[r].err.c_str()); ok = false; }
    if (!ok) continue;
    for (uint32_t u = 0; u < U; ++u) {
      std::vector<int32_t> lab;
      for (int r = 0; r < world; ++r) {
        const uint64_t lo = uint64_t(n) * r / world, hi = uint64_t(n) * (r + 1) / world;
        const size_t nl = size_t(hi - lo);
        lab.insert(lab.end(), out[r].labels.begin() + u * nl, out[r].labels.begin() + (u + 1) * nl);
        CHECK(std::memcmp(&out[r].cents[size_t(u) * C * d], oc[u].data(), size_t(C) * d * 4) == 0,
              "world %d rank %d unit %u: centroids differ", world, r, u);
        CHECK(out[r].info[u].iterations_used == oi[u].iterations_used &&
                  out[r].info[u].converged == oi[u].converged &&
                  out[r].info[u].n_repair == oi[u].n_repair,
              "world %d rank %d unit %u: iterations %u/%u converged %d/%d repairs %u/%u", world, r, u,
              out[r].info[u].iterations_used, oi[u].iterations_used, out[r].info[u].converged,
              oi[u].converged, out[r].info[u].n_repair, oi[u].n_repair);
      }
      CHECK(lab == ol[u], "world %d unit %u: labels differ", world, u);
    }
    std::printf("world %d (%s): iterations %u %u\n", world, nccl ? "NCCL" : "LOCAL",
                out[0].info[0].iterations_used, out[0].info[1].iterations_used);
  }
  if (failures) { std::printf("sharded_native: %d failures\n", failures); return 1; }
  std::printf("sharded_native: OK\n");
  return 0;
}

// ckv_comm.cu — collectives of the sequence-sharded paths (SURVEY §8e,
// config E) and the native host driver of the sharded k-means, so a C/C++
// host runs kmeans_cosine (clustering.hpp:160-263) over position shards
// without PyTorch.
//
// Two communicator backends behind one interface:
//   NCCL   one rank per GPU (a process or a thread each), ncclCommInitRank
//          from an ncclUniqueId the caller distributes; the collectives run
//          on the device buffers in place over NVLink / NVSwitch, ordered on
//          the context's stream.  libnccl is resolved at run time (dlopen),
//          so libckv_b200.so loads on hosts without it.
//   LOCAL  the ranks are threads of one process sharing a ckv_local_group:
//          the collectives stage through host memory behind a barrier.  For
//          several ranks on one GPU (tests) — NCCL refuses duplicate devices.
//
// ckv_kmeans_sharded is sharded.py's kmeans_cosine_sharded in C++: the
// per-shard device steps of ckv_kmshard.cu with an all-reduce SUM of the f64
// member sums and counts, an all-reduce MAX of the "changed" flags and one
// all-gather of (distance, row) per empty-cluster repair.  f64 sums of bf16
// keys are exact in any order, so every rank ends with the
// single-process reference's centroids, labels and iteration counts.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "ckv_internal.cuh"

namespace ckvb {
void host_init_rows_batch(uint32_t n_units, uint32_t n, uint32_t C, const uint64_t* seeds,
                          uint32_t* rows);
}

// ---------------------------------------------------------------------------
// NCCL, resolved at run time
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};
const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(h, "ncclAllGather"));
    a.getErrorString = reinterpret_cast<decltype(a.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.allReduce && a.allGather &&
           a.getErrorString;
    return a;
  }();
  return api;
}
#define CKV_NCCL_TRY(x)                                                                  \
  do {                                                                                   \
    ncclResult_t r_ = (x);                                                               \
    if (r_ != ncclSuccess) {                                                             \
      ckvb::set_error(std::string("nccl: ") + nccl().getErrorString(r_) + " (" #x ")");  \
      return CKV_ENCCL;                                                                  \
    }                                                                                    \
  } while (0)
}  // namespace

// ---------------------------------------------------------------------------
// LOCAL backend: ranks are threads sharing a group
// ---------------------------------------------------------------------------
struct ckv_local_group {
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<std::vector<unsigned char>> slot;  // per rank staging
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct ckv_comm {
  ckv_ctx* ctx = nullptr;
  int world = 1, rank = 0;
  ncclComm_t nc = nullptr;           // NCCL backend
  ckv_local_group* local = nullptr;  // LOCAL backend
};

namespace {
size_t dtype_bytes(int dt) { return dt == CKV_DT_F64 ? 8 : 4; }

template <typename T>
void host_reduce(T* acc, const T* x, size_t n, int op) {
  if (op == CKV_OP_MAX)
    for (size_t i = 0; i < n; ++i) acc[i] = std::max(acc[i], x[i]);
  else
    for (size_t i = 0; i < n; ++i) acc[i] += x[i];
}
}  // namespace

using ckvb::D;

extern "C" {

int ckv_comm_nccl_id(unsigned char* id_out) {
  if (!nccl().ok) { ckvb::set_error("ckv_comm: libnccl.so.2 not available"); return CKV_ENCCL; }
  ncclUniqueId id;
  CKV_NCCL_TRY(nccl().getUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return CKV_OK;
}

int ckv_comm_create_nccl(ckv_ctx* ctx, int world, int rank, const unsigned char* id,
                         ckv_comm** out) {
  if (!ctx || !out || world < 1 || rank < 0 || rank >= world) {
    ckvb::set_error("ckv_comm_create_nccl: bad arguments");
    return CKV_EINVAL;
  }
  if (!nccl().ok) { ckvb::set_error("ckv_comm: libnccl.so.2 not available"); return CKV_ENCCL; }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  auto* c = new ckv_comm;
  c->ctx = ctx;
  c->world = world;
  c->rank = rank;
  CKV_CUDA_TRY(cudaSetDevice(ctx->device));
  const ncclResult_t r = nccl().commInitRank(&c->nc, world, uid, rank);
  if (r != ncclSuccess) {
    ckvb::set_error(std::string("nccl: ") + nccl().getErrorString(r) + " (ncclCommInitRank)");
    delete c;
    return CKV_ENCCL;
  }
  *out = c;
  return CKV_OK;
}

int ckv_local_group_create(int world, ckv_local_group** out) {
  if (world < 1 || !out) { ckvb::set_error("ckv_local_group_create: world >= 1"); return CKV_EINVAL; }
  auto* g = new ckv_local_group;
  g->world = world;
  g->slot.resize(world);
  *out = g;
  return CKV_OK;
}

int ckv_local_group_destroy(ckv_local_group* g) {
  delete g;
  return CKV_OK;
}

int ckv_comm_create_local(ckv_ctx* ctx, ckv_local_group* g, int rank, ckv_comm** out) {
  if (!ctx || !g || !out || rank < 0 || rank >= g->world) {
    ckvb::set_error("ckv_comm_create_local: bad arguments");
    return CKV_EINVAL;
  }
  auto* c = new ckv_comm;
  c->ctx = ctx;
  c->world = g->world;
  c->rank = rank;
  c->local = g;
  *out = c;
  return CKV_OK;
}

int ckv_comm_destroy(ckv_comm* c) {
  if (!c) return CKV_OK;
  if (c->nc) nccl().commDestroy(c->nc);
  delete c;
  return CKV_OK;
}

int ckv_comm_world(const ckv_comm* c, int* world, int* rank) {
  *world = c->world;
  *rank = c->rank;
  return CKV_OK;
}

// in place on a device buffer, ordered on the context's stream
int ckv_comm_allreduce(ckv_comm* c, void* dev, size_t count, int dtype, int op) {
  if (c->world == 1 || count == 0) return CKV_OK;
  if ((dtype != CKV_DT_I32 && dtype != CKV_DT_F64) || (op != CKV_OP_SUM && op != CKV_OP_MAX)) {
    ckvb::set_error("ckv_comm_allreduce: dtype CKV_DT_I32 / CKV_DT_F64, op SUM / MAX");
    return CKV_EINVAL;
  }
  cudaStream_t st = c->ctx->stream;
  if (c->nc) {
    CKV_NCCL_TRY(nccl().allReduce(dev, dev, count, dtype == CKV_DT_F64 ? ncclFloat64 : ncclInt32,
                                  op == CKV_OP_MAX ? ncclMax : ncclSum, c->nc, st));
    return CKV_OK;
  }
  ckv_local_group* g = c->local;
  const size_t bytes = count * dtype_bytes(dtype);
  std::vector<unsigned char>& mine = g->slot[c->rank];
  mine.resize(bytes);
  CKV_CUDA_TRY(cudaMemcpyAsync(mine.data(), dev, bytes, cudaMemcpyDeviceToHost, st));
  CKV_CUDA_TRY(cudaStreamSynchronize(st));
  g->barrier();
  // every rank reduces all slots in rank order (identical results)
  std::vector<unsigned char> acc(g->slot[0]);
  for (int r = 1; r < c->world; ++r) {
    if (dtype == CKV_DT_F64)
      host_reduce(reinterpret_cast<double*>(acc.data()),
                  reinterpret_cast<const double*>(g->slot[r].data()), count, op);
    else
      host_reduce(reinterpret_cast<int32_t*>(acc.data()),
                  reinterpret_cast<const int32_t*>(g->slot[r].data()), count, op);
  }
  g->barrier();  // every rank has read every slot before any is reused
  CKV_CUDA_TRY(cudaMemcpyAsync(dev, acc.data(), bytes, cudaMemcpyHostToDevice, st));
  CKV_CUDA_TRY(cudaStreamSynchronize(st));
  return CKV_OK;
}

// recv = [world][bytes] of every rank's send, device buffers
int ckv_comm_allgather(ckv_comm* c, const void* send, void* recv, size_t bytes) {
  cudaStream_t st = c->ctx->stream;
  if (c->world == 1) {
    if (recv != send) CKV_CUDA_TRY(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st));
    return CKV_OK;
  }
  if (c->nc) {
    CKV_NCCL_TRY(nccl().allGather(send, recv, bytes, ncclUint8, c->nc, st));
    return CKV_OK;
  }
  ckv_local_group* g = c->local;
  std::vector<unsigned char>& mine = g->slot[c->rank];
  mine.resize(bytes);
  CKV_CUDA_TRY(cudaMemcpyAsync(mine.data(), send, bytes, cudaMemcpyDeviceToHost, st));
  CKV_CUDA_TRY(cudaStreamSynchronize(st));
  g->barrier();
  std::vector<unsigned char> all(bytes * c->world);
  for (int r = 0; r < c->world; ++r) std::memcpy(all.data() + r * bytes, g->slot[r].data(), bytes);
  g->barrier();
  CKV_CUDA_TRY(cudaMemcpyAsync(recv, all.data(), all.size(), cudaMemcpyHostToDevice, st));
  CKV_CUDA_TRY(cudaStreamSynchronize(st));
  return CKV_OK;
}

// ---------------------------------------------------------------------------
// the sharded kmeans_cosine (clustering.hpp:160-263; sharded.py mirrors it)
// ---------------------------------------------------------------------------
int ckv_kmeans_sharded(ckv_comm* comm, const ckv_kmshard_desc* d, const uint16_t* keys,
                       uint64_t n_total, uint64_t row_lo, const uint64_t* seeds_host,
                       const uint32_t* init_rows_host, uint32_t max_iters, float* centroids,
                       int32_t* labels, ckv_kmeans_info* info_host) {
  if (!comm || !d || !keys || !centroids || !labels) {
    ckvb::set_error("ckv_kmeans_sharded: NULL argument");
    return CKV_EINVAL;
  }
  const uint32_t U = d->n_units, C = d->C;
  if (C < 1 || uint64_t(C) > n_total || n_total > 0xffffffffull) {
    ckvb::set_error("kmeans: need 1 <= C <= N");
    return CKV_EINVAL;
  }
  if (max_iters < 1) { ckvb::set_error("ClusterConfig: max_iters must be >= 1"); return CKV_EINVAL; }
  if (!seeds_host && !init_rows_host) {
    ckvb::set_error("ckv_kmeans_sharded: seeds or init_rows required");
    return CKV_EINVAL;
  }
  ckv_ctx* ctx = comm->ctx;
  cudaStream_t st = ctx->stream;
  const int world = comm->world;
  // collective buffers: device, owned here for the call
  double *sums = nullptr, *objective = nullptr, *far_x = nullptr, *far_all = nullptr;
  int32_t *counts = nullptr, *stat = nullptr;
  ckv_kmshard* sh = nullptr;
  int rc = CKV_OK;
  auto cleanup = [&]() {
    if (sh) ckv_kmshard_destroy(sh);
    for (void* p : {static_cast<void*>(sums), static_cast<void*>(objective), static_cast<void*>(far_x),
                    static_cast<void*>(counts), static_cast<void*>(stat)})
      if (p) cudaFree(p);
  };
#define KS_TRY(x)               \
  do {                          \
    rc = (x);                   \
    if (rc) { cleanup(); return rc; } \
  } while (0)
#define KS_CUDA(x)                                                         \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      ckvb::set_error(std::string("ckv_kmeans_sharded: ") + cudaGetErrorString(e_)); \
      cleanup();                                                           \
      return CKV_ECUDA;                                                    \
    }                                                                      \
  } while (0)
  KS_CUDA(cudaMalloc(&sums, sizeof(double) * size_t(U) * C * D));
  KS_CUDA(cudaMalloc(&counts, sizeof(int32_t) * size_t(U) * C));
  KS_CUDA(cudaMalloc(&stat, sizeof(int32_t) * size_t(U) * 4));
  KS_CUDA(cudaMalloc(&objective, sizeof(double) * U));
  KS_CUDA(cudaMalloc(&far_x, sizeof(double) * 2 * (1 + size_t(world))));  // mine, then [world][2]
  far_all = far_x + 2;
  KS_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * size_t(U) * C * D, st));
  KS_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * size_t(U) * C, st));
  KS_CUDA(cudaMemsetAsync(stat, 0, sizeof(int32_t) * size_t(U) * 4, st));
  KS_CUDA(cudaMemsetAsync(objective, 0, sizeof(double) * U, st));
  ckv_kmshard_bufs bufs{sums, counts, stat, objective};
  KS_TRY(ckv_kmshard_create(ctx, d, keys, &bufs, &sh));

  // kmeans_cosine's input checks (clustering.hpp:166-172) over all shards
  std::vector<int32_t> hstat(size_t(U) * 4);
  KS_TRY(ckv_kmshard_validate(sh));
  KS_TRY(ckv_comm_allreduce(comm, stat, size_t(U) * 4, CKV_DT_I32, CKV_OP_MAX));
  KS_CUDA(cudaMemcpyAsync(hstat.data(), stat, 4 * hstat.size(), cudaMemcpyDeviceToHost, st));
  KS_CUDA(cudaStreamSynchronize(st));
  for (uint32_t u = 0; u < U; ++u)
    if (hstat[size_t(u) * 4 + 1]) { ckvb::set_error("kmeans: keys must be finite"); cleanup(); return CKV_EINVAL; }
  for (uint32_t u = 0; u < U; ++u)
    if (!hstat[size_t(u) * 4 + 2]) {
      ckvb::set_error("kmeans: degenerate input, all keys zero-norm");
      cleanup();
      return CKV_EINVAL;
    }
  std::vector<uint32_t> rows(size_t(U) * C);
  if (init_rows_host) std::memcpy(rows.data(), init_rows_host, 4 * rows.size());
  else ckvb::host_init_rows_batch(U, uint32_t(n_total), C, seeds_host, rows.data());
  KS_TRY(ckv_kmshard_init(sh, rows.data(), row_lo));
  KS_TRY(ckv_comm_allreduce(comm, sums, size_t(U) * C * D, CKV_DT_F64, CKV_OP_SUM));
  KS_TRY(ckv_kmshard_update(sh, 1));

  std::vector<int32_t> active(U, 1), converged(U, 0), any_empty(U, 0), hcounts(C);
  std::vector<uint32_t> iters(U, 0), n_rep(U, 0);
  const uint32_t n_local = d->n_local;
  // repair_empty_clusters (clustering.hpp:128-153) over the global counts:
  // every rank takes the same decisions; the victim is the farthest member
  // of the largest cluster, lowest global row on ties (one all-gather each)
  auto repair = [&]() -> int {
    CKV_TRY(ckv_kmshard_empty(sh, any_empty.data()));
    for (uint32_t u = 0; u < U; ++u) {
      if (!any_empty[u] || !active[u]) continue;
      CKV_CUDA_TRY(cudaMemcpyAsync(hcounts.data(), counts + size_t(u) * C, 4 * size_t(C),
                                   cudaMemcpyDeviceToHost, st));
      CKV_CUDA_TRY(cudaStreamSynchronize(st));
      bool repaired = false;
      for (uint32_t c = 0; c < C; ++c) {
        if (hcounts[c] > 0) continue;
        const uint32_t largest =
            uint32_t(std::max_element(hcounts.begin(), hcounts.end()) - hcounts.begin());
        if (hcounts[largest] <= 1) continue;
        double dist = 0.0;
        int64_t r = -1;
        CKV_TRY(ckv_kmshard_farthest(sh, u, largest, &dist, &r));
        const double mine[2] = {dist, r >= 0 ? double(row_lo + uint64_t(r)) : -1.0};
        CKV_CUDA_TRY(cudaMemcpyAsync(far_x, mine, 16, cudaMemcpyHostToDevice, st));
        CKV_TRY(ckv_comm_allgather(comm, far_x, far_all, 16));
        std::vector<double> all(2 * size_t(world));
        CKV_CUDA_TRY(cudaMemcpyAsync(all.data(), far_all, 16 * size_t(world), cudaMemcpyDeviceToHost, st));
        CKV_CUDA_TRY(cudaStreamSynchronize(st));
        double best = -1.0;
        int64_t victim = -1;
        for (int k = 0; k < world; ++k) {
          const double dd = all[2 * k];
          const int64_t gg = int64_t(all[2 * k + 1]);
          if (gg >= 0 && (dd > best || (dd == best && gg < victim))) { best = dd; victim = gg; }
        }
        if (victim < 0) victim = 0;  // no member beat distance -1: the reference keeps 0
        if (uint64_t(victim) >= row_lo && uint64_t(victim) < row_lo + n_local)
          CKV_TRY(ckv_kmshard_move(sh, u, uint32_t(uint64_t(victim) - row_lo), c));
        hcounts[largest]--;
        hcounts[c]++;
        repaired = true;
      }
      if (repaired) {
        ++n_rep[u];
        CKV_CUDA_TRY(cudaMemcpyAsync(counts + size_t(u) * C, hcounts.data(), 4 * size_t(C),
                                     cudaMemcpyHostToDevice, st));
        CKV_CUDA_TRY(cudaStreamSynchronize(st));
      }
    }
    return CKV_OK;
  };
  auto assign_pass = [&](uint32_t t) -> int {
    CKV_TRY(ckv_kmshard_assign(sh, t));
    CKV_TRY(ckv_comm_allreduce(comm, counts, size_t(U) * C, CKV_DT_I32, CKV_OP_SUM));
    CKV_TRY(repair());
    CKV_TRY(ckv_kmshard_finish(sh, t, 0));
    if (t > 0) CKV_TRY(ckv_comm_allreduce(comm, stat, size_t(U) * 4, CKV_DT_I32, CKV_OP_MAX));
    return CKV_OK;
  };
  KS_TRY(assign_pass(0));
  for (uint32_t t = 1; t <= max_iters; ++t) {
    KS_TRY(ckv_kmshard_partial_sums(sh));
    KS_TRY(ckv_comm_allreduce(comm, sums, size_t(U) * C * D, CKV_DT_F64, CKV_OP_SUM));
    KS_TRY(ckv_kmshard_update(sh, 0));
    KS_TRY(assign_pass(t));
    KS_CUDA(cudaMemcpyAsync(hstat.data(), stat, 4 * hstat.size(), cudaMemcpyDeviceToHost, st));
    KS_CUDA(cudaStreamSynchronize(st));
    bool any = false;
    for (uint32_t u = 0; u < U; ++u) {
      if (!active[u]) continue;
      if (!hstat[size_t(u) * 4]) { converged[u] = 1; iters[u] = t; active[u] = 0; }
      else if (t == max_iters) { iters[u] = t; active[u] = 0; }
      any |= active[u] != 0;
    }
    if (!any) break;
    KS_TRY(ckv_kmshard_set_active(sh, active.data()));
  }
  KS_TRY(ckv_kmshard_result(sh, iters.data(), centroids, labels));
  KS_CUDA(cudaStreamSynchronize(st));
  if (info_host)
    for (uint32_t u = 0; u < U; ++u) info_host[u] = {iters[u], converged[u], n_rep[u], 0u};
  cleanup();
  return CKV_OK;
#undef KS_TRY
#undef KS_CUDA
}

}  // extern "C"

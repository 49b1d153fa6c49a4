// ckv_kmshard.cu — per-shard steps of the sequence-sharded cosine k-means
// (protocol in include/ckv_cuda.h).
//
// One very long head's N keys are split into contiguous position shards, one
// per rank.  The assignment of a shard's keys needs only the (replicated)
// centroids, so it runs the single-GPU kernels unchanged (tensor-core filter
// + exact f64 fix-up, ckv_assign_tc.cu, or the exact CUDA-core pass).  What
// changes is the update: each shard sums its members in f64 and the caller
// all-reduces the sums and counts.  A sum of bf16 values in f64 is exact in
// any order, so the reduced sums equal the reference's
// position-ordered accumulation (clustering.hpp:207-216) bit for bit, and the
// centroids computed from them by finish_centroid (shared with k_update) are
// the reference's.  Empty-cluster repair (clustering.hpp:128-153) is driven
// by the caller through farthest() / move(), one all-gather per repair.
#include <cstdio>
#include <vector>

#include "ckv_internal.cuh"
#include "ckv_kmeans_dev.cuh"

struct ckv_kmshard {
  ckv_ctx* ctx = nullptr;
  ckv_kmshard_desc d{};
  const uint16_t* keys = nullptr;
  ckv_kmshard_bufs b{};
  uint32_t c_pad = 0;
  bool use_tc = false;
  uint32_t cur = 0;  // labels buffer of the latest assignment
  // device state
  float* cents = nullptr;     // [U][C][128]
  int32_t* lab[2] = {nullptr, nullptr};  // [U][n_local]
  uint32_t* lsizes = nullptr;  // local index [U][C], [U][C+1], [U][n_local]
  uint32_t* lstarts = nullptr;
  uint32_t* lsorted = nullptr;
  float* dirs = nullptr;       // [U][c_pad][128]
  uint16_t* dirs16 = nullptr;
  double* cnorm = nullptr;     // [U][c_pad]
  float* deps = nullptr;
  int32_t* active = nullptr;   // [U]
  int32_t* changed = nullptr;  // [U]
  int32_t* vflags = nullptr;   // [U] validation bits
  uint32_t* init_rows = nullptr;  // [U][C]
  double* far_d = nullptr;     // farthest(): distance, row
  int64_t* far_r = nullptr;
  void* tc = nullptr;
  size_t tc_bytes = 0;
  std::vector<void*> owned;
};

namespace ckvb {
namespace {

// sums[u][c] = key row r - row_lo if this shard owns r, else 0
__global__ void k_shard_init(const uint16_t* __restrict__ keys, uint64_t key_stride,
                             uint32_t n_local, uint64_t row_lo, const uint32_t* __restrict__ rows,
                             uint32_t C, double* __restrict__ sums) {
  const uint32_t u = blockIdx.y, c = blockIdx.x;
  const uint64_t r = rows[size_t(u) * C + c];
  const bool own = r >= row_lo && r < row_lo + n_local;
  double* dst = sums + (size_t(u) * C + c) * D;
  for (int j = threadIdx.x; j < D; j += blockDim.x)
    dst[j] = own ? double(bf16_to_f32(keys[u * key_stride + (r - row_lo) * D + j])) : 0.0;
}

// f64 member sums per (unit, cluster), one warp, lane = 4 dims; any order
// is exact (N3), the member order is kept anyway
__global__ void __launch_bounds__(256)
k_shard_sums(const uint16_t* __restrict__ keys, uint64_t key_stride, uint32_t C,
             uint32_t n_local, const uint32_t* __restrict__ sizes,
             const uint32_t* __restrict__ starts, const uint32_t* __restrict__ sorted,
             double* __restrict__ sums, const int32_t* __restrict__ active) {
  const uint32_t u = blockIdx.y;
  if (!active[u]) return;
  const uint32_t c = blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (c >= C) return;
  const int lane = lane_id();
  const uint32_t cnt = sizes[size_t(u) * C + c];
  const uint32_t* ids = sorted + size_t(u) * n_local + starts[size_t(u) * (C + 1) + c];
  const uint2* kb = reinterpret_cast<const uint2*>(keys + u * key_stride) + lane;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (uint32_t m0 = 0; m0 < cnt; m0 += 32) {
    const uint32_t nb = min(32u, cnt - m0);
    const uint32_t myid = uint32_t(lane) < nb ? __ldg(ids + m0 + lane) : 0u;
    for (uint32_t k0 = 0; k0 < nb; k0 += 8) {
      uint2 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t id = __shfl_sync(0xffffffffu, myid, (k0 + k) & 31);
        v[k] = k0 + k < nb ? __ldg(kb + size_t(id) * (D / 4)) : make_uint2(0, 0);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        a0 += double(__uint_as_float(v[k].x << 16));
        a1 += double(__uint_as_float(v[k].x & 0xffff0000u));
        a2 += double(__uint_as_float(v[k].y << 16));
        a3 += double(__uint_as_float(v[k].y & 0xffff0000u));
      }
    }
  }
  reinterpret_cast<double4*>(sums + (size_t(u) * C + c) * D)[lane] = make_double4(a0, a1, a2, a3);
}

// centroid + next directions from the all-reduced sums and counts
__global__ void __launch_bounds__(256)
k_shard_finalize(const double* __restrict__ sums, const int32_t* __restrict__ counts, uint32_t C,
                 uint32_t c_pad, float* __restrict__ cents, float* __restrict__ dirs,
                 uint16_t* __restrict__ dirs16, double* __restrict__ cnorm,
                 float* __restrict__ deps, const int32_t* __restrict__ active) {
  const uint32_t u = blockIdx.y;
  if (!active[u]) return;
  const uint32_t c = blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (c >= c_pad) return;
  const int lane = lane_id();
  float* dr = dirs + (size_t(u) * c_pad + c) * D;
  uint16_t* db = dirs16 + (size_t(u) * c_pad + c) * D;
  if (c >= C) {  // padding columns of the MMA operand
    for (int j = lane; j < D; j += 32) { dr[j] = 0.f; db[j] = 0; }
    if (lane == 0) deps[size_t(u) * c_pad + c] = 0.f;
    return;
  }
  const double4 s = reinterpret_cast<const double4*>(sums + (size_t(u) * C + c) * D)[lane];
  const double cnt = counts ? double(uint32_t(counts[size_t(u) * C + c])) : 1.0;
  finish_centroid(s.x, s.y, s.z, s.w, cnt, cents + (size_t(u) * C + c) * D, dr, db,
                  cnorm + size_t(u) * c_pad + c, deps + size_t(u) * c_pad + c);
}

__global__ void k_shard_empty(const int32_t* __restrict__ counts, uint32_t C,
                              const int32_t* __restrict__ active, int32_t* __restrict__ out) {
  const uint32_t u = blockIdx.x;
  int e = 0;
  if (active[u])
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) e |= counts[size_t(u) * C + c] == 0;
  e = __syncthreads_or(e);
  if (threadIdx.x == 0) out[u] = e;
}

// farthest local member of `cluster` (first maximum, distance > -1 only, as
// repair_empty_clusters' `dist > worst` scan with worst = -1)
__global__ void __launch_bounds__(256)
k_shard_farthest(const uint16_t* __restrict__ keys, uint64_t key_stride, uint32_t n_local,
                 const int32_t* __restrict__ labels, uint32_t u, uint32_t cluster, uint32_t C,
                 uint32_t c_pad, const float* __restrict__ cents, const double* __restrict__ cnorm,
                 double* __restrict__ out_d, int64_t* __restrict__ out_r) {
  __shared__ double s_d[8];
  __shared__ uint32_t s_i[8];
  const int32_t* lab = labels + size_t(u) * n_local;
  const uint16_t* kb = keys + u * key_stride;
  const float* cl = cents + (size_t(u) * C + cluster) * D;
  const double nb = cnorm[size_t(u) * c_pad + cluster];
  double bd = -1.0;
  uint32_t bv = 0xffffffffu;
  for (uint32_t i = threadIdx.x; i < n_local; i += blockDim.x) {
    if (uint32_t(lab[i]) != cluster) continue;
    const double dd = cosine_distance_dev(kb + size_t(i) * D, cl, nb);
    if (dd > bd) { bd = dd; bv = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
    const uint32_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
    if (od > bd || (od == bd && ov < bv)) { bd = od; bv = ov; }
  }
  if (lane_id() == 0) { s_d[warp_id()] = bd; s_i[warp_id()] = bv; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = s_d[0];
    uint32_t v = s_i[0];
    for (int w = 1; w < int(blockDim.x >> 5); ++w)
      if (s_d[w] > b || (s_d[w] == b && s_i[w] < v)) { b = s_d[w]; v = s_i[w]; }
    *out_d = b;
    *out_r = v == 0xffffffffu ? int64_t(-1) : int64_t(v);
  }
}

// local member counts -> the collective buffer (0 for frozen units, so their
// rows stay bounded through the all-reduces)
__global__ void k_shard_counts(const uint32_t* __restrict__ lsizes, uint32_t C,
                               const int32_t* __restrict__ active, int32_t* __restrict__ counts) {
  const uint32_t u = blockIdx.y;
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) counts[size_t(u) * C + c] = active[u] ? int32_t(lsizes[size_t(u) * C + c]) : 0;
}

__global__ void k_shard_stat_changed(const int32_t* __restrict__ changed, uint32_t U,
                                     int32_t* __restrict__ stat, const int32_t* __restrict__ active) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < U) stat[size_t(u) * 4] = active[u] ? changed[u] : 0;
}

__global__ void k_shard_stat_valid(const int32_t* __restrict__ vflags, uint32_t U,
                                   int32_t* __restrict__ stat) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < U) {
    stat[size_t(u) * 4 + 1] = vflags[u] & 1;
    stat[size_t(u) * 4 + 2] = (vflags[u] >> 1) & 1;
  }
}

int salloc(ckv_kmshard* s, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    *p = nullptr;
    return cuda_status(e, "kmshard: cudaMalloc");
  }
  s->owned.push_back(*p);
  return CKV_OK;
}
template <typename T>
int salloc(ckv_kmshard* s, T** p, size_t n) {
  return salloc(s, reinterpret_cast<void**>(p), n * sizeof(T));
}

}  // namespace
}  // namespace ckvb

using namespace ckvb;

extern "C" {

int ckv_kmshard_destroy(ckv_kmshard* s) {
  if (!s) return CKV_OK;
  if (s->ctx) cudaStreamSynchronize(s->ctx->stream);
  for (void* p : s->owned) cudaFree(p);
  delete s;
  return CKV_OK;
}

int ckv_kmshard_create(ckv_ctx* ctx, const ckv_kmshard_desc* d, const uint16_t* keys,
                       const ckv_kmshard_bufs* bufs, ckv_kmshard** out) {
  if (!ctx || !d || !keys || !bufs || !out) {
    set_error("ckv_kmshard_create: NULL argument");
    return CKV_EINVAL;
  }
  if (d->n_units == 0 || d->n_local == 0 || d->C == 0) {
    set_error("ckv_kmshard_create: need n_units, n_local, C >= 1");
    return CKV_EINVAL;
  }
  if (d->key_stride < uint64_t(d->n_local) * D || d->key_stride % D) {
    set_error("ckv_kmshard_create: key_stride must be whole rows >= n_local");
    return CKV_EINVAL;
  }
  if (!bufs->sums || !bufs->counts || !bufs->stat || !bufs->objective) {
    set_error("ckv_kmshard_create: every collective buffer is required");
    return CKV_EINVAL;
  }
  auto* s = new ckv_kmshard();
  s->ctx = ctx;
  s->d = *d;
  s->keys = keys;
  s->b = *bufs;
  const uint32_t U = d->n_units, C = d->C, n = d->n_local;
  s->c_pad = (C + 31) / 32 * 32;
  s->use_tc = !(d->flags & CKV_KM_EXACT_ONLY) && assign_tc_supported(n, C);
  int rc = CKV_OK;
  auto A = [&](int r) { if (rc == CKV_OK) rc = r; };
  A(salloc(s, &s->cents, size_t(U) * C * D));
  A(salloc(s, &s->lab[0], size_t(U) * n));
  A(salloc(s, &s->lab[1], size_t(U) * n));
  A(salloc(s, &s->lsizes, size_t(U) * C));
  A(salloc(s, &s->lstarts, size_t(U) * (C + 1)));
  A(salloc(s, &s->lsorted, size_t(U) * n));
  A(salloc(s, &s->dirs, size_t(U) * s->c_pad * D));
  A(salloc(s, &s->dirs16, size_t(U) * s->c_pad * D));
  A(salloc(s, &s->cnorm, size_t(U) * s->c_pad));
  A(salloc(s, &s->deps, size_t(U) * s->c_pad));
  A(salloc(s, &s->active, U));
  A(salloc(s, &s->changed, U));
  A(salloc(s, &s->vflags, U));
  A(salloc(s, &s->init_rows, size_t(U) * C));
  A(salloc(s, &s->far_d, 1));
  A(salloc(s, &s->far_r, 1));
  if (s->use_tc) {
    s->tc_bytes = assign_tc_scratch_bytes(U, n, C);
    A(salloc(s, &s->tc, s->tc_bytes));
  }
  if (rc != CKV_OK) { ckv_kmshard_destroy(s); return rc; }
  std::vector<int32_t> ones(U, 1);
  rc = cudaMemcpy(s->active, ones.data(), 4 * U, cudaMemcpyHostToDevice) == cudaSuccess
           ? CKV_OK : CKV_ECUDA;
  if (rc != CKV_OK) { set_error("kmshard: init copy failed"); ckv_kmshard_destroy(s); return rc; }
  // key norms for the tensor-core band (keys never change)
  if (s->use_tc) {
    const TcKeyPrep prep = assign_tc_keyprep(s->tc, U, n);
    rc = launch_scan_keys(ctx->stream, keys, d->key_stride, n, U, nullptr, &prep);
    if (rc != CKV_OK) { ckv_kmshard_destroy(s); return rc; }
    ctx->launches++;
  }
  *out = s;
  return CKV_OK;
}

int ckv_kmshard_validate(ckv_kmshard* s) {
  cudaStream_t st = s->ctx->stream;
  const uint32_t U = s->d.n_units;
  CKV_CUDA_TRY(cudaMemsetAsync(s->vflags, 0, 4 * U, st));
  CKV_TRY(launch_scan_keys(st, s->keys, s->d.key_stride, s->d.n_local, U, s->vflags, nullptr));
  k_shard_stat_valid<<<(U + 127) / 128, 128, 0, st>>>(s->vflags, U, s->b.stat);
  CKV_LAUNCH_CHECK("k_shard_stat_valid");
  s->ctx->launches += 3;
  return CKV_OK;
}

int ckv_kmshard_init(ckv_kmshard* s, const uint32_t* rows_host, uint64_t row_lo) {
  cudaStream_t st = s->ctx->stream;
  const uint32_t U = s->d.n_units, C = s->d.C;
  CKV_CUDA_TRY(cudaMemcpyAsync(s->init_rows, rows_host, 4 * size_t(U) * C,
                               cudaMemcpyHostToDevice, st));
  k_shard_init<<<dim3(C, U), 128, 0, st>>>(s->keys, s->d.key_stride, s->d.n_local, row_lo,
                                           s->init_rows, C, s->b.sums);
  CKV_LAUNCH_CHECK("k_shard_init");
  s->ctx->launches++;
  return cudaStreamSynchronize(st) == cudaSuccess ? CKV_OK : CKV_ECUDA;  // rows_host may go
}

int ckv_kmshard_set_active(ckv_kmshard* s, const int32_t* active_host) {
  CKV_CUDA_TRY(cudaMemcpyAsync(s->active, active_host, 4 * size_t(s->d.n_units),
                               cudaMemcpyHostToDevice, s->ctx->stream));
  return cudaStreamSynchronize(s->ctx->stream) == cudaSuccess ? CKV_OK : CKV_ECUDA;
}

int ckv_kmshard_update(ckv_kmshard* s, int from_init) {
  cudaStream_t st = s->ctx->stream;
  const uint32_t U = s->d.n_units, C = s->d.C;
  k_shard_finalize<<<dim3((s->c_pad + 7) / 8, U), 256, 0, st>>>(
      s->b.sums, from_init ? nullptr : s->b.counts, C, s->c_pad, s->cents, s->dirs, s->dirs16,
      s->cnorm, s->deps, s->active);
  CKV_LAUNCH_CHECK("k_shard_finalize");
  s->ctx->launches++;
  return CKV_OK;
}

int ckv_kmshard_assign(ckv_kmshard* s, uint32_t pass) {
  cudaStream_t st = s->ctx->stream;
  const uint32_t U = s->d.n_units, C = s->d.C, n = s->d.n_local;
  s->cur = pass & 1;
  CKV_TRY(launch_assign(st, s->use_tc, s->keys, s->d.key_stride, n, C, s->c_pad, U, s->dirs16,
                        s->deps, s->dirs, s->lab[s->cur], n, s->active, s->tc, s->tc_bytes,
                        &s->ctx->launches));
  CKV_TRY(launch_index(st, U, s->lab[s->cur], n, n, C, nullptr, C, s->lsizes, s->lstarts,
                       s->lsorted, nullptr, nullptr, s->active, nullptr));
  k_shard_counts<<<dim3((C + 255) / 256, U), 256, 0, st>>>(s->lsizes, C, s->active, s->b.counts);
  CKV_LAUNCH_CHECK("k_shard_counts");
  s->ctx->launches += 2;
  return CKV_OK;
}

int ckv_kmshard_empty(ckv_kmshard* s, int32_t* any_empty_host) {
  cudaStream_t st = s->ctx->stream;
  const uint32_t U = s->d.n_units;
  k_shard_empty<<<U, 256, 0, st>>>(s->b.counts, s->d.C, s->active, s->changed);
  CKV_LAUNCH_CHECK("k_shard_empty");
  s->ctx->launches++;
  CKV_CUDA_TRY(cudaMemcpyAsync(any_empty_host, s->changed, 4 * size_t(U),
                               cudaMemcpyDeviceToHost, st));
  CKV_CUDA_TRY(cudaStreamSynchronize(st));
  return CKV_OK;
}

int ckv_kmshard_farthest(ckv_kmshard* s, uint32_t unit, uint32_t cluster, double* dist_host,
                         int64_t* row_host) {
  if (unit >= s->d.n_units || cluster >= s->d.C) {
    set_error("kmshard_farthest: unit / cluster out of range");
    return CKV_EINVAL;
  }
  cudaStream_t st = s->ctx->stream;
  k_shard_farthest<<<1, 256, 0, st>>>(s->keys, s->d.key_stride, s->d.n_local, s->lab[s->cur],
                                      unit, cluster, s->d.C, s->c_pad, s->cents, s->cnorm,
                                      s->far_d, s->far_r);
  CKV_LAUNCH_CHECK("k_shard_farthest");
  s->ctx->launches++;
  CKV_CUDA_TRY(cudaMemcpyAsync(dist_host, s->far_d, 8, cudaMemcpyDeviceToHost, st));
  CKV_CUDA_TRY(cudaMemcpyAsync(row_host, s->far_r, 8, cudaMemcpyDeviceToHost, st));
  CKV_CUDA_TRY(cudaStreamSynchronize(st));
  return CKV_OK;
}

int ckv_kmshard_move(ckv_kmshard* s, uint32_t unit, uint32_t row, uint32_t cluster) {
  if (unit >= s->d.n_units || row >= s->d.n_local || cluster >= s->d.C) {
    set_error("kmshard_move: unit / row / cluster out of range");
    return CKV_EINVAL;
  }
  const int32_t v = int32_t(cluster);
  CKV_CUDA_TRY(cudaMemcpyAsync(s->lab[s->cur] + size_t(unit) * s->d.n_local + row, &v, 4,
                               cudaMemcpyHostToDevice, s->ctx->stream));
  CKV_CUDA_TRY(cudaStreamSynchronize(s->ctx->stream));
  return CKV_OK;
}

int ckv_kmshard_finish(ckv_kmshard* s, uint32_t pass, int want_objective) {
  cudaStream_t st = s->ctx->stream;
  const uint32_t U = s->d.n_units, C = s->d.C, n = s->d.n_local;
  const int32_t* prev = pass > 0 ? s->lab[s->cur ^ 1] : nullptr;
  CKV_CUDA_TRY(cudaMemsetAsync(s->changed, 0, 4 * size_t(U), st));
  CKV_TRY(launch_index(st, U, s->lab[s->cur], n, n, C, nullptr, C, s->lsizes, s->lstarts,
                       s->lsorted, prev, s->changed, s->active, nullptr));
  k_shard_stat_changed<<<(U + 127) / 128, 128, 0, st>>>(s->changed, U, s->b.stat, s->active);
  CKV_LAUNCH_CHECK("k_shard_stat_changed");
  s->ctx->launches += 2;
  if (want_objective) {
    CKV_CUDA_TRY(cudaMemsetAsync(s->b.objective, 0, 8 * size_t(U), st));
    CKV_TRY(launch_objective(st, s->keys, s->d.key_stride, n, U, C, s->c_pad, s->lab[s->cur], n,
                             s->cents, s->cnorm, s->b.objective, s->active));
    s->ctx->launches++;
  }
  return CKV_OK;
}

int ckv_kmshard_partial_sums(ckv_kmshard* s) {
  cudaStream_t st = s->ctx->stream;
  const uint32_t U = s->d.n_units, C = s->d.C;
  k_shard_sums<<<dim3((C + 7) / 8, U), 256, 0, st>>>(s->keys, s->d.key_stride, C, s->d.n_local,
                                                     s->lsizes, s->lstarts, s->lsorted, s->b.sums,
                                                     s->active);
  CKV_LAUNCH_CHECK("k_shard_sums");
  s->ctx->launches++;
  return CKV_OK;
}

int ckv_kmshard_result(ckv_kmshard* s, const uint32_t* iters_host, float* centroids,
                       int32_t* labels) {
  cudaStream_t st = s->ctx->stream;
  const uint32_t U = s->d.n_units, C = s->d.C, n = s->d.n_local;
  if (centroids)
    CKV_CUDA_TRY(cudaMemcpyAsync(centroids, s->cents, 4 * size_t(U) * C * D,
                                 cudaMemcpyDeviceToDevice, st));
  if (labels)
    for (uint32_t u = 0; u < U; ++u)
      CKV_CUDA_TRY(cudaMemcpyAsync(labels + size_t(u) * n, s->lab[iters_host[u] & 1] + size_t(u) * n,
                                   4 * size_t(n), cudaMemcpyDeviceToDevice, st));
  return CKV_OK;
}

}  // extern "C"

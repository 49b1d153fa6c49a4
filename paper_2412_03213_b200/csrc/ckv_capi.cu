// ckv_capi.cu — the extern "C" boundary (include/ckv_cuda.h) and the
// device-resident decode session.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <deque>
#include <atomic>
#include <mutex>
#include <random>
#include <set>
#include <tuple>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "ckv_internal.cuh"

namespace ckvb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int cuda_status(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? CKV_ENOMEM : CKV_ECUDA;
}
// grow-only scratch slot of the context (slots 0-20: k-means, 24-26: attend);
// zero_new: zero the bytes when (re)allocated
int ctx_scratch(ckv_ctx* ctx, int slot, size_t bytes, bool zero_new, void** out) {
  if (bytes == 0) bytes = 16;
  if (ctx->scratch_cap[slot] < bytes) {
    if (ctx->scratch[slot]) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->scratch[slot]);
      ctx->scratch[slot] = nullptr;
      ctx->scratch_cap[slot] = 0;
    }
    cudaError_t e = cudaMalloc(&ctx->scratch[slot], bytes);
    if (e != cudaSuccess) {
      ctx->scratch[slot] = nullptr;
      return cuda_status(e, "context scratch allocation");
    }
    ctx->scratch_cap[slot] = bytes;
    if (zero_new) CKV_CUDA_TRY(cudaMemsetAsync(ctx->scratch[slot], 0, bytes, ctx->stream));
  }
  *out = ctx->scratch[slot];
  return CKV_OK;
}

// persistent split-K partials, merge tickets (zeroed once; k_attend re-arms
// them) and the parity-mode logits of ckv_attend / ckv_attend_partial
int attend_scratch(ckv_ctx* ctx, const ckv_attend_desc& d, bool weights, float** part,
                   uint32_t** tickets, float** lw) {
  void *p = nullptr, *t = nullptr, *w = nullptr;
  CKV_TRY(ctx_scratch(ctx, 24, attend_part_floats(d.n_q, d.max_tokens) * 4 + 16, false, &p));
  CKV_TRY(ctx_scratch(ctx, 25, size_t(d.n_q) * 4 + 4, true, &t));
  if (weights) CKV_TRY(ctx_scratch(ctx, 26, size_t(d.n_q) * d.sel_cap * 4 + 16, false, &w));
  *part = static_cast<float*>(p);
  *tickets = static_cast<uint32_t*>(t);
  *lw = static_cast<float*>(w);
  return CKV_OK;
}

int num_sms() {  // per device, queried once (called several times per launch)
  static std::atomic<int> sms[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int n = sms[dev & 63].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    sms[dev & 63].store(n, std::memory_order_relaxed);
  }
  return n;
}

// common.hpp:100-113
static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
bool trace_on() {
  static const bool on = getenv("CKV_TRACE_HOST") != nullptr;
  return on;
}
static thread_local std::chrono::steady_clock::time_point g_trace_t0;
void trace_begin(const char* what) {
  if (!trace_on()) return;
  g_trace_t0 = std::chrono::steady_clock::now();
  fprintf(stderr, "[ckv trace] %s: begin\n", what);
}
void trace_mark(const char* what, long arg) {
  if (!trace_on()) return;
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                              g_trace_t0).count();
  if (arg >= 0) fprintf(stderr, "[ckv trace] %9.3f ms %s %ld\n", ms, what, arg);
  else fprintf(stderr, "[ckv trace] %9.3f ms %s\n", ms, what);
}

cudaError_t smem_optin(const void* fn, int bytes, bool max_carveout) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  const auto key = std::make_tuple(fn, dev, bytes);
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && max_carveout)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) done.insert(key);
  return e;
}

uint64_t host_mix_seed(uint64_t seed, uint64_t a, uint64_t b) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ (a + 0x9e3779b97f4a7c15ull));
  return splitmix64(h ^ (b + 0xbf58476d1ce4e5b9ull));
}
// clustering.hpp:186-193 (std::mt19937_64 is bit-specified by the standard;
// uniform_below is rng() % n, common.hpp:124-126)
void host_init_rows(uint32_t n, uint32_t C, uint64_t seed, uint32_t* rows) {
  // the reference's partial Fisher-Yates over pool = 0..n-1, with the pool
  // kept sparse (only the <= 2C touched slots, an open-addressing table), so
  // a unit costs O(C) not O(n)
  std::mt19937_64 rng(seed);
  uint32_t cap = 64;
  while (cap < 4 * C) cap <<= 1;
  std::vector<uint32_t> key(cap, 0xffffffffu), val(cap);
  auto slot = [&](uint32_t i) {
    uint32_t h = (i * 2654435761u) & (cap - 1);
    while (key[h] != 0xffffffffu && key[h] != i) h = (h + 1) & (cap - 1);
    return h;
  };
  auto get = [&](uint32_t i) {
    const uint32_t h = slot(i);
    return key[h] == i ? val[h] : i;
  };
  auto put = [&](uint32_t i, uint32_t v) {
    const uint32_t h = slot(i);
    key[h] = i;
    val[h] = v;
  };
  for (uint32_t c = 0; c < C; ++c) {
    const uint32_t j = c + uint32_t(rng() % uint64_t(n - c));
    const uint32_t pc = get(c), pj = get(j);
    put(c, pj);
    put(j, pc);
    rows[c] = pj;
  }
}

// host_init_rows for many units on host threads (units are independent)
void host_init_rows_batch(uint32_t n_units, uint32_t n, uint32_t C, const uint64_t* seeds,
                          uint32_t* rows) {
  const uint32_t hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const uint32_t nt = std::min(hw, std::max(1u, n_units / 8));
  auto work = [&](uint32_t t0) {
    for (uint32_t u = t0; u < n_units; u += nt) host_init_rows(n, C, seeds[u], rows + size_t(u) * C);
  };
  if (nt == 1) { work(0); return; }
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < nt; ++t) th.emplace_back(work, t);
  for (auto& x : th) x.join();
}

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__global__ void k_f32_to_bf16(const float* __restrict__ src, uint16_t* __restrict__ dst,
                              size_t n, int* __restrict__ inexact) {
  int bad = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    float x = src[i];
    uint16_t b = f32_to_bf16_rn(x);
    dst[i] = b;
    if (__float_as_uint(x) != (uint32_t(b) << 16) && !isnan(x)) bad = 1;
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(inexact, 1);
}

__global__ void k_fill_i32(int32_t* __restrict__ p, uint32_t n, uint32_t stride, int32_t v) {
  const uint32_t u = blockIdx.y;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[size_t(u) * stride + i] = v;
}

__global__ void k_set_u32(uint32_t* __restrict__ p, uint32_t n, uint32_t v) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// append decode-batch clusters: centroids / labels at each unit's n_clusters
__global__ void k_append_clusters(const float* __restrict__ tmp_c, const int32_t* __restrict__ tmp_l,
                                  uint32_t cplus, uint32_t rows, uint32_t pos0, uint32_t c_cap,
                                  uint32_t p_cap, float* __restrict__ cents,
                                  int32_t* __restrict__ labels, uint32_t* __restrict__ n_clusters) {
  const uint32_t u = blockIdx.x;
  const uint32_t base = n_clusters[u];
  for (uint32_t i = threadIdx.x; i < cplus * D; i += blockDim.x)
    cents[(size_t(u) * c_cap + base) * D + i] = tmp_c[size_t(u) * cplus * D + i];
  for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x)
    labels[size_t(u) * p_cap + pos0 + i] = tmp_l[size_t(u) * rows + i] + int32_t(base);
  __syncthreads();
  if (threadIdx.x == 0) n_clusters[u] = base + cplus;
}

// append one token's K/V row per unit at position pos
// (and advance the StepSync epoch: the step's selection / attention are done)
__global__ void k_append_kv(const uint16_t* __restrict__ kn, const uint16_t* __restrict__ vn,
                            uint16_t* __restrict__ K, uint16_t* __restrict__ V, uint32_t pos,
                            uint32_t p_cap, uint32_t* __restrict__ epoch,
                            uint32_t* __restrict__ work) {
  const uint32_t u = blockIdx.x, j = threadIdx.x;  // 16 threads x 16 B
  // the next step's selection (PDL) may start streaming its centroids now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (epoch && u == 0 && j == 0) ++*epoch;
  if (work && j == 0) work[u] = 0u;  // the attention work counters (per slice start unit)
  if (!kn) return;  // the fused selection appended the row
  const uint4* ks = reinterpret_cast<const uint4*>(kn + size_t(u) * D);
  const uint4* vs = reinterpret_cast<const uint4*>(vn + size_t(u) * D);
  reinterpret_cast<uint4*>(K + (size_t(u) * p_cap + pos) * D)[j] = ks[j];
  reinterpret_cast<uint4*>(V + (size_t(u) * p_cap + pos) * D)[j] = vs[j];
}

__global__ void k_epoch_advance(uint32_t* epoch, uint32_t* work, uint32_t n) {
  for (uint32_t u = threadIdx.x; u < n; u += blockDim.x) work[u] = 0u;
  if (threadIdx.x == 0) ++*epoch;
}

// cluster-major relayout of the prompt KV (after the prefill index):
// dst row r = src position  r              for r < sink or r >= labeled_end
//                           sorted[r-sink] for sink <= r < labeled_end
__global__ void k_relayout(const uint16_t* __restrict__ K, const uint16_t* __restrict__ V,
                           uint16_t* __restrict__ K2, uint16_t* __restrict__ V2,
                           const uint32_t* __restrict__ sorted, uint32_t p_cap, uint32_t sink,
                           uint32_t labeled_end, uint32_t n_ctx) {
  const uint32_t u = blockIdx.y;
  const uint32_t r = blockIdx.x * 8 + (threadIdx.x >> 4);  // 16 threads x 16 B per row
  const uint32_t j = threadIdx.x & 15;
  if (r >= n_ctx) return;
  uint32_t src = r;
  if (r >= sink && r < labeled_end) src = __ldg(sorted + size_t(u) * p_cap + (r - sink));
  const size_t base = size_t(u) * p_cap;
  reinterpret_cast<uint4*>(K2 + (base + r) * D)[j] =
      __ldg(reinterpret_cast<const uint4*>(K + (base + src) * D) + j);
  reinterpret_cast<uint4*>(V2 + (base + r) * D)[j] =
      __ldg(reinterpret_cast<const uint4*>(V + (base + src) * D) + j);
}

// relayout of one clustered decode batch: rows [le0, le0+m) get the batch's
// tokens in index order (sorted entries le0-sink .. le0-sink+m-1)
__global__ void k_relayout_batch(uint16_t* __restrict__ K, uint16_t* __restrict__ V,
                                 uint16_t* __restrict__ tK, uint16_t* __restrict__ tV,
                                 const uint32_t* __restrict__ sorted, uint32_t p_cap,
                                 uint32_t sink, uint32_t le0, uint32_t m) {
  const uint32_t u = blockIdx.x;
  const size_t base = size_t(u) * p_cap;
  uint4* tk = reinterpret_cast<uint4*>(tK + size_t(u) * m * D);
  uint4* tv = reinterpret_cast<uint4*>(tV + size_t(u) * m * D);
  for (uint32_t e = threadIdx.x; e < m * 16; e += blockDim.x) {
    tk[e] = reinterpret_cast<const uint4*>(K + (base + le0) * D)[e];
    tv[e] = reinterpret_cast<const uint4*>(V + (base + le0) * D)[e];
  }
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < m * 16; e += blockDim.x) {
    const uint32_t r = e >> 4, j = e & 15;
    const uint32_t src = sorted[base + (le0 - sink) + r] - le0;
    reinterpret_cast<uint4*>(K + (base + le0 + r) * D)[j] = tk[src * 16 + j];
    reinterpret_cast<uint4*>(V + (base + le0 + r) * D)[j] = tv[src * 16 + j];
  }
}

// ---- cluster_decode_batch's init rows on the device ----------------------
// clustering.hpp:186-193 with seed mix_seed(seed_u, 0xdecade, pos0)
// (clustering.hpp:318-320): a partial Fisher-Yates over 0..n-1 driven by
// std::mt19937_64 (bit-specified by the C++ standard; uniform_below = rng() %
// m, common.hpp:124-126).  Only the first C <= 32 outputs are drawn, and the
// first twist's output k needs just the seeded words k, k+1 and k+156, so a
// thread per unit computes them in one pass of the seeding recurrence; the
// pool is kept sparse (the <= 2C touched slots).
constexpr uint32_t DI_MAX_C = 32;

__device__ __forceinline__ uint64_t d_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void k_decode_init_rows(const uint64_t* __restrict__ seeds, uint32_t n_units,
                                   uint64_t pos0, uint32_t n, uint32_t C,
                                   uint32_t* __restrict__ rows) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  // mix_seed(seed, 0xdecade, pos0) (common.hpp:108-113)
  uint64_t h = d_splitmix64(seeds[u]);
  h = d_splitmix64(h ^ (0xdecadeull + 0x9e3779b97f4a7c15ull));
  const uint64_t seed = d_splitmix64(h ^ (pos0 + 0xbf58476d1ce4e5b9ull));
  uint64_t lo[DI_MAX_C + 1], hi[DI_MAX_C];
  uint64_t x = seed;
  lo[0] = x;
  for (uint32_t i = 1; i < 156 + C; ++i) {
    x = 6364136223846793005ull * (x ^ (x >> 62)) + i;
    if (i <= C) lo[i] = x;
    if (i >= 156) hi[i - 156] = x;
  }
  uint32_t key[2 * DI_MAX_C], val[2 * DI_MAX_C];
  uint32_t nk = 0;
  auto get = [&](uint32_t i) {
    for (uint32_t k = 0; k < nk; ++k) if (key[k] == i) return val[k];
    return i;
  };
  auto put = [&](uint32_t i, uint32_t v) {
    for (uint32_t k = 0; k < nk; ++k) if (key[k] == i) { val[k] = v; return; }
    key[nk] = i;
    val[nk] = v;
    ++nk;
  };
  for (uint32_t c = 0; c < C; ++c) {
    const uint64_t y = (lo[c] & 0xFFFFFFFF80000000ull) | (lo[c + 1] & 0x000000007FFFFFFFull);
    uint64_t z = hi[c] ^ (y >> 1);
    if (y & 1ull) z ^= 0xB5026F5AA96619E9ull;
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    const uint32_t j = c + uint32_t(z % uint64_t(n - c));
    const uint32_t pc = get(c), pj = get(j);
    put(c, pj);
    put(j, pc);
    rows[size_t(u) * C + c] = pj;
  }
}

// ---- commit of one clustered decode batch ---------------------------------
// The batch's clusters are fresh ids [base, base + C) and their members are
// exactly the batch rows [le0, le0 + m), so build_index over the whole
// context (selection.hpp:29-48) only APPENDS: sizes / starts of the new ids
// and their sorted entries (positions in order) after the existing
// le0 - sink ones.  The same pass re-lays the batch's K/V rows cluster-major
// (row le0 + i <- position sorted[le0 - sink + i]) through a staging copy, and
// publishes n_clusters (base + C) from ncl_src.  One CTA per unit.
constexpr int BC_THREADS = 512;
__global__ void __launch_bounds__(BC_THREADS)
k_batch_commit(uint16_t* __restrict__ K, uint16_t* __restrict__ V, uint16_t* __restrict__ tK,
               uint16_t* __restrict__ tV, const int32_t* __restrict__ labels, uint32_t p_cap,
               uint32_t c_cap, uint32_t sink, uint32_t le0, uint32_t m, uint32_t C,
               const uint32_t* __restrict__ ncl_src, uint32_t* __restrict__ n_clusters,
               uint32_t* __restrict__ sizes, uint32_t* __restrict__ starts,
               uint32_t* __restrict__ sorted) {
  const uint32_t u = blockIdx.x;
  const int tid = threadIdx.x, lane = lane_id(), wid = warp_id();
  __shared__ uint32_t wc[BC_THREADS / 32][DI_MAX_C];
  __shared__ uint32_t off[DI_MAX_C + 1];
  __shared__ uint16_t dest[BC_THREADS];
  const uint32_t base = ncl_src[u] - C;
  const size_t urow = size_t(u) * p_cap;
  const uint32_t first = le0 - sink;  // sorted entries before the batch's
  const uint4* Ksrc = reinterpret_cast<const uint4*>(K + (urow + le0) * D);
  const uint4* Vsrc = reinterpret_cast<const uint4*>(V + (urow + le0) * D);
  uint4* tk = reinterpret_cast<uint4*>(tK + size_t(u) * m * D);
  uint4* tv = reinterpret_cast<uint4*>(tV + size_t(u) * m * D);
  for (uint32_t e = tid; e < m * 16; e += BC_THREADS) {  // stage the batch rows
    tk[e] = Ksrc[e];
    tv[e] = Vsrc[e];
  }
  for (uint32_t r0 = 0; r0 < m; r0 += BC_THREADS) {
    const uint32_t r = r0 + tid;
    const int32_t k = r < m ? labels[urow + le0 + r] - int32_t(base) : -1;
    for (uint32_t c = 0; c < C; ++c) {
      const unsigned b = __ballot_sync(0xffffffffu, k == int32_t(c));
      if (lane == 0) wc[wid][c] = __popc(b);
    }
    __syncthreads();
    if (tid < int(C)) {  // exclusive over warps; totals
      uint32_t sum = 0;
      for (int w = 0; w < BC_THREADS / 32; ++w) { const uint32_t x = wc[w][tid]; wc[w][tid] = sum; sum += x; }
      off[tid] = sum;
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t b = 0;
      for (uint32_t c = 0; c < C; ++c) {
        const uint32_t x = off[c];
        if (r0 == 0) sizes[size_t(u) * c_cap + base + c] = x;
        else sizes[size_t(u) * c_cap + base + c] += x;
        off[c] = b;
        b += x;
      }
      off[C] = b;
    }
    __syncthreads();
    const unsigned same = __match_any_sync(0xffffffffu, k);
    if (k >= 0) {
      // members of cluster k before this chunk come first (rows ascending)
      const uint32_t prior = r0 ? sizes[size_t(u) * c_cap + base + k] - off[k + 1] + off[k] : 0;
      (void)prior;
    }
    __syncthreads();
    if (k >= 0 && m <= BC_THREADS) {
      const uint32_t slot = off[k] + wc[wid][k] + __popc(same & ((1u << lane) - 1u));
      sorted[urow + first + slot] = le0 + r;
      dest[r] = uint16_t(slot);
    }
    __syncthreads();
  }
  if (tid <= int(C)) starts[size_t(u) * (c_cap + 1) + base + tid] = first + off[tid];
  __syncthreads();
  uint4* Kd = reinterpret_cast<uint4*>(K + (urow + le0) * D);
  uint4* Vd = reinterpret_cast<uint4*>(V + (urow + le0) * D);
  for (uint32_t e = tid; e < m * 16; e += BC_THREADS) {
    const uint32_t r = e >> 4, j = e & 15;
    Kd[size_t(dest[r]) * 16 + j] = tk[e];
    Vd[size_t(dest[r]) * 16 + j] = tv[e];
  }
  if (tid == 0) n_clusters[u] = base + C;
}

}  // namespace ckvb

using namespace ckvb;

// ===========================================================================
// context + memory
// ===========================================================================
extern "C" {

const char* ckv_last_error(void) { return g_err.c_str(); }

int ckv_ctx_create(int device, void* stream, ckv_ctx** out) {
  if (!out) { set_error("ckv_ctx_create: out is NULL"); return CKV_EINVAL; }
  CKV_CUDA_TRY(cudaSetDevice(device));
  ckv_ctx* c = new ckv_ctx();
  for (int i = 0; i < ckv_ctx::kScratchSlots; ++i) { c->scratch[i] = nullptr; c->scratch_cap[i] = 0; }
  c->device = device;
  // NULL is the CUDA legacy default stream (torch's default stream too), so
  // work launched here is ordered with the caller's default-stream work.
  c->stream = static_cast<cudaStream_t>(stream);
  *out = c;
  return CKV_OK;
}

int ckv_ctx_destroy(ckv_ctx* ctx) {
  if (!ctx) return CKV_OK;
  cudaSetDevice(ctx->device);
  if (ctx->aux) ckv_ctx_destroy(ctx->aux);
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
  for (int i = 0; i < ckv_ctx::kScratchSlots; ++i)
    if (ctx->scratch[i]) cudaFree(ctx->scratch[i]);
  delete ctx;
  return CKV_OK;
}

int ckv_ctx_sync(ckv_ctx* ctx) {
  CKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CKV_OK;
}
void* ckv_ctx_stream(ckv_ctx* ctx) { return ctx->stream; }
uint64_t ckv_ctx_launch_count(ckv_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ckv_malloc(ckv_ctx* ctx, void** ptr, size_t bytes) {
  (void)ctx;
  CKV_CUDA_TRY(cudaMalloc(ptr, bytes ? bytes : 16));
  return CKV_OK;
}
int ckv_free(ckv_ctx* ctx, void* ptr) {
  (void)ctx;
  if (ptr) CKV_CUDA_TRY(cudaFree(ptr));
  return CKV_OK;
}
int ckv_memcpy_h2d(ckv_ctx* ctx, void* dst, const void* src, size_t bytes) {
  CKV_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  CKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CKV_OK;
}
int ckv_memcpy_d2h(ckv_ctx* ctx, void* dst, const void* src, size_t bytes) {
  CKV_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CKV_OK;
}
int ckv_memset(ckv_ctx* ctx, void* dst, int value, size_t bytes) {
  CKV_CUDA_TRY(cudaMemsetAsync(dst, value, bytes, ctx->stream));
  return CKV_OK;
}

int ckv_f32_to_bf16(ckv_ctx* ctx, const float* src, uint16_t* dst, size_t n, int* all_exact) {
  void* fv = nullptr;
  CKV_TRY(ctx_scratch(ctx, 37, sizeof(int), false, &fv));
  int* flag = static_cast<int*>(fv);
  CKV_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  if (n) {
    int blocks = int(std::min<size_t>((n + 255) / 256, size_t(num_sms()) * 8));
    k_f32_to_bf16<<<blocks, 256, 0, ctx->stream>>>(src, dst, n, flag);
    CKV_LAUNCH_CHECK("k_f32_to_bf16");
    ctx->launches++;
  }
  int h = 0;
  CKV_CUDA_TRY(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (all_exact) *all_exact = h ? 0 : 1;
  return CKV_OK;
}

// ===========================================================================
// k-means
// ===========================================================================
uint64_t ckv_mix_seed(uint64_t seed, uint64_t a, uint64_t b) { return host_mix_seed(seed, a, b); }

int ckv_kmeans_init_rows(uint32_t n, uint32_t C, uint64_t seed, uint32_t* rows_out) {
  if (C < 1 || C > n) { set_error("kmeans: need 1 <= C <= N"); return CKV_EINVAL; }
  host_init_rows(n, C, seed, rows_out);
  return CKV_OK;
}

int ckv_kmeans(ckv_ctx* ctx, const ckv_kmeans_desc* d, const uint16_t* keys,
               const uint32_t* init_rows, float* centroids, int32_t* labels,
               ckv_kmeans_info* info_host, double* objective_host, uint32_t* repair_host) {
  if (!ctx || !d) { set_error("ckv_kmeans: NULL argument"); return CKV_EINVAL; }
  KMeansArgs a;
  a.n_units = d->n_units;
  a.n = d->n;
  a.C = d->C;
  a.max_iters = d->max_iters;
  a.key_stride = d->key_stride;
  a.c_stride = d->c_stride;
  a.label_stride = d->label_stride;
  a.flags = d->flags;
  a.keys = keys;
  a.init_rows = init_rows;
  a.centroids = centroids;
  a.labels = labels;
  if (a.c_stride < a.C || a.label_stride < a.n) {
    set_error("ckv_kmeans: strides smaller than C / n");
    return CKV_EINVAL;
  }
  return kmeans_run(ctx, a, info_host, objective_host, repair_host);
}

uint32_t ckv_prefill_cluster_count(uint32_t L, uint32_t divisor, uint32_t sink, uint32_t ovr) {
  if (L <= sink) return 0;
  const uint32_t n = L - sink;
  uint32_t c0 = ovr ? ovr : uint32_t(std::llround(double(n) / double(divisor ? divisor : 1)));
  return std::clamp<uint32_t>(c0, 1, n);
}

int ckv_cluster_prefill(ckv_ctx* ctx, const ckv_prefill_desc* d, const uint16_t* keys,
                        const uint64_t* seeds, float* centroids, int32_t* labels,
                        uint32_t* n_clusters, ckv_kmeans_info* info_host, double* objective_host,
                        uint32_t* repair_host) {
  if (d->c0_divisor < 1) { set_error("ClusterConfig: c0_divisor must be >= 1"); return CKV_EINVAL; }
  if (d->max_iters < 1) { set_error("ClusterConfig: max_iters must be >= 1"); return CKV_EINVAL; }
  const uint32_t U = d->n_units, L = d->L, sink = d->sink_tokens;
  const uint32_t C0 = ckv_prefill_cluster_count(L, d->c0_divisor, sink, d->c0_override);
  cudaStream_t st = ctx->stream;
  // labels: -1 everywhere first (sinks, and anything beyond L)
  k_fill_i32<<<dim3(std::max<uint32_t>(1, std::min<uint32_t>((d->p_cap + 255) / 256, 64)), U),
               256, 0, st>>>(labels, d->p_cap, d->p_cap, -1);
  CKV_LAUNCH_CHECK("k_fill_i32");
  k_set_u32<<<(U + 127) / 128, 128, 0, st>>>(n_clusters, U, C0);
  CKV_LAUNCH_CHECK("k_set_u32");
  ctx->launches += 2;
  if (C0 == 0) {
    for (uint32_t u = 0; info_host && u < U; ++u) info_host[u] = {0, 1, 0, 0};
    return ckv_ctx_sync(ctx);
  }
  if (C0 > d->c_cap) { set_error("cluster_prefill: C0 exceeds c_cap"); return CKV_EINVAL; }
  const uint32_t n = L - sink;
  trace_begin("cluster_prefill");
  std::vector<uint32_t> rows(size_t(U) * C0);
  host_init_rows_batch(U, n, C0, seeds, rows.data());
  trace_mark("init rows sampled");
  void* d_rows_v = nullptr;  // context scratch: no stream-ordered pool trim on the sync
  CKV_TRY(ctx_scratch(ctx, 29, rows.size() * 4, false, &d_rows_v));
  uint32_t* d_rows = static_cast<uint32_t*>(d_rows_v);
  CKV_CUDA_TRY(cudaMemcpyAsync(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, st));
  trace_mark("init rows queued");
  KMeansArgs a;
  a.n_units = U;
  a.n = n;
  a.C = C0;
  a.max_iters = d->max_iters;
  a.key_stride = uint64_t(d->p_cap) * D;
  a.c_stride = d->c_cap;
  a.label_stride = d->p_cap;
  a.flags = d->flags;
  a.keys = keys + size_t(sink) * D;
  a.init_rows = d_rows;
  a.centroids = centroids;
  a.labels = labels + sink;
  int rc = kmeans_run(ctx, a, info_host, objective_host, repair_host);
  if (rc) return rc;
  rc = ckv_ctx_sync(ctx);
  trace_mark("done");
  return rc;
}

// device init rows of a decode batch (k_decode_init_rows) into `rows`
static int launch_decode_init_rows(cudaStream_t st, const uint64_t* seeds_dev, uint32_t n_units,
                            uint32_t pos0, uint32_t n, uint32_t C, uint32_t* rows) {
  if (C > DI_MAX_C || C > n) { set_error("decode init rows: need C <= min(32, rows)"); return CKV_EINVAL; }
  k_decode_init_rows<<<(n_units + 127) / 128, 128, 0, st>>>(seeds_dev, n_units, pos0, n, C, rows);
  CKV_LAUNCH_CHECK("k_decode_init_rows");
  return CKV_OK;
}

int ckv_cluster_decode_batch(ckv_ctx* ctx, const ckv_decode_cluster_desc* d,
                             const uint16_t* keys, const uint64_t* seeds, float* centroids,
                             int32_t* labels, uint32_t* n_clusters, uint32_t* iterations_host) {
  const uint32_t U = d->n_units, rows = d->rows;
  if (rows == 0 || U == 0) return CKV_OK;  // clustering.hpp:311
  if (d->c_plus < 1) { set_error("ClusterConfig: c_plus must be >= 1"); return CKV_EINVAL; }
  if (d->max_iters < 1) { set_error("ClusterConfig: max_iters must be >= 1"); return CKV_EINVAL; }
  cudaStream_t st = ctx->stream;
  const uint32_t C = std::min(d->c_plus, rows);
  void *v_init = nullptr, *v_c = nullptr, *v_l = nullptr, *v_seed = nullptr;
  CKV_TRY(ctx_scratch(ctx, 30, size_t(U) * C * 4, false, &v_init));
  CKV_TRY(ctx_scratch(ctx, 31, size_t(U) * C * D * 4, false, &v_c));
  CKV_TRY(ctx_scratch(ctx, 32, size_t(U) * std::max(rows, 2u) * 4, false, &v_l));
  uint32_t* d_init = static_cast<uint32_t*>(v_init);
  float* tmp_c = static_cast<float*>(v_c);
  int32_t* tmp_l = static_cast<int32_t*>(v_l);
  if (kmeans_small_supported(rows, C)) {
    // init rows on the device, then the whole k-means of every unit's batch
    // in one launch (ckv_kmeans.cu); one read-back for the input checks
    CKV_TRY(ctx_scratch(ctx, 33, size_t(U) * 8, false, &v_seed));
    CKV_CUDA_TRY(cudaMemcpyAsync(v_seed, seeds, size_t(U) * 8, cudaMemcpyHostToDevice, st));
    CKV_TRY(launch_decode_init_rows(st, static_cast<const uint64_t*>(v_seed), U, d->pos0, rows,
                                    C, d_init));
    uint32_t* d_it = reinterpret_cast<uint32_t*>(tmp_l);  // scratch reuse: [U] + [U]
    int32_t* d_st = tmp_l + U;
    CKV_TRY(launch_kmeans_small(st, keys + size_t(d->pos0) * D, uint64_t(d->p_cap) * D, U, rows,
                                C, d->max_iters, d_init, centroids, d->c_cap, labels + d->pos0,
                                d->p_cap, n_clusters, d_it, d_st));
    ctx->launches += 2;
    std::vector<int32_t> hb(2 * size_t(U));
    CKV_CUDA_TRY(cudaMemcpyAsync(hb.data(), tmp_l, 8 * size_t(U), cudaMemcpyDeviceToHost, st));
    CKV_CUDA_TRY(cudaStreamSynchronize(st));
    for (uint32_t u = 0; u < U; ++u) {
      if (hb[U + u] == 1) { set_error("kmeans: keys must be finite"); return CKV_EINVAL; }
      if (hb[U + u] == 2) {
        set_error("kmeans: degenerate input, all keys zero-norm");
        return CKV_EINVAL;
      }
      if (iterations_host) iterations_host[u] = uint32_t(hb[u]) & 0x7fffffffu;
    }
    return CKV_OK;
  }
  // large batches (rows > 512 or C+ > 32): the generic k-means driver
  std::vector<uint32_t> init(size_t(U) * C);
  for (uint32_t u = 0; u < U; ++u)
    host_init_rows(rows, C, host_mix_seed(seeds[u], 0xdecadeull, d->pos0),
                   init.data() + size_t(u) * C);
  CKV_CUDA_TRY(cudaMemcpyAsync(d_init, init.data(), init.size() * 4, cudaMemcpyHostToDevice, st));
  KMeansArgs a;
  a.n_units = U;
  a.n = rows;
  a.C = C;
  a.max_iters = d->max_iters;
  a.key_stride = uint64_t(d->p_cap) * D;
  a.c_stride = C;
  a.label_stride = rows;
  a.flags = CKV_KM_EXACT_ONLY;
  a.keys = keys + size_t(d->pos0) * D;
  a.init_rows = d_init;
  a.centroids = tmp_c;
  a.labels = tmp_l;
  std::vector<ckv_kmeans_info> info(U);
  CKV_TRY(kmeans_run(ctx, a, info.data(), nullptr, nullptr));
  k_append_clusters<<<U, 256, 0, st>>>(tmp_c, tmp_l, C, rows, d->pos0, d->c_cap, d->p_cap,
                                       centroids, labels, n_clusters);
  CKV_LAUNCH_CHECK("k_append_clusters");
  ctx->launches++;
  if (iterations_host)
    for (uint32_t u = 0; u < U; ++u) iterations_host[u] = info[u].iterations_used;
  return ckv_ctx_sync(ctx);
}

// ===========================================================================
// index, select, cache, attend
// ===========================================================================
int ckv_build_index(ckv_ctx* ctx, uint32_t n_units, uint32_t n_pos, uint32_t p_cap,
                    uint32_t c_cap, const int32_t* labels, const uint32_t* n_clusters,
                    uint32_t* sizes, uint32_t* starts, uint32_t* sorted_ids) {
  if (n_pos > p_cap) { set_error("build_index: n_pos > p_cap"); return CKV_EINVAL; }
  CKV_TRY(launch_index(ctx->stream, n_units, labels, n_pos, p_cap, c_cap, n_clusters, 0, sizes,
                       starts, sorted_ids, nullptr, nullptr, nullptr, nullptr));
  ctx->launches++;
  return CKV_OK;
}

static CacheDev null_cache() {
  CacheDev c;
  std::memset(&c, 0, sizeof c);
  return c;
}

static ckv_runs null_runs() {
  ckv_runs r;
  std::memset(&r, 0, sizeof r);
  return r;
}

int ckv_select(ckv_ctx* ctx, const ckv_select_desc* d, const float* q, const float* centroids,
               const uint32_t* n_clusters, const uint32_t* sizes, const uint32_t* starts,
               const uint32_t* sorted_ids, uint32_t* token_ids, uint32_t* rows,
               const ckv_runs* runs, uint32_t* n_tokens, uint32_t* n_taken, uint32_t* trimmed,
               uint32_t* ranked, double* scores, ckv_cache* cache) {
  if (!ranked || !n_tokens || !n_taken || !trimmed) {
    set_error("ckv_select: ranked / n_tokens / n_taken / trimmed are required");
    return CKV_EINVAL;
  }
  if (cache && cache->dev.n_slots < d->n_q) {
    set_error("ckv_select: cache has fewer slots than q heads");
    return CKV_EINVAL;
  }
  if (runs && runs->run_cap < d->c_cap + 2) {
    set_error("ckv_select: runs.run_cap must be >= c_cap + 2");
    return CKV_EINVAL;
  }
  if (cache && cache->dev.c_cap < d->c_cap) {
    set_error("ckv_select: cache c_cap is smaller than the selection's c_cap");
    return CKV_EINVAL;
  }
  if (token_ids || rows) {  // |I_T| <= min(B, labeled) + sinks + recency (selection.hpp:88-89)
    const uint64_t need = uint64_t(std::min(d->budget, d->p_cap)) + d->sink_count +
                          (d->rec_end > d->rec_begin ? d->rec_end - d->rec_begin : 0);
    if (d->sel_cap < need) {
      set_error("ckv_select: sel_cap < min(budget, p_cap) + sink_count + (rec_end - rec_begin)");
      return CKV_EINVAL;
    }
  }
  void* scratch = nullptr;
  CKV_TRY(ctx_scratch(ctx, 34, select_scratch_bytes(d->n_q, d->c_cap), false, &scratch));
  int rc = launch_select(ctx->stream, *d, q, centroids, n_clusters, sizes, starts, sorted_ids,
                         token_ids, rows, runs ? *runs : null_runs(), d->row_base, n_tokens,
                         n_taken, trimmed, ranked, scores, cache ? cache->dev : null_cache(),
                         scratch);
  ctx->launches += 2;
  return rc;
}

int ckv_cache_create(ckv_ctx* ctx, uint32_t n_slots, uint32_t c_cap, uint32_t retention,
                     uint32_t d, ckv_cache** out) {
  if (retention < 1) { set_error("ClusterCache: retention must be >= 1"); return CKV_EINVAL; }
  ckv_cache* c = new ckv_cache();
  c->ctx = ctx;
  c->dev.n_slots = n_slots;
  c->dev.c_cap = c_cap;
  c->dev.retention = retention;
  c->dev.d = d;
  c->dev.words = (c_cap + 31) / 32;
  size_t bits = size_t(n_slots) * retention * c->dev.words * 4;
  cudaError_t e = cudaMalloc(&c->dev.bits, bits ? bits : 4);
  if (e == cudaSuccess) e = cudaMalloc(&c->dev.ring, size_t(n_slots) * 8 + 8);
  if (e == cudaSuccess) e = cudaMalloc(&c->dev.counters, size_t(n_slots) * 32 + 32);
  if (e != cudaSuccess) { delete c; return cuda_status(e, "ckv_cache_create"); }
  cudaMemsetAsync(c->dev.bits, 0, bits ? bits : 4, ctx->stream);
  cudaMemsetAsync(c->dev.ring, 0, size_t(n_slots) * 8 + 8, ctx->stream);
  cudaMemsetAsync(c->dev.counters, 0, size_t(n_slots) * 32 + 32, ctx->stream);
  *out = c;
  return CKV_OK;
}

int ckv_cache_destroy(ckv_cache* c) {
  if (!c) return CKV_OK;
  cudaStreamSynchronize(c->ctx->stream);
  cudaFree(c->dev.bits);
  cudaFree(c->dev.ring);
  cudaFree(c->dev.counters);
  delete c;
  return CKV_OK;
}

int ckv_cache_counters(ckv_cache* c, uint64_t* out) {
  CKV_CUDA_TRY(cudaMemcpyAsync(out, c->dev.counters, size_t(c->dev.n_slots) * 32,
                               cudaMemcpyDeviceToHost, c->ctx->stream));
  CKV_CUDA_TRY(cudaStreamSynchronize(c->ctx->stream));
  return CKV_OK;
}

int ckv_cache_lookup(ckv_ctx* ctx, ckv_cache* c, uint32_t slot, const uint32_t* selected,
                     uint32_t n_sel, const uint32_t* sizes, uint32_t* hit, uint32_t* miss,
                     uint32_t* counts_host) {
  if (slot >= c->dev.n_slots) { set_error("cache: slot out of range"); return CKV_EINVAL; }
  void* dcv = nullptr;
  CKV_TRY(ctx_scratch(ctx, 35, 8, false, &dcv));
  uint32_t* dcounts = static_cast<uint32_t*>(dcv);
  CKV_TRY(launch_cache_lookup(ctx->stream, c->dev, slot, selected, n_sel, sizes, hit, miss,
                              dcounts));
  ctx->launches++;
  CKV_CUDA_TRY(cudaMemcpyAsync(counts_host, dcounts, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CKV_OK;
}

int ckv_cache_invalidate(ckv_ctx* ctx, ckv_cache* c, uint32_t slot, const uint32_t* retired,
                         uint32_t n) {
  if (n == 0) return CKV_OK;
  void* dv = nullptr;
  CKV_TRY(ctx_scratch(ctx, 36, size_t(n) * 4, false, &dv));
  uint32_t* d = static_cast<uint32_t*>(dv);
  CKV_CUDA_TRY(cudaMemcpyAsync(d, retired, size_t(n) * 4, cudaMemcpyHostToDevice, ctx->stream));
  CKV_TRY(launch_cache_invalidate(ctx->stream, c->dev, slot, d, n));
  ctx->launches++;
  CKV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CKV_OK;
}

int ckv_relayout_kv(ckv_ctx* ctx, uint32_t n_units, uint32_t p_cap, const uint16_t* K,
                    const uint16_t* V, uint16_t* K2, uint16_t* V2, const uint32_t* sorted_ids,
                    uint32_t sink, uint32_t labeled_end, uint32_t n_rows) {
  if (!ctx || !K || !V || !K2 || !V2 || !sorted_ids) {
    set_error("ckv_relayout_kv: NULL argument");
    return CKV_EINVAL;
  }
  if (sink > labeled_end || labeled_end > n_rows || n_rows > p_cap) {
    set_error("ckv_relayout_kv: need sink <= labeled_end <= n_rows <= p_cap");
    return CKV_EINVAL;
  }
  if ((K2 == K) != (V2 == V)) {
    set_error("ckv_relayout_kv: K and V must both be in place or both out of place");
    return CKV_EINVAL;
  }
  if (n_units == 0 || n_rows == 0) return CKV_OK;
  cudaStream_t st = ctx->stream;
  if (K2 != K) {
    dim3 g((n_rows + 7) / 8, n_units);
    k_relayout<<<g, 128, 0, st>>>(K, V, K2, V2, sorted_ids, p_cap, sink, labeled_end, n_rows);
    CKV_LAUNCH_CHECK("k_relayout");
    ctx->launches++;
    return CKV_OK;
  }
  // in place: chunks of units through a bounded staging buffer, so a store
  // that fills most of HBM (config C: 128 GiB of KV) never needs a second
  // copy.  The staging is the context's grow-only slot 22 (a stream-ordered
  // allocation per call re-commits its pages every prefill: ~170 ms at
  // config B for 2 GiB).
  const size_t unit_bytes = size_t(p_cap) * D * 2;
  const uint32_t chunk = uint32_t(std::max<size_t>(1, std::min<size_t>(
      n_units, (size_t(256) << 20) / unit_bytes)));
  void* stage = nullptr;
  CKV_TRY(ctx_scratch(ctx, 22, 2 * size_t(chunk) * unit_bytes, false, &stage));
  uint16_t* tK = static_cast<uint16_t*>(stage);
  uint16_t* tV = tK + size_t(chunk) * p_cap * D;
  int rc = CKV_OK;
  for (uint32_t u0 = 0; u0 < n_units && rc == CKV_OK; u0 += chunk) {
    const uint32_t nu = std::min(chunk, n_units - u0);
    const size_t off = size_t(u0) * p_cap * D;
    dim3 g((n_rows + 7) / 8, nu);
    k_relayout<<<g, 128, 0, st>>>(K + off, V + off, tK, tV, sorted_ids + size_t(u0) * p_cap,
                                  p_cap, sink, labeled_end, n_rows);
    if (cudaGetLastError() != cudaSuccess) { rc = cuda_status(cudaErrorLaunchFailure, "k_relayout"); break; }
    ctx->launches++;
    for (int kv = 0; kv < 2 && rc == CKV_OK; ++kv) {
      cudaError_t e = cudaMemcpy2DAsync(kv ? K2 + off : V2 + off, unit_bytes, kv ? tK : tV,
                                        unit_bytes, size_t(n_rows) * D * 2, nu,
                                        cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) rc = cuda_status(e, "ckv_relayout_kv copy-back");
    }
  }
  return rc;
}

int ckv_attend(ckv_ctx* ctx, const ckv_attend_desc* d, const float* q, const uint16_t* K,
               const uint16_t* V, const uint32_t* rows, const ckv_runs* runs,
               const uint32_t* n_tokens, float* out, float* weights) {
  cudaStream_t st = ctx->stream;
  if (weights && d->max_tokens > d->sel_cap) {  // weights rows are sel_cap apart
    set_error("ckv_attend: max_tokens > sel_cap with a weights output");
    return CKV_EINVAL;
  }
  if (weights) {  // parity mode: approx_attention's empty-selection check
    std::vector<uint32_t> nt(d->n_q);
    CKV_CUDA_TRY(cudaMemcpyAsync(nt.data(), n_tokens, 4 * size_t(d->n_q),
                                 cudaMemcpyDeviceToHost, st));
    CKV_CUDA_TRY(cudaStreamSynchronize(st));
    for (uint32_t v : nt)
      if (v == 0) { set_error("approx_attention: empty selection"); return CKV_EINVAL; }
  }
  float *part = nullptr, *lw = nullptr;
  uint32_t* tickets = nullptr;
  CKV_TRY(attend_scratch(ctx, *d, weights != nullptr, &part, &tickets, &lw));
  int rc = launch_attend(st, *d, q, K, V, rows, runs ? *runs : null_runs(), n_tokens, out,
                         weights, lw, part, tickets);
  ctx->launches++;
  return rc;
}

}  // extern "C"

// ===========================================================================
// session
// ===========================================================================
struct ckv_session {
  ckv_ctx* ctx = nullptr;
  ckv_session_desc d{};
  uint32_t U = 0, n_q = 0, p_cap = 0, c_cap = 0, sel_cap = 0;
  uint16_t *K = nullptr, *V = nullptr;
  float* cents = nullptr;
  // CKV_SESSION_F16_SCORES=1: the fused selection's approximate scores from an
  // fp16 centroid copy (SelC16), refreshed before the first selection after
  // anything rewrote the centroids.  Opt-in: measured no faster at config B
  // (114.0 vs 113.9 us/step) and slower in layer mode (0.79 vs 0.75 ms/step)
  // -- the scoring phase is not bound by the centroid bytes.
  bool use_c16 = false;
  uint16_t* c16 = nullptr;
  float* cerr = nullptr;
  bool c16_dirty = true;  // all rows
  uint32_t c16_tail = 0;  // or only each unit's last c16_tail rows (committed decode batches)
  int32_t* labels = nullptr;
  uint32_t *n_clusters = nullptr, *sizes = nullptr, *starts = nullptr, *sorted = nullptr;
  uint32_t *token_ids = nullptr, *rows = nullptr, *n_tokens = nullptr, *n_taken = nullptr,
           *trimmed = nullptr, *ranked = nullptr;
  void* sel_scratch = nullptr;
  ckv_runs runs{};
  uint16_t *tmpK = nullptr, *tmpV = nullptr;  // decode-batch relayout staging
  float* part = nullptr;
  uint32_t* tickets = nullptr;
  // StepSync (ckv_internal.cuh): per-q-head selection -> attention flags
  // and their epoch; off with CKV_SESSION_NO_STEPSYNC=1
  uint32_t *step_ready = nullptr, *step_epoch = nullptr, *step_work = nullptr;
  StepSync sync{};
  float *q_dev = nullptr, *out_dev = nullptr;
  uint16_t *kn_dev = nullptr, *vn_dev = nullptr;
  ckv_cache* cache = nullptr;
  std::vector<uint64_t> seeds;
  uint32_t n_ctx = 0, labeled_end = 0, steps = 0, pending = 0, C_cur = 0;
  bool prefilled = false;
  bool l2_persist = false;
  // decode-batch clustering, device-resident (harness.hpp:318-337): per-unit
  // seeds, init rows, the kernel's iteration / status words and their
  // pinned host copy (checked lazily: no sync on the decode path)
  uint64_t* d_seeds = nullptr;
  uint32_t* db_init = nullptr;
  int32_t* db_stat = nullptr;   // [2U]: iterations | converged bit, status
  int32_t* h_stat = nullptr;    // pinned [2U]
  cudaEvent_t ev_stat = nullptr;
  bool stat_pending = false;
  uint32_t pend_pos0 = 0;       // first position of the batch being collected
  // async mode (harness.hpp:236-243, 327-329): the batch's k-means runs on a
  // side stream and is committed async_delay steps later
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_done = nullptr;
  // the batched step's second selection stream (session_select_attend)
  cudaStream_t sel_stream = nullptr;
  cudaEvent_t ev_sel_fork = nullptr, ev_sel_join = nullptr;
  uint32_t* stage_ncl = nullptr;  // n_clusters as the side stream's k-means leaves it
  struct Queued { uint32_t ready, pos0, rows, C; };
  std::deque<Queued> queue;
  uint32_t layer_units = 0;  // 0: one select + attend for all units; else per slice
  // no kernel has written the centroids / sizes / starts / n_clusters since
  // the previous selection, and the stream's last kernel is the append
  // (CKV_SEL_EARLY for the next step's selections)
  bool sel_early = false;
  // this step's new K/V rows while its selection is launched (the fused
  // selection appends them; app_done: every slice's launch did)
  const uint16_t* app_k = nullptr;
  const uint16_t* app_v = nullptr;
  bool app_done = false;
  bool step_early = false;  // this step's selections may start early
  // physical two-tier cache (CKV_SESSION_TIERED / _TIER_HOST, ckv_tier.cu)
  bool tiered = false;
  TierArgs tier{};
  ckv_runs truns{};            // page runs the attention reads in tiered mode
  uint16_t *hK = nullptr, *hV = nullptr;  // host-pinned backing mirror (TIER_HOST)
  uint32_t n_batches = 0;    // decode batches launched (device path)
};

namespace {
template <typename T>
int salloc(T** p, size_t count) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count * sizeof(T), 16));
  if (e != cudaSuccess) return cuda_status(e, "ckv_session alloc");
  return CKV_OK;
}
}  // namespace

extern "C" {

// The persisting-L2 limit is device-wide state: reference-count the sessions
// that raised it, remember the caller's value before the first one, and
// restore it (and drop the persisting lines) only when the last one goes.
static std::mutex g_l2_mu;
static int g_l2_refs[64];
static size_t g_l2_saved[64];

// the device's persisting-L2 limit as this library last read or set it (the
// selection's access-policy window sizes its hit ratio from it every launch;
// SIZE_MAX: not read yet)
static std::atomic<size_t> g_l2_limit[64];
static bool g_l2_limit_init = [] {
  for (auto& x : g_l2_limit) x.store(SIZE_MAX);
  return true;
}();

extern "C++" {
size_t ckvb::l2_persist_limit() {
  int dev = 0;
  cudaGetDevice(&dev);
  size_t v = g_l2_limit[dev & 63].load(std::memory_order_relaxed);
  if (v == SIZE_MAX) {
    if (cudaDeviceGetLimit(&v, cudaLimitPersistingL2CacheSize) != cudaSuccess) return 0;
    g_l2_limit[dev & 63].store(v, std::memory_order_relaxed);
  }
  return v;
}
}  // extern "C++"

static bool l2_persist_acquire(int dev, size_t want) {
  std::lock_guard<std::mutex> lock(g_l2_mu);
  const int i = dev & 63;
  size_t cur = 0;
  if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) != cudaSuccess) return false;
  if (g_l2_refs[i] == 0) g_l2_saved[i] = cur;
  if (want > cur && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess)
    return false;
  size_t now = cur;
  if (cudaDeviceGetLimit(&now, cudaLimitPersistingL2CacheSize) == cudaSuccess)
    g_l2_limit[i].store(now, std::memory_order_relaxed);
  ++g_l2_refs[i];
  return true;
}

static void l2_persist_release(int dev) {
  std::lock_guard<std::mutex> lock(g_l2_mu);
  const int i = dev & 63;
  if (g_l2_refs[i] > 0 && --g_l2_refs[i] == 0) {
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, g_l2_saved[i]);
    g_l2_limit[i].store(SIZE_MAX, std::memory_order_relaxed);  // re-read on next use
  }
}

int ckv_session_create(ckv_ctx* ctx, const ckv_session_desc* d, ckv_session** out) {
  if (d->group < 1 || d->budget < 1 || d->decode_batch < 1 || d->c_plus < 1 ||
      d->max_iters < 1 || d->c0_divisor < 1) {
    set_error("ckv_session_create: invalid configuration");
    return CKV_EINVAL;
  }
  if (d->async_delay &&
      (d->async_delay >= d->decode_batch ||
       !kmeans_small_supported(d->decode_batch, std::min(d->c_plus, d->decode_batch)))) {
    set_error("ckv_session_create: async clustering needs async_delay < decode_batch <= 512 "
              "and c_plus <= 32");
    return CKV_EINVAL;
  }
  ckv_session* s = new ckv_session();
  s->ctx = ctx;
  s->d = *d;
  s->U = d->n_units;
  s->n_q = d->n_units * d->group;
  s->p_cap = d->prompt_len + d->max_decode;
  const uint32_t C0 = ckv_prefill_cluster_count(d->prompt_len, d->c0_divisor, d->sink_tokens,
                                                d->c0_override);
  s->c_cap = C0 + d->c_plus * (d->max_decode / d->decode_batch + 1);
  // recency: the collecting batch (< m rows) plus, in async mode, a batch
  // waiting async_delay steps for its commit
  s->sel_cap = d->budget + d->sink_tokens + d->decode_batch + 1 +
               (d->async_delay ? d->decode_batch + d->async_delay : 0);
  s->tiered = (d->flags & (CKV_SESSION_TIERED | CKV_SESSION_TIER_HOST)) != 0;
  // tiered: every unit's page pool sits after all units' store rows (pool
  // rows are addressed relative to a unit's store base, ckv_tier.cu); sized
  // for R steps of the unit's heads' selections (whole clusters, page
  // rounding) with slack — the fetch evicts harder before it ever fails
  uint32_t np = 0;
  if (s->tiered)
    np = std::max<uint32_t>(1, d->retention) * d->group * ((d->budget + 512) / TIER_PAGE_ROWS + 64) +
         64;
  const size_t kv = size_t(s->U) * (s->p_cap + size_t(np) * TIER_PAGE_ROWS) * D;
  int rc = CKV_OK;
  rc |= salloc(&s->K, kv);
  rc |= salloc(&s->V, kv);
  rc |= salloc(&s->cents, size_t(s->U) * s->c_cap * D);
  s->use_c16 = getenv("CKV_SESSION_F16_SCORES") != nullptr;
  if (s->use_c16) {
    rc |= salloc(&s->c16, size_t(s->U) * s->c_cap * D);
    rc |= salloc(&s->cerr, size_t(s->U) * s->c_cap);
  }
  rc |= salloc(&s->labels, size_t(s->U) * s->p_cap);
  rc |= salloc(&s->n_clusters, s->U);
  rc |= salloc(&s->sizes, size_t(s->U) * s->c_cap);
  rc |= salloc(&s->starts, size_t(s->U) * (s->c_cap + 1));
  rc |= salloc(&s->sorted, size_t(s->U) * s->p_cap);
  rc |= salloc(&s->token_ids, size_t(s->n_q) * s->sel_cap);
  rc |= salloc(&s->rows, size_t(s->n_q) * s->sel_cap);
  rc |= salloc(reinterpret_cast<unsigned char**>(&s->sel_scratch),
               select_scratch_bytes(s->n_q, s->c_cap));
  s->runs.run_cap = s->c_cap + 2;
  rc |= salloc(&s->runs.row, size_t(s->n_q) * s->runs.run_cap);
  rc |= salloc(&s->runs.off, size_t(s->n_q) * (s->runs.run_cap + 1));
  rc |= salloc(&s->runs.count, s->n_q);
  rc |= salloc(&s->tmpK, size_t(s->U) * d->decode_batch * D);
  rc |= salloc(&s->tmpV, size_t(s->U) * d->decode_batch * D);
  rc |= salloc(&s->n_tokens, s->n_q);
  rc |= salloc(&s->n_taken, s->n_q);
  rc |= salloc(&s->trimmed, s->n_q);
  rc |= salloc(&s->ranked, size_t(s->n_q) * s->c_cap);
  rc |= salloc(&s->part, attend_part_floats(s->n_q, s->sel_cap));
  rc |= salloc(&s->tickets, s->n_q);
  rc |= salloc(&s->step_ready, s->n_q);
  rc |= salloc(&s->step_epoch, 1);
  rc |= salloc(&s->step_work, s->U);
  rc |= salloc(&s->q_dev, size_t(s->n_q) * D);
  rc |= salloc(&s->out_dev, size_t(s->n_q) * D);
  rc |= salloc(&s->kn_dev, size_t(s->U) * D);
  rc |= salloc(&s->vn_dev, size_t(s->U) * D);
  rc |= salloc(&s->d_seeds, s->U);
  rc |= salloc(&s->db_init, size_t(s->U) * std::min(d->c_plus, d->decode_batch));
  rc |= salloc(&s->db_stat, 2 * size_t(s->U));
  rc |= salloc(&s->stage_ncl, s->U);
  if (!rc && cudaMallocHost(&s->h_stat, 8 * size_t(s->U)) != cudaSuccess) rc = 1;
  if (!rc && cudaEventCreateWithFlags(&s->ev_stat, cudaEventDisableTiming) != cudaSuccess) rc = 1;
  if (!rc && (cudaStreamCreateWithFlags(&s->sel_stream, cudaStreamNonBlocking) != cudaSuccess ||
              cudaEventCreateWithFlags(&s->ev_sel_fork, cudaEventDisableTiming) != cudaSuccess ||
              cudaEventCreateWithFlags(&s->ev_sel_join, cudaEventDisableTiming) != cudaSuccess))
    rc = 1;
  if (!rc && d->async_delay) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&s->side, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev_done, cudaEventDisableTiming) != cudaSuccess)
      rc = 1;
  }
  if (!rc && s->tiered) {
    TierArgs& t = s->tier;
    t.n_units_total = s->U;
    t.p_cap = s->p_cap;
    t.c_cap = s->c_cap;
    t.np = np;
    t.group = d->group;
    t.retention = std::max<uint32_t>(1, d->retention);
    t.sink = std::min(d->sink_tokens, d->prompt_len);
    t.n_clusters = s->n_clusters;
    t.sizes = s->sizes;
    t.starts = s->starts;
    rc |= salloc(&t.cpage, size_t(s->U) * s->c_cap);
    rc |= salloc(&t.last, size_t(s->U) * s->c_cap);
    rc |= salloc(&t.next, size_t(s->U) * np);
    rc |= salloc(&t.free_stack, size_t(s->U) * np);
    rc |= salloc(&t.n_free, s->U);
    rc |= salloc(&t.stats, size_t(s->U) * 4);
    rc |= salloc(&t.status, 1);
    s->truns.run_cap = s->c_cap + (d->budget + TIER_PAGE_ROWS - 1) / TIER_PAGE_ROWS + 3;
    rc |= salloc(&s->truns.row, size_t(s->n_q) * s->truns.run_cap);
    rc |= salloc(&s->truns.off, size_t(s->n_q) * (s->truns.run_cap + 1));
    rc |= salloc(&s->truns.count, s->n_q);
    if (!rc && (d->flags & CKV_SESSION_TIER_HOST)) {
      const size_t bytes = size_t(s->U) * s->p_cap * D * 2;
      void *hk = nullptr, *hv = nullptr, *dk = nullptr, *dv = nullptr;
      if (cudaHostAlloc(&hk, bytes, cudaHostAllocMapped) != cudaSuccess ||
          cudaHostAlloc(&hv, bytes, cudaHostAllocMapped) != cudaSuccess ||
          cudaHostGetDevicePointer(&dk, hk, 0) != cudaSuccess ||
          cudaHostGetDevicePointer(&dv, hv, 0) != cudaSuccess)
        rc = 1;
      s->hK = static_cast<uint16_t*>(hk);
      s->hV = static_cast<uint16_t*>(hv);
      t.back_K = static_cast<const uint16_t*>(dk);
      t.back_V = static_cast<const uint16_t*>(dv);
    } else {
      t.back_K = s->K;  // secondary-HBM backing: the store itself
      t.back_V = s->V;
    }
    if (!rc) cudaMemsetAsync(t.status, 0, 4, ctx->stream);
  }
  if (rc) { ckv_session_destroy(s); return CKV_ENOMEM; }
  cudaMemsetAsync(s->tickets, 0, size_t(s->n_q) * 4, ctx->stream);
  cudaMemsetAsync(s->step_ready, 0, size_t(s->n_q) * 4, ctx->stream);
  cudaMemsetAsync(s->step_epoch, 0, 4, ctx->stream);
  cudaMemsetAsync(s->step_work, 0, size_t(s->U) * 4, ctx->stream);
  cudaMemsetAsync(s->n_clusters, 0, size_t(s->U) * 4, ctx->stream);
  if (d->flags & CKV_SESSION_L2_PERSIST) {  // device-wide; restored by the last user
    int maxp = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
    const size_t want = std::min<size_t>(size_t(maxp), size_t(s->U) * s->c_cap * D * 4);
    s->l2_persist = want && l2_persist_acquire(ctx->device, want);
    cudaGetLastError();
  }
  if (d->retention > 0) {
    rc = ckv_cache_create(ctx, s->n_q, s->c_cap, d->retention, D, &s->cache);
    if (rc) { ckv_session_destroy(s); return rc; }
  }
  s->seeds.resize(s->U);
  const uint32_t kvh = std::max<uint32_t>(1, d->kv_heads);
  // unit u = layer * kv_heads + head (batch folded into the layer index)
  for (uint32_t u = 0; u < s->U; ++u)
    s->seeds[u] = host_mix_seed(d->cluster_seed, u / kvh, u % kvh);  // harness.hpp:195
  {
    const cudaError_t e = cudaMemcpyAsync(s->d_seeds, s->seeds.data(), 8 * size_t(s->U),
                                          cudaMemcpyHostToDevice, ctx->stream);
    rc = e == cudaSuccess ? ckv_ctx_sync(ctx) : cuda_status(e, "session seeds");
  }
  if (rc) { ckv_session_destroy(s); return rc; }
  s->n_ctx = d->prompt_len;
  s->labeled_end = d->prompt_len;
  s->pend_pos0 = d->prompt_len;
  *out = s;
  return CKV_OK;
}

int ckv_session_destroy(ckv_session* s) {
  if (!s) return CKV_OK;
  cudaStreamSynchronize(s->ctx->stream);
  cudaFree(s->K); cudaFree(s->V); cudaFree(s->cents); cudaFree(s->labels);
  cudaFree(s->c16); cudaFree(s->cerr);
  cudaFree(s->n_clusters); cudaFree(s->sizes); cudaFree(s->starts); cudaFree(s->sorted);
  cudaFree(s->token_ids); cudaFree(s->rows); cudaFree(s->sel_scratch); cudaFree(s->tmpK);
  cudaFree(s->runs.row); cudaFree(s->runs.off); cudaFree(s->runs.count);
  cudaFree(s->tmpV); cudaFree(s->n_tokens); cudaFree(s->n_taken); cudaFree(s->trimmed);
  cudaFree(s->ranked); cudaFree(s->part); cudaFree(s->tickets); cudaFree(s->q_dev);
  cudaFree(s->step_ready); cudaFree(s->step_epoch); cudaFree(s->step_work);
  cudaFree(s->out_dev); cudaFree(s->kn_dev); cudaFree(s->vn_dev);
  if (s->side) { cudaStreamSynchronize(s->side); cudaStreamDestroy(s->side); }
  if (s->sel_stream) { cudaStreamSynchronize(s->sel_stream); cudaStreamDestroy(s->sel_stream); }
  if (s->ev_sel_fork) cudaEventDestroy(s->ev_sel_fork);
  if (s->ev_sel_join) cudaEventDestroy(s->ev_sel_join);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_done) cudaEventDestroy(s->ev_done);
  if (s->ev_stat) cudaEventDestroy(s->ev_stat);
  if (s->h_stat) cudaFreeHost(s->h_stat);
  cudaFree(s->d_seeds); cudaFree(s->db_init); cudaFree(s->db_stat); cudaFree(s->stage_ncl);
  cudaFree(s->tier.cpage); cudaFree(s->tier.last); cudaFree(s->tier.next);
  cudaFree(s->tier.free_stack); cudaFree(s->tier.n_free); cudaFree(s->tier.stats);
  cudaFree(s->tier.status);
  cudaFree(s->truns.row); cudaFree(s->truns.off); cudaFree(s->truns.count);
  if (s->hK) cudaFreeHost(s->hK);
  if (s->hV) cudaFreeHost(s->hV);
  ckv_cache_destroy(s->cache);
  if (s->l2_persist) l2_persist_release(s->ctx->device);
  delete s;
  return CKV_OK;
}

int ckv_session_kv(ckv_session* s, uint16_t** K, uint16_t** V, uint32_t* p_cap) {
  *K = s->K;
  *V = s->V;
  *p_cap = s->p_cap;
  return CKV_OK;
}

int ckv_session_load_prompt(ckv_session* s, const uint16_t* Kh, const uint16_t* Vh) {
  const size_t row = size_t(s->d.prompt_len) * D * 2;
  CKV_CUDA_TRY(cudaMemcpy2DAsync(s->K, size_t(s->p_cap) * D * 2, Kh, row, row, s->U,
                                 cudaMemcpyHostToDevice, s->ctx->stream));
  CKV_CUDA_TRY(cudaMemcpy2DAsync(s->V, size_t(s->p_cap) * D * 2, Vh, row, row, s->U,
                                 cudaMemcpyHostToDevice, s->ctx->stream));
  CKV_CUDA_TRY(cudaStreamSynchronize(s->ctx->stream));
  return CKV_OK;
}

int ckv_session_prefill(ckv_session* s, ckv_kmeans_info* info) {
  s->sel_early = false;  // the prefill writes the centroids and the index
  ckv_prefill_desc pd{};
  pd.n_units = s->U;
  pd.L = s->d.prompt_len;
  pd.p_cap = s->p_cap;
  pd.c_cap = s->c_cap;
  pd.c0_divisor = s->d.c0_divisor;
  pd.sink_tokens = s->d.sink_tokens;
  pd.max_iters = s->d.max_iters;
  pd.c0_override = s->d.c0_override;
  pd.flags = s->d.flags;
  // CKV_DEBUG_TIMING=1: host wall time of the three phases on stderr
  static const bool dbg = getenv("CKV_DEBUG_TIMING") != nullptr;
  auto now = [&]() {
    if (dbg) cudaStreamSynchronize(s->ctx->stream);
    return std::chrono::steady_clock::now();
  };
  const auto t0 = now();
  CKV_TRY(ckv_cluster_prefill(s->ctx, &pd, s->K, s->seeds.data(), s->cents, s->labels,
                              s->n_clusters, info, nullptr, nullptr));
  const auto t1 = now();
  s->C_cur = ckv_prefill_cluster_count(pd.L, pd.c0_divisor, pd.sink_tokens, pd.c0_override);
  CKV_TRY(ckv_build_index(s->ctx, s->U, s->labeled_end, s->p_cap, s->c_cap, s->labels,
                          s->n_clusters, s->sizes, s->starts, s->sorted));
  const auto t2 = now();
  // relay the KV store cluster-major: row sink + j <- position sorted[j]
  const uint32_t sink = std::min(s->d.sink_tokens, s->d.prompt_len);
  const uint32_t N = s->labeled_end - sink;
  if (N > 0)  // in place (bounded staging), so the store is never held twice
    CKV_TRY(ckv_relayout_kv(s->ctx, s->U, s->p_cap, s->K, s->V, s->K, s->V, s->sorted, sink,
                            s->labeled_end, s->n_ctx));
  if (s->tiered) {
    CKV_TRY(launch_tier_init(s->ctx->stream, s->tier, s->U));
    if (s->hK) {  // the clustered store to the host tier
      const size_t bytes = size_t(s->U) * s->p_cap * D * 2;
      CKV_CUDA_TRY(cudaMemcpyAsync(s->hK, s->K, bytes, cudaMemcpyDeviceToHost, s->ctx->stream));
      CKV_CUDA_TRY(cudaMemcpyAsync(s->hV, s->V, bytes, cudaMemcpyDeviceToHost, s->ctx->stream));
    }
  }
  s->prefilled = true;
  s->c16_dirty = true;
  const int rc = ckv_ctx_sync(s->ctx);
  if (dbg) {
    const auto t3 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "[session prefill] kmeans %.2f ms, index %.2f ms, relayout %.2f ms\n",
            ms(t0, t1), ms(t1, t2), ms(t2, t3));
  }
  return rc;
}

// select + attend of units [u0, u0 + nu) (all offsets are per unit / per q
// head, so a slice is a sub-session).  q_copy: when q is mapped host memory,
// the selection leaves a device copy of it there and the attention reads that
// (its bulk copies stay on HBM).  The two halves take a stream each so the
// batched step can overlap one slice's selection with another's attention.
static bool session_no_early() {
  static const bool off = getenv("CKV_SESSION_NO_EARLY") != nullptr;
  return off;
}

// CKV_SESSION_NO_FOLD_APPEND=1: the append kernel copies the new K/V rows
// (instead of the fused selection)
static bool session_no_fold_append() {
  static const bool v = getenv("CKV_SESSION_NO_FOLD_APPEND") != nullptr;
  return v;
}
static bool session_no_stepsync() {
  static const bool off = getenv("CKV_SESSION_NO_STEPSYNC") != nullptr;
  return off;
}

static int session_select_slice(ckv_session* s, cudaStream_t st, uint32_t u0, uint32_t nu,
                                const float* q_dev, float* q_copy, bool force_fused,
                                StepSync* sync = nullptr) {
  const uint32_t G = s->d.group, h0 = u0 * G;
  ckv_select_desc sd{};
  sd.n_q = nu * G;
  sd.group = G;
  sd.budget = s->d.budget;
  sd.sink_count = std::min(s->d.sink_tokens, s->d.prompt_len);
  sd.p_cap = s->p_cap;
  sd.c_cap = s->c_cap;
  sd.sel_cap = s->sel_cap;
  sd.rec_begin = s->labeled_end;
  sd.rec_end = s->n_ctx;
  sd.flags = (s->d.flags & CKV_SESSION_L2_PERSIST) ? CKV_SEL_L2_PERSIST : 0u;
  if (force_fused) sd.flags |= CKV_SEL_FORCE_FUSED;
  if (s->step_early) sd.flags |= CKV_SEL_EARLY;
  sd.row_base = sd.sink_count;
  const bool want_ids = (s->d.flags & CKV_SESSION_TOKEN_IDS) != 0;
  ckv_runs runs = s->runs;
  runs.row += size_t(h0) * runs.run_cap;
  runs.off += size_t(h0) * (runs.run_cap + 1);
  runs.count += h0;
  CacheDev cache = s->cache ? s->cache->dev : null_cache();
  if (cache.bits) {
    cache.bits += size_t(h0) * cache.retention * cache.words;
    cache.ring += size_t(h0) * 2;
    cache.counters += size_t(h0) * 4;
    cache.n_slots = sd.n_q;
  }
  const float* qs = q_dev + size_t(h0) * D;
  float* qc = q_copy ? q_copy + size_t(h0) * D : nullptr;
  StepSync ls;  // the slice's flags (q heads from h0)
  if (sync) {
    ls = *sync;
    ls.ready += h0;
    if (s->app_k) {  // this slice's units append their new rows
      ls.app_k = s->app_k + size_t(u0) * D;
      ls.app_v = s->app_v + size_t(u0) * D;
      ls.K = s->K + size_t(u0) * s->p_cap * D;
      ls.V = s->V + size_t(u0) * s->p_cap * D;
      ls.app_pos = s->n_ctx;
      ls.p_cap = s->p_cap;
    }
  }
  const SelC16 hc{s->use_c16 ? s->c16 + size_t(u0) * s->c_cap * D : nullptr,
                  s->use_c16 ? s->cerr + size_t(u0) * s->c_cap : nullptr};
  CKV_TRY(launch_select(st, sd, qs, s->cents + size_t(u0) * s->c_cap * D,
                        s->n_clusters + u0, s->sizes + size_t(u0) * s->c_cap,
                        s->starts + size_t(u0) * (s->c_cap + 1), s->sorted + size_t(u0) * s->p_cap,
                        want_ids ? s->token_ids + size_t(h0) * s->sel_cap : nullptr, nullptr, runs,
                        sd.row_base, s->n_tokens + h0, s->n_taken + h0, s->trimmed + h0,
                        s->ranked + size_t(h0) * s->c_cap, nullptr, cache, s->sel_scratch, qc,
                        sync ? &ls : nullptr, s->use_c16 ? &hc : nullptr));
  if (sync) {
    sync->published = ls.published;
    s->app_done = s->app_done && ls.appended;
  } else {
    s->app_done = false;
  }
  s->ctx->launches += 2;
  return CKV_OK;
}

static int session_attend_slice(ckv_session* s, cudaStream_t st, uint32_t u0, uint32_t nu,
                                const float* q_dev, float* out_dev, float* q_copy,
                                const StepSync* sync = nullptr) {
  const uint32_t G = s->d.group, h0 = u0 * G;
  const uint32_t sink = std::min(s->d.sink_tokens, s->d.prompt_len);
  ckv_runs runs = s->runs;
  runs.row += size_t(h0) * runs.run_cap;
  runs.off += size_t(h0) * (runs.run_cap + 1);
  runs.count += h0;
  const float* qs = q_dev + size_t(h0) * D;
  float* qc = q_copy ? q_copy + size_t(h0) * D : nullptr;
  ckv_attend_desc ad{};
  ad.n_q = nu * G;
  ad.group = G;
  ad.p_cap = s->p_cap;
  ad.sel_cap = s->sel_cap;
  ad.max_tokens = std::min(s->d.budget, s->labeled_end) + sink + (s->n_ctx - s->labeled_end);
  if (s->tiered) {  // misses backing -> page pool; the attention reads page runs
    ckv_runs tr = s->truns;
    tr.row += size_t(h0) * tr.run_cap;
    tr.off += size_t(h0) * (tr.run_cap + 1);
    tr.count += h0;
    CKV_TRY(launch_tier_fetch(st, s->tier, u0, nu, s->steps, runs, tr,
                              s->ranked + size_t(h0) * s->c_cap, s->n_taken + h0, s->K, s->V));
    s->ctx->launches++;
    runs = tr;
  }
  StepSync ls;
  if (sync) {
    ls = *sync;
    ls.ready += h0;
    if (ls.work) ls.work += u0;  // one counter per slice (first unit)
  }
  CKV_TRY(launch_attend(st, ad, qc ? qc : qs, s->K + size_t(u0) * s->p_cap * D,
                        s->V + size_t(u0) * s->p_cap * D, nullptr, runs, s->n_tokens + h0,
                        out_dev + size_t(h0) * D, nullptr, nullptr, s->part, s->tickets,
                        nullptr, sync ? &ls : nullptr));
  s->ctx->launches++;
  return CKV_OK;
}

// one step's select + attend: every unit in one launch pair, or (layer mode,
// ckv_session_set_layer_units) one pair per layer slice in layer order — the
// dependency order of a model, where layer l+1's queries need layer l's output.
// CKV_SESSION_SPLIT=1 (experiment, off): batched mode splits the units in
// two (the first 1/8 and the rest) and runs the large slice's selection on a
// second stream beside the small slice's attention, to overlap the
// selection's latency tail with HBM work.  Measured slower at config B (144
// vs 120 us/step: the concurrent kernels contend and the small attention
// lands on the critical path).  Every attention follows its own selection;
// the two attentions share the split-K scratch, so they run in order.
static int session_select_attend(ckv_session* s, const float* q_dev, float* out_dev,
                                 float* q_copy = nullptr) {
  cudaStream_t st = s->ctx->stream;
  if (s->use_c16 && (s->c16_dirty || s->c16_tail)) {  // centroids changed since the last selection
    CKV_TRY(launch_cents_f16(st, s->cents, s->n_clusters, s->U, s->c_cap, s->c16, s->cerr,
                             s->c16_dirty ? 0u : s->c16_tail));
    s->ctx->launches++;
    s->c16_dirty = false;
    s->c16_tail = 0;
    s->step_early = false;  // the selection reads what this kernel writes
  }
  const uint32_t lu = s->layer_units;
  if (lu == 0 || lu >= s->U) {
    static const bool split = getenv("CKV_SESSION_SPLIT") != nullptr;
    const uint32_t u1 = s->U / 8;
    if (!split || s->tiered || !s->sel_stream || u1 < 8) {
      // StepSync: the attention starts on each q head as soon as its
      // selection is published, overlapping the selection's tail (not with
      // the tier fetch between them)
      StepSync* sy = nullptr;
      if (!session_no_stepsync() && !s->tiered) {
        s->sync.ready = s->step_ready;
        s->sync.epoch = s->step_epoch;
        s->sync.work = s->step_work;
        sy = &s->sync;
      }
      CKV_TRY(session_select_slice(s, st, 0, s->U, q_dev, q_copy, false, sy));
      return session_attend_slice(s, st, 0, s->U, q_dev, out_dev, q_copy, sy);
    }
    CKV_CUDA_TRY(cudaEventRecord(s->ev_sel_fork, st));
    CKV_CUDA_TRY(cudaStreamWaitEvent(s->sel_stream, s->ev_sel_fork, 0));
    CKV_TRY(session_select_slice(s, s->sel_stream, u1, s->U - u1, q_dev, q_copy, true));
    CKV_CUDA_TRY(cudaEventRecord(s->ev_sel_join, s->sel_stream));
    CKV_TRY(session_select_slice(s, st, 0, u1, q_dev, q_copy, true));
    CKV_TRY(session_attend_slice(s, st, 0, u1, q_dev, out_dev, q_copy));
    CKV_CUDA_TRY(cudaStreamWaitEvent(st, s->ev_sel_join, 0));
    return session_attend_slice(s, st, u1, s->U - u1, q_dev, out_dev, q_copy);
  }
  // layer slices: disjoint q heads, so one epoch per step serves them all
  StepSync* sy = nullptr;
  if (!session_no_stepsync() && !s->tiered) {
    s->sync.ready = s->step_ready;
    s->sync.epoch = s->step_epoch;
    s->sync.work = nullptr;  // layer slices: the fixed item stride (measured faster here)
    sy = &s->sync;
  }
  for (uint32_t u0 = 0; u0 < s->U; u0 += lu) {
    const uint32_t nu = std::min(lu, s->U - u0);
    CKV_TRY(session_select_slice(s, st, u0, nu, q_dev, q_copy, false, sy));
    CKV_TRY(session_attend_slice(s, st, u0, nu, q_dev, out_dev, q_copy, sy));
  }
  return CKV_OK;
}

int ckv_session_set_layer_units(ckv_session* s, uint32_t layer_units) {
  if (layer_units && s->U % layer_units) {
    set_error("ckv_session_set_layer_units: must divide n_units");
    return CKV_EINVAL;
  }
  s->layer_units = layer_units;
  return CKV_OK;
}

int ckv_session_attend_only(ckv_session* s, const float* q_dev, float* out_dev) {
  if (!s->prefilled) { set_error("session: prefill first"); return CKV_EINVAL; }
  CKV_TRY(session_select_attend(s, q_dev, out_dev));
  // no append follows: advance the StepSync epoch here
  s->sel_early = false;
  k_epoch_advance<<<1, 256, 0, s->ctx->stream>>>(s->step_epoch, s->step_work, s->U);
  CKV_LAUNCH_CHECK("k_epoch_advance");
  s->ctx->launches++;
  return CKV_OK;
}

// The decode-batch k-means reports kmeans_cosine's input errors
// (clustering.hpp:166-172) through a status word copied to pinned host memory
// behind an event; it is read when the event has completed (the next step
// that finds it done, or blocking at stats / destroy), so the decode path
// never waits on it.  A failed batch poisons the session (CKV_EINVAL from
// then on), the way the reference's cluster_decode_batch throws.
static int session_check_status(ckv_session* s, bool block) {
  if (!s->stat_pending) return CKV_OK;
  if (block) {
    CKV_CUDA_TRY(cudaEventSynchronize(s->ev_stat));
  } else {
    const cudaError_t e = cudaEventQuery(s->ev_stat);
    if (e == cudaErrorNotReady) return CKV_OK;
    if (e != cudaSuccess) return cuda_status(e, "session decode-batch status");
  }
  s->stat_pending = false;
  for (uint32_t u = 0; u < s->U; ++u) {
    const int32_t st = s->h_stat[s->U + u];
    if (st == 1) { set_error("kmeans: keys must be finite"); s->prefilled = false; return CKV_EINVAL; }
    if (st == 2) {
      set_error("kmeans: degenerate input, all keys zero-norm");
      s->prefilled = false;
      return CKV_EINVAL;
    }
  }
  return CKV_OK;
}

// cluster_decode_batch (clustering.hpp:310-332) of every unit's rows
// [pos0, pos0 + m) on stream st: init rows and the whole k-means on the
// device (centroids at ncl[u], labels +ncl[u], ncl[u] += C), no host work
static int session_cluster_batch(ckv_session* s, cudaStream_t st, uint32_t pos0, uint32_t m,
                                 uint32_t* ncl) {
  const uint32_t C = std::min(s->d.c_plus, m);
  CKV_TRY(session_check_status(s, true));  // the previous batch's (long finished)
  CKV_TRY(launch_decode_init_rows(st, s->d_seeds, s->U, pos0, m, C, s->db_init));
  CKV_TRY(launch_kmeans_small(st, s->K + size_t(pos0) * D, uint64_t(s->p_cap) * D, s->U, m, C,
                              s->d.max_iters, s->db_init, s->cents, s->c_cap, s->labels + pos0,
                              s->p_cap, ncl, reinterpret_cast<uint32_t*>(s->db_stat),
                              s->db_stat + s->U));
  CKV_CUDA_TRY(cudaMemcpyAsync(s->h_stat, s->db_stat, 8 * size_t(s->U), cudaMemcpyDeviceToHost,
                               st));
  CKV_CUDA_TRY(cudaEventRecord(s->ev_stat, st));
  s->stat_pending = true;
  s->n_batches++;
  s->ctx->launches += 2;
  return CKV_OK;
}

// the clustered batch joins the model: index entries appended, the batch's
// K/V rows re-laid cluster-major, n_clusters published (k_batch_commit)
static int session_commit_batch(ckv_session* s, uint32_t pos0, uint32_t m, uint32_t C,
                                const uint32_t* ncl_src) {
  cudaStream_t st = s->ctx->stream;
  const uint32_t sink = std::min(s->d.sink_tokens, s->d.prompt_len);
  if (pos0 != s->labeled_end) { set_error("session: batch commit out of order"); return CKV_EINVAL; }
  k_batch_commit<<<s->U, BC_THREADS, 0, st>>>(s->K, s->V, s->tmpK, s->tmpV, s->labels, s->p_cap,
                                              s->c_cap, sink, pos0, m, C, ncl_src, s->n_clusters,
                                              s->sizes, s->starts, s->sorted);
  CKV_LAUNCH_CHECK("k_batch_commit");
  s->ctx->launches++;
  if (s->hK) {  // the re-laid batch rows join the host tier
    const size_t pitch = size_t(s->p_cap) * D * 2, w = size_t(m) * D * 2, o = size_t(pos0) * D;
    CKV_CUDA_TRY(cudaMemcpy2DAsync(s->hK + o, pitch, s->K + o, pitch, w, s->U,
                                   cudaMemcpyDeviceToHost, st));
    CKV_CUDA_TRY(cudaMemcpy2DAsync(s->hV + o, pitch, s->V + o, pitch, w, s->U,
                                   cudaMemcpyDeviceToHost, st));
  }
  s->labeled_end += m;
  s->C_cur += C;
  s->c16_tail += C;  // the batch's centroids are each unit's last C rows
  return CKV_OK;
}

int ckv_session_step(ckv_session* s, const float* q, const uint16_t* kn, const uint16_t* vn,
                     float* out, int on_device) {
  if (!s->prefilled) { set_error("session: prefill first (or a failed decode batch)"); return CKV_EINVAL; }
  if (s->n_ctx >= s->p_cap) { set_error("session: decode capacity exhausted"); return CKV_EINVAL; }
  CKV_TRY(session_check_status(s, false));
  cudaStream_t st = s->ctx->stream;
  // async mode: batches whose delay has run out join before this step's
  // selection (harness.hpp:237-243)
  bool early = s->sel_early && !session_no_early();
  s->sel_early = false;
  while (!s->queue.empty() && s->queue.front().ready <= s->steps) {
    const auto b = s->queue.front();
    CKV_CUDA_TRY(cudaStreamWaitEvent(st, s->ev_done, 0));
    CKV_TRY(session_commit_batch(s, b.pos0, b.rows, b.C, s->stage_ncl));
    s->queue.pop_front();
    early = false;  // the commit wrote the centroids and the index
  }
  const float* qd = q;
  const uint16_t *kd = kn, *vd = vn;
  float* od = out;
  float* q_copy = nullptr;
  bool zero_copy = false;
  if (!on_device) {
    // pinned (page-locked, device-mapped) host buffers are read and written
    // by the kernels in place over PCIe: the selection reads q and leaves a
    // device copy, the attention writes out, the append reads the new k/v;
    // no copy-engine transfers or their latencies on the step's path.
    // Pageable buffers take the staged copies.
    auto mapped = [](const void* p) -> const void* {
      cudaPointerAttributes a{};
      if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return nullptr; }
      return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
    };
    const void *mq = mapped(q), *mk = mapped(kn), *mv = mapped(vn), *mo = mapped(out);
    zero_copy = mq && mk && mv && mo && mq == q && mk == kn && mv == vn && mo == out;
    if (zero_copy) {
      q_copy = s->q_dev;
    } else {
      CKV_CUDA_TRY(cudaMemcpyAsync(s->q_dev, q, size_t(s->n_q) * D * 4, cudaMemcpyHostToDevice, st));
      CKV_CUDA_TRY(cudaMemcpyAsync(s->kn_dev, kn, size_t(s->U) * D * 2, cudaMemcpyHostToDevice, st));
      CKV_CUDA_TRY(cudaMemcpyAsync(s->vn_dev, vn, size_t(s->U) * D * 2, cudaMemcpyHostToDevice, st));
      qd = s->q_dev;
      kd = s->kn_dev;
      vd = s->vn_dev;
      od = s->out_dev;
    }
  }
  s->step_early = early;
  // the fused selection copies the new K/V rows when every slice takes them
  s->app_k = session_no_fold_append() ? nullptr : kd;
  s->app_v = vd;
  s->app_done = s->app_k != nullptr;
  const int rc_sa = session_select_attend(s, qd, od, q_copy);
  s->step_early = false;
  s->app_k = s->app_v = nullptr;
  CKV_TRY(rc_sa);
  const bool appended = s->app_done;
  // append this step's token (harness.hpp:318-320), unless the selection did;
  // the kernel still advances the StepSync epoch and zeroes the work counters
  k_append_kv<<<s->U, 16, 0, st>>>(appended ? nullptr : kd, vd, s->K, s->V, s->n_ctx, s->p_cap,
                                   s->step_epoch, s->step_work);
  CKV_LAUNCH_CHECK("k_append_kv");
  s->ctx->launches++;
  s->n_ctx++;
  s->pending++;
  s->steps++;
  s->sel_early = true;  // cleared below if a synchronous decode batch follows
  if (s->pending == s->d.decode_batch) {  // harness.hpp:321-336
    const uint32_t m = s->pending, pos0 = s->pend_pos0;
    const uint32_t C = std::min(s->d.c_plus, m);
    s->pending = 0;
    s->pend_pos0 += m;
    if (s->d.async_delay) {
      // the k-means on the side stream, from n_clusters as it stands (no
      // other batch commits before this one), into a staging copy of it
      CKV_CUDA_TRY(cudaEventRecord(s->ev_fork, st));
      CKV_CUDA_TRY(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
      CKV_CUDA_TRY(cudaMemcpyAsync(s->stage_ncl, s->n_clusters, 4 * size_t(s->U),
                                   cudaMemcpyDeviceToDevice, s->side));
      CKV_TRY(session_cluster_batch(s, s->side, pos0, m, s->stage_ncl));
      CKV_CUDA_TRY(cudaEventRecord(s->ev_done, s->side));
      s->queue.push_back({s->steps - 1 + s->d.async_delay, pos0, m, C});
    } else if (kmeans_small_supported(m, C) && m <= uint32_t(BC_THREADS)) {
      s->sel_early = false;
      CKV_TRY(session_cluster_batch(s, st, pos0, m, s->n_clusters));
      CKV_TRY(session_commit_batch(s, pos0, m, C, s->n_clusters));
    } else {  // large batches: the generic driver, full index, staged relayout
      s->sel_early = false;
      ckv_decode_cluster_desc dd{};
      dd.n_units = s->U;
      dd.pos0 = pos0;
      dd.rows = m;
      dd.p_cap = s->p_cap;
      dd.c_cap = s->c_cap;
      dd.c_plus = s->d.c_plus;
      dd.max_iters = s->d.max_iters;
      CKV_TRY(ckv_cluster_decode_batch(s->ctx, &dd, s->K, s->seeds.data(), s->cents, s->labels,
                                       s->n_clusters, nullptr));
      s->labeled_end += m;
      s->C_cur += C;
      s->c16_dirty = true;
      CKV_TRY(ckv_build_index(s->ctx, s->U, s->labeled_end, s->p_cap, s->c_cap, s->labels,
                              s->n_clusters, s->sizes, s->starts, s->sorted));
      const uint32_t sink = std::min(s->d.sink_tokens, s->d.prompt_len);
      k_relayout_batch<<<s->U, 256, 0, st>>>(s->K, s->V, s->tmpK, s->tmpV, s->sorted, s->p_cap,
                                             sink, pos0, m);
      CKV_LAUNCH_CHECK("k_relayout_batch");
      s->ctx->launches++;
    }
  }
  if (!on_device) {
    if (!zero_copy)
      CKV_CUDA_TRY(cudaMemcpyAsync(out, s->out_dev, size_t(s->n_q) * D * 4,
                                   cudaMemcpyDeviceToHost, st));
    CKV_CUDA_TRY(cudaStreamSynchronize(st));
  }
  return CKV_OK;
}

int ckv_session_stats_get(ckv_session* s, ckv_session_stats* st) {
  CKV_TRY(session_check_status(s, true));
  st->n_ctx = s->n_ctx;
  st->labeled_end = s->labeled_end;
  st->steps = s->steps;
  st->max_clusters = s->C_cur;
  st->launches = s->ctx->launches;
  return CKV_OK;
}

int ckv_session_state(ckv_session* s, float** cents, int32_t** labels, uint32_t** n_clusters,
                      uint32_t** sizes, uint32_t** starts, uint32_t** sorted,
                      uint32_t** token_ids, uint32_t** n_tokens, uint32_t* c_cap,
                      uint32_t* sel_cap) {
  if (cents) *cents = s->cents;
  if (labels) *labels = s->labels;
  if (n_clusters) *n_clusters = s->n_clusters;
  if (sizes) *sizes = s->sizes;
  if (starts) *starts = s->starts;
  if (sorted) *sorted = s->sorted;
  if (token_ids) *token_ids = s->token_ids;
  if (n_tokens) *n_tokens = s->n_tokens;
  if (c_cap) *c_cap = s->c_cap;
  if (sel_cap) *sel_cap = s->sel_cap;
  return CKV_OK;
}

int ckv_session_batch_iterations(ckv_session* s, uint32_t* iterations_host) {
  if (s->n_batches == 0) { set_error("session: no decode batch yet"); return CKV_EINVAL; }
  CKV_TRY(session_check_status(s, true));
  for (uint32_t u = 0; u < s->U; ++u)
    iterations_host[u] = uint32_t(s->h_stat[u]) & 0x7fffffffu;
  return CKV_OK;
}

ckv_cache* ckv_session_cache(ckv_session* s) { return s->cache; }

int ckv_session_tier_stats(ckv_session* s, uint64_t* out) {
  if (!s->tiered) { set_error("session: not tiered"); return CKV_EINVAL; }
  std::vector<unsigned long long> st(size_t(s->U) * 4);
  int32_t status = 0;
  CKV_CUDA_TRY(cudaMemcpyAsync(st.data(), s->tier.stats, st.size() * 8, cudaMemcpyDeviceToHost,
                               s->ctx->stream));
  CKV_CUDA_TRY(cudaMemcpyAsync(&status, s->tier.status, 4, cudaMemcpyDeviceToHost, s->ctx->stream));
  CKV_CUDA_TRY(cudaStreamSynchronize(s->ctx->stream));
  if (status) { set_error("session: tier page pool exhausted"); return CKV_EINVAL; }
  for (int k = 0; k < 4; ++k) out[k] = 0;
  for (uint32_t u = 0; u < s->U; ++u)
    for (int k = 0; k < 4; ++k) out[k] += st[size_t(u) * 4 + k];
  out[4] = uint64_t(s->tier.np) * TIER_PAGE_ROWS;  // pool rows per unit
  return CKV_OK;
}

}  // extern "C"

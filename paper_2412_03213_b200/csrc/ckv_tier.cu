// ckv_tier.cu — the physical two-tier cluster-granular KV cache (SURVEY §8f
// row 1; cache.hpp:25-93; the paper's offloaded KV with GPU-resident recently
// selected clusters).
//
// Backing tier: the cluster-major KV store, either the device store itself
// (secondary HBM) or a host-pinned, device-mapped mirror of it (the offload
// setting: every miss is a PCIe read).  Primary tier: a per-unit pool of
// 16-row pages in HBM, after all units' store rows in the same allocation,
// so the attention reads pool pages through ordinary run lists.
//
// k_tier_fetch runs between the selection and the attention of a step, one
// CTA per unit:
//   1. the clusters the unit's q heads took this step (union);
//   2. eviction: resident clusters not selected in the last R steps give
//      their pages back (R = the session's cache retention, applied per unit
//      — the reference's resident set is per q head, cache.hpp:38-57; its
//      counters stay bit-exact in the selection kernel, this is the physical
//      residency serving them);
//   3. allocation: each selected, non-resident cluster gets ceil(size/16)
//      pages (a page chain) off the unit's free stack; if the pool runs dry,
//      every resident cluster not selected this step is evicted first;
//   4. the misses' rows are copied backing -> pool (whole clusters, as the
//      reference charges them, cache.hpp:48-50), 16-B loads, all in flight;
//   5. each head's cluster runs are rewritten into page runs (same rows in
//      the same order, so the attention output is bit-identical).
// Physical counters per unit: rows and clusters fetched, clusters hit.
#include "ckv_internal.cuh"

namespace ckvb {
namespace {

constexpr int TF_THREADS = 256;
constexpr uint32_t TF_PAGE = TIER_PAGE_ROWS;

// pool row (relative to unit u's store base) of page p, slot s
__device__ __forceinline__ uint32_t pool_row(uint32_t u, uint32_t U, uint32_t p_cap,
                                             uint32_t np, uint32_t page, uint32_t slot) {
  return (U - u) * p_cap + u * np * TF_PAGE + page * TF_PAGE + slot;
}

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp,
                                                    uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < TF_THREADS / 32 ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < TF_THREADS / 32) s_warp[lane] = w;
  }
  __syncthreads();
  const uint32_t base = (wid ? s_warp[wid - 1] : 0u) + x - v;
  *total = s_warp[TF_THREADS / 32 - 1];
  __syncthreads();
  return base;
}

__global__ void __launch_bounds__(TF_THREADS)
k_tier_fetch(TierArgs a, uint32_t u0, uint32_t step, ckv_runs runs, ckv_runs out,
             const uint32_t* __restrict__ ranked, const uint32_t* __restrict__ n_taken,
             uint16_t* __restrict__ K, uint16_t* __restrict__ V) {
  extern __shared__ __align__(16) uint32_t tf_sm[];
  const uint32_t u = u0 + blockIdx.x;  // global unit
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t C = a.n_clusters[u], W = (a.c_cap + 31) / 32;
  uint32_t* sel = tf_sm;                 // [W] selected bitmap
  uint32_t* mbase = sel + W;             // [c_cap + 1] page base of each missing cluster
  uint32_t* rbase = mbase + a.c_cap + 1; // [c_cap + 1] row prefix of the missing clusters
  uint16_t* mlist = reinterpret_cast<uint16_t*>(rbase + a.c_cap + 1);  // [c_cap]
  __shared__ uint32_t s_warp[TF_THREADS / 32], s_nmiss, s_force, s_fail;
  __shared__ int32_t s_nfree;
  int32_t* cpage = a.cpage + size_t(u) * a.c_cap;
  uint32_t* last = a.last + size_t(u) * a.c_cap;
  int32_t* next = a.next + size_t(u) * a.np;
  int32_t* fstack = a.free_stack + size_t(u) * a.np;
  const uint32_t* sz = a.sizes + size_t(u) * a.c_cap;
  const uint32_t* st = a.starts + size_t(u) * (a.c_cap + 1);
  // runs / ranked / n_taken are the launch's (a slice in layer mode): its
  // q heads are blockIdx.x * group + g; metadata and K/V are global by unit
  const uint32_t hq0 = blockIdx.x * a.group;

  // ---- 1. this step's clusters (union over the unit's q heads) -------------
  for (uint32_t i = tid; i < W; i += TF_THREADS) sel[i] = 0u;
  if (tid == 0) { s_nfree = a.n_free[u]; s_force = 0; s_fail = 0; }
  __syncthreads();
  for (uint32_t g = 0; g < a.group; ++g) {
    const uint32_t h = hq0 + g, nt = n_taken[h];
    for (uint32_t i = tid; i < nt; i += TF_THREADS) {
      const uint32_t c = ranked[size_t(h) * a.c_cap + i];
      atomicOr(&sel[c >> 5], 1u << (c & 31));
    }
  }
  __syncthreads();
  auto is_sel = [&](uint32_t c) { return (sel[c >> 5] >> (c & 31)) & 1u; };
  // ---- 2. eviction -----------------------------------------------------------
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1 && !s_force) break;
    for (uint32_t c = tid; c < C; c += TF_THREADS) {
      const int32_t p0 = cpage[c];
      if (p0 < 0 || is_sel(c)) continue;
      if (pass == 0 && last[c] + a.retention > step) continue;  // still in the window
      const uint32_t np = (sz[c] + TF_PAGE - 1) / TF_PAGE;
      const int32_t at = atomicAdd(&s_nfree, int32_t(np));
      int32_t p = p0;
      for (uint32_t k = 0; k < np; ++k) { fstack[at + k] = p; p = next[p]; }
      cpage[c] = -1;
      atomicAdd(&a.stats[size_t(u) * 4 + 3], 1ull);  // evictions
    }
    __syncthreads();
    // ---- 3. pages for the selected, non-resident clusters --------------------
    const uint32_t per = (C + TF_THREADS - 1) / TF_THREADS;
    const uint32_t c0 = min(C, tid * per), c1 = min(C, c0 + per);
    uint32_t need = 0, nm = 0, rows = 0;
    for (uint32_t c = c0; c < c1; ++c)
      if (is_sel(c) && cpage[c] < 0) {
        need += (sz[c] + TF_PAGE - 1) / TF_PAGE;
        rows += sz[c];
        ++nm;
      }
    uint32_t tot_need, tot_m, tot_rows;
    uint32_t pb = block_excl_scan(need, s_warp, &tot_need);
    uint32_t mb = block_excl_scan(nm, s_warp, &tot_m);
    uint32_t rb = block_excl_scan(rows, s_warp, &tot_rows);
    if (tot_need > uint32_t(s_nfree)) {
      if (pass == 0) {
        if (tid == 0) s_force = 1;
        __syncthreads();
        continue;  // evict everything not selected now, then retry
      }
      if (tid == 0) { s_fail = 1; atomicExch(a.status, 1); }
      __syncthreads();
      break;
    }
    // pop tot_need pages off the stack top; cluster k takes its slice
    const int32_t top = s_nfree - int32_t(tot_need);
    for (uint32_t c = c0; c < c1; ++c) {
      if (!(is_sel(c) && cpage[c] < 0)) continue;
      const uint32_t np = (sz[c] + TF_PAGE - 1) / TF_PAGE;
      for (uint32_t k = 0; k < np; ++k) {
        const int32_t p = fstack[top + int32_t(pb + k)];
        next[p] = k + 1 < np ? fstack[top + int32_t(pb + k + 1)] : -1;
      }
      mlist[mb] = uint16_t(c);
      mbase[mb] = uint32_t(top) + pb;
      rbase[mb] = rb;
      pb += np;
      rb += sz[c];
      ++mb;
    }
    if (tid == 0) { s_nmiss = tot_m; rbase[tot_m] = tot_rows; }
    __syncthreads();
    // ---- 4. copy the misses' rows backing -> pool ------------------------------
    const uint32_t nmiss = s_nmiss, nchunk = tot_rows * 16;  // 16-B chunks per row: 16
    const uint16_t* bK = a.back_K + size_t(u) * a.p_cap * D;
    const uint16_t* bV = a.back_V + size_t(u) * a.p_cap * D;
    uint16_t* dK = K + size_t(u) * a.p_cap * D;
    uint16_t* dV = V + size_t(u) * a.p_cap * D;
    for (uint32_t e0 = tid; e0 < nchunk; e0 += TF_THREADS * 4) {
      uint4 xk[4], xv[4];
      uint32_t dst[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t e = e0 + j * TF_THREADS;
        dst[j] = ~0u;
        if (e >= nchunk) continue;
        const uint32_t r = e >> 4, q = e & 15;
        uint32_t lo = 0, hi = nmiss;  // missing cluster holding flat row r
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (rbase[mid] <= r) lo = mid; else hi = mid;
        }
        const uint32_t c = mlist[lo], rr = r - rbase[lo];
        const uint32_t page = uint32_t(fstack[mbase[lo] + rr / TF_PAGE]);
        const size_t src = (size_t(a.sink) + st[c] + rr) * D;
        xk[j] = __ldcs(reinterpret_cast<const uint4*>(bK + src) + q);
        xv[j] = __ldcs(reinterpret_cast<const uint4*>(bV + src) + q);
        dst[j] = pool_row(u, a.n_units_total, a.p_cap, a.np, page, rr % TF_PAGE) * 16 + q;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (dst[j] == ~0u) continue;
        reinterpret_cast<uint4*>(dK)[dst[j]] = xk[j];
        reinterpret_cast<uint4*>(dV)[dst[j]] = xv[j];
      }
    }
    // chains become visible to the run rewrite below
    for (uint32_t k = tid; k < nmiss; k += TF_THREADS) cpage[mlist[k]] = fstack[mbase[k]];
    if (tid == 0) {
      s_nfree = top;
      a.n_free[u] = top;
      atomicAdd(&a.stats[size_t(u) * 4 + 0], (unsigned long long)tot_rows);
      atomicAdd(&a.stats[size_t(u) * 4 + 1], (unsigned long long)tot_m);
    }
    __syncthreads();
    break;
  }
  if (s_fail) return;  // pool exhausted: the status word poisons the session
  // ---- 5. hits, recency of use ----------------------------------------------
  uint32_t hits = 0;
  for (uint32_t c = tid; c < C; c += TF_THREADS)
    if (is_sel(c)) { hits += 1; last[c] = step; }
  hits = warp_sum(hits);
  if (lane == 0) atomicAdd(&a.stats[size_t(u) * 4 + 2], (unsigned long long)hits);
  // (stats[2] counts selected clusters; hits = selected - fetched, on the host)
  __syncthreads();
  // ---- 6. cluster runs -> page runs (a separate list), one warp per head ----
  for (uint32_t g = wid; g < a.group; g += TF_THREADS / 32) {
    const uint32_t h = hq0 + g, nt = n_taken[h];
    const uint32_t* rr = runs.row + size_t(h) * runs.run_cap;
    const uint32_t* ro = runs.off + size_t(h) * (runs.run_cap + 1);
    uint32_t* wr = out.row + size_t(h) * out.run_cap;
    uint32_t* wo = out.off + size_t(h) * (out.run_cap + 1);
    const uint32_t nr = runs.count[h];
    // page runs of slice i: ceil(count_i / 16), in slice order; then the
    // rows outside the clusters (sinks, recency) as they were
    uint32_t carry = 0;
    for (uint32_t b = 0; b < nt; b += 32) {
      const uint32_t i = b + lane;
      uint32_t c = 0, off = 0, cnt = 0, npg = 0;
      if (i < nt) {
        c = ranked[size_t(h) * a.c_cap + i];
        off = ro[i];
        cnt = ro[i + 1] - off;
        npg = (cnt + TF_PAGE - 1) / TF_PAGE;
      }
      uint32_t x = npg;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t first = carry + x - npg;
      carry += __shfl_sync(0xffffffffu, x, 31);
      if (i < nt) {
        int32_t p = cpage[c];
        for (uint32_t k = 0; k < npg; ++k) {
          wr[first + k] = pool_row(u, a.n_units_total, a.p_cap, a.np, uint32_t(p), 0);
          wo[first + k] = off + k * TF_PAGE;
          p = next[p];
        }
      }
    }
    for (uint32_t k = nt + lane; k < nr; k += 32) {
      wr[carry + k - nt] = rr[k];
      wo[carry + k - nt] = ro[k];
    }
    if (lane == 0) {
      wo[carry + nr - nt] = ro[nr];
      out.count[h] = carry + nr - nt;
    }
  }
}

}  // namespace

int launch_tier_fetch(cudaStream_t st, const TierArgs& a, uint32_t u0, uint32_t n_units,
                      uint32_t step, const ckv_runs& runs, const ckv_runs& out,
                      const uint32_t* ranked, const uint32_t* n_taken, uint16_t* K,
                      uint16_t* V) {
  if (n_units == 0) return CKV_OK;
  const uint32_t W = (a.c_cap + 31) / 32;
  const size_t smem = size_t(W) * 4 + 2 * size_t(a.c_cap + 1) * 4 + size_t(a.c_cap) * 2 + 16;
  CKV_CUDA_TRY(smem_optin((const void*)k_tier_fetch, int(std::max<size_t>(smem, 48 * 1024))));
  k_tier_fetch<<<n_units, TF_THREADS, smem, st>>>(a, u0, step, runs, out, ranked, n_taken, K, V);
  CKV_LAUNCH_CHECK("k_tier_fetch");
  return CKV_OK;
}

__global__ void k_tier_init(TierArgs a, uint32_t n_units) {
  const uint32_t u = blockIdx.x;
  if (u >= n_units) return;
  for (uint32_t c = threadIdx.x; c < a.c_cap; c += blockDim.x) {
    a.cpage[size_t(u) * a.c_cap + c] = -1;
    a.last[size_t(u) * a.c_cap + c] = 0;
  }
  for (uint32_t p = threadIdx.x; p < a.np; p += blockDim.x) {
    a.free_stack[size_t(u) * a.np + p] = int32_t(a.np - 1 - p);
    a.next[size_t(u) * a.np + p] = -1;
  }
  if (threadIdx.x == 0) a.n_free[u] = int32_t(a.np);
  if (threadIdx.x < 4) a.stats[size_t(u) * 4 + threadIdx.x] = 0ull;
}

int launch_tier_init(cudaStream_t st, const TierArgs& a, uint32_t n_units) {
  k_tier_init<<<n_units, 256, 0, st>>>(a, n_units);
  CKV_LAUNCH_CHECK("k_tier_init");
  return CKV_OK;
}

}  // namespace ckvb

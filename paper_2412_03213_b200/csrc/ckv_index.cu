// ckv_index.cu — K5: stable counting sort of cluster labels into the
// ClusterIndex layout (selection.hpp:16-48 build_index).
//
// One CTA per unit.  W warps each own a contiguous segment of positions:
//   1. per-warp histograms hist[w][c] (smem atomics);
//   2. column scan: starts[c] = sum_{c'<c} size[c'], and per-warp write
//      cursors off[w][c] = starts[c] + sum_{w'<w} hist[w'][c] (columns in
//      parallel, the scan over clusters by one warp);
//   3. each warp walks its segment in order, 32 positions at a time, ranks
//      equal labels with __match_any_sync and scatters position ids.
// Warp w's ids precede warp w+1's for every cluster and each warp scatters
// in position order, so the sort is stable: identical to the reference's
// sequential cursor loop (selection.hpp:41-46), bit for bit.
//
// The same kernel produces the member lists and counts the k-means update
// needs (ckv_kmeans.cu) and, optionally, compares the labels against a
// previous assignment (the convergence test, clustering.hpp:252).
#include "ckv_internal.cuh"

namespace ckvb {

__global__ void __launch_bounds__(1024)
k_index(const int32_t* __restrict__ labels, uint32_t n_pos, uint32_t p_cap, uint32_t c_cap,
        const uint32_t* __restrict__ n_clusters, uint32_t c_uniform,
        uint32_t* __restrict__ sizes, uint32_t* __restrict__ starts,
        uint32_t* __restrict__ sorted_ids, const int32_t* __restrict__ prev_labels,
        int32_t* __restrict__ changed, const int32_t* __restrict__ active,
        int32_t* __restrict__ any_empty, uint8_t* __restrict__ dirty) {
  const uint32_t u = blockIdx.x;
  if (active && !active[u]) return;
  const uint32_t C = n_clusters ? n_clusters[u] : c_uniform;
  const int W = blockDim.x >> 5;
  const int w = warp_id(), lane = lane_id();
  extern __shared__ uint32_t sm[];
  uint32_t* hist = sm;                       // [W][C]
  __shared__ uint32_t s_total;
  __shared__ int s_changed, s_empty;

  const int32_t* lab = labels + size_t(u) * p_cap;
  for (uint32_t i = threadIdx.x; i < uint32_t(W) * C; i += blockDim.x) hist[i] = 0;
  // dirty[c]: cluster c's member set differs from the previous labels' (the
  // k-means update recomputes only those centroids; the others are
  // bit-identical by construction)
  uint8_t* dty = dirty ? dirty + size_t(u) * c_cap : nullptr;
  if (dty)
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) dty[c] = 0;
  if (threadIdx.x == 0) { s_changed = 0; s_empty = 0; }
  __syncthreads();

  const uint32_t seg = (n_pos + W - 1) / W;
  const uint32_t p0 = min(n_pos, seg * w), p1 = min(n_pos, p0 + seg);
  int my_changed = 0;
  const int32_t* prev = prev_labels ? prev_labels + size_t(u) * p_cap : nullptr;
  if (dty) __syncthreads();  // zeroed before any mark
  // IX_BATCH rounds of 32 labels (and previous labels) are loaded before
  // any is used, so a warp keeps that many loads in flight
  constexpr int IX_BATCH = 8;
  for (uint32_t p = p0 + lane; p < p1; p += 32 * IX_BATCH) {
    int32_t l[IX_BATCH], pv[IX_BATCH];
#pragma unroll
    for (int k = 0; k < IX_BATCH; ++k) {
      const uint32_t q = p + 32 * k;
      l[k] = q < p1 ? __ldg(lab + q) : -1;
      pv[k] = prev && q < p1 ? __ldg(prev + q) : -1;
    }
#pragma unroll
    for (int k = 0; k < IX_BATCH; ++k) {
      if (l[k] >= 0) atomicAdd(&hist[w * C + l[k]], 1u);
      if (prev && pv[k] != l[k]) {
        my_changed = 1;
        if (dty) {
          if (l[k] >= 0) dty[l[k]] = 1;
          if (pv[k] >= 0) dty[pv[k]] = 1;
        }
      }
    }
  }
  if (prev && __any_sync(0xffffffffu, my_changed) && lane == 0) s_changed = 1;
  __syncthreads();

  // column totals and intra-column offsets (every thread, one column at a
  // time), then the exclusive scan of the totals over clusters (warp 0,
  // 32 clusters per step), then the starts added back into the offsets
  uint32_t* sz = sizes + size_t(u) * c_cap;
  uint32_t* st = starts + size_t(u) * (c_cap + 1);
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
    uint32_t run = 0;
    for (int ww = 0; ww < W; ++ww) {
      const uint32_t h = hist[ww * C + c];
      hist[ww * C + c] = run;  // becomes the intra-column offset
      run += h;
    }
    sz[c] = run;  // the column total (this block reads it back below)
  }
  __syncthreads();
  if (w == 0) {
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < C; c0 += 32) {
      const uint32_t c = c0 + lane;
      const uint32_t tot = c < C ? sz[c] : 0u;
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const uint32_t excl = carry + incl - tot;
      if (c < C) {
        st[c] = excl;
        if (tot == 0) s_empty = 1;
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) { st[C] = carry; s_total = carry; }
  }
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
    const uint32_t e = st[c];
    for (int ww = 0; ww < W; ++ww) hist[ww * C + c] += e;
  }
  __syncthreads();

  // stable scatter: warp w walks its segment in order (sorted_ids NULL:
  // the caller needs only the sizes / starts / flags)
  uint32_t* out = sorted_ids ? sorted_ids + size_t(u) * p_cap : nullptr;
  uint32_t* cur = hist + w * C;
  for (uint32_t b0 = p0; out && b0 < p1; b0 += 32 * IX_BATCH) {
    int32_t lb[IX_BATCH];
#pragma unroll
    for (int k = 0; k < IX_BATCH; ++k) {
      const uint32_t q = b0 + 32 * k + lane;
      lb[k] = q < p1 ? __ldg(lab + q) : -1;
    }
#pragma unroll
    for (int k = 0; k < IX_BATCH; ++k) {
      const uint32_t p = b0 + 32 * k + lane;
      const int32_t l = lb[k];
      unsigned valid = __ballot_sync(0xffffffffu, l >= 0);
      if (l >= 0) {
        unsigned peers = __match_any_sync(valid, l);
        unsigned rank = __popc(peers & ((1u << lane) - 1u));
        out[cur[l] + rank] = p;
        __syncwarp(valid);
        if (rank == 0) cur[l] += __popc(peers);
      }
      __syncwarp();
    }
  }
  if (threadIdx.x == 0) {
    if (changed && prev) changed[u] = s_changed;
    if (any_empty && s_empty) any_empty[u] = 1;
  }
}

int launch_index(cudaStream_t st, uint32_t n_units, const int32_t* labels, uint32_t n_pos,
                 uint32_t p_cap, uint32_t c_cap, const uint32_t* n_clusters,
                 uint32_t c_uniform, uint32_t* sizes, uint32_t* starts, uint32_t* sorted_ids,
                 const int32_t* prev_labels, int32_t* changed, const int32_t* active,
                 int32_t* any_empty, uint8_t* dirty) {
  if (n_units == 0) return CKV_OK;
  // warps per CTA limited by the smem histogram [W][c_cap]
  const size_t budget = 200 * 1024;
  int W = 32;
  while (W > 1 && size_t(W) * c_cap * 4 > budget) W >>= 1;
  if (size_t(W) * c_cap * 4 > budget) {
    set_error("build_index: cluster capacity exceeds the 51200-cluster smem limit");
    return CKV_EINVAL;
  }
  size_t smem = size_t(W) * c_cap * 4;
  CKV_CUDA_TRY(smem_optin((const void*)k_index, int(budget)));
  k_index<<<n_units, W * 32, smem, st>>>(labels, n_pos, p_cap, c_cap, n_clusters, c_uniform,
                                         sizes, starts, sorted_ids, prev_labels, changed, active,
                                         any_empty, dirty);
  CKV_LAUNCH_CHECK("k_index");
  return CKV_OK;
}

}  // namespace ckvb

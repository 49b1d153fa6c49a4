// ckv_select.cu — K6 + K8: score_clusters + select_tokens + ClusterCache,
// fused, for every q head of a decode step (selection.hpp:50-111,
// cache.hpp:38-57).
//
// One CTA per kv unit; warp g serves q head (unit*group + g).
//   1. scores: every (q head, cluster) pair is a sequential f64 FMA chain
//      over d = 128 (bit-identical to dot_f64).  Centroids are
//      staged 32 at a time through smem, transposed, so one centroid read
//      from HBM feeds all `group` q heads of the unit.
//   2. ranking: each lane insertion-sorts its strided share of the clusters
//      by (score desc, id asc), then a 32-way warp tournament pops clusters
//      in global rank order until the running size reaches the budget (or
//      all C for CKV_SEL_FULL_RANK).  Same total order as the reference's
//      std::sort comparator (selection.hpp:83-87), so ties break to the
//      lowest id.
//   3. gather: the taken slices (last one trimmed to its lowest positions),
//      then sinks 0..S-1, then the recency window — I_T in reference order.
//   4. cache: taken ids vs the union of the last R taken-sets (bitmap ring),
//      counters updated exactly as lookup_and_update does.
#include "ckv_internal.cuh"

namespace ckvb {



constexpr int SEL_MAX_GROUP = 8;
constexpr int SEL_CHUNK = 32;

__device__ __forceinline__ unsigned long long rank_key(double s) {
  // NaN scores (only from empty-cluster NaN centroids) rank last
  return isnan(s) ? 0ull : dkey(s);
}

// dynamic smem: keys [group][c_pad] u64 | order [group][c_pad] u32 |
//               per-warp centroid chunk [NW][D][33] f32
__global__ void __launch_bounds__(256)
k_select(ckv_select_desc desc, const float* __restrict__ q, const float* __restrict__ cents,
         const uint32_t* __restrict__ n_clusters, const uint32_t* __restrict__ sizes,
         const uint32_t* __restrict__ starts, const uint32_t* __restrict__ sorted_ids,
         uint32_t* __restrict__ token_ids, uint32_t* __restrict__ n_tokens,
         uint32_t* __restrict__ n_taken_out, uint32_t* __restrict__ trimmed_out,
         uint32_t* __restrict__ ranked_out, double* __restrict__ scores_out, CacheDev cache,
         uint32_t c_pad) {
  const uint32_t unit = blockIdx.x;
  const uint32_t G = desc.group;
  const int w = warp_id(), lane = lane_id();
  const int NW = blockDim.x >> 5;
  const uint32_t C = n_clusters[unit];
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smraw);      // [G][c_pad]
  uint32_t* order = reinterpret_cast<uint32_t*>(keys + size_t(G) * c_pad);      // [G][c_pad]
  float* chunk = reinterpret_cast<float*>(order + size_t(G) * c_pad);           // [NW][D][33]
  __shared__ float qs[SEL_MAX_GROUP][D];

  for (uint32_t i = threadIdx.x; i < G * D; i += blockDim.x)
    qs[i / D][i % D] = q[(size_t(unit) * G + i / D) * D + i % D];
  __syncthreads();

  // ---- 1. scores --------------------------------------------------------
  const float* cu = cents + size_t(unit) * desc.c_cap * D;
  float* my_chunk = chunk + size_t(w) * D * 33;
  for (uint32_t c0 = uint32_t(w) * SEL_CHUNK; c0 < C; c0 += uint32_t(NW) * SEL_CHUNK) {
    // coalesced load of 32 centroid rows, transposed into smem
    for (int r = 0; r < SEL_CHUNK; ++r) {
      uint32_t c = c0 + r;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < C) v = __ldg(reinterpret_cast<const float4*>(cu + size_t(c) * D) + lane);
      my_chunk[(4 * lane + 0) * 33 + r] = v.x;
      my_chunk[(4 * lane + 1) * 33 + r] = v.y;
      my_chunk[(4 * lane + 2) * 33 + r] = v.z;
      my_chunk[(4 * lane + 3) * 33 + r] = v.w;
    }
    __syncwarp();
    const uint32_t c = c0 + lane;
    double acc[SEL_MAX_GROUP];
#pragma unroll
    for (int g = 0; g < SEL_MAX_GROUP; ++g) acc[g] = 0.0;
#pragma unroll 4
    for (int j = 0; j < D; ++j) {
      const double m = double(my_chunk[j * 33 + lane]);
#pragma unroll
      for (int g = 0; g < SEL_MAX_GROUP; ++g)
        if (g < int(G)) acc[g] = __fma_rn(double(qs[g][j]), m, acc[g]);
    }
    if (c < C) {
#pragma unroll
      for (int g = 0; g < SEL_MAX_GROUP; ++g)
        if (g < int(G)) {
          keys[size_t(g) * c_pad + c] = rank_key(acc[g]);
          if (scores_out) scores_out[(size_t(unit) * G + g) * desc.c_cap + c] = acc[g];
        }
    }
    __syncwarp();
  }
  __syncthreads();

  // ---- 2-4. one warp per q head -----------------------------------------
  for (uint32_t g = w; g < G; g += NW) {
    const uint32_t h = unit * G + g;
    unsigned long long* kg = keys + size_t(g) * c_pad;
    uint32_t* og = order + size_t(g) * c_pad;
    // per-lane insertion sort of clusters c = lane + 32k (k-major layout)
    const uint32_t cnt = C > uint32_t(lane) ? (C - lane + 31) / 32 : 0;
    for (uint32_t k = 0; k < cnt; ++k) {
      const uint32_t c = lane + 32 * k;
      const unsigned long long kc = kg[c];
      uint32_t pos = k;
      while (pos > 0) {
        uint32_t prev = og[(pos - 1) * 32 + lane];
        unsigned long long kp = kg[prev];
        if (kp > kc || (kp == kc && prev < c)) break;
        og[pos * 32 + lane] = prev;
        --pos;
      }
      og[pos * 32 + lane] = c;
    }
    __syncwarp();
    // tournament
    const uint32_t* sz = sizes + size_t(unit) * desc.c_cap;
    const uint32_t* stt = starts + size_t(unit) * (desc.c_cap + 1);
    const uint32_t* sid = sorted_ids + size_t(unit) * desc.p_cap;
    uint32_t* out = token_ids + size_t(h) * desc.sel_cap;
    uint32_t* rk = ranked_out ? ranked_out + size_t(h) * desc.c_cap : nullptr;
    const bool full = (desc.flags & CKV_SEL_FULL_RANK) != 0;
    uint32_t head = 0;
    uint32_t cum = 0, taken = 0, trimmed = 0, r = 0;
    uint32_t my_c = cnt > 0 ? og[lane] : 0xffffffffu;
    unsigned long long my_k = cnt > 0 ? kg[my_c] : 0ull;
    bool my_valid = cnt > 0;
    for (; r < C; ++r) {
      if (!full && cum >= desc.budget) break;
      unsigned long long bk = my_valid ? my_k : 0ull;
      uint32_t bc = my_valid ? my_c : 0xffffffffu;
      // best = max key, ties -> lowest id; invalid lanes lose to everything
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
        uint32_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (ok > bk || (ok == bk && oc < bc)) { bk = ok; bc = oc; }
      }
      if (my_valid && bc == my_c) {
        ++head;
        my_valid = head < cnt;
        if (my_valid) { my_c = og[head * 32 + lane]; my_k = kg[my_c]; }
      }
      if (rk && lane == 0) rk[r] = bc;
      if (cum < desc.budget) {
        // take cluster bc (selection.hpp:92-106)
        const uint32_t s = sz[bc], rem = desc.budget - cum;
        const uint32_t take = s <= rem ? s : rem;
        const uint32_t* src = sid + stt[bc];
        for (uint32_t i = lane; i < take; i += 32) out[cum + i] = src[i];
        if (s > rem) trimmed = s - rem;
        cum += take;
        ++taken;
      }
    }
    // (the cache step below reads the taken prefix back from rk)
    uint32_t n = cum;
    for (uint32_t s = lane; s < desc.sink_count; s += 32) out[n + s] = s;
    n += desc.sink_count;
    const uint32_t nrec = desc.rec_end > desc.rec_begin ? desc.rec_end - desc.rec_begin : 0;
    for (uint32_t i = lane; i < nrec; i += 32) out[n + i] = desc.rec_begin + i;
    n += nrec;
    if (lane == 0) {
      n_tokens[h] = n;
      n_taken_out[h] = taken;
      trimmed_out[h] = trimmed;
    }
    // ---- cache (cache.hpp:38-57) ------------------------------------------
    if (cache.bits) {
      __syncwarp();
      const uint32_t W = cache.words, R = cache.retention;
      uint32_t* bits = cache.bits + size_t(h) * R * W;
      uint32_t* ring = cache.ring + size_t(h) * 2;
      uint32_t rhead = ring[0], rlen = ring[1];
      uint32_t hits = 0;
      unsigned long long miss_tokens = 0;
      for (uint32_t t = lane; t < taken; t += 32) {
        const uint32_t c = rk[t];
        bool res = false;
        for (uint32_t k = 0; k < R; ++k) res |= (bits[size_t(k) * W + (c >> 5)] >> (c & 31)) & 1u;
        if (res) ++hits; else miss_tokens += sz[c];
      }
      hits = __reduce_add_sync(0xffffffffu, hits);
      miss_tokens = warp_sum(miss_tokens);
      // push the new set into the ring (pop the oldest when full)
      uint32_t slot;
      if (rlen < R) { slot = (rhead + rlen) % R; rlen++; }
      else { slot = rhead; rhead = (rhead + 1) % R; }
      __syncwarp();
      uint32_t* sb = bits + size_t(slot) * W;
      for (uint32_t i = lane; i < W; i += 32) sb[i] = 0u;
      __syncwarp();
      for (uint32_t t = lane; t < taken; t += 32) atomicOr(&sb[rk[t] >> 5], 1u << (rk[t] & 31));
      if (lane == 0) {
        ring[0] = rhead;
        ring[1] = rlen;
        unsigned long long* ctr = cache.counters + size_t(h) * 4;
        ctr[0] += taken;
        ctr[1] += hits;
        ctr[2] += miss_tokens;
        ctr[3] = ctr[2] * 2ull * cache.d * 4ull;
      }
    }
  }
}

int launch_select(cudaStream_t st, const ckv_select_desc& desc, const float* q,
                  const float* cents, const uint32_t* n_clusters, const uint32_t* sizes,
                  const uint32_t* starts, const uint32_t* sorted_ids, uint32_t* token_ids,
                  uint32_t* n_tokens, uint32_t* n_taken, uint32_t* trimmed, uint32_t* ranked,
                  double* scores, const CacheDev& cache) {
  if (desc.group < 1 || desc.group > SEL_MAX_GROUP || desc.n_q % desc.group) {
    set_error("select: group must divide n_q and be <= 8");
    return CKV_EINVAL;
  }
  if (desc.budget < 1) { set_error("select: budget must be >= 1"); return CKV_EINVAL; }
  const uint32_t units = desc.n_q / desc.group;
  const uint32_t c_pad = (desc.c_cap + 31) / 32 * 32;
  const int threads = 128;
  const size_t smem = size_t(desc.group) * c_pad * (8 + 4) + size_t(threads / 32) * D * 33 * 4;
  if (smem > 227 * 1024) {
    set_error("select: cluster capacity too large for the smem ranking buffers");
    return CKV_EINVAL;
  }
  CKV_CUDA_TRY(cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem)));
  k_select<<<units, threads, smem, st>>>(desc, q, cents, n_clusters, sizes, starts, sorted_ids,
                                         token_ids, n_tokens, n_taken, trimmed, ranked, scores,
                                         cache, c_pad);
  CKV_LAUNCH_CHECK("k_select");
  return CKV_OK;
}

// ---------------------------------------------------------------------------
// standalone ClusterCache::lookup_and_update for one slot (cache.hpp:38-57),
// preserving the caller's order in the hit / miss lists.  Single warp.
// ---------------------------------------------------------------------------
__global__ void k_cache_lookup(CacheDev cache, uint32_t slot_h, const uint32_t* __restrict__ sel,
                               uint32_t n_sel, const uint32_t* __restrict__ sizes,
                               uint32_t* __restrict__ hit_ids, uint32_t* __restrict__ miss_ids,
                               uint32_t* __restrict__ counts) {
  const int lane = lane_id();
  const uint32_t W = cache.words, R = cache.retention;
  uint32_t* bits = cache.bits + size_t(slot_h) * R * W;
  uint32_t* ring = cache.ring + size_t(slot_h) * 2;
  uint32_t nh = 0, nm = 0;
  unsigned long long miss_tokens = 0;
  for (uint32_t b = 0; b < n_sel; b += 32) {
    uint32_t i = b + lane;
    bool valid = i < n_sel;
    uint32_t c = valid ? sel[i] : 0;
    bool res = false;
    if (valid && c < cache.c_cap)
      for (uint32_t k = 0; k < R; ++k) res |= (bits[size_t(k) * W + (c >> 5)] >> (c & 31)) & 1u;
    unsigned hm = __ballot_sync(0xffffffffu, valid && res);
    unsigned mm = __ballot_sync(0xffffffffu, valid && !res);
    unsigned lt = (1u << lane) - 1u;
    if (valid && res) hit_ids[nh + __popc(hm & lt)] = c;
    if (valid && !res) { miss_ids[nm + __popc(mm & lt)] = c; miss_tokens += sizes[c]; }
    nh += __popc(hm);
    nm += __popc(mm);
  }
  miss_tokens = warp_sum(miss_tokens);
  uint32_t rhead = ring[0], rlen = ring[1], slot;
  if (rlen < R) { slot = (rhead + rlen) % R; rlen++; }
  else { slot = rhead; rhead = (rhead + 1) % R; }
  __syncwarp();
  uint32_t* sb = bits + size_t(slot) * W;
  for (uint32_t i = lane; i < W; i += 32) sb[i] = 0u;
  __syncwarp();
  for (uint32_t i = lane; i < n_sel; i += 32)
    if (sel[i] < cache.c_cap) atomicOr(&sb[sel[i] >> 5], 1u << (sel[i] & 31));
  if (lane == 0) {
    ring[0] = rhead;
    ring[1] = rlen;
    unsigned long long* ctr = cache.counters + size_t(slot_h) * 4;
    ctr[0] += n_sel;
    ctr[1] += nh;
    ctr[2] += miss_tokens;
    ctr[3] = ctr[2] * 2ull * cache.d * 4ull;
    counts[0] = nh;
    counts[1] = nm;
  }
}

// invalidate_on_recluster (cache.hpp:67-76): clear retired ids in every set
__global__ void k_cache_invalidate(CacheDev cache, uint32_t slot_h,
                                   const uint32_t* __restrict__ retired, uint32_t n) {
  const uint32_t W = cache.words, R = cache.retention;
  uint32_t* bits = cache.bits + size_t(slot_h) * R * W;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    uint32_t c = retired[i];
    if (c >= cache.c_cap) continue;
    for (uint32_t k = 0; k < R; ++k) atomicAnd(&bits[size_t(k) * W + (c >> 5)], ~(1u << (c & 31)));
  }
}

int launch_cache_lookup(cudaStream_t st, const CacheDev& cache, uint32_t slot,
                        const uint32_t* sel, uint32_t n_sel, const uint32_t* sizes,
                        uint32_t* hit, uint32_t* miss, uint32_t* counts) {
  k_cache_lookup<<<1, 32, 0, st>>>(cache, slot, sel, n_sel, sizes, hit, miss, counts);
  CKV_LAUNCH_CHECK("k_cache_lookup");
  return CKV_OK;
}

int launch_cache_invalidate(cudaStream_t st, const CacheDev& cache, uint32_t slot,
                            const uint32_t* retired, uint32_t n) {
  k_cache_invalidate<<<1, 256, 0, st>>>(cache, slot, retired, n);
  CKV_LAUNCH_CHECK("k_cache_invalidate");
  return CKV_OK;
}

}  // namespace ckvb

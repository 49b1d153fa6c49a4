// ckv_select.cu — K6 + K8: score_clusters + select_tokens + ClusterCache
// for every q head of a decode step (selection.hpp:50-111, cache.hpp:38-57).
//
// Two launches:
//  k_score : one thread per (kv unit, cluster) runs the `group` q heads'
//            sequential f64 FMA chains over d = 128 (bit-identical to
//            dot_f64) and writes order-preserving u64 rank
//            keys.  Each centroid row is read once per unit, every q head of
//            the GQA group reuses it from registers.
//  k_rank  : one warp per q head.  Each lane insertion-sorts its strided
//            share of the keys by (score desc, id asc) — the reference's
//            std::sort comparator (selection.hpp:83-87) — then a 32-way warp
//            tournament pops clusters in global rank order until the running
//            size reaches the budget (all C for CKV_SEL_FULL_RANK).  The taken
//            slices (last one trimmed to its lowest positions), sinks and the
//            recency window are then written in parallel:
//              token_ids : reference I_T positions (selection.hpp:91-109)
//              rows      : the same entries as rows of the cluster-major KV
//                          store (row = row_base + starts[c] + i for cluster
//                          tokens, the position for sinks / recency), i.e.
//                          contiguous runs for the attention kernel.
//            The cache step (bitmap ring of the last R taken-sets) is fused.
#include "ckv_internal.cuh"

namespace ckvb {

__device__ __forceinline__ unsigned long long rank_key(double s) {
  // NaN scores (only from empty-cluster NaN centroids) rank last
  return isnan(s) ? 0ull : dkey(s);
}

constexpr int SC_ROWS = 64;       // clusters per k_score CTA (one per thread)
constexpr int SC_STRIDE = D + 4;  // padded smem row: conflict-free 16-B reads

__device__ __forceinline__ void cp_async16_sel(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(valid ? 16 : 0));
}

template <int G>
__global__ void __launch_bounds__(SC_ROWS)
k_score(const float* __restrict__ q, const float* __restrict__ cents,
        const uint32_t* __restrict__ n_clusters, uint32_t c_cap, uint32_t c_pad,
        unsigned long long* __restrict__ keys, double* __restrict__ scores_out) {
  const uint32_t unit = blockIdx.x;
  const uint32_t c0 = blockIdx.y * SC_ROWS;
  const uint32_t C = n_clusters[unit];
  if (c0 >= C) return;
  __shared__ __align__(16) float cs[SC_ROWS][SC_STRIDE];
  __shared__ double qs[G][D];
  // stage this CTA's centroid rows: coalesced 16-B cp.async, one latency
  const float* src = cents + (size_t(unit) * c_cap + c0) * D;
  for (int e = threadIdx.x; e < SC_ROWS * (D / 4); e += SC_ROWS) {
    const int r = e / (D / 4), c4 = e % (D / 4);
    const bool ok = c0 + r < C;
    cp_async16_sel(&cs[r][4 * c4], src + size_t(ok ? r : 0) * D + 4 * c4, ok);
  }
  asm volatile("cp.async.commit_group;\n");
  for (int i = threadIdx.x; i < G * D; i += SC_ROWS)
    qs[i / D][i % D] = double(q[(size_t(unit) * G + i / D) * D + i % D]);
  asm volatile("cp.async.wait_group 0;\n");
  __syncthreads();
  const uint32_t c = c0 + threadIdx.x;
  if (c >= C) return;
  double acc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g] = 0.0;
  const float4* row = reinterpret_cast<const float4*>(&cs[threadIdx.x][0]);
#pragma unroll 8
  for (int j4 = 0; j4 < D / 4; ++j4) {
    const float4 m = row[j4];
    const double m0 = m.x, m1 = m.y, m2 = m.z, m3 = m.w;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      acc[g] = __fma_rn(qs[g][4 * j4 + 0], m0, acc[g]);
      acc[g] = __fma_rn(qs[g][4 * j4 + 1], m1, acc[g]);
      acc[g] = __fma_rn(qs[g][4 * j4 + 2], m2, acc[g]);
      acc[g] = __fma_rn(qs[g][4 * j4 + 3], m3, acc[g]);
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const size_t h = size_t(unit) * G + g;
    keys[h * c_pad + c] = rank_key(acc[g]);
    if (scores_out) scores_out[h * c_cap + c] = acc[g];
  }
}

__global__ void __launch_bounds__(128)
k_rank(ckv_select_desc desc, uint32_t c_pad, uint32_t row_base,
       const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ n_clusters,
       const uint32_t* __restrict__ sizes, const uint32_t* __restrict__ starts,
       const uint32_t* __restrict__ sorted_ids, uint32_t* __restrict__ token_ids,
       uint32_t* __restrict__ rows_out, uint32_t* __restrict__ n_tokens,
       uint32_t* __restrict__ n_taken_out, uint32_t* __restrict__ trimmed_out,
       uint32_t* __restrict__ ranked_out, CacheDev cache) {
  const int lane = lane_id();
  const int wpb = blockDim.x >> 5;
  const uint32_t h = blockIdx.x * wpb + warp_id();
  if (h >= desc.n_q) return;
  const uint32_t unit = h / desc.group;
  const uint32_t C = n_clusters[unit];
  extern __shared__ __align__(16) unsigned char smraw[];
  // per warp: keys u64[c_pad] | order u32[c_pad] | taken u32[c_pad] | offsets u32[c_pad]
  unsigned long long* kg = reinterpret_cast<unsigned long long*>(smraw) + size_t(warp_id()) * c_pad;
  uint32_t* og = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned long long*>(smraw) +
                                             size_t(wpb) * c_pad) + size_t(warp_id()) * 3 * c_pad;
  uint32_t* taken_c = og + c_pad;
  uint32_t* taken_off = og + 2 * c_pad;

  const unsigned long long* kin = keys + size_t(h) * c_pad;
  for (uint32_t c = lane; c < C; c += 32) kg[c] = kin[c];
  __syncwarp();
  // per-lane insertion sort of clusters c = lane + 32k (k-major layout)
  const uint32_t cnt = C > uint32_t(lane) ? (C - lane + 31) / 32 : 0;
  for (uint32_t k = 0; k < cnt; ++k) {
    const uint32_t c = lane + 32 * k;
    const unsigned long long kc = kg[c];
    uint32_t pos = k;
    while (pos > 0) {
      const uint32_t prev = og[(pos - 1) * 32 + lane];
      const unsigned long long kp = kg[prev];
      if (kp > kc || (kp == kc && prev < c)) break;
      og[pos * 32 + lane] = prev;
      --pos;
    }
    og[pos * 32 + lane] = c;
  }
  __syncwarp();

  const uint32_t* sz = sizes + size_t(unit) * desc.c_cap;
  const uint32_t* stt = starts + size_t(unit) * (desc.c_cap + 1);
  uint32_t* rk = ranked_out + size_t(h) * desc.c_cap;
  const bool full = (desc.flags & CKV_SEL_FULL_RANK) != 0;
  uint32_t head = 0, cum = 0, taken = 0, trimmed = 0;
  uint32_t my_c = cnt > 0 ? og[lane] : 0xffffffffu;
  unsigned long long my_k = cnt > 0 ? kg[my_c] : 0ull;
  uint32_t my_sz = cnt > 0 ? sz[my_c] : 0u;
  bool my_valid = cnt > 0;
  for (uint32_t r = 0; r < C; ++r) {
    if (!full && cum >= desc.budget) break;
    unsigned long long bk = my_valid ? my_k : 0ull;
    uint32_t bc = my_valid ? my_c : 0xffffffffu;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const uint32_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ok > bk || (ok == bk && oc < bc)) { bk = ok; bc = oc; }
    }
    const bool mine = my_valid && bc == my_c;
    const uint32_t s = __shfl_sync(0xffffffffu, my_sz, __ffs(__ballot_sync(0xffffffffu, mine)) - 1);
    if (mine) {
      ++head;
      my_valid = head < cnt;
      if (my_valid) { my_c = og[head * 32 + lane]; my_k = kg[my_c]; my_sz = sz[my_c]; }
    }
    if (lane == 0) rk[r] = bc;
    if (cum < desc.budget) {  // take cluster bc (selection.hpp:92-106)
      const uint32_t rem = desc.budget - cum;
      const uint32_t take = s <= rem ? s : rem;
      if (lane == 0) { taken_c[taken] = bc; taken_off[taken] = cum; }
      if (s > rem) trimmed = s - rem;
      cum += take;
      ++taken;
    }
  }
  __syncwarp();
  // flat parallel fill of the taken slices: entry e (< cum) belongs to the
  // last taken cluster whose offset is <= e (binary search in smem)
  uint32_t* out = token_ids ? token_ids + size_t(h) * desc.sel_cap : nullptr;
  uint32_t* rows = rows_out ? rows_out + size_t(h) * desc.sel_cap : nullptr;
  const uint32_t* sid = sorted_ids + size_t(unit) * desc.p_cap;
  for (uint32_t t = lane; t < taken; t += 32) taken_c[t] = stt[taken_c[t]];  // -> slice start
  __syncwarp();
  for (uint32_t e0 = 0; e0 < cum; e0 += 128) {
    uint32_t src[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t e = e0 + 32 * k + lane;
      uint32_t lo = 0, hi = taken;  // largest t with taken_off[t] <= e
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (taken_off[mid] <= e) lo = mid; else hi = mid;
      }
      src[k] = taken_c[lo] + (e - taken_off[lo]);
    }
    uint32_t pos[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t e = e0 + 32 * k + lane;
      pos[k] = (out && e < cum) ? __ldg(sid + src[k]) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t e = e0 + 32 * k + lane;
      if (e < cum) {
        if (rows) rows[e] = row_base + src[k];
        if (out) out[e] = pos[k];
      }
    }
  }
  uint32_t n = cum;
  for (uint32_t s = lane; s < desc.sink_count; s += 32) {
    if (rows) rows[n + s] = s;
    if (out) out[n + s] = s;
  }
  n += desc.sink_count;
  const uint32_t nrec = desc.rec_end > desc.rec_begin ? desc.rec_end - desc.rec_begin : 0;
  for (uint32_t i = lane; i < nrec; i += 32) {
    if (rows) rows[n + i] = desc.rec_begin + i;
    if (out) out[n + i] = desc.rec_begin + i;
  }
  n += nrec;
  if (lane == 0) {
    n_tokens[h] = n;
    n_taken_out[h] = taken;
    trimmed_out[h] = trimmed;
  }
  // ---- cache (cache.hpp:38-57) ----------------------------------------------
  if (cache.bits) {
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

size_t select_scratch_bytes(uint32_t n_q, uint32_t c_cap) {
  return size_t(n_q) * ((c_cap + 31) / 32 * 32) * 8 + 16;
}

int launch_select(cudaStream_t st, const ckv_select_desc& desc, const float* q,
                  const float* cents, const uint32_t* n_clusters, const uint32_t* sizes,
                  const uint32_t* starts, const uint32_t* sorted_ids, uint32_t* token_ids,
                  uint32_t* rows, uint32_t row_base, uint32_t* n_tokens, uint32_t* n_taken,
                  uint32_t* trimmed, uint32_t* ranked, double* scores, const CacheDev& cache,
                  void* scratch) {
  const uint32_t G = desc.group;
  if (G < 1 || desc.n_q % G || !(G == 1 || G == 2 || G == 4 || G == 8)) {
    set_error("select: group must be 1, 2, 4 or 8 and divide n_q");
    return CKV_EINVAL;
  }
  if (desc.budget < 1) { set_error("select: budget must be >= 1"); return CKV_EINVAL; }
  const uint32_t units = desc.n_q / G;
  const uint32_t c_pad = (desc.c_cap + 31) / 32 * 32;
  auto* keys = static_cast<unsigned long long*>(scratch);
  const dim3 gs(units, (c_pad + SC_ROWS - 1) / SC_ROWS);
  switch (G) {
    case 1: k_score<1><<<gs, SC_ROWS, 0, st>>>(q, cents, n_clusters, desc.c_cap, c_pad, keys, scores); break;
    case 2: k_score<2><<<gs, SC_ROWS, 0, st>>>(q, cents, n_clusters, desc.c_cap, c_pad, keys, scores); break;
    case 4: k_score<4><<<gs, SC_ROWS, 0, st>>>(q, cents, n_clusters, desc.c_cap, c_pad, keys, scores); break;
    default: k_score<8><<<gs, SC_ROWS, 0, st>>>(q, cents, n_clusters, desc.c_cap, c_pad, keys, scores); break;
  }
  CKV_LAUNCH_CHECK("k_score");
  const size_t per_warp = size_t(c_pad) * (8 + 12);
  int wpb = 4;
  while (wpb > 1 && per_warp * wpb > 200 * 1024) wpb >>= 1;
  if (per_warp * wpb > 200 * 1024) {
    set_error("select: cluster capacity too large for the smem ranking buffers");
    return CKV_EINVAL;
  }
  const size_t smem = per_warp * wpb;
  if (smem > 48 * 1024)
    CKV_CUDA_TRY(cudaFuncSetAttribute(k_rank, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem)));
  k_rank<<<(desc.n_q + wpb - 1) / wpb, wpb * 32, smem, st>>>(
      desc, c_pad, row_base, keys, n_clusters, sizes, starts, sorted_ids, token_ids, rows,
      n_tokens, n_taken, trimmed, ranked, cache);
  CKV_LAUNCH_CHECK("k_rank");
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
    const uint32_t i = b + lane;
    const bool valid = i < n_sel;
    const uint32_t c = valid ? sel[i] : 0;
    bool res = false;
    if (valid && c < cache.c_cap)
      for (uint32_t k = 0; k < R; ++k) res |= (bits[size_t(k) * W + (c >> 5)] >> (c & 31)) & 1u;
    const unsigned hm = __ballot_sync(0xffffffffu, valid && res);
    const unsigned mm = __ballot_sync(0xffffffffu, valid && !res);
    const unsigned lt = (1u << lane) - 1u;
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
    const uint32_t c = retired[i];
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

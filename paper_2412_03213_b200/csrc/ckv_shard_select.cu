// ckv_shard_select.cu — decode-step kernels of the sequence-sharded path
// (SURVEY §8e, config E): centroid-sharded scoring, the global budgeted
// top-k over the all-gathered scores, and the log-sum-exp merge of the
// ranks' partial attention outputs.
//
//   k_score_range   exact f64 score_clusters (selection.hpp:51-57) of this
//                   rank's centroid slice for all q heads: the sequential
//                   dot_f64 chain, bit-identical to the reference (N2/N6).
//                   Centroid rows and the unit's G queries are staged in
//                   smem; one thread per (q head, cluster).
//   (caller)        all-gather of the slices -> [world][n_q][slice] f64.
//   k_select_scored one CTA per q head: block bitonic sort of all C scores by
//                   (score desc, id asc) — select_tokens' comparator
//                   (selection.hpp:83-87) — prefix of the GLOBAL sizes,
//                   cut at the budget, and this rank's share of every taken
//                   cluster: the reference takes a cluster's lowest positions
//                   first and shards are contiguous in position, so shard s
//                   keeps clamp(allow_c - prefix_s(c), 0, size_s(c)) of
//                   cluster c, allow_c = its size, or B - cum for the trimmed
//                   last one (selection.hpp:91-106).  Emits I_T as runs of
//                   the local cluster-major store (ckv_attend's input).
//   k_lse_merge     out = sum_s 2^(lse_s - M) o_s / sum_s 2^(lse_s - M) over
//                   the ranks' (o_s, lse_s) from ckv_attend_partial; the
//                   local weights are rescaled to global softmax weights.
#include "ckv_internal.cuh"

namespace ckvb {
namespace {

constexpr int SR_THREADS = 256;

__device__ __forceinline__ unsigned long long rank_key_s(double s) {
  return isnan(s) ? 0ull : dkey(s);  // NaN (empty-cluster centroids) ranks last
}
__device__ __forceinline__ uint32_t fkey32(float x) {  // order-preserving f32 -> u32
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ bool before(unsigned long long ka, uint32_t ia, unsigned long long kb,
                                       uint32_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}

// blockIdx.x = unit, blockIdx.y = a tile of SR_ROWS centroid rows.  A thread
// owns one centroid row and runs the G heads' sequential f64 chains side by
// side (G independent FMA chains hide the f64 latency; one 16-B smem load of
// the row feeds 4G FMAs, the query quads are broadcasts).
constexpr int SR_ROWS = 128;
constexpr int SR_LD = D + 4;  // row stride in floats: 16-B aligned rows
__device__ __forceinline__ void sr_cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}

template <int G>
__global__ void __launch_bounds__(SR_ROWS)
k_score_range(const float* __restrict__ q, const float* __restrict__ cents, uint32_t c_cap,
              uint32_t C, uint32_t c_lo, uint32_t c_hi, uint32_t slice,
              double* __restrict__ scores) {
  extern __shared__ __align__(16) float sr_sm[];
  float* crow = sr_sm;                  // [SR_ROWS][SR_LD]
  float* qs = sr_sm + SR_ROWS * SR_LD;  // [G][D]
  const uint32_t u = blockIdx.x;
  const uint32_t t0 = c_lo + blockIdx.y * SR_ROWS;
  const uint32_t hi = min(c_hi, C);
  if (t0 >= hi) return;
  const uint32_t nrow = min(uint32_t(SR_ROWS), hi - t0);
  const float4* cu = reinterpret_cast<const float4*>(cents + (size_t(u) * c_cap + t0) * D);
  // tile and q to shared memory by cp.async, all pieces in flight at once
  for (uint32_t e = threadIdx.x; e < nrow * (D / 4); e += SR_ROWS)
    sr_cp_async16(crow + (e / (D / 4)) * SR_LD + 4 * (e % (D / 4)), cu + e);
  const float4* qu = reinterpret_cast<const float4*>(q + size_t(u) * G * D);
  for (uint32_t e = threadIdx.x; e < G * D / 4; e += SR_ROWS)
    sr_cp_async16(qs + 4 * e, qu + e);
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  const uint32_t r = threadIdx.x;
  if (r >= nrow) return;
  double s[G];
#pragma unroll
  for (int g = 0; g < G; ++g) s[g] = 0.0;
  const float* row = crow + r * SR_LD;
#pragma unroll 2
  for (int j = 0; j < D; j += 4) {
    const float4 m = *reinterpret_cast<const float4*>(row + j);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float4 x = *reinterpret_cast<const float4*>(qs + g * D + j);
      s[g] = __fma_rn(double(x.x), double(m.x), s[g]);
      s[g] = __fma_rn(double(x.y), double(m.y), s[g]);
      s[g] = __fma_rn(double(x.z), double(m.z), s[g]);
      s[g] = __fma_rn(double(x.w), double(m.w), s[g]);
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) scores[(size_t(u) * G + g) * slice + (t0 + r - c_lo)] = s[g];
}

// block-wide inclusive scan of one u32 per thread (SR_THREADS threads)
__device__ __forceinline__ uint32_t block_incl_scan(uint32_t x, uint32_t* wsum,
                                                    uint32_t* total = nullptr) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  uint32_t pre = 0, tot = 0;
  for (int w = 0; w < SR_THREADS / 32; ++w) {
    if (w < wid) pre += wsum[w];
    tot += wsum[w];
  }
  __syncthreads();
  if (total) *total = tot;
  return x + pre;
}

// block bitonic sort of key[0..n2) / id[0..n2) by before() (n2 a power of 2)
__device__ __forceinline__ void block_sort(unsigned long long* key, uint32_t* id, uint32_t n2) {
  for (uint32_t k = 2; k <= n2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < n2; i += SR_THREADS) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long ka = key[i], kb = key[ixj];
          const uint32_t ia = id[i], ib = id[ixj];
          const bool asc = (i & k) == 0;
          const bool swap = asc ? before(kb, ib, ka, ia) : before(ka, ia, kb, ib);
          if (swap) { key[i] = kb; key[ixj] = ka; id[i] = ib; id[ixj] = ia; }
        }
      }
      __syncthreads();
    }
  }
}

// approximate scores of a centroid slice for the sharded decode step: the
// same smem-staged layout as k_score_range (a thread per centroid row, the G
// heads' chains side by side) in f32, plus the rigorous bound
// e = 2^-14 |q| |mu| >= |a - dot_f64| (an f32 chain of 128 products errs by
// <= 127 u sum |q_j mu_j| <= 2^-17 |q| |mu|; the factor 8 covers the rounding
// of the norms).  out [2][n_q][slice]: a, then e.
constexpr float SA_ERR = 1.0f / 16384.0f;
template <int G>
__global__ void __launch_bounds__(SR_ROWS)
k_score_range_f32(const float* __restrict__ q, const float* __restrict__ cents, uint32_t c_cap,
                  uint32_t C, uint32_t c_lo, uint32_t c_hi, uint32_t slice, uint32_t n_q,
                  float* __restrict__ out) {
  extern __shared__ __align__(16) float sr_sm[];
  float* crow = sr_sm;                  // [SR_ROWS][SR_LD]
  float* qs = sr_sm + SR_ROWS * SR_LD;  // [G][D]
  __shared__ float qn[G];
  const uint32_t u = blockIdx.x;
  const uint32_t t0 = c_lo + blockIdx.y * SR_ROWS;
  const uint32_t hi = min(c_hi, C);
  if (t0 >= hi) return;
  const uint32_t nrow = min(uint32_t(SR_ROWS), hi - t0);
  const float4* cu = reinterpret_cast<const float4*>(cents + (size_t(u) * c_cap + t0) * D);
  // the tile and q go to shared memory by cp.async: every 16-B piece of the
  // 64 KB tile is in flight at once (a load-then-store loop keeps one)
  for (uint32_t e = threadIdx.x; e < nrow * (D / 4); e += SR_ROWS)
    sr_cp_async16(crow + (e / (D / 4)) * SR_LD + 4 * (e % (D / 4)), cu + e);
  const float4* qu = reinterpret_cast<const float4*>(q + size_t(u) * G * D);
  for (uint32_t e = threadIdx.x; e < G * D / 4; e += SR_ROWS)
    sr_cp_async16(qs + 4 * e, qu + e);
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  // |q| of each head by a warp (a lane per 4 dims + shuffles), not one
  // thread's 128-long dependent chain that the whole block would wait for
  for (int g = threadIdx.x >> 5; g < G; g += SR_ROWS / 32) {
    const float4 x = reinterpret_cast<const float4*>(qs + g * D)[threadIdx.x & 31];
    float n2 = fmaf(x.x, x.x, fmaf(x.y, x.y, fmaf(x.z, x.z, x.w * x.w)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    if ((threadIdx.x & 31) == 0) qn[g] = SA_ERR * sqrtf(n2);
  }
  __syncthreads();
  const uint32_t r = threadIdx.x;
  if (r >= nrow) return;
  float sacc[G], mn2 = 0.f;
#pragma unroll
  for (int g = 0; g < G; ++g) sacc[g] = 0.f;
  const float* row = crow + r * SR_LD;
#pragma unroll 4
  for (int j = 0; j < D; j += 4) {
    const float4 m = *reinterpret_cast<const float4*>(row + j);
    mn2 = fmaf(m.x, m.x, fmaf(m.y, m.y, fmaf(m.z, m.z, fmaf(m.w, m.w, mn2))));
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float4 x = *reinterpret_cast<const float4*>(qs + g * D + j);
      sacc[g] = fmaf(x.x, m.x, sacc[g]);
      sacc[g] = fmaf(x.y, m.y, sacc[g]);
      sacc[g] = fmaf(x.z, m.z, sacc[g]);
      sacc[g] = fmaf(x.w, m.w, sacc[g]);
    }
  }
  const float mn = sqrtf(mn2);
  const size_t plane = size_t(n_q) * slice;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const size_t o = (size_t(u) * G + g) * slice + (t0 + r - c_lo);
    out[o] = sacc[g];
    out[plane + o] = fmaf(qn[g], mn, 1e-30f);
  }
}

__global__ void __launch_bounds__(SR_THREADS)
k_select_scored(ckv_shard_select_desc d, uint32_t p2, const double* __restrict__ scores,
                const uint32_t* __restrict__ gsize, const uint32_t* __restrict__ lsize,
                const uint32_t* __restrict__ lstart, const uint32_t* __restrict__ prefix,
                const uint32_t* __restrict__ lsorted, ckv_runs runs,
                uint32_t* __restrict__ token_ids, uint32_t* __restrict__ n_tokens,
                uint32_t* __restrict__ n_taken, uint32_t* __restrict__ trimmed_out,
                uint32_t* __restrict__ ranked) {
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smraw);  // [p2]
  uint32_t* id = reinterpret_cast<uint32_t*>(key + p2);                     // [p2]
  uint32_t* incl = id + p2;                                                 // [p2]
  uint32_t* loc = incl + p2;                                                // [p2 + 1]
  uint32_t* sz = loc + p2 + 1;                                              // [p2]
  uint32_t* tid2 = sz + p2;                                                 // [p2]
  unsigned long long* tk = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(tid2 + p2) + 7) & ~uintptr_t(7));        // [p2]
  __shared__ uint32_t s_taken, s_wsum[SR_THREADS / 32], s_hist[256], s_n, s_bin, s_above;
  const uint32_t h = blockIdx.x, unit = h / d.group;
  const uint32_t C = d.C, B = d.budget;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t* gs = gsize + size_t(unit) * d.c_cap;
  // gathered scores: cluster c lives in rank c / slice at offset c % slice
  uint32_t tot = 0;
  for (uint32_t c = tid; c < p2; c += SR_THREADS) {
    if (c < C) {
      const uint32_t r = c / d.slice, o = c % d.slice;
      key[c] = rank_key_s(scores[(size_t(r) * d.n_q + h) * d.slice + o]);
      id[c] = c;
      sz[c] = __ldg(gs + c);
      tot += sz[c];
    } else {
      key[c] = 0ull;
      id[c] = 0xffffffffu;  // padding sorts after every real cluster
      sz[c] = 0u;
    }
  }
  tot = __reduce_add_sync(0xffffffffu, tot);
  if ((tid & 31) == 0) s_wsum[tid >> 5] = tot;
  __syncthreads();
  tot = 0;
  for (int w = 0; w < SR_THREADS / 32; ++w) tot += s_wsum[w];
  __syncthreads();
  uint32_t n_sorted = C;
  if (!(d.flags & CKV_SEL_FULL_RANK) && B > 0 && tot >= B) {
    // ---- size-weighted radix select on the 64-bit rank keys: tau with
    // W(key > tau) < B <= W(key >= tau); only the clusters ranked at or above
    // the cutoff need sorting (~B / mean size of them, not all C)
    unsigned long long prefix_k = 0ull;
    uint32_t above = 0;
    s_hist[tid] = 0u;  // SR_THREADS == 256 bins; warp 0 re-zeroes them per pass
    __syncthreads();
    for (int pass = 0; pass < 8; ++pass) {
      const int sh = 56 - 8 * pass;
      const unsigned long long hm = pass == 0 ? 0ull : (~0ull << (sh + 8));
      // warp-aggregated: the scores share their high bytes, so most lanes hit
      // the same bin; one smem atomic per distinct bin per warp
      for (uint32_t c0 = tid - lane; c0 < C; c0 += SR_THREADS) {
        const uint32_t c = c0 + lane;
        const bool in = c < C && sz[c] && ((key[c] ^ prefix_k) & hm) == 0ull;
        const uint32_t bin = in ? uint32_t(key[c] >> sh) & 255u : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, bin);
        const uint32_t w = __reduce_add_sync(peers, in ? sz[c] : 0u);
        if (in && lane == __ffs(peers) - 1) atomicAdd(&s_hist[bin], w);
      }
      __syncthreads();
      if (wid == 0) {
        // one warp scans the 256 bins from high to low: lane L holds bins
        // 255 - 8L .. 248 - 8L; the first bin where the running weight
        // reaches B holds the cutoff
        uint32_t v[8], ls = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          v[k] = s_hist[255 - 8 * lane - k];
          s_hist[255 - 8 * lane - k] = 0u;  // ready for the next pass
          ls += v[k];
        }
        uint32_t x = ls;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        uint32_t run = above + x - ls;  // weight of the bins above my 8
        int found = -1;
        uint32_t above_sel = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (found < 0 && run + v[k] >= B) { found = 255 - 8 * lane - k; above_sel = run; }
          run += v[k];
        }
        const unsigned f = __ballot_sync(0xffffffffu, found >= 0);
        const int src = __ffs(f) - 1;  // the highest bin reaching B
        if (lane == src) { s_bin = uint32_t(found); s_above = above_sel; }
      }
      __syncthreads();
      prefix_k |= (unsigned long long)s_bin << sh;
      above = s_above;
    }
    // T = {key > tau} plus the ties at tau, in id order, until the budget
    __shared__ uint32_t s_nt;
    if (tid == 0) { s_n = 0; s_nt = 0; }
    __syncthreads();
    for (uint32_t c = tid; c < C; c += SR_THREADS) {
      if (key[c] > prefix_k) {
        const uint32_t slot = atomicAdd(&s_n, 1u);
        tk[slot] = key[c];
        tid2[slot] = c;
      } else if (key[c] == prefix_k) {
        loc[atomicAdd(&s_nt, 1u)] = c;  // the ties at tau (usually one)
      }
    }
    __syncthreads();
    const uint32_t nt = s_nt;
    if (nt > 1) {  // ascending id: rank by counting (incl[] is free scratch here)
      for (uint32_t i = tid; i < nt; i += SR_THREADS) {
        const uint32_t ci = loc[i];
        uint32_t r = 0;
        for (uint32_t j = 0; j < nt; ++j) r += loc[j] < ci;
        incl[r] = ci;
      }
      __syncthreads();
      for (uint32_t i = tid; i < nt; i += SR_THREADS) loc[i] = incl[i];
      __syncthreads();
    }
    if (tid == 0) {
      // the reference's walk takes the ties while cum < B (selection.hpp:90-104)
      uint32_t cum = above, n = s_n;
      for (uint32_t i = 0; i < nt && cum < B; ++i) {
        const uint32_t c = loc[i];
        tk[n] = key[c];
        tid2[n] = c;
        ++n;
        cum += sz[c];
      }
      s_n = n;
    }
    __syncthreads();
    n_sorted = s_n;
    uint32_t n2 = 32;
    while (n2 < n_sorted) n2 <<= 1;
    for (uint32_t i = tid; i < n2; i += SR_THREADS) {
      const bool v2 = i < n_sorted;
      key[i] = v2 ? tk[i] : 0ull;
      id[i] = v2 ? tid2[i] : 0xffffffffu;
    }
    __syncthreads();
    if (n2 <= 256) {  // the taken prefix is small: one warp sorts it, no block barriers
      if (wid == 0) {
        for (uint32_t k = 2; k <= n2; k <<= 1) {
          for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = lane; i < n2; i += 32) {
              const uint32_t ixj = i ^ j;
              if (ixj > i) {
                const unsigned long long ka = key[i], kb = key[ixj];
                const uint32_t ia = id[i], ib = id[ixj];
                const bool asc = (i & k) == 0;
                const bool swap = asc ? before(kb, ib, ka, ia) : before(ka, ia, kb, ib);
                if (swap) { key[i] = kb; key[ixj] = ka; id[i] = ib; id[ixj] = ia; }
              }
            }
            __syncwarp();
          }
        }
      }
      __syncthreads();
    } else {
      block_sort(key, id, n2);
    }
  } else {
    block_sort(key, id, p2);
  }
  // inclusive prefix of the global sizes in rank order (chunks of 256)
  if (tid == 0) s_taken = B == 0 ? 0u : n_sorted;  // the reference breaks at cum >= B
  if (n_sorted <= 256) {  // one warp, no block barriers
    if (wid == 0) {
      uint32_t c2 = 0;
      for (uint32_t b = 0; b < n_sorted; b += 32) {
        const uint32_t i = b + lane;
        uint32_t x = i < n_sorted ? sz[id[i]] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (i < n_sorted) incl[i] = c2 + x;
        c2 += __shfl_sync(0xffffffffu, x, 31);
      }
    }
  } else {
    uint32_t carry = 0;
    for (uint32_t b = 0; b < n_sorted; b += SR_THREADS) {
      const uint32_t i = b + tid;
      uint32_t chunk_tot;
      const uint32_t x = block_incl_scan(i < n_sorted ? __ldg(gs + id[i]) : 0u, s_wsum, &chunk_tot);
      if (i < n_sorted) incl[i] = x + carry;
      carry += chunk_tot;
    }
  }
  __syncthreads();
  // taken = first i with incl[i] >= B, plus one (all of C when the total < B)
  for (uint32_t i = tid; i < n_sorted; i += SR_THREADS)
    if (B > 0 && incl[i] >= B && (i == 0 || incl[i - 1] < B)) s_taken = i + 1;
  __syncthreads();
  const uint32_t taken = s_taken;
  const uint32_t full_cum = taken ? incl[taken - 1] : 0;
  const uint32_t trimmed = full_cum > B ? full_cum - B : 0;
  // this rank's share of each taken cluster
  const uint32_t* ls = lsize + size_t(unit) * d.c_cap;
  const uint32_t* pf = prefix + size_t(unit) * d.c_cap;
  for (uint32_t i = tid; i < taken; i += SR_THREADS) {
    const uint32_t c = id[i];
    const uint32_t allow = (i + 1 == taken && trimmed) ? B - (i ? incl[i - 1] : 0u) : __ldg(gs + c);
    const uint32_t p = __ldg(pf + c), l = __ldg(ls + c);
    loc[i] = allow > p ? min(allow - p, l) : 0u;
  }
  __syncthreads();
  // exclusive prefix of the local shares -> run offsets (reuse incl[] as out)
  if (wid == 0) {
    uint32_t c2 = 0;
    for (uint32_t b = 0; b < taken; b += 32) {
      const uint32_t i = b + lane;
      uint32_t x = i < taken ? loc[i] : 0u;
      const uint32_t own = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (i < taken) loc[i] = c2 + x - own;  // exclusive
      c2 += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) loc[taken] = c2;
  }
  __syncthreads();
  const uint32_t cum = loc[taken];
  const uint32_t n = cum + d.sink_rows + d.n_rec;
  const uint32_t* lst = lstart + size_t(unit) * (d.c_cap + 1);
  uint32_t* rr = runs.row + size_t(h) * runs.run_cap;
  uint32_t* ro = runs.off + size_t(h) * (runs.run_cap + 1);
  for (uint32_t i = tid; i < taken; i += SR_THREADS) {
    rr[i] = d.row_base + __ldg(lst + id[i]);
    ro[i] = loc[i];
  }
  if (tid == 0) {
    uint32_t nr = taken;
    if (d.sink_rows) { rr[nr] = 0; ro[nr] = cum; ++nr; }
    if (d.n_rec) { rr[nr] = d.rec_row; ro[nr] = cum + d.sink_rows; ++nr; }
    ro[nr] = n;
    runs.count[h] = nr;
    n_tokens[h] = n;
    n_taken[h] = taken;
    trimmed_out[h] = trimmed;
  }
  const uint32_t n_rank = (d.flags & CKV_SEL_FULL_RANK) ? C : taken;
  for (uint32_t i = tid; i < n_rank; i += SR_THREADS) ranked[size_t(h) * d.c_cap + i] = id[i];
  if (token_ids) {  // reference positions of this rank's I_T entries
    uint32_t* out = token_ids + size_t(h) * d.sel_cap;
    const uint32_t* sid = lsorted + size_t(unit) * d.n_local;
    for (uint32_t e = tid; e < cum; e += SR_THREADS) {
      uint32_t lo = 0, hi = taken;  // last run i with loc[i] <= e
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (loc[mid] <= e) lo = mid; else hi = mid;
      }
      while (loc[lo + 1] <= e) ++lo;  // skip empty shares
      out[e] = d.pos_base + __ldg(sid + __ldg(lst + id[lo]) + (e - loc[lo]));
    }
    for (uint32_t s2 = tid; s2 < d.sink_rows; s2 += SR_THREADS) out[cum + s2] = s2;
    for (uint32_t i = tid; i < d.n_rec; i += SR_THREADS) out[cum + d.sink_rows + i] = d.rec_pos + i;
  }
}

__global__ void __launch_bounds__(SR_THREADS)
k_select_approx(ckv_shard_select_desc d, uint32_t p2, const float* __restrict__ ascores,
                const float* __restrict__ q, const float* __restrict__ cents,
                const uint32_t* __restrict__ gsize, const uint32_t* __restrict__ lsize,
                const uint32_t* __restrict__ lstart, const uint32_t* __restrict__ prefix,
                const uint32_t* __restrict__ lsorted, ckv_runs runs,
                uint32_t* __restrict__ token_ids, uint32_t* __restrict__ n_tokens,
                uint32_t* __restrict__ n_taken, uint32_t* __restrict__ trimmed_out,
                uint32_t* __restrict__ ranked) {
  // ascores: [world][2][n_q][slice] — approximate score a and its rigorous
  // bound e (|a - s| <= e, s = dot_f64) of every cluster, all-gathered.  The
  // cutoff is found on a (size-weighted radix select), then only the
  // clusters that can reach the exact taken prefix, S = {c : a_c + e_c >= L}
  // with L = min over the approximate top set of (a - e), are re-scored
  // exactly (the replicated centroids) and ranked: the exact prefix lies in S
  // and ranks before everything outside it (the argument of k_select_warp,
  // ckv_select.cu).  FULL_RANK, non-finite scores, a total below B or an
  // oversized S take the exhaustive exact path.
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smraw);  // [p2]
  uint32_t* id = reinterpret_cast<uint32_t*>(key + p2);                     // [p2]
  uint32_t* incl = id + p2;                                                 // [p2]
  uint32_t* loc = incl + p2;                                                // [p2 + 1]
  uint32_t* sz = loc + p2 + 1;                                              // [p2]
  // the approximate scores and bounds share the key array's bytes: they are
  // last read (the candidate set S) before the barrier that precedes the
  // first key write, and the exhaustive path never reads them (a quarter
  // less shared memory per head: 4 instead of 3 heads per SM at C = 1638)
  float* av = reinterpret_cast<float*>(smraw);                              // [p2]
  float* ev = av + p2;                                                      // [p2]
  __shared__ uint32_t s_taken, s_wsum[SR_THREADS / 32], s_hist[256], s_n, s_bin, s_above;
  __shared__ float s_lo[SR_THREADS / 32];
  __shared__ int s_bad;
  __shared__ float qsm[D];
  const uint32_t h = blockIdx.x, unit = h / d.group;
  const uint32_t C = d.C, B = d.budget;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t* gs = gsize + size_t(unit) * d.c_cap;
  const float* cu = cents + size_t(unit) * d.c_cap * D;
  if (tid < D) qsm[tid] = q[size_t(h) * D + tid];
  if (tid == 0) s_bad = 0;
  __syncthreads();
  uint32_t tot = 0;
  int bad = 0;
  for (uint32_t c = tid; c < C; c += SR_THREADS) {
    const uint32_t r = c / d.slice, o = c % d.slice;
    const float a = ascores[((size_t(r) * 2 + 0) * d.n_q + h) * d.slice + o];
    const float e = ascores[((size_t(r) * 2 + 1) * d.n_q + h) * d.slice + o];
    av[c] = a;
    ev[c] = e;
    sz[c] = __ldg(gs + c);
    tot += sz[c];
    bad |= !(isfinite(a) && isfinite(e));
  }
  tot = __reduce_add_sync(0xffffffffu, tot);
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) { s_wsum[wid] = tot; if (bad) s_bad = 1; }
  __syncthreads();
  tot = 0;
  for (int w = 0; w < SR_THREADS / 32; ++w) tot += s_wsum[w];
  __syncthreads();
  auto exact = [&](uint32_t c) {  // dot_f64's sequential chain
    const float4* row = reinterpret_cast<const float4*>(cu + size_t(c) * D);
    double acc = 0.0;
#pragma unroll 4
    for (int j4 = 0; j4 < D / 4; ++j4) {
      const float4 m = __ldg(row + j4);
      acc = __fma_rn(double(qsm[4 * j4 + 0]), double(m.x), acc);
      acc = __fma_rn(double(qsm[4 * j4 + 1]), double(m.y), acc);
      acc = __fma_rn(double(qsm[4 * j4 + 2]), double(m.z), acc);
      acc = __fma_rn(double(qsm[4 * j4 + 3]), double(m.w), acc);
    }
    return acc;
  };
  uint32_t n_sorted = C;
  bool fast = !(d.flags & CKV_SEL_FULL_RANK) && B > 0 && tot >= B && !s_bad;
  if (fast) {
    // ---- size-weighted radix select on the fp32 approximate keys ----------
    uint32_t prefix_k = 0, above = 0;
    s_hist[tid] = 0u;
    __syncthreads();
    for (int pass = 0; pass < 4; ++pass) {
      const int sh = 24 - 8 * pass;
      const uint32_t hm = pass == 0 ? 0u : (~0u << (sh + 8));
      for (uint32_t c = tid; c < C; c += SR_THREADS) {
        const uint32_t k = fkey32(av[c]);
        if (sz[c] && ((k ^ prefix_k) & hm) == 0u) atomicAdd(&s_hist[(k >> sh) & 255u], sz[c]);
      }
      __syncthreads();
      if (wid == 0) {
        uint32_t v[8], ls = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          v[k] = s_hist[255 - 8 * lane - k];
          s_hist[255 - 8 * lane - k] = 0u;
          ls += v[k];
        }
        uint32_t x = ls;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        uint32_t run = above + x - ls;
        int found = -1;
        uint32_t above_sel = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (found < 0 && run + v[k] >= B) { found = 255 - 8 * lane - k; above_sel = run; }
          run += v[k];
        }
        const unsigned f = __ballot_sync(0xffffffffu, found >= 0);
        const int src = __ffs(f) - 1;
        if (lane == src) { s_bin = uint32_t(found); s_above = above_sel; }
      }
      __syncthreads();
      prefix_k |= s_bin << sh;
      above = s_above;
    }
    // ---- L = min over U = {key >= tau} of (a - e); S = {c : a + e >= L} ------
    float lo = INFINITY;
    for (uint32_t c = tid; c < C; c += SR_THREADS)
      if (fkey32(av[c]) >= prefix_k) lo = fminf(lo, av[c] - ev[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    if (lane == 0) s_lo[wid] = lo;
    if (tid == 0) s_n = 0;
    __syncthreads();
    lo = s_lo[0];
    for (int w = 1; w < SR_THREADS / 32; ++w) lo = fminf(lo, s_lo[w]);
    for (uint32_t c = tid; c < C; c += SR_THREADS)
      if (av[c] + ev[c] >= lo) {
        const uint32_t slot = atomicAdd(&s_n, 1u);
        if (slot < uint32_t(SR_THREADS)) loc[slot] = c;
      }
    __syncthreads();
    const uint32_t ns = s_n;
    if (ns <= uint32_t(SR_THREADS)) {
      // ---- exact f64 re-score of S, then its exact order --------------------
      uint32_t n2 = 32;
      while (n2 < ns) n2 <<= 1;
      if (uint32_t(tid) < n2) {
        if (uint32_t(tid) < ns) {
          const uint32_t c = loc[tid];
          key[tid] = rank_key_s(exact(c));
          id[tid] = c;
        } else {
          key[tid] = 0ull;
          id[tid] = 0xffffffffu;
        }
      }
      __syncthreads();
      if (wid == 0) {
        for (uint32_t k = 2; k <= n2; k <<= 1) {
          for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = lane; i < n2; i += 32) {
              const uint32_t ixj = i ^ j;
              if (ixj > i) {
                const unsigned long long ka = key[i], kb = key[ixj];
                const uint32_t ia = id[i], ib = id[ixj];
                const bool asc = (i & k) == 0;
                const bool swap = asc ? before(kb, ib, ka, ia) : before(ka, ia, kb, ib);
                if (swap) { key[i] = kb; key[ixj] = ka; id[i] = ib; id[ixj] = ia; }
              }
            }
            __syncwarp();
          }
        }
      }
      __syncthreads();
      n_sorted = ns;
    } else {
      fast = false;
    }
  }
  if (!fast) {
    // ---- exhaustive: exact f64 scores of every cluster, full sort -------------
    for (uint32_t c = tid; c < p2; c += SR_THREADS) {
      if (c < C) { key[c] = rank_key_s(exact(c)); id[c] = c; }
      else { key[c] = 0ull; id[c] = 0xffffffffu; }
    }
    __syncthreads();
    block_sort(key, id, p2);
    n_sorted = C;
  }
  // inclusive prefix of the global sizes in rank order (chunks of 256)
  if (tid == 0) s_taken = B == 0 ? 0u : n_sorted;  // the reference breaks at cum >= B
  if (n_sorted <= 256) {  // one warp, no block barriers
    if (wid == 0) {
      uint32_t c2 = 0;
      for (uint32_t b = 0; b < n_sorted; b += 32) {
        const uint32_t i = b + lane;
        uint32_t x = i < n_sorted ? sz[id[i]] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (i < n_sorted) incl[i] = c2 + x;
        c2 += __shfl_sync(0xffffffffu, x, 31);
      }
    }
  } else {
    uint32_t carry = 0;
    for (uint32_t b = 0; b < n_sorted; b += SR_THREADS) {
      const uint32_t i = b + tid;
      uint32_t chunk_tot;
      const uint32_t x = block_incl_scan(i < n_sorted ? __ldg(gs + id[i]) : 0u, s_wsum, &chunk_tot);
      if (i < n_sorted) incl[i] = x + carry;
      carry += chunk_tot;
    }
  }
  __syncthreads();
  // taken = first i with incl[i] >= B, plus one (all of C when the total < B)
  for (uint32_t i = tid; i < n_sorted; i += SR_THREADS)
    if (B > 0 && incl[i] >= B && (i == 0 || incl[i - 1] < B)) s_taken = i + 1;
  __syncthreads();
  const uint32_t taken = s_taken;
  const uint32_t full_cum = taken ? incl[taken - 1] : 0;
  const uint32_t trimmed = full_cum > B ? full_cum - B : 0;
  // this rank's share of each taken cluster
  const uint32_t* ls = lsize + size_t(unit) * d.c_cap;
  const uint32_t* pf = prefix + size_t(unit) * d.c_cap;
  for (uint32_t i = tid; i < taken; i += SR_THREADS) {
    const uint32_t c = id[i];
    const uint32_t allow = (i + 1 == taken && trimmed) ? B - (i ? incl[i - 1] : 0u) : __ldg(gs + c);
    const uint32_t p = __ldg(pf + c), l = __ldg(ls + c);
    loc[i] = allow > p ? min(allow - p, l) : 0u;
  }
  __syncthreads();
  // exclusive prefix of the local shares -> run offsets (reuse incl[] as out)
  if (wid == 0) {
    uint32_t c2 = 0;
    for (uint32_t b = 0; b < taken; b += 32) {
      const uint32_t i = b + lane;
      uint32_t x = i < taken ? loc[i] : 0u;
      const uint32_t own = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (i < taken) loc[i] = c2 + x - own;  // exclusive
      c2 += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) loc[taken] = c2;
  }
  __syncthreads();
  const uint32_t cum = loc[taken];
  const uint32_t n = cum + d.sink_rows + d.n_rec;
  const uint32_t* lst = lstart + size_t(unit) * (d.c_cap + 1);
  uint32_t* rr = runs.row + size_t(h) * runs.run_cap;
  uint32_t* ro = runs.off + size_t(h) * (runs.run_cap + 1);
  for (uint32_t i = tid; i < taken; i += SR_THREADS) {
    rr[i] = d.row_base + __ldg(lst + id[i]);
    ro[i] = loc[i];
  }
  if (tid == 0) {
    uint32_t nr = taken;
    if (d.sink_rows) { rr[nr] = 0; ro[nr] = cum; ++nr; }
    if (d.n_rec) { rr[nr] = d.rec_row; ro[nr] = cum + d.sink_rows; ++nr; }
    ro[nr] = n;
    runs.count[h] = nr;
    n_tokens[h] = n;
    n_taken[h] = taken;
    trimmed_out[h] = trimmed;
  }
  const uint32_t n_rank = (d.flags & CKV_SEL_FULL_RANK) ? C : taken;
  for (uint32_t i = tid; i < n_rank; i += SR_THREADS) ranked[size_t(h) * d.c_cap + i] = id[i];
  if (token_ids) {  // reference positions of this rank's I_T entries
    uint32_t* out = token_ids + size_t(h) * d.sel_cap;
    const uint32_t* sid = lsorted + size_t(unit) * d.n_local;
    for (uint32_t e = tid; e < cum; e += SR_THREADS) {
      uint32_t lo = 0, hi = taken;  // last run i with loc[i] <= e
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (loc[mid] <= e) lo = mid; else hi = mid;
      }
      while (loc[lo + 1] <= e) ++lo;  // skip empty shares
      out[e] = d.pos_base + __ldg(sid + __ldg(lst + id[lo]) + (e - loc[lo]));
    }
    for (uint32_t s2 = tid; s2 < d.sink_rows; s2 += SR_THREADS) out[cum + s2] = s2;
    for (uint32_t i = tid; i < d.n_rec; i += SR_THREADS) out[cum + d.sink_rows + i] = d.rec_pos + i;
  }
}


__global__ void k_lse_merge(uint32_t n_q, uint32_t world, uint32_t rank,
                            const float* __restrict__ outs, const float* __restrict__ lses,
                            float* __restrict__ out, float* __restrict__ weights,
                            const uint32_t* __restrict__ n_tokens, uint32_t sel_cap) {
  const uint32_t h = blockIdx.x;
  const int t = threadIdx.x;  // 128 threads = D
  float M = -INFINITY;
  for (uint32_t s = 0; s < world; ++s) M = fmaxf(M, lses[size_t(s) * n_q + h]);
  float L = 0.f, o = 0.f;
  for (uint32_t s = 0; s < world; ++s) {
    const float ls = lses[size_t(s) * n_q + h];
    const float w = ls == -INFINITY ? 0.f : exp2f(ls - M);
    L += w;
    o += w * outs[(size_t(s) * n_q + h) * D + t];
  }
  out[size_t(h) * D + t] = o / L;
  if (weights) {
    const float ls = lses[size_t(rank) * n_q + h];
    const float sc = ls == -INFINITY ? 0.f : exp2f(ls - M) / L;
    float* w = weights + size_t(h) * sel_cap;
    for (uint32_t j = t; j < n_tokens[h]; j += blockDim.x) w[j] *= sc;
  }
}

__global__ void k_fill_empty(uint32_t n_q, float* __restrict__ out, float* __restrict__ lse) {
  const uint32_t h = blockIdx.x;
  out[size_t(h) * D + threadIdx.x] = 0.f;
  if (threadIdx.x == 0) lse[h] = -INFINITY;
}

}  // namespace
}  // namespace ckvb

using namespace ckvb;

extern "C" {

int ckv_score_range(ckv_ctx* ctx, uint32_t n_units, uint32_t group, const float* q,
                    const float* centroids, uint32_t c_cap, uint32_t C, uint32_t c_lo,
                    uint32_t slice, double* scores) {
  if (!ctx || !q || !centroids || !scores) { set_error("ckv_score_range: NULL argument"); return CKV_EINVAL; }
  if (c_cap < C || slice == 0) { set_error("ckv_score_range: need c_cap >= C, slice >= 1"); return CKV_EINVAL; }
  const uint32_t c_hi = c_lo + slice;
  if (n_units == 0 || c_lo >= C) return CKV_OK;
  cudaStream_t st = ctx->stream;
#define CKV_SR(GG)                                                                           \
  case GG: {                                                                                 \
    dim3 grid(n_units, (slice + SR_ROWS - 1) / SR_ROWS);                                     \
    const size_t sm = (SR_ROWS * SR_LD + GG * D) * 4;                                        \
    k_score_range<GG><<<grid, SR_ROWS, sm, st>>>(q, centroids, c_cap, C, c_lo, c_hi, slice,   \
                                                 scores);                                    \
    break;                                                                                   \
  }
  for (const void* fn : {(const void*)k_score_range<1>, (const void*)k_score_range<2>,
                         (const void*)k_score_range<4>, (const void*)k_score_range<8>})
    CKV_CUDA_TRY(smem_optin(fn, (SR_ROWS * SR_LD + 8 * D) * 4));
  switch (group) {
    CKV_SR(1) CKV_SR(2) CKV_SR(4) CKV_SR(8)
    default: set_error("ckv_score_range: group must be 1, 2, 4 or 8"); return CKV_EINVAL;
  }
#undef CKV_SR
  CKV_LAUNCH_CHECK("k_score_range");
  ctx->launches++;
  return CKV_OK;
}

int ckv_select_scored(ckv_ctx* ctx, const ckv_shard_select_desc* d, const double* scores,
                      const uint32_t* gsize, const uint32_t* lsize, const uint32_t* lstart,
                      const uint32_t* prefix, const uint32_t* lsorted, const ckv_runs* runs,
                      uint32_t* token_ids, uint32_t* n_tokens, uint32_t* n_taken,
                      uint32_t* trimmed, uint32_t* ranked) {
  if (!ctx || !d || !scores || !gsize || !lsize || !lstart || !prefix || !runs || !runs->row ||
      !n_tokens || !n_taken || !trimmed || !ranked) {
    set_error("ckv_select_scored: NULL argument");
    return CKV_EINVAL;
  }
  if (d->C == 0 || d->C > 4096 || d->c_cap < d->C || runs->run_cap < d->C + 2 ||
      d->slice * d->world < d->C || (token_ids && !lsorted)) {
    set_error("ckv_select_scored: need 1 <= C <= 4096 <= c_cap, run_cap >= C + 2, "
              "slice * world >= C, lsorted with token_ids");
    return CKV_EINVAL;
  }
  if (token_ids && uint64_t(d->sel_cap) < uint64_t(d->budget) + d->sink_rows + d->n_rec) {
    set_error("ckv_select_scored: sel_cap < budget + sink_rows + n_rec");
    return CKV_EINVAL;
  }
  if (d->n_q == 0) return CKV_OK;
  uint32_t p2 = 32;
  while (p2 < d->C) p2 <<= 1;
  const size_t smem = size_t(p2) * 8 * 2 + size_t(p2) * 4 * 5 + 4 + 8;
  CKV_CUDA_TRY(smem_optin((const void*)k_select_scored, 200 * 1024));
  k_select_scored<<<d->n_q, SR_THREADS, smem, ctx->stream>>>(
      *d, p2, scores, gsize, lsize, lstart, prefix, lsorted, *runs, token_ids, n_tokens, n_taken,
      trimmed, ranked);
  CKV_LAUNCH_CHECK("k_select_scored");
  ctx->launches++;
  return CKV_OK;
}

int ckv_score_range_approx(ckv_ctx* ctx, uint32_t n_units, uint32_t group, const float* q,
                           const float* centroids, uint32_t c_cap, uint32_t C, uint32_t c_lo,
                           uint32_t slice, float* out) {
  if (!ctx || !q || !centroids || !out) {
    set_error("ckv_score_range_approx: NULL argument");
    return CKV_EINVAL;
  }
  if (c_cap < C || slice == 0) {
    set_error("ckv_score_range_approx: need c_cap >= C, slice >= 1");
    return CKV_EINVAL;
  }
  if (n_units == 0 || c_lo >= C) return CKV_OK;
  cudaStream_t st = ctx->stream;
  const uint32_t n_q = n_units * group, c_hi = c_lo + slice;
  for (const void* fn : {(const void*)k_score_range_f32<1>, (const void*)k_score_range_f32<2>,
                         (const void*)k_score_range_f32<4>, (const void*)k_score_range_f32<8>})
    CKV_CUDA_TRY(smem_optin(fn, (SR_ROWS * SR_LD + 8 * D) * 4));
#define CKV_SA(GG)                                                                           \
  case GG: {                                                                                 \
    dim3 grid(n_units, (slice + SR_ROWS - 1) / SR_ROWS);                                     \
    const size_t sm = (SR_ROWS * SR_LD + GG * D) * 4;                                        \
    k_score_range_f32<GG><<<grid, SR_ROWS, sm, st>>>(q, centroids, c_cap, C, c_lo, c_hi,      \
                                                     slice, n_q, out);                       \
    break;                                                                                   \
  }
  switch (group) {
    CKV_SA(1) CKV_SA(2) CKV_SA(4) CKV_SA(8)
    default: set_error("ckv_score_range_approx: group must be 1, 2, 4 or 8"); return CKV_EINVAL;
  }
#undef CKV_SA
  CKV_LAUNCH_CHECK("k_score_range_f32");
  ctx->launches++;
  return CKV_OK;
}

int ckv_select_approx(ckv_ctx* ctx, const ckv_shard_select_desc* d, const float* ascores,
                      const float* q, const float* centroids, const uint32_t* gsize,
                      const uint32_t* lsize, const uint32_t* lstart, const uint32_t* prefix,
                      const uint32_t* lsorted, const ckv_runs* runs, uint32_t* token_ids,
                      uint32_t* n_tokens, uint32_t* n_taken, uint32_t* trimmed,
                      uint32_t* ranked) {
  if (!ctx || !d || !ascores || !q || !centroids || !gsize || !lsize || !lstart || !prefix ||
      !runs || !runs->row || !n_tokens || !n_taken || !trimmed || !ranked) {
    set_error("ckv_select_approx: NULL argument");
    return CKV_EINVAL;
  }
  if (d->C == 0 || d->C > 4096 || d->c_cap < d->C || runs->run_cap < d->C + 2 ||
      d->slice * d->world < d->C || (token_ids && !lsorted)) {
    set_error("ckv_select_approx: need 1 <= C <= 4096 <= c_cap, run_cap >= C + 2, "
              "slice * world >= C, lsorted with token_ids");
    return CKV_EINVAL;
  }
  if (token_ids && uint64_t(d->sel_cap) < uint64_t(d->budget) + d->sink_rows + d->n_rec) {
    set_error("ckv_select_approx: sel_cap < budget + sink_rows + n_rec");
    return CKV_EINVAL;
  }
  if (d->n_q == 0) return CKV_OK;
  uint32_t p2 = 32;
  while (p2 < d->C) p2 <<= 1;
  const size_t smem = size_t(p2) * 8 + size_t(p2) * 4 * 4 + 4 + 16;  // av/ev alias key
  CKV_CUDA_TRY(smem_optin((const void*)k_select_approx, 200 * 1024));
  k_select_approx<<<d->n_q, SR_THREADS, smem, ctx->stream>>>(
      *d, p2, ascores, q, centroids, gsize, lsize, lstart, prefix, lsorted, *runs, token_ids,
      n_tokens, n_taken, trimmed, ranked);
  CKV_LAUNCH_CHECK("k_select_approx");
  ctx->launches++;
  return CKV_OK;
}

int ckv_attend_partial(ckv_ctx* ctx, const ckv_attend_desc* d, const float* q,
                       const uint16_t* K, const uint16_t* V, const ckv_runs* runs,
                       const uint32_t* n_tokens, float* out, float* lse, float* weights) {
  if (!ctx || !d || !runs || !out || !lse) { set_error("ckv_attend_partial: NULL argument"); return CKV_EINVAL; }
  cudaStream_t st = ctx->stream;
  if (d->n_q == 0) return CKV_OK;
  if (d->max_tokens == 0) {  // no local tokens for any q head
    k_fill_empty<<<d->n_q, D, 0, st>>>(d->n_q, out, lse);
    CKV_LAUNCH_CHECK("k_fill_empty");
    ctx->launches++;
    return CKV_OK;
  }
  float *part = nullptr, *lw = nullptr;
  uint32_t* tickets = nullptr;
  CKV_TRY(attend_scratch(ctx, *d, weights != nullptr, &part, &tickets, &lw));
  int rc = launch_attend(st, *d, q, K, V, nullptr, *runs, n_tokens, out, weights, lw, part,
                         tickets, lse);
  ctx->launches++;
  return rc;
}

int ckv_attend_merge(ckv_ctx* ctx, uint32_t n_q, uint32_t world, uint32_t rank,
                     const float* outs, const float* lses, float* out, float* weights,
                     const uint32_t* n_tokens, uint32_t sel_cap) {
  if (!ctx || !outs || !lses || !out || (weights && !n_tokens) || rank >= world) {
    set_error("ckv_attend_merge: bad argument");
    return CKV_EINVAL;
  }
  if (n_q == 0) return CKV_OK;
  k_lse_merge<<<n_q, D, 0, ctx->stream>>>(n_q, world, rank, outs, lses, out, weights, n_tokens,
                                          sel_cap);
  CKV_LAUNCH_CHECK("k_lse_merge");
  ctx->launches++;
  return CKV_OK;
}

}  // extern "C"

// ckv_select.cu — K6 + K8: score_clusters + select_tokens + ClusterCache
// for every q head of a decode step (selection.hpp:50-111, cache.hpp:38-57).
//
// K1 k_score_approx — fp32 GEMV, one warp per 8 centroid rows of a kv unit
//   (one coalesced 512-B row per warp load, 8 rows in flight), all G q heads
//   of the unit per row, so every centroid is read from HBM once.  For each
//   (q head, cluster) it writes the fp32 dot a and a rigorous bound
//   E = 2^-14 |q| |mu| >= |a - s|, where s is the reference's sequential
//   f64 dot_f64 (the fp32 error is <= gamma_9 sum|q_j mu_j|
//   <= gamma_9 |q||mu| by Cauchy-Schwarz, ~60x below E).
// K2 k_select_warp — one warp per q head:
//   1. pop clusters in approximate (a desc, id asc) order until the running
//      size reaches the budget: set U, L = min_{c in U}(a_c - E_c).
//   2. Every cluster of the reference's exact prefix has s >= L (otherwise
//      all of U, whose sizes sum to >= B, would rank before it and it would
//      not be taken), and every cluster with a + E < L ranks strictly after
//      all of them.  So S = {c : a_c + E_c >= L} contains the exact prefix
//      and is exactly ordered against everything outside it.
//   3. S (|U| + a few near-ties) is re-scored with the sequential f64 FMA
//      chain — bit-identical to dot_f64 — ranked by (s desc, id asc), the
//      reference's std::sort comparator (selection.hpp:83-87), and cut at
//      the budget (selection.hpp:91-106).
//   CKV_SEL_FULL_RANK / CKV_SEL_SCORES (the parity API), C > 512, > 64 pops
//   or > 64 candidates take the exhaustive path: exact f64 scores for every
//   cluster and a warp bitonic sort.
//   Output: I_T as runs of the cluster-major KV store (one run per taken
//   cluster, last one trimmed to its lowest positions, then the sink and
//   recency runs), optionally the reference's position list and per-entry
//   rows; the R-step cluster cache (bitmap ring, cache.hpp:38-57) is fused.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ckv_internal.cuh"

namespace ckvb {

constexpr int SC_WARPS = 4;            // K1 warps per CTA
constexpr int SC_ROWS = 8;             // K1 rows per warp
constexpr int SW_WARPS = 4;            // K2 warps (q heads) per CTA
constexpr int SW_KPL = 16;             // approx keys per lane in registers (C <= 512)
constexpr int SW_MAXCAND = 64;         // exact candidates before the exhaustive path
constexpr int SW_STAGE = 32;           // candidate rows staged per pass (16 KB)
constexpr float SEL_ERR = 1.0f / 16384.0f;

__device__ __forceinline__ unsigned long long rank_key(double s) {
  return isnan(s) ? 0ull : dkey(s);  // NaN (empty-cluster centroids) ranks last
}
__device__ __forceinline__ uint32_t fkey(float s) {  // order-preserving f32 -> u32
  const uint32_t u = __float_as_uint(s);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ bool rank_before(unsigned long long ka, uint32_t ia,
                                            unsigned long long kb, uint32_t ib) {
  return ka > kb || (ka == kb && ia < ib);  // selection.hpp:83-87
}
__device__ __forceinline__ void cp_async16_sel(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(valid ? 16 : 0));
}

// ---------------------------------------------------------------------------
// K1
// ---------------------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(SC_WARPS * 32)
k_score_approx(const float* __restrict__ q, const float* __restrict__ cents,
               const uint32_t* __restrict__ n_clusters, uint32_t c_cap, uint32_t c_pad,
               float* __restrict__ aval, float* __restrict__ aerr) {
  const uint32_t unit = blockIdx.x;
  const int lane = lane_id();
  const uint32_t c0 = (blockIdx.y * SC_WARPS + warp_id()) * SC_ROWS;
  // programmatic launch (layer mode): everything read here may come from the
  // previous kernels; the selection kernel may start its own prologue now
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t C = n_clusters[unit];
  if (c0 >= C) return;
  const float* cu = cents + size_t(unit) * c_cap * D;
  float4 m[SC_ROWS];
#pragma unroll
  for (int r = 0; r < SC_ROWS; ++r)
    m[r] = c0 + r < C ? __ldg(reinterpret_cast<const float4*>(cu + size_t(c0 + r) * D) + lane)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 qv[G];
  float qn[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    qv[g] = __ldg(reinterpret_cast<const float4*>(q + (size_t(unit) * G + g) * D) + lane);
    qn[g] = qv[g].x * qv[g].x + qv[g].y * qv[g].y + qv[g].z * qv[g].z + qv[g].w * qv[g].w;
  }
  float dg[SC_ROWS][G], mn[SC_ROWS];
#pragma unroll
  for (int r = 0; r < SC_ROWS; ++r) {
    mn[r] = m[r].x * m[r].x + m[r].y * m[r].y + m[r].z * m[r].z + m[r].w * m[r].w;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float d = qv[g].x * m[r].x;
      d = fmaf(qv[g].y, m[r].y, d);
      d = fmaf(qv[g].z, m[r].z, d);
      dg[r][g] = fmaf(qv[g].w, m[r].w, d);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int g = 0; g < G; ++g) qn[g] += __shfl_xor_sync(0xffffffffu, qn[g], o);
#pragma unroll
    for (int r = 0; r < SC_ROWS; ++r) {
      mn[r] += __shfl_xor_sync(0xffffffffu, mn[r], o);
#pragma unroll
      for (int g = 0; g < G; ++g) dg[r][g] += __shfl_xor_sync(0xffffffffu, dg[r][g], o);
    }
  }
  // every lane holds every sum; lane (r*G + g) stores (row r, head g)
  float qs[G];
#pragma unroll
  for (int g = 0; g < G; ++g) qs[g] = SEL_ERR * sqrtf(qn[g]);
#pragma unroll
  for (int r = 0; r < SC_ROWS; ++r) {
    const float ms = sqrtf(mn[r]);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (lane == ((r * G + g) & 31) && c0 + r < C) {
        const size_t o = (size_t(unit) * G + g) * c_pad + c0 + r;
        aval[o] = dg[r][g];
        aerr[o] = fmaf(qs[g], ms, 1e-30f);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K2
// ---------------------------------------------------------------------------
struct WarpSel {  // per-warp static bookkeeping
  uint32_t cand[SW_MAXCAND];
  unsigned long long ckey[SW_MAXCAND];
  float ca[SW_MAXCAND], ce[SW_MAXCAND];  // the candidates' approximate scores / bounds
  uint32_t hist[256];
};

// per-warp phase timestamps, compiled in with -DCKV_SEL_DEBUG and enabled by
// CKV_DEBUG_TIMING=1 (diagnostics only; absent from the product build)
__device__ unsigned long long* g_sel_dbg = nullptr;
__device__ __forceinline__ void dbg_stamp(uint32_t h, int slot) {
#ifdef CKV_SEL_DEBUG
  if (g_sel_dbg && lane_id() == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_sel_dbg[size_t(h) * 16 + slot] = t;
  }
#else
  (void)h;
  (void)slot;
#endif
}

// The cache state of head h, loaded once up front so the lookups and the
// update need no dependent global round trips: lane w < words holds word w of
// every retained bitmap (R <= 4; more retention reads global memory), lane
// j < 4 holds counter j.
struct SelCachePre {
  uint32_t cbits[4];
  uint32_t rhead, rlen;
  unsigned long long ctr;
  bool creg;
};
__device__ __forceinline__ SelCachePre cache_prefetch(uint32_t h, const CacheDev& cache) {
  SelCachePre p{{0u, 0u, 0u, 0u}, 0u, 0u, 0ull, false};
  if (!cache.bits) return p;
  const int lane = lane_id();
  p.creg = cache.retention <= 4 && cache.words <= 32;
  const uint32_t* bits = cache.bits + size_t(h) * cache.retention * cache.words;
  if (p.creg && uint32_t(lane) < cache.words)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (uint32_t(k) < cache.retention) p.cbits[k] = bits[size_t(k) * cache.words + lane];
  p.rhead = cache.ring[size_t(h) * 2];
  p.rlen = cache.ring[size_t(h) * 2 + 1];
  if (lane < 4) p.ctr = cache.counters[size_t(h) * 4 + lane];
  return p;
}

// The selection of one q head h by one warp.  av / ae: the head's approximate
// scores and their bounds (global scratch after K1, or shared memory in the
// fused kernel); wbase: the warp's private smem (warp_bytes).
// SM_META: sizes / starts point at the unit's shared-memory copies (the
// fused kernel stages them while it scores), else at global memory.
template <bool SM_META>
__device__ __forceinline__ uint32_t meta_ld(const uint32_t* p) {
  if constexpr (SM_META) return *p; else return __ldg(p);
}
template <bool SM_META>
__device__ __forceinline__ void select_head(
    uint32_t h, const ckv_select_desc& desc, uint32_t p2, uint32_t row_base,
    const float* __restrict__ q, const float* __restrict__ cents, const float* av,
    const float* ae, const uint32_t* __restrict__ n_clusters, const uint32_t* __restrict__ sizes,
    const uint32_t* __restrict__ starts, const uint32_t* __restrict__ sorted_ids,
    uint32_t* __restrict__ token_ids, uint32_t* __restrict__ rows_out, const ckv_runs& runs,
    uint32_t* __restrict__ n_tokens, uint32_t* __restrict__ n_taken_out,
    uint32_t* __restrict__ trimmed_out, uint32_t* __restrict__ ranked_out,
    double* __restrict__ scores_out, const CacheDev& cache, const SelCachePre& cpre,
    unsigned char* wbase, WarpSel& ws, uint32_t* ready = nullptr, uint32_t ready_val = 0u) {
  const int lane = lane_id();
  dbg_stamp(h, 0);
  const uint32_t unit = h / desc.group;
  const uint32_t C = n_clusters[unit];
  const uint32_t B = desc.budget;
  unsigned long long* xkey = reinterpret_cast<unsigned long long*>(wbase);  // [p2]
  uint32_t* ids = reinterpret_cast<uint32_t*>(xkey + p2);                    // [p2]
  uint32_t* incl = ids + p2;                                                 // [p2]
  float (*stage)[D] = reinterpret_cast<float (*)[D]>(wbase);                 // [SW_STAGE][D]

  const float* cu = cents + size_t(unit) * desc.c_cap * D;
  const uint32_t* sz = SM_META ? sizes : sizes + size_t(unit) * desc.c_cap;
  const uint32_t* stt = SM_META ? starts : starts + size_t(unit) * (desc.c_cap + 1);
  // SM_META: q points at the head's row in shared memory (the fused kernel
  // staged it), else at the q array in global memory
  const float4* qh4 = reinterpret_cast<const float4*>(SM_META ? q : q + size_t(h) * D);
  auto qld = [&](int j4) -> float4 { if constexpr (SM_META) return qh4[j4]; else return __ldg(qh4 + j4); };
  const bool exhaustive_req = (desc.flags & (CKV_SEL_FULL_RANK | CKV_SEL_SCORES)) != 0;
  // budget 0 takes no cluster (selection.hpp:91: the loop breaks at once);
  // the exhaustive path still ranks every cluster for CKV_SEL_FULL_RANK
  bool fast = !exhaustive_req && C <= 32u * SW_KPL && B > 0;
  uint32_t taken = 0;

  // cluster starts of this lane's 16 columns (runs output; fast path only)
  uint32_t str[SW_KPL];
  const bool creg = cpre.creg;
  uint32_t rhead = cpre.rhead, rlen = cpre.rlen;
  const bool have_str = fast;  // str[] filled below
  if (fast) {
    // ---- 1. a set U of top clusters whose sizes reach B ----------------------
    // Any U with total size >= B gives a valid L = min_U (a - E) (step 2), so
    // U need not be the minimal prefix: a 64-bin histogram of the approximate
    // scores over [min, max] (one pass, a second one inside the boundary bin
    // when it holds many clusters) replaces an exact size-weighted select.
    float ar[SW_KPL], er[SW_KPL];
    uint32_t szr[SW_KPL];
    bool bad = false;  // non-finite scores (NaN centroids): exhaustive path
    float amax = -INFINITY, amin = INFINITY;
    uint32_t total = 0;
#pragma unroll
    for (int k = 0; k < SW_KPL; ++k) {
      const uint32_t c = lane + 32 * k;
      const bool v = c < C;
      ar[k] = v ? av[c] : 0.f;
      er[k] = v ? ae[c] : 0.f;
      szr[k] = v ? meta_ld<SM_META>(sz + c) : 0u;
      str[k] = v ? meta_ld<SM_META>(stt + c) : 0u;
      bad |= v && !(isfinite(ar[k]) && isfinite(er[k]));
      if (v) { amax = fmaxf(amax, ar[k]); amin = fminf(amin, ar[k]); }
      total += szr[k];
    }
    total = __reduce_add_sync(0xffffffffu, total);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      amin = fminf(amin, __shfl_xor_sync(0xffffffffu, amin, o));
    }
    fast = !__any_sync(0xffffffffu, bad);
    dbg_stamp(h, 4);
    // membership code per column: bin (0..63) in pass 1; 64 + sub-bin (0..63)
    // for the boundary bin after pass 2; members: code >= cut
    uint32_t code[SW_KPL];
    uint32_t cut = 0;  // everyone (total <= B, or all scores equal)
    uint32_t* hist = ws.hist;
    // weighted histogram of codes[k] in [base, base + 64) -> the highest bin
    // whose suffix weight (plus `above`) reaches B
    auto pick = [&](uint32_t base, uint32_t above) -> uint32_t {
      hist[2 * lane] = 0u;
      hist[2 * lane + 1] = 0u;
      __syncwarp();
#pragma unroll
      for (int k = 0; k < SW_KPL; ++k)
        if (szr[k] && code[k] >= base && code[k] < base + 64u) atomicAdd(&hist[code[k] - base], szr[k]);
      __syncwarp();
      const uint32_t h0 = hist[2 * lane], h1 = hist[2 * lane + 1];
      uint32_t suf = h0 + h1;  // suffix over lanes >= mine
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf += y;
      }
      suf += above;
      const int my = (suf - h0 >= B) ? 2 * lane + 1 : (suf >= B ? 2 * lane : -1);
      const unsigned f = __ballot_sync(0xffffffffu, my >= 0);
      __syncwarp();
      return f ? base + uint32_t(__shfl_sync(0xffffffffu, my, 31 - __clz(f))) : base;
    };
    if (fast && total > B && amax > amin) {
      const float inv = 64.f / (amax - amin);
#pragma unroll
      for (int k = 0; k < SW_KPL; ++k)
        code[k] = lane + 32 * k < C ? min(63u, uint32_t((ar[k] - amin) * inv)) : 0u;
      const uint32_t b1 = pick(0u, 0u);
      dbg_stamp(h, 5);
      // the boundary bin's population and the weight strictly above it
      uint32_t n_at = 0, above = 0;
      float lo2 = INFINITY, hi2 = -INFINITY;
#pragma unroll
      for (int k = 0; k < SW_KPL; ++k) {
        const bool v = lane + 32 * k < C;
        if (v && code[k] == b1) { ++n_at; lo2 = fminf(lo2, ar[k]); hi2 = fmaxf(hi2, ar[k]); }
        if (v && code[k] > b1) above += szr[k];
      }
      n_at = __reduce_add_sync(0xffffffffu, n_at);
      above = __reduce_add_sync(0xffffffffu, above);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo2 = fminf(lo2, __shfl_xor_sync(0xffffffffu, lo2, o));
        hi2 = fmaxf(hi2, __shfl_xor_sync(0xffffffffu, hi2, o));
      }
      cut = b1;
      if (n_at > 8u && hi2 > lo2) {  // pass 2 inside the boundary bin
        const float inv2 = 64.f / (hi2 - lo2);
#pragma unroll
        for (int k = 0; k < SW_KPL; ++k) {
          const bool v = lane + 32 * k < C;
          code[k] = !v ? 0u : code[k] > b1 ? 128u
                  : code[k] == b1 ? 64u + min(63u, uint32_t((ar[k] - lo2) * inv2)) : 0u;
        }
        cut = pick(64u, above);
      }
    } else {
#pragma unroll
      for (int k = 0; k < SW_KPL; ++k) code[k] = 0u;
    }
    dbg_stamp(h, 6);
    if (fast) {
      // L = min over U of (a - E)
      float lower = INFINITY;
#pragma unroll
      for (int k = 0; k < SW_KPL; ++k) {
        const uint32_t c = lane + 32 * k;
        if (c < C && code[k] >= cut) lower = fminf(lower, ar[k] - er[k]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lower = fminf(lower, __shfl_xor_sync(0xffffffffu, lower, o));
      // ---- 2. candidates S = {c : a + E >= L} -----------------------------------
      uint32_t nc = 0;
#pragma unroll
      for (int k = 0; k < SW_KPL; ++k) {
        const uint32_t c = lane + 32 * k;
        bool in = false;
        if (c < C) in = ar[k] + er[k] >= lower;
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        const uint32_t pos = nc + __popc(bal & ((1u << lane) - 1u));
        if (in && pos < uint32_t(SW_MAXCAND)) {
          ws.cand[pos] = c;
          ws.ca[pos] = ar[k];
          ws.ce[pos] = er[k];
        }
        nc += __popc(bal);
      }
      fast = nc <= uint32_t(SW_MAXCAND);
      __syncwarp();
      // ---- 3a. disjoint bounds: the approximate order IS the exact order ------
      // s_c lies in [a_c - E_c, a_c + E_c]; when no two candidates' intervals
      // meet, s orders S exactly as a does (and no two s tie), so the f64
      // re-score is skipped.  Rank by a (index breaks ties), then test
      // adjacent intervals in that order: if any two intervals meet, some
      // adjacent pair does (an interval meeting a non-neighbour also meets an
      // interval between them).  The test runs in f64, where a_i - a_j and
      // E_i + E_j of fp32 values are exact.
      bool approx_order = false;
      if (fast) {
        float* sa = reinterpret_cast<float*>(ws.ckey);  // [nc] a in rank order
        float* se = sa + SW_MAXCAND;                     // [nc] E in rank order
        for (uint32_t i = lane; i < nc; i += 32) {
          const float ai = ws.ca[i];
          uint32_t r = 0;
          for (uint32_t j = 0; j < nc; ++j) r += ws.ca[j] > ai || (ws.ca[j] == ai && j < i);
          ids[r] = ws.cand[i];
          sa[r] = ai;
          se[r] = ws.ce[i];
        }
        __syncwarp();
        bool meet = false;
        for (uint32_t r = lane; r + 1 < nc; r += 32)
          meet |= double(sa[r]) - double(se[r]) <= double(sa[r + 1]) + double(se[r + 1]);
        approx_order = !__any_sync(0xffffffffu, meet);
        __syncwarp();
      }
      if (fast) {
        dbg_stamp(h, 1);
        // ---- 3. exact f64 re-score of S (rows staged through smem) ---------------
        for (uint32_t b = 0; !approx_order && b < nc; b += SW_STAGE) {
          const uint32_t nb = min(uint32_t(SW_STAGE), nc - b);
          for (uint32_t r = 0; r < nb; ++r)
            cp_async16_sel(&stage[r][4 * lane], cu + size_t(ws.cand[b + r]) * D + 4 * lane, true);
          asm volatile("cp.async.commit_group;\n");
          asm volatile("cp.async.wait_group 0;\n");
          __syncwarp();
          if (uint32_t(lane) < nb) {
            double acc = 0.0;
            const float4* row = reinterpret_cast<const float4*>(&stage[lane][0]);
#pragma unroll 8
            for (int j4 = 0; j4 < D / 4; ++j4) {
              const float4 m = row[j4], qq = qld(j4);
              acc = __fma_rn(double(qq.x), double(m.x), acc);
              acc = __fma_rn(double(qq.y), double(m.y), acc);
              acc = __fma_rn(double(qq.z), double(m.z), acc);
              acc = __fma_rn(double(qq.w), double(m.w), acc);
            }
            ws.ckey[b + lane] = rank_key(acc);
          }
          __syncwarp();
        }
        // exact rank of every candidate within S -> ids[rank]
        for (uint32_t i = lane; !approx_order && i < nc; i += 32) {
          const unsigned long long ki = ws.ckey[i];
          const uint32_t ci = ws.cand[i];
          uint32_t r = 0;
          for (uint32_t j = 0; j < nc; ++j) r += rank_before(ws.ckey[j], ws.cand[j], ki, ci);
          ids[r] = ci;
        }
        __syncwarp();
        // sizes in exact order -> inclusive prefix, cutoff at the budget
        uint32_t carry = 0;
        taken = nc;
        for (uint32_t b = 0; b < nc; b += 32) {
          const uint32_t i = b + lane;
          uint32_t x = i < nc ? meta_ld<SM_META>(sz + ids[i]) : 0u;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          x += carry;
          if (i < nc) incl[i] = x;
          const unsigned hit = __ballot_sync(0xffffffffu, i < nc && x >= B);
          if (hit && taken == nc) taken = b + __ffs(hit);  // first r with incl >= B, plus one
          carry = __shfl_sync(0xffffffffu, x, 31);
        }
        __syncwarp();
      }
    }
  }

  if (!fast) {
    // ---- exhaustive: exact f64 scores for all C + warp bitonic sort -----------
    for (uint32_t c = lane; c < p2; c += 32) {
      if (c < C) {
        const float4* row = reinterpret_cast<const float4*>(cu + size_t(c) * D);
        double acc = 0.0;
#pragma unroll 4
        for (int j4 = 0; j4 < D / 4; ++j4) {
          const float4 m = __ldg(row + j4), qq = qld(j4);
          acc = __fma_rn(double(qq.x), double(m.x), acc);
          acc = __fma_rn(double(qq.y), double(m.y), acc);
          acc = __fma_rn(double(qq.z), double(m.z), acc);
          acc = __fma_rn(double(qq.w), double(m.w), acc);
        }
        xkey[c] = rank_key(acc);
        ids[c] = c;
        if (scores_out) scores_out[size_t(h) * desc.c_cap + c] = acc;
      } else {
        xkey[c] = 0ull;
        ids[c] = 0xffffffffu;  // padding sorts after every real cluster
      }
    }
    __syncwarp();
    for (uint32_t k = 2; k <= p2; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = lane; i < p2; i += 32) {
          const uint32_t ixj = i ^ j;
          if (ixj > i) {
            const unsigned long long ka = xkey[i], kb = xkey[ixj];
            const uint32_t ia = ids[i], ib = ids[ixj];
            const bool asc = (i & k) == 0;
            const bool swap = asc ? rank_before(kb, ib, ka, ia) : rank_before(ka, ia, kb, ib);
            if (swap) { xkey[i] = kb; xkey[ixj] = ka; ids[i] = ib; ids[ixj] = ia; }
          }
        }
        __syncwarp();
      }
    }
    uint32_t carry = 0;
    taken = C;
    for (uint32_t b = 0; b < C; b += 32) {
      const uint32_t i = b + lane;
      uint32_t x = i < C ? meta_ld<SM_META>(sz + ids[i]) : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      x += carry;
      if (i < C) incl[i] = x;
      const unsigned hit = __ballot_sync(0xffffffffu, i < C && x >= B);
      if (hit && taken == C) taken = b + __ffs(hit);
      carry = __shfl_sync(0xffffffffu, x, 31);
    }
    __syncwarp();
  }
  dbg_stamp(h, 2);

  // ---- outputs ---------------------------------------------------------------
  if (B == 0) taken = 0;
  const uint32_t full_cum = taken ? incl[taken - 1] : 0;
  const uint32_t cum = full_cum < B ? full_cum : B;
  const uint32_t trimmed = full_cum > B ? full_cum - B : 0;
  uint32_t* rk = ranked_out + size_t(h) * desc.c_cap;
  const uint32_t n_rank = (!fast && (desc.flags & CKV_SEL_FULL_RANK)) ? C : taken;
  for (uint32_t i = lane; i < n_rank; i += 32) rk[i] = ids[i];
  const uint32_t sinks = desc.sink_count;
  const uint32_t nrec = desc.rec_end > desc.rec_begin ? desc.rec_end - desc.rec_begin : 0;
  const uint32_t n = cum + sinks + nrec;
  // runs: one per taken cluster, then sinks, then recency (selection.hpp:91-109)
  // the start row of cluster c from this warp's registers (lane c % 32 holds
  // str[c / 32]); every lane calls it (shuffles), c ignored when !valid
  auto start_of = [&](uint32_t c, bool valid) -> uint32_t {
    uint32_t v = 0u;
    const uint32_t src = c & 31u, kk = c >> 5;
#pragma unroll
    for (int k = 0; k < SW_KPL; ++k) {
      const uint32_t t2 = __shfl_sync(0xffffffffu, str[k], src);
      if (valid && uint32_t(k) == kk) v = t2;
    }
    return v;
  };
  if (runs.row) {
    uint32_t* rr = runs.row + size_t(h) * runs.run_cap;
    uint32_t* ro = runs.off + size_t(h) * (runs.run_cap + 1);
    if (have_str) {
      for (uint32_t i0 = 0; i0 < taken; i0 += 32) {
        const uint32_t i = i0 + lane;
        const bool v = i < taken;
        const uint32_t st0 = start_of(v ? ids[i] : 0u, v);
        if (v) { rr[i] = row_base + st0; ro[i] = i ? incl[i - 1] : 0u; }
      }
    } else {
      for (uint32_t i = lane; i < taken; i += 32) {
        rr[i] = row_base + meta_ld<SM_META>(stt + ids[i]);
        ro[i] = i ? incl[i - 1] : 0u;
      }
    }
    if (lane == 0) {
      uint32_t nr = taken;
      if (sinks) { rr[nr] = 0; ro[nr] = cum; ++nr; }
      if (nrec) { rr[nr] = desc.rec_begin; ro[nr] = cum + sinks; ++nr; }
      ro[nr] = n;
      runs.count[h] = nr;
    }
  }
  // per-entry outputs (parity / position-ordered stores): flat fill
  uint32_t* out = token_ids ? token_ids + size_t(h) * desc.sel_cap : nullptr;
  uint32_t* rows = rows_out ? rows_out + size_t(h) * desc.sel_cap : nullptr;
  if (out || rows) {
    const uint32_t* sid = sorted_ids + size_t(unit) * desc.p_cap;
    for (uint32_t e0 = 0; e0 < cum; e0 += 128) {
      uint32_t src[4], pos[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t e = e0 + 32 * k + lane;
        uint32_t lo = 0, hi = taken;  // first r with incl[r] > e
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (incl[mid] > e) hi = mid; else lo = mid + 1;
        }
        const uint32_t before = lo ? incl[lo - 1] : 0;
        src[k] = (e < cum && lo < taken) ? meta_ld<SM_META>(stt + ids[lo]) + (e - before) : 0u;
      }
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
    for (uint32_t s2 = lane; s2 < sinks; s2 += 32) {
      if (rows) rows[cum + s2] = s2;
      if (out) out[cum + s2] = s2;
    }
    for (uint32_t i = lane; i < nrec; i += 32) {
      if (rows) rows[cum + sinks + i] = desc.rec_begin + i;
      if (out) out[cum + sinks + i] = desc.rec_begin + i;
    }
  }
  if (lane == 0) {
    n_tokens[h] = n;
    n_taken_out[h] = taken;
    trimmed_out[h] = trimmed;
  }
  // hand head h to the attention (StepSync): every lane's run / count stores
  // are fenced before lane 0's release of the flag
  if (ready) {
    __threadfence();
    __syncwarp();
    if (lane == 0)
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ready + h), "r"(ready_val)
                   : "memory");
  }
  // ---- cache (cache.hpp:38-57) -------------------------------------------------
  // lookup of the taken clusters in the R retained bitmaps, then the taken
  // set replaces the oldest slot (the ring was prefetched with the bitmaps)
  if (cache.bits) {
    const uint32_t W = cache.words, R = cache.retention;
    uint32_t* bits = cache.bits + size_t(h) * R * W;
    uint32_t hits = 0;
    unsigned long long miss_tokens = 0;
    uint32_t slot;
    if (rlen < R) { slot = (rhead + rlen) % R; rlen++; }
    else { slot = rhead; rhead = (rhead + 1) % R; }
    if (creg) {
      uint32_t nw = 0u;  // lane w < W: the new bitmap's word w
      for (uint32_t i0 = 0; i0 < taken; i0 += 32) {
        const uint32_t i = i0 + lane;
        const bool v = i < taken;
        const uint32_t c = v ? ids[i] : 0u;
        bool res = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t wk = __shfl_sync(0xffffffffu, cpre.cbits[k], (c >> 5) & 31u);
          res |= uint32_t(k) < R && ((wk >> (c & 31u)) & 1u);
        }
        if (v) { if (res) ++hits; else miss_tokens += meta_ld<SM_META>(sz + c); }
        for (uint32_t w = 0; w < W; ++w) {
          const uint32_t mw = __reduce_or_sync(0xffffffffu, (v && (c >> 5) == w) ? 1u << (c & 31u) : 0u);
          if (uint32_t(lane) == w) nw |= mw;
        }
      }
      if (uint32_t(lane) < W) bits[size_t(slot) * W + lane] = nw;
    } else {
      for (uint32_t i = lane; i < taken; i += 32) {
        const uint32_t c = ids[i];
        bool res = false;
        for (uint32_t k = 0; k < R; ++k) res |= (bits[size_t(k) * W + (c >> 5)] >> (c & 31)) & 1u;
        if (res) ++hits; else miss_tokens += sz[c];
      }
      __syncwarp();
      uint32_t* sb = bits + size_t(slot) * W;
      for (uint32_t i = lane; i < W; i += 32) sb[i] = 0u;
      __syncwarp();
      for (uint32_t i = lane; i < taken; i += 32) atomicOr(&sb[ids[i] >> 5], 1u << (ids[i] & 31));
    }
    hits = __reduce_add_sync(0xffffffffu, hits);
    miss_tokens = warp_sum(miss_tokens);
    // lane j < 4 holds counter j (prefetched): taken, hits, miss tokens, bytes
    unsigned long long cv = cpre.ctr;
    if (lane == 0) cv += taken;
    if (lane == 1) cv += hits;
    if (lane == 2) cv += miss_tokens;
    const unsigned long long c2 = __shfl_sync(0xffffffffu, cv, 2);
    if (lane == 3) cv = c2 * 2ull * cache.d * 4ull;
    if (lane < 4) cache.counters[size_t(h) * 4 + lane] = cv;
    if (lane == 0) {
      cache.ring[size_t(h) * 2] = rhead;
      cache.ring[size_t(h) * 2 + 1] = rlen;
    }
  }
  dbg_stamp(h, 3);
}

__global__ void __launch_bounds__(SW_WARPS * 32)
k_select_warp(ckv_select_desc desc, uint32_t p2, uint32_t c_pad, uint32_t row_base,
              const float* __restrict__ q, const float* __restrict__ cents,
              const float* __restrict__ aval, const float* __restrict__ aerr,
              const uint32_t* __restrict__ n_clusters, const uint32_t* __restrict__ sizes,
              const uint32_t* __restrict__ starts, const uint32_t* __restrict__ sorted_ids,
              uint32_t* __restrict__ token_ids, uint32_t* __restrict__ rows_out, ckv_runs runs,
              uint32_t* __restrict__ n_tokens, uint32_t* __restrict__ n_taken_out,
              uint32_t* __restrict__ trimmed_out, uint32_t* __restrict__ ranked_out,
              double* __restrict__ scores_out, CacheDev cache, uint32_t warp_bytes,
              uint32_t* __restrict__ ready, const uint32_t* __restrict__ epoch) {
  const int wid = warp_id();
  const uint32_t h = blockIdx.x * SW_WARPS + wid;
  if (h >= desc.n_q) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ WarpSel wsa[SW_WARPS];
  // the cache state is not written by K1: fetched before waiting for it
  const SelCachePre cpre = cache_prefetch(h, cache);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t ready_val = ready ? *epoch + 1u : 0u;  // StepSync (see k_select_fused)
  select_head<false>(h, desc, p2, row_base, q, cents, aval + size_t(h) * c_pad,
                     aerr + size_t(h) * c_pad, n_clusters, sizes, starts, sorted_ids, token_ids,
                     rows_out, runs, n_tokens, n_taken_out, trimmed_out, ranked_out, scores_out,
                     cache, cpre, smraw + size_t(wid) * warp_bytes, wsa[wid], ready, ready_val);
}

// ---------------------------------------------------------------------------
// K1+K2 fused (the decode path): one CTA per kv unit.  All SF_WARPS warps
// score the unit's centroids for its G q heads into shared memory — lane per
// centroid row, a sequential fp32 chain per head (any summation order is
// covered by E, see K1) — then warps 0..G-1 each select one head from those
// scores.  No score round trip through HBM, and 8 warps per unit stream the
// centroids instead of 1 per head.
// ---------------------------------------------------------------------------
constexpr int SF_WARPS = 8;
#ifndef CKV_SEL_FFMA2
#define CKV_SEL_FFMA2 1
#endif
// the unit's centroid block streams through a ring of SF_NS bulk-copied
// stages of SF_ROWS rows (TMA bulk copies: many bytes in flight per CTA
// without registers; the ring aliases the selection warps' buffers, which
// are free while scoring)
constexpr int SF_ROWS = 32;                          // rows per stage (16 KB)
constexpr int SF_NS = 5;                             // stages
constexpr size_t SF_RING = size_t(SF_NS) * SF_ROWS * D * 4;
__device__ __forceinline__ uint32_t sel_su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void sel_mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sel_su32(b)), "r"(n));
}
__device__ __forceinline__ void sel_mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sel_su32(b)) : "memory");
}
__device__ __forceinline__ void sel_mb_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(sel_su32(b)), "r"(parity) : "memory");
  } while (!done);
}
// Ring stages of the unit's centroid block.  The centroids are re-read every
// step: the copy marks them evict_last in L2 (the attention's one-pass KV
// stream is marked evict_first), so they stay resident between steps.
__device__ __forceinline__ void sel_stage_bytes(void* dst, const void* src, uint32_t bytes,
                                                uint64_t* bar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sel_su32(bar)),
               "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(sel_su32(dst)), "l"(src), "r"(bytes), "r"(sel_su32(bar)),
      "l"(pol)
      : "memory");
}
// ring stage k of a unit: rows [k * RPS, k * RPS + RPS) of its f32 (or, H, fp16) block
template <bool H>
__device__ __forceinline__ void sel_stage_chunk(void* ring, uint32_t slot, const float* cu,
                                                const uint16_t* hu, uint32_t k, uint32_t C,
                                                uint64_t* bar) {
  constexpr uint32_t RPS = H ? 64u : 32u, RB = H ? D * 2u : D * 4u;
  const uint32_t n = min(RPS, C - k * RPS);
  char* dst = static_cast<char*>(ring) + size_t(slot) * RPS * RB;
  const char* src = H ? reinterpret_cast<const char*>(hu) : reinterpret_cast<const char*>(cu);
  sel_stage_bytes(dst, src + size_t(k) * RPS * RB, n * RB, bar);
}

// NC > 1 (few units, e.g. one layer's launch): a cluster of NC CTAs per
// unit; CTA r scores the ring chunks r, r + NC, ... and stores its scores
// straight into the leader CTA's shared memory (DSMEM), then the leader's
// G warps select after one cluster barrier.
//
// H (the session's step): the approximate scores come from the fp16 copy of
// the centroids (SelC16: 256 B per row instead of 512, 64 rows per ring
// stage) and each row's bound adds |q| * cerr_c >= |q . (mu_c - h(mu_c))|;
// the exact phase still re-scores from the f32 centroids, so the selection
// is unchanged -- only the candidate band is wider.
template <int G, int NC, bool H>
__global__ void __launch_bounds__(SF_WARPS * 32, 2)  // two units per SM: one wave at config B
k_select_fused(ckv_select_desc desc, uint32_t p2, uint32_t c_pad, uint32_t row_base,
               const float* __restrict__ q, const float* __restrict__ cents,
               const uint16_t* __restrict__ c16, const float* __restrict__ cerr,
               const uint32_t* __restrict__ n_clusters, const uint32_t* __restrict__ sizes,
               const uint32_t* __restrict__ starts, const uint32_t* __restrict__ sorted_ids,
               uint32_t* __restrict__ token_ids, uint32_t* __restrict__ rows_out, ckv_runs runs,
               uint32_t* __restrict__ n_tokens, uint32_t* __restrict__ n_taken_out,
               uint32_t* __restrict__ trimmed_out, uint32_t* __restrict__ ranked_out,
               CacheDev cache, uint32_t warp_bytes, uint32_t mode, float* __restrict__ q_copy,
               uint32_t* __restrict__ ready, const uint32_t* __restrict__ epoch,
               SelAppend app) {
  static_assert(G <= SF_WARPS, "one select warp per head");
  const uint32_t unit = blockIdx.x / NC;
  uint32_t crank = 0;
  if constexpr (NC > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const bool leader = crank == 0;
  const int lane = lane_id(), wid = warp_id();
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ WarpSel wsa[G];
  __shared__ float qn2[G];
  // programmatic stream serialization: launched while the previous kernel
  // (the last step's append / clustering) drains; nothing it writes is read
  // before it completes (a no-op for a normal launch).  CKV_SEL_EARLY: the
  // centroid ring and the sizes / starts are issued before the wait (nothing
  // since the previous selection wrote them).
  const bool early = (desc.flags & CKV_SEL_EARLY) != 0;
  if (!early) asm volatile("griddepcontrol.wait;" ::: "memory");
  const size_t ring_bytes = max(size_t(G) * warp_bytes, SF_RING);
  float* ring = reinterpret_cast<float*>(smraw);                          // [SF_NS][SF_ROWS][D]
  float* av_s = reinterpret_cast<float*>(smraw + ring_bytes);              // [G][c_pad]
  float* ae_s = av_s + size_t(G) * c_pad;                                  // [G][c_pad]
  uint32_t* sz_s = reinterpret_cast<uint32_t*>(ae_s + size_t(G) * c_pad);  // [c_pad]
  uint32_t* st_s = sz_s + c_pad;                                           // [c_pad]
  const uint32_t C = n_clusters[unit];
  const float* cu = cents + size_t(unit) * desc.c_cap * D;
  const uint16_t* hu = H ? c16 + size_t(unit) * desc.c_cap * D : nullptr;
  const float* eu = H ? cerr + size_t(unit) * desc.c_cap : nullptr;
  constexpr uint32_t RPS = H ? 64u : uint32_t(SF_ROWS);  // rows per ring stage (16 KB)
  __shared__ uint64_t full[SF_NS], empty[SF_NS];
  // this CTA's ring chunks: global chunk crank + NC j for j < nloc
  const uint32_t nch = (C + RPS - 1) / RPS;
  const uint32_t nloc = nch > crank ? (nch - crank + NC - 1) / NC : 0u;
  if (threadIdx.x == 0) {
    for (int k = 0; k < SF_NS; ++k) { sel_mb_init(&full[k], 1); sel_mb_init(&empty[k], SF_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint32_t j = 0; j < nloc && j < uint32_t(SF_NS); ++j)
      sel_stage_chunk<H>(ring, j, cu, hu, crank + j * NC, C, &full[j]);
  }
  // the scores go to the leader's copy of av_s / ae_s (its own for NC = 1)
  auto put_score = [&](float* p, float v) {
    if constexpr (NC > 1) {
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ra) : "r"(sel_su32(p)));
      asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(v) : "memory");
    } else {
      *p = v;
    }
  };
  // the unit's sizes / starts land in shared memory while the warps score
  // (4-byte cp.async: the per-unit arrays are not 16-byte aligned)
  if (leader) {
    const uint32_t* szg = sizes + size_t(unit) * desc.c_cap;
    const uint32_t* stg = starts + size_t(unit) * (desc.c_cap + 1);
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(sz_s + c))), "l"(szg + c));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(st_s + c))), "l"(stg + c));
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  if (early) asm volatile("griddepcontrol.wait;" ::: "memory");
  // the step's append (after the wait: the previous step's kernels are done
  // with row pos's neighbours): the last warp copies the unit's new k / v row
  // (16 lanes x 16 B each), in flight beside the q reads below
  if (app.k && leader && wid == SF_WARPS - 1) {
    const uint32_t j = uint32_t(lane) & 15u;
    const uint16_t* src = (lane < 16 ? app.k : app.v) + size_t(unit) * D;
    uint16_t* dst = (lane < 16 ? app.K : app.V) + (size_t(unit) * app.p_cap + app.pos) * D;
    reinterpret_cast<uint4*>(dst)[j] = __ldg(reinterpret_cast<const uint4*>(src) + j);
  }
  // StepSync: the attention may launch now (every CTA of this grid is
  // resident once all have passed here); it waits per q head on ready[]
  uint32_t ready_val = 0u;
  if (ready) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    ready_val = *epoch + 1u;
  }
  if (leader && wid < G) dbg_stamp(unit * G + wid, 7);
  SelCachePre cpre{{0u, 0u, 0u, 0u}, 0u, 0u, 0ull, false};
  if (leader && wid < G && mode != 1) cpre = cache_prefetch(unit * G + wid, cache);
  const float* qu = q + size_t(unit) * G * D;
  // 8 lanes per centroid row (lane sub holds float4 columns sub, sub+8, +16,
  // +24: 128 contiguous bytes per row per load), 4 rows per warp step.
  // The unit's G q rows are read ONCE (warp g reads row g: over PCIe in the
  // session's zero-copy step, where 8 warps each re-reading them cost ~8x
  // the bytes) into shared memory, then every warp takes its operand there.
  __shared__ __align__(16) float q_s[G][D];
  const int sub = lane & 7, rsel = lane >> 3;
  if (wid < G) {
    const float4 qw = __ldg(reinterpret_cast<const float4*>(qu + size_t(wid) * D) + lane);
    reinterpret_cast<float4*>(q_s[wid])[lane] = qw;
    const float s2 = warp_sum(qw.x * qw.x + qw.y * qw.y + qw.z * qw.z + qw.w * qw.w);
    if (lane == 0) qn2[wid] = s2;
    // q read from mapped host memory (the session's zero-copy step): leave a
    // device copy for the attention kernel
    if (q_copy && leader) reinterpret_cast<float4*>(q_copy + (size_t(unit) * G + wid) * D)[lane] = qw;
  }
  __syncthreads();
  // f32 rows: lane sub holds float4 columns sub, sub + 8, + 16, + 24; fp16
  // rows (H): dims [8 sub, 8 sub + 8) and [64 + 8 sub, 64 + 8 sub + 8)
  float4 qv[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      qv[g][k] = reinterpret_cast<const float4*>(q_s[g])[H ? 2 * sub + (k & 1) + 16 * (k >> 1)
                                                           : sub + 8 * k];
  float qnrm[G], qabs[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    qnrm[g] = SEL_ERR * sqrtf(qn2[g]);
    qabs[g] = 1.0001f * sqrtf(qn2[g]);  // >= |q| (the f32 sum's rounding is < 2^-17)
  }
  if (leader && wid < G) dbg_stamp(unit * G + wid, 8);
  // stage k: rows [RPS k, RPS k + RPS); warp w takes rows 4w..4w+3 of it
  // (f32) or 8w..8w+7 as two groups of 4 (H); 8 lanes per row
  constexpr int NSUB = H ? 2 : 1;
  for (uint32_t j = 0; j < nloc; ++j) {
    const uint32_t k = crank + j * NC;
    const uint32_t stg = j % SF_NS, ph = (j / SF_NS) & 1u;
    const uint32_t c0 = k * RPS + uint32_t(wid) * (4 * NSUB);
    float ecv[NSUB];
    if constexpr (H) {
#pragma unroll
      for (int s2 = 0; s2 < NSUB; ++s2) {
        const uint32_t c = c0 + rsel + 4 * s2;
        ecv[s2] = c < C ? __ldg(eu + c) : 0.f;
      }
    }
    float4 m[NSUB][4];
    sel_mb_wait(&full[stg], ph);
    if constexpr (H) {
      const uint16_t* rs = reinterpret_cast<const uint16_t*>(ring) + size_t(stg) * RPS * D;
#pragma unroll
      for (int s2 = 0; s2 < NSUB; ++s2) {
        const uint32_t rr = uint32_t(wid) * 8 + 4 * s2 + rsel;
        uint4 hx[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
        if (c0 + 4 * s2 + rsel < C) {
          hx[0] = reinterpret_cast<const uint4*>(rs + size_t(rr) * D)[sub];
          hx[1] = reinterpret_cast<const uint4*>(rs + size_t(rr) * D)[8 + sub];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 x0 = __half22float2(*reinterpret_cast<const __half2*>(&hx[h].x));
          const float2 x1 = __half22float2(*reinterpret_cast<const __half2*>(&hx[h].y));
          const float2 x2 = __half22float2(*reinterpret_cast<const __half2*>(&hx[h].z));
          const float2 x3 = __half22float2(*reinterpret_cast<const __half2*>(&hx[h].w));
          m[s2][2 * h] = make_float4(x0.x, x0.y, x1.x, x1.y);
          m[s2][2 * h + 1] = make_float4(x2.x, x2.y, x3.x, x3.y);
        }
      }
    } else {
      const float* rs = ring + size_t(stg) * SF_ROWS * D;
      const uint32_t rr = uint32_t(wid) * 4 + rsel;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4)
        m[0][q4] = c0 + rsel < C ? reinterpret_cast<const float4*>(rs + size_t(rr) * D)[sub + 8 * q4]
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // the stage is in registers: release it; thread 0 refills it with
    // stage k + SF_NS once every warp has released it
    __syncwarp();
    if (lane == 0) sel_mb_arrive(&empty[stg]);
    if (threadIdx.x == 0 && j + SF_NS < nloc) {
      sel_mb_wait(&empty[stg], ph);
      sel_stage_chunk<H>(ring, stg, cu, hu, k + SF_NS * NC, C, &full[stg]);
    }
#pragma unroll
    for (int st2 = 0; st2 < NSUB; ++st2) {
      float acc[G], mn;
#if CKV_SEL_FFMA2
      // packed f32 FMAs (FFMA2): even / odd dims in the two halves, one
      // instruction per two products; any summation order stays inside the
      // 2^-14 |q| |row| bound
      {
        float2 a2[G], n2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int g = 0; g < G; ++g) a2[g] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 x = m[st2][k];
          const float2 xl = make_float2(x.x, x.y), xh = make_float2(x.z, x.w);
          n2 = __ffma2_rn(xl, xl, n2);
          n2 = __ffma2_rn(xh, xh, n2);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float4 y = qv[g][k];
            a2[g] = __ffma2_rn(xl, make_float2(y.x, y.y), a2[g]);
            a2[g] = __ffma2_rn(xh, make_float2(y.z, y.w), a2[g]);
          }
        }
        mn = n2.x + n2.y;
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = a2[g].x + a2[g].y;
      }
#else
      mn = 0.f;
#pragma unroll
      for (int g = 0; g < G; ++g) acc[g] = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 x = m[st2][k];
        mn = fmaf(x.x, x.x, fmaf(x.y, x.y, fmaf(x.z, x.z, fmaf(x.w, x.w, mn))));
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float4 y = qv[g][k];
          acc[g] = fmaf(x.x, y.x, fmaf(x.y, y.y, fmaf(x.z, y.z, fmaf(x.w, y.w, acc[g]))));
        }
      }
#endif
      const uint32_t c = c0 + rsel + 4 * st2;
      // the row's bound: 2^-14 |q| |row| (f32 arithmetic) + |q| cerr_c (H: fp16 rows)
      auto bound = [&](float qn, float qa, float mnf) {
        if constexpr (H) return fmaf(qn, sqrtf(mnf), fmaf(qa, ecv[st2], 1e-30f));
        else return fmaf(qn, sqrtf(mnf), 1e-30f);
      };
      if constexpr (G <= 4) {
        // reduce-scatter over the row's 8 lanes: {acc[0..G), mn, 0...} -> lane
        // sub holds the sum of value sub (7 shuffles instead of 3 (G + 1)),
        // then mn is broadcast from lane 4 of the group
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = i < G ? acc[i] : (i == 4 ? mn : 0.f);
        float w[4], x2[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool hi = sub & 4;
          w[i] = (hi ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, hi ? v[i] : v[i + 4], 4);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const bool hi = sub & 2;
          x2[i] = (hi ? w[i + 2] : w[i]) + __shfl_xor_sync(0xffffffffu, hi ? w[i] : w[i + 2], 2);
        }
        const bool hi = sub & 1;
        const float y = (hi ? x2[1] : x2[0]) + __shfl_xor_sync(0xffffffffu, hi ? x2[0] : x2[1], 1);
        const float mnf = __shfl_sync(0xffffffffu, y, (lane & ~7) | 4);
        if (c < C && sub < G) {
          float qn = qnrm[0], qa = qabs[0];
#pragma unroll
          for (int g = 1; g < G; ++g) if (sub == g) { qn = qnrm[g]; qa = qabs[g]; }
          put_score(av_s + size_t(sub) * c_pad + c, y);
          put_score(ae_s + size_t(sub) * c_pad + c, bound(qn, qa, mnf));
        }
        continue;
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        mn += __shfl_xor_sync(0xffffffffu, mn, o);
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], o);
      }
      if (c < C && sub < G) {  // lane sub writes head sub (G <= 8)
        float a = acc[0];
#pragma unroll
        for (int g = 1; g < G; ++g) if (sub == g) a = acc[g];
        float qn = qnrm[0], qa = qabs[0];
#pragma unroll
        for (int g = 1; g < G; ++g) if (sub == g) { qn = qnrm[g]; qa = qabs[g]; }
        put_score(av_s + size_t(sub) * c_pad + c, a);
        put_score(ae_s + size_t(sub) * c_pad + c, bound(qn, qa, mn));
      }
    }
  }
  if (leader && wid < G) dbg_stamp(unit * G + wid, 9);
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  if constexpr (NC > 1) {
    // every CTA's remote score stores are visible to the leader after this
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
    if (!leader) return;
  } else {
    __syncthreads();
  }
  if (wid >= G || mode == 1) return;
  const uint32_t h = unit * G + wid;
  dbg_stamp(h, 10);
  select_head<true>(h, desc, p2, row_base, q_s[wid], cents, av_s + size_t(wid) * c_pad,
                    ae_s + size_t(wid) * c_pad, n_clusters, sz_s, st_s, sorted_ids, token_ids,
                    rows_out, runs, n_tokens, n_taken_out, trimmed_out, ranked_out, nullptr, cache,
                    cpre, smraw + size_t(wid) * warp_bytes, wsa[wid], ready, ready_val);
}

// the fp16 centroid copy of the fused selection (SelC16): one warp per
// centroid row, lane L converts dims 4L..4L+3.  h = RN_fp16(mu) (saturated,
// below-normal flushed: f32_to_f16_tc), and mu - h is exact in f32 for every
// unsaturated component, so cerr = |mu - h|_2 carries only the f32 rounding
// of the sum of squares (< 2^-17 relative; the 1.0001 margin covers it).
__global__ void __launch_bounds__(256)
k_cents_f16(const float* __restrict__ cents, const uint32_t* __restrict__ n_clusters,
            uint32_t c_cap, uint32_t tail, uint16_t* __restrict__ c16, float* __restrict__ cerr) {
  const uint32_t u = blockIdx.y, nc = min(n_clusters[u], c_cap);
  uint32_t c = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (tail) {
    if (c >= tail || c >= nc) return;
    c = nc - 1 - c;
  } else if (c >= nc) {
    return;
  }
  const size_t r = size_t(u) * c_cap + c;
  const float4 x = reinterpret_cast<const float4*>(cents + r * D)[lane];
  const float xs[4] = {x.x, x.y, x.z, x.w};
  uint16_t h[4];
  float e2 = 0.f, e1 = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h[i] = f32_to_f16_tc(xs[i]);
    const float d = __fsub_rn(xs[i], f16_to_f32(h[i]));
    e2 = fmaf(d, d, e2);
    e1 += fabsf(d);
  }
  e2 = warp_sum(e2);
  e1 = warp_sum(e1);
  reinterpret_cast<uint2*>(c16 + r * D)[lane] =
      make_uint2(uint32_t(h[0]) | uint32_t(h[1]) << 16, uint32_t(h[2]) | uint32_t(h[3]) << 16);
  if (lane == 0) {
    // |d|_1 >= |d|_2 stands in where the squares underflow (flushed tiny components)
    float e = e2 >= 1e-30f ? sqrtf(e2) * 1.0001f : e1 * 1.0001f;
    if (!(e <= 3.0e38f)) e = INFINITY;  // overflowed or non-finite: no usable bound
    cerr[r] = e;
  }
}

int launch_cents_f16(cudaStream_t st, const float* cents, const uint32_t* n_clusters,
                     uint32_t n_units, uint32_t c_cap, uint16_t* c16, float* cerr,
                     uint32_t tail) {
  if (n_units == 0 || c_cap == 0) return CKV_OK;
  tail = std::min(tail, c_cap);
  k_cents_f16<<<dim3(((tail ? tail : c_cap) + 7) / 8, n_units), 256, 0, st>>>(
      cents, n_clusters, c_cap, tail, c16, cerr);
  CKV_LAUNCH_CHECK("k_cents_f16");
  return CKV_OK;
}

size_t select_scratch_bytes(uint32_t n_q, uint32_t c_cap) {
  const uint32_t c_pad = (c_cap + 31) / 32 * 32;
  return size_t(n_q) * c_pad * 8 + 64;  // aval + aerr
}

// the fused kernel's per-head stamps: 7 = CTA start, 0 = scores ready,
// 1 = order known, 3 = head done
static void dbg_report_fused(uint32_t n, const unsigned long long* dbuf, float ms) {
  std::vector<unsigned long long> hb(size_t(n) * 16);
  cudaMemcpy(hb.data(), dbuf, hb.size() * 8, cudaMemcpyDeviceToHost);
  double sc = 0, pop = 0, rest = 0;
  unsigned long long t_lo = ~0ull, t_hi = 0, s_hi = 0;
  for (uint32_t h = 0; h < n; ++h) {
    const unsigned long long* x = &hb[size_t(h) * 16];
    sc += double(x[0] - x[7]);
    pop += double(x[1] - x[0]);
    rest += double(x[3] - x[1]);
    t_lo = std::min(t_lo, x[7]);
    t_hi = std::max(t_hi, x[3]);
    s_hi = std::max(s_hi, x[7]);
  }
  fprintf(stderr, "[k_select_fused dbg] %.1f us | per head us: score %.2f pop %.2f rest %.2f | "
          "span %.2f us, last CTA start +%.2f us\n", ms * 1e3, sc / n * 1e-3, pop / n * 1e-3,
          rest / n * 1e-3, double(t_hi - t_lo) * 1e-3, double(s_hi - t_lo) * 1e-3);
  // select_head phases (stamps 0 start, 4 loads, 6 histogram, 1 candidates,
  // 2 exact re-score + prefix, 3 outputs): means, and the heads whose
  // exact phase took > 0.5 us (the f64 re-score ran)
  double ph[5] = {0, 0, 0, 0, 0};
  uint32_t nf = 0, slow = 0;
  for (uint32_t h = 0; h < n; ++h) {
    const unsigned long long* x = &hb[size_t(h) * 16];
    if (!x[1] || !x[4] || !x[6]) continue;
    ++nf;
    ph[0] += double(x[4] - x[0]);
    ph[1] += double(x[6] - x[4]);
    ph[2] += double(x[1] - x[6]);
    ph[3] += double(x[2] - x[1]);
    ph[4] += double(x[3] - x[2]);
    slow += (x[2] - x[1]) > 500ull;
  }
  double pre = 0, loop = 0, bar = 0;
  for (uint32_t h = 0; h < n; ++h) {
    const unsigned long long* x = &hb[size_t(h) * 16];
    pre += double(x[8] - x[7]);
    loop += double(x[9] - x[8]);
    bar += double(x[10] - x[9]);
  }
  fprintf(stderr, "[k_select_fused dbg] scoring phase per head: q / cache prefetch %.2f, "
          "ring loop %.2f, cp.async wait + CTA barrier %.2f us\n", pre / n * 1e-3,
          loop / n * 1e-3, bar / n * 1e-3);
  if (nf)
    fprintf(stderr, "[k_select_fused dbg] fast heads %u/%u: loads %.2f hist %.2f cand %.2f "
            "exact+prefix %.2f outputs %.2f us; exact re-score ran in %u\n", nf, n,
            ph[0] / nf * 1e-3, ph[1] / nf * 1e-3, ph[2] / nf * 1e-3, ph[3] / nf * 1e-3,
            ph[4] / nf * 1e-3, slow);
}

static void dbg_report(uint32_t n, const unsigned long long* dbuf, float k1_ms, float k2_ms) {
  std::vector<unsigned long long> hb(size_t(n) * 16);
  cudaMemcpy(hb.data(), dbuf, hb.size() * 8, cudaMemcpyDeviceToHost);
  double ph[3] = {0, 0, 0};
  uint32_t nfast = 0;
  for (uint32_t b = 0; b < n; ++b) {
    const unsigned long long* x = &hb[size_t(b) * 16];
    if (x[1]) { ph[0] += double(x[1] - x[0]); ph[1] += double(x[2] - x[1]); ++nfast; }
    ph[2] += double(x[3] - x[2]);
  }
  double q[3] = {0, 0, 0};  // loads, pass 1, pass 2 (fast heads)
  for (uint32_t b = 0; b < n; ++b) {
    const unsigned long long* x = &hb[size_t(b) * 16];
    if (x[1] && x[4] && x[6]) {
      q[0] += double(x[4] - x[0]);
      if (x[5]) { q[1] += double(x[5] - x[4]); q[2] += double(x[6] - x[5]); }
    }
  }
  fprintf(stderr, "[k_select dbg] K1 %.1f us K2 %.1f us | K2 per-warp us: pop %.2f (loads %.2f "
          "pass1 %.2f pass2 %.2f) exact %.2f out %.2f | fast %u/%u\n", k1_ms * 1e3, k2_ms * 1e3,
          nfast ? ph[0] / nfast * 1e-3 : 0, nfast ? q[0] / nfast * 1e-3 : 0,
          nfast ? q[1] / nfast * 1e-3 : 0, nfast ? q[2] / nfast * 1e-3 : 0,
          nfast ? ph[1] / nfast * 1e-3 : 0, ph[2] / n * 1e-3, nfast, n);
}

// approximate scores + rigorous bounds of a centroid block (the sharded
// decode step's per-rank slice): cents points at the block's first row of
// unit 0 (unit stride c_cap rows), counts[u] = rows of the block, outputs
// [n_q][c_pad] (K1 above)
int launch_score_approx(cudaStream_t st, uint32_t G, uint32_t n_units, const float* q,
                        const float* cents, const uint32_t* counts, uint32_t c_cap,
                        uint32_t c_pad, float* aval, float* aerr) {
  const dim3 g1(n_units, (c_pad + SC_WARPS * SC_ROWS - 1) / (SC_WARPS * SC_ROWS));
  switch (G) {
    case 1: k_score_approx<1><<<g1, SC_WARPS * 32, 0, st>>>(q, cents, counts, c_cap, c_pad, aval, aerr); break;
    case 2: k_score_approx<2><<<g1, SC_WARPS * 32, 0, st>>>(q, cents, counts, c_cap, c_pad, aval, aerr); break;
    case 4: k_score_approx<4><<<g1, SC_WARPS * 32, 0, st>>>(q, cents, counts, c_cap, c_pad, aval, aerr); break;
    case 8: k_score_approx<8><<<g1, SC_WARPS * 32, 0, st>>>(q, cents, counts, c_cap, c_pad, aval, aerr); break;
    default: set_error("score_approx: group must be 1, 2, 4 or 8"); return CKV_EINVAL;
  }
  CKV_LAUNCH_CHECK("k_score_approx");
  return CKV_OK;
}

int launch_select(cudaStream_t st, const ckv_select_desc& desc, const float* q,
                  const float* cents, const uint32_t* n_clusters, const uint32_t* sizes,
                  const uint32_t* starts, const uint32_t* sorted_ids, uint32_t* token_ids,
                  uint32_t* rows, const ckv_runs& runs, uint32_t row_base, uint32_t* n_tokens,
                  uint32_t* n_taken, uint32_t* trimmed, uint32_t* ranked, double* scores,
                  const CacheDev& cache, void* scratch, float* q_copy, StepSync* sync,
                  const SelC16* c16) {
  const uint32_t G = desc.group;
  if (sync) sync->published = sync->appended = false;
  if (G < 1 || desc.n_q % G || !(G == 1 || G == 2 || G == 4 || G == 8)) {
    set_error("select: group must be 1, 2, 4 or 8 and divide n_q");
    return CKV_EINVAL;
  }
  const uint32_t units = desc.n_q / G;
  const uint32_t c_pad = (desc.c_cap + 31) / 32 * 32;
  float* aval = static_cast<float*>(scratch);
  float* aerr = aval + size_t(desc.n_q) * c_pad;
  static const bool dbg = getenv("CKV_DEBUG_TIMING") != nullptr;
  cudaEvent_t ev[3];
  if (dbg) for (auto& e : ev) cudaEventCreate(&e);
  if (dbg) cudaEventRecord(ev[0], st);
  uint32_t p2 = 64;
  while (p2 < desc.c_cap) p2 <<= 1;
  const uint32_t warp_bytes =
      uint32_t(std::max<size_t>(size_t(p2) * 16, size_t(SW_STAGE) * D * 4));
  // fused (one CTA per unit: score + select) when the units fill the GPU;
  // a layer-sized launch (few units) scores with many CTAs per unit instead
  static const bool unfused = getenv("CKV_SELECT_UNFUSED") != nullptr;
  static const int few_env = getenv("CKV_SEL_FEW") ? atoi(getenv("CKV_SEL_FEW")) : -1;
  // few units: a cluster of nc CTAs per unit (k_select_fused<G, NC>)
  uint32_t nc = 1;
  while (nc < 8 && units * nc * 2 <= uint32_t(num_sms())) nc *= 2;
  static const int nc_env = getenv("CKV_SEL_NC") ? atoi(getenv("CKV_SEL_NC")) : 0;
  if (nc_env == 1 || nc_env == 2 || nc_env == 4 || nc_env == 8) nc = uint32_t(nc_env);
  if (desc.flags & CKV_SEL_FORCE_FUSED) nc = 1;
  const bool few_units = (desc.flags & CKV_SEL_FORCE_FUSED) ? false
                         : few_env >= 0 ? few_env != 0 : (units * 2 < uint32_t(num_sms()) && nc == 1);
  if (!(desc.flags & (CKV_SEL_FULL_RANK | CKV_SEL_SCORES)) && !unfused && !few_units) {
    const size_t smem_f = std::max(size_t(G) * warp_bytes, SF_RING) + size_t(G) * c_pad * 8 +
                          size_t(c_pad) * 8;
    if (smem_f <= 200 * 1024) {
      // the opt-in for the one instantiation launched (a per-call host cost)
      // H: approximate scores from the fp16 centroid copy (session steps)
      const bool hc = c16 && c16->c16 && c16->cerr;
      const uint16_t* c16p = hc ? c16->c16 : nullptr;
      const float* cerrp = hc ? c16->cerr : nullptr;
      {
#define CKV_SF_FN(H_, NC_)                                                                    \
  {(const void*)k_select_fused<1, NC_, H_>, (const void*)k_select_fused<2, NC_, H_>,          \
   (const void*)k_select_fused<4, NC_, H_>, (const void*)k_select_fused<8, NC_, H_>}
        const void* fns[2][4][4] = {
            {CKV_SF_FN(false, 1), CKV_SF_FN(false, 2), CKV_SF_FN(false, 4), CKV_SF_FN(false, 8)},
            {CKV_SF_FN(true, 1), CKV_SF_FN(true, 2), CKV_SF_FN(true, 4), CKV_SF_FN(true, 8)}};
#undef CKV_SF_FN
        const int ni = nc == 1 ? 0 : nc == 2 ? 1 : nc == 4 ? 2 : 3;
        const int gi = G == 1 ? 0 : G == 2 ? 1 : G == 4 ? 2 : 3;
        CKV_CUDA_TRY(smem_optin(fns[hc ? 1 : 0][ni][gi], 200 * 1024));
      }
#define CKV_SF_ARGS desc, p2, c_pad, row_base, q, cents, c16p, cerrp, n_clusters, sizes, starts, sorted_ids, \
    token_ids, rows, runs, n_tokens, n_taken, trimmed, ranked, cache, warp_bytes, sel_mode, q_copy, \
    rdy, ep, sa
      static const uint32_t sel_mode = getenv("CKV_SEL_MODE") ? uint32_t(atoi(getenv("CKV_SEL_MODE"))) : 0u;
      // mode 1 (experiment: scoring only) publishes nothing
      const bool pub = sync && sync->ready && sync->epoch && sel_mode != 1;
      uint32_t* rdy = pub ? sync->ready : nullptr;
      const uint32_t* ep = pub ? sync->epoch : nullptr;
      // the step's append rides along (StepSync sessions only)
      SelAppend sa{nullptr, nullptr, nullptr, nullptr, 0u, 0u};
      if (sync && sync->app_k) {
        sa = SelAppend{sync->app_k, sync->app_v, sync->K, sync->V, sync->app_pos, sync->p_cap};
        sync->appended = true;
      }
      // CKV_SEL_L2_PERSIST: the centroids (read by every step, ~60 MB at
      // config B) are accessed through a persisting L2 window, so the KV
      // stream of the attention between two steps does not evict them and the
      // next select reads them from L2 instead of HBM.
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(units * nc);
      cfg.blockDim = dim3(SF_WARPS * 32);
      cfg.dynamicSmemBytes = smem_f;
      cfg.stream = st;
      // attr[0] the optional L2 window, [1] PDL, [2] the cluster shape
      cudaLaunchAttribute attr[3];
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = 1;
      attr[2].id = cudaLaunchAttributeClusterDimension;
      attr[2].val.clusterDim.x = nc;
      attr[2].val.clusterDim.y = 1;
      attr[2].val.clusterDim.z = 1;
      cfg.attrs = attr + 1;
      cfg.numAttrs = 2;
      if (desc.flags & CKV_SEL_L2_PERSIST) {
        // the device's window limit is fixed: queried once per device
        static int win_dev[64];
        int dev_w = 0;
        cudaGetDevice(&dev_w);
        int& v = win_dev[dev_w & 63];
        if (v == 0) cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, dev_w);
        const size_t max_win = size_t(v);
        const size_t persist = l2_persist_limit();
        const size_t bytes = std::min(max_win, size_t(units) * desc.c_cap * D * (hc ? 2 : 4));
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr =
            hc ? const_cast<void*>(static_cast<const void*>(c16p))
               : const_cast<void*>(static_cast<const void*>(cents));
        attr[0].val.accessPolicyWindow.num_bytes = bytes;
        attr[0].val.accessPolicyWindow.hitRatio =
            bytes ? float(std::min(1.0, double(persist) / double(bytes))) : 0.f;
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = attr;
        cfg.numAttrs = persist && bytes ? 3 : 2;
        if (cfg.numAttrs == 2) cfg.attrs = attr + 1;
      }
      unsigned long long* fbuf = nullptr;
      if (dbg) {
        cudaMalloc(&fbuf, size_t(desc.n_q) * 128);
        cudaMemset(fbuf, 0, size_t(desc.n_q) * 128);
        cudaMemcpyToSymbol(g_sel_dbg, &fbuf, sizeof(fbuf));
      }
#define CKV_SF_CASE(NC_, H_)                                                                     \
  switch (G) {                                                                                   \
    case 1: CKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_select_fused<1, NC_, H_>, CKV_SF_ARGS)); break; \
    case 2: CKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_select_fused<2, NC_, H_>, CKV_SF_ARGS)); break; \
    case 4: CKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_select_fused<4, NC_, H_>, CKV_SF_ARGS)); break; \
    default: CKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_select_fused<8, NC_, H_>, CKV_SF_ARGS)); break; \
  }
#define CKV_SF_NC(H_)                  \
  switch (nc) {                        \
    case 1: CKV_SF_CASE(1, H_) break;  \
    case 2: CKV_SF_CASE(2, H_) break;  \
    case 4: CKV_SF_CASE(4, H_) break;  \
    default: CKV_SF_CASE(8, H_) break; \
  }
      if (hc) { CKV_SF_NC(true) } else { CKV_SF_NC(false) }
#undef CKV_SF_NC
#undef CKV_SF_CASE
#undef CKV_SF_ARGS
      CKV_LAUNCH_CHECK("k_select_fused");
      if (dbg) {
        cudaEventRecord(ev[1], st);
        cudaEventSynchronize(ev[1]);
        float a = 0;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        dbg_report_fused(desc.n_q, fbuf, a);
        unsigned long long z = 0;
        cudaMemcpyToSymbol(g_sel_dbg, &z, sizeof(z));
        cudaFree(fbuf);
        for (auto& e : ev) cudaEventDestroy(e);
      }
      if (pub) sync->published = true;
      return CKV_OK;
    }
  }
  if (q_copy) {  // the unfused kernels read q from the device copy
    CKV_CUDA_TRY(cudaMemcpyAsync(q_copy, q, size_t(desc.n_q) * D * 4, cudaMemcpyDefault, st));
    q = q_copy;
  }
  if (!(desc.flags & (CKV_SEL_FULL_RANK | CKV_SEL_SCORES))) {
    const dim3 g1(units, (c_pad + SC_WARPS * SC_ROWS - 1) / (SC_WARPS * SC_ROWS));
    cudaLaunchConfig_t c1 = {};
    c1.gridDim = g1;
    c1.blockDim = dim3(SC_WARPS * 32);
    c1.stream = st;
    cudaLaunchAttribute a1[1];
    a1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a1[0].val.programmaticStreamSerializationAllowed = 1;
    c1.attrs = a1;
    c1.numAttrs = 1;
    const uint32_t cc = desc.c_cap;
    switch (G) {
      case 1: CKV_CUDA_TRY(cudaLaunchKernelEx(&c1, k_score_approx<1>, q, cents, n_clusters, cc, c_pad, aval, aerr)); break;
      case 2: CKV_CUDA_TRY(cudaLaunchKernelEx(&c1, k_score_approx<2>, q, cents, n_clusters, cc, c_pad, aval, aerr)); break;
      case 4: CKV_CUDA_TRY(cudaLaunchKernelEx(&c1, k_score_approx<4>, q, cents, n_clusters, cc, c_pad, aval, aerr)); break;
      default: CKV_CUDA_TRY(cudaLaunchKernelEx(&c1, k_score_approx<8>, q, cents, n_clusters, cc, c_pad, aval, aerr)); break;
    }
    CKV_LAUNCH_CHECK("k_score_approx");
  }
  if (dbg) cudaEventRecord(ev[1], st);
  const size_t smem = size_t(warp_bytes) * SW_WARPS;
  if (smem > 200 * 1024) {
    set_error("select: cluster capacity too large for the smem ranking buffers");
    return CKV_EINVAL;
  }
  CKV_CUDA_TRY(smem_optin((const void*)k_select_warp, 200 * 1024));
  unsigned long long* dbuf = nullptr;
  if (dbg) {
    cudaMalloc(&dbuf, size_t(desc.n_q) * 128);
    cudaMemset(dbuf, 0, size_t(desc.n_q) * 128);
    cudaMemcpyToSymbol(g_sel_dbg, &dbuf, sizeof(dbuf));
  }
  {
    cudaLaunchConfig_t c2 = {};
    c2.gridDim = dim3((desc.n_q + SW_WARPS - 1) / SW_WARPS);
    c2.blockDim = dim3(SW_WARPS * 32);
    c2.dynamicSmemBytes = smem;
    c2.stream = st;
    cudaLaunchAttribute a2[1];
    a2[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a2[0].val.programmaticStreamSerializationAllowed = 1;
    c2.attrs = a2;
    c2.numAttrs = 1;
    // StepSync as in the fused kernel (not for the parity API's full ranking)
    const bool pub = sync && sync->ready && sync->epoch &&
                     !(desc.flags & (CKV_SEL_FULL_RANK | CKV_SEL_SCORES));
    uint32_t* rdy = pub ? sync->ready : nullptr;
    const uint32_t* ep = pub ? sync->epoch : nullptr;
    CKV_CUDA_TRY(cudaLaunchKernelEx(&c2, k_select_warp, desc, p2, c_pad, row_base, q, cents,
                                    static_cast<const float*>(aval), static_cast<const float*>(aerr),
                                    n_clusters, sizes, starts, sorted_ids, token_ids, rows, runs,
                                    n_tokens, n_taken, trimmed, ranked, scores, cache, warp_bytes,
                                    rdy, ep));
    if (pub) sync->published = true;
  }
  CKV_LAUNCH_CHECK("k_select_warp");
  if (dbg) {
    cudaEventRecord(ev[2], st);
    cudaEventSynchronize(ev[2]);
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    dbg_report(desc.n_q, dbuf, a, b);
    unsigned long long z = 0;
    cudaMemcpyToSymbol(g_sel_dbg, &z, sizeof(z));
    cudaFree(dbuf);
    for (auto& e : ev) cudaEventDestroy(e);
  }
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

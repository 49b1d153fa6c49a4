// ckv_metrics.cu — the harness's quality metrics on the GPU (SURVEY §8f row
// 3; harness.hpp:228-310): the exact top-B ground truth (selection.hpp:
// 115-132 exact_topb), recall (attention.hpp:70-93 recall_rate), full
// attention (attention.hpp:53-60, via ckv_attend over one run) and the output
// error (attention.hpp:101-131 output_error), so quality sweeps over many
// steps and heads run at GPU speed.
//
//   k_exact_topb  one CTA per q head over a POSITION-ordered store: f32
//                 scores of every key with a uniform rigorous bound E =
//                 2^-14 |q| max|k| (>= |a - dot_f64|), a count radix select
//                 of the approximate top-B, then exact f64 re-scoring of
//                 S = {a >= a_cut - 2E} only (it contains the exact top-B and
//                 ranks before everything outside it), an exact radix select
//                 by (score desc, id asc) within S, and the ids ascending.
//                 Bit-exact against the reference (tests/test_gpu_metrics.py).
//   k_recall, k_output_error, k_full_runs: per q head.
#include "ckv_internal.cuh"

namespace ckvb {
namespace {

constexpr int MT_THREADS = 512;
constexpr float MT_ERR = 1.0f / 16384.0f;

__device__ __forceinline__ uint32_t fkey32m(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ffrom32(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ unsigned long long rkey(double s) {
  return isnan(s) ? 0ull : dkey(s);
}

// block-wide count of the selection threshold over `n` keys (8-bit passes,
// `bits` wide keys): the largest k with #(key >= k) >= B; returns k and the
// count strictly above it.  hist: 256 shared counters; one warp scans.
template <typename K, int BITS>
__device__ uint32_t radix_count_select(const K* keys, uint32_t n, uint32_t B, K* cut,
                                       uint32_t* hist) {
  __shared__ uint32_t s_bin, s_above;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  K prefix = 0;
  uint32_t above = 0;
  for (uint32_t i = tid; i < 256; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int pass = 0; pass < BITS / 8; ++pass) {
    const int sh = BITS - 8 - 8 * pass;
    const K hm = pass == 0 ? K(0) : K(~K(0) << (sh + 8));
    for (uint32_t i = tid; i < n; i += blockDim.x)
      if (((keys[i] ^ prefix) & hm) == 0) atomicAdd(&hist[uint32_t(keys[i] >> sh) & 255u], 1u);
    __syncthreads();
    if (wid == 0) {
      uint32_t v[8], ls = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        v[k] = hist[255 - 8 * lane - k];
        hist[255 - 8 * lane - k] = 0u;
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
      if (lane == __ffs(f) - 1) { s_bin = uint32_t(found); s_above = above_sel; }
    }
    __syncthreads();
    prefix |= K(s_bin) << sh;
    above = s_above;
    __syncthreads();
  }
  *cut = prefix;
  return above;
}

__global__ void __launch_bounds__(MT_THREADS)
k_exact_topb(uint32_t group, uint32_t n, uint32_t p_cap, const float* __restrict__ q,
             const uint16_t* __restrict__ keys, uint32_t B, uint32_t* __restrict__ ids_out,
             uint32_t ids_cap, unsigned long long* __restrict__ s_key_g,
             uint32_t* __restrict__ s_id_g) {
  extern __shared__ __align__(16) uint32_t akey[];  // [n] approximate keys
  __shared__ float qs[D];
  __shared__ uint32_t hist[256], s_ns, s_nsel, s_nt;
  __shared__ float s_red[MT_THREADS / 32];
  const uint32_t h = blockIdx.x, unit = h / group;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t Bn = min(B, n);
  if (tid < D) qs[tid] = q[size_t(h) * D + tid];
  __syncthreads();
  // ---- approximate scores: a half-warp per key row (16 lanes x 8 dims) -------
  const uint16_t* ku = keys + size_t(unit) * p_cap * D;
  const int hl = lane & 15;
  float qv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) qv[k] = qs[8 * hl + k];
  float kmax2 = 0.f;
  // both half-warps stay in the loop to the end (the shuffles are warp-wide);
  // a half-warp past the last row scores zeros and stores nothing
  for (uint32_t r0 = (tid >> 5) * 2; r0 < n; r0 += MT_THREADS / 16) {
    const uint32_t r = r0 + ((tid >> 4) & 1);
    const uint4 kv = r < n ? __ldg(reinterpret_cast<const uint4*>(ku + size_t(r) * D) + hl)
                           : make_uint4(0u, 0u, 0u, 0u);
    const float x[8] = {__uint_as_float(kv.x << 16), __uint_as_float(kv.x & 0xffff0000u),
                        __uint_as_float(kv.y << 16), __uint_as_float(kv.y & 0xffff0000u),
                        __uint_as_float(kv.z << 16), __uint_as_float(kv.z & 0xffff0000u),
                        __uint_as_float(kv.w << 16), __uint_as_float(kv.w & 0xffff0000u)};
    float a = 0.f, k2 = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) { a = fmaf(qv[k], x[k], a); k2 = fmaf(x[k], x[k], k2); }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      k2 += __shfl_xor_sync(0xffffffffu, k2, o);
    }
    if (hl == 0 && r < n) akey[r] = fkey32m(a);
    kmax2 = fmaxf(kmax2, k2);
  }
  kmax2 = warp_max(kmax2);
  if (lane == 0) s_red[wid] = kmax2;
  __syncthreads();
  float km = 0.f;
  for (int w = 0; w < MT_THREADS / 32; ++w) km = fmaxf(km, s_red[w]);
  float qn2 = 0.f;
  for (int j = 0; j < D; ++j) qn2 = fmaf(qs[j], qs[j], qn2);
  // |a - s| <= 127 u sum |q_j k_j| <= 2^-17 |q||k|; 2^-14 covers the roundings
  const float E = MT_ERR * sqrtf(qn2) * sqrtf(km) * 1.01f + 1e-30f;
  // ---- approximate cut, then the candidate set S ------------------------------
  uint32_t cut = 0;
  if (Bn < n) radix_count_select<uint32_t, 32>(akey, n, Bn, &cut, hist);
  const float a_cut = Bn < n ? ffrom32(cut) : -INFINITY;
  const float lo = a_cut - 2.f * E;
  if (tid == 0) { s_ns = 0; s_nsel = 0; s_nt = 0; }
  __syncthreads();
  unsigned long long* sk = s_key_g + size_t(h) * n;  // per-head global scratch
  uint32_t* si = s_id_g + size_t(h) * n;
  for (uint32_t r = tid; r < n; r += MT_THREADS) {
    if (Bn < n && !(ffrom32(akey[r]) >= lo)) continue;
    si[atomicAdd(&s_ns, 1u)] = r;
  }
  __syncthreads();
  const uint32_t ns = s_ns;
  // ---- exact f64 scores of S (dot_f64's sequential chain) -------------------
  for (uint32_t i = tid; i < ns; i += MT_THREADS) {
    const uint32_t r = si[i];
    const uint4* kr = reinterpret_cast<const uint4*>(ku + size_t(r) * D);
    double s = 0.0;
    for (int b = 0; b < D / 8; ++b) {
      const uint4 kv = __ldg(kr + b);
      const uint32_t w[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        s = __fma_rn(double(qs[8 * b + 2 * k]), double(__uint_as_float(w[k] << 16)), s);
        s = __fma_rn(double(qs[8 * b + 2 * k + 1]), double(__uint_as_float(w[k] & 0xffff0000u)), s);
      }
    }
    sk[i] = rkey(s);
  }
  __syncthreads();
  // ---- exact top-Bn within S by (score desc, id asc) -------------------------
  unsigned long long ecut = 0;
  uint32_t above = 0;
  if (Bn < ns) above = radix_count_select<unsigned long long, 64>(sk, ns, Bn, &ecut, hist);
  uint32_t* out = ids_out + size_t(h) * ids_cap;
  uint32_t* tie = reinterpret_cast<uint32_t*>(akey);  // akey is free now
  for (uint32_t i = tid; i < ns; i += MT_THREADS) {
    if (Bn >= ns || sk[i] > ecut) out[atomicAdd(&s_nsel, 1u)] = si[i];
    else if (sk[i] == ecut) tie[atomicAdd(&s_nt, 1u)] = si[i];
  }
  __syncthreads();
  if (tid == 0 && Bn < ns) {  // the cut's ties by ascending id (rare beyond one)
    uint32_t k = s_nsel;
    while (k < Bn) {
      uint32_t best = 0xffffffffu, bi = 0;
      for (uint32_t i = 0; i < s_nt; ++i)
        if (tie[i] < best) { best = tie[i]; bi = i; }
      tie[bi] = 0xffffffffu;
      out[k++] = best;
    }
    s_nsel = k;
  }
  __syncthreads();
  (void)above;
  // ---- ids ascending (block bitonic in smem) -----------------------------------
  uint32_t n2 = 1;
  while (n2 < Bn) n2 <<= 1;
  uint32_t* srt = reinterpret_cast<uint32_t*>(akey);
  for (uint32_t i = tid; i < n2; i += MT_THREADS) srt[i] = i < Bn ? out[i] : 0xffffffffu;
  __syncthreads();
  for (uint32_t k = 2; k <= n2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = tid; i < n2; i += MT_THREADS) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint32_t x = srt[i], y = srt[ixj];
          if (((i & k) == 0) == (x > y)) { srt[i] = y; srt[ixj] = x; }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = tid; i < Bn; i += MT_THREADS) out[i] = srt[i];
}

// recall_rate (attention.hpp:70-93): |selected ∩ truth| / |truth|; truth is
// ascending (exact_topb's order), selected ids are distinct
__global__ void k_recall(uint32_t n_q, const uint32_t* __restrict__ sel, uint32_t sel_cap,
                         const uint32_t* __restrict__ n_sel, const uint32_t* __restrict__ truth,
                         uint32_t truth_cap, uint32_t n_truth, double* __restrict__ recall) {
  const uint32_t h = blockIdx.x;
  const uint32_t* t = truth + size_t(h) * truth_cap;
  const uint32_t ns = n_sel[h];
  uint32_t hits = 0;
  for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) {
    const uint32_t x = sel[size_t(h) * sel_cap + i];
    uint32_t lo = 0, hi = n_truth;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (t[mid] < x) lo = mid + 1; else hi = mid;
    }
    hits += lo < n_truth && t[lo] == x;
  }
  hits = __reduce_add_sync(0xffffffffu, hits);
  __shared__ uint32_t s_h[32];
  if (lane_id() == 0) s_h[warp_id()] = hits;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) tot += s_h[w];
    recall[h] = double(tot) / double(n_truth);
  }
}

// output_error (attention.hpp:101-131), the reference's sequential f64 sums
__global__ void k_output_error(uint32_t n_q, const float* __restrict__ approx,
                               const float* __restrict__ exact, double* __restrict__ l2_rel,
                               double* __restrict__ cos_sim) {
  const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= n_q) return;
  double diff2 = 0.0, e2 = 0.0, a2 = 0.0, dot = 0.0;
  for (int i = 0; i < D; ++i) {
    const double a = approx[size_t(h) * D + i], e = exact[size_t(h) * D + i];
    diff2 += (a - e) * (a - e);
    e2 += e * e;
    a2 += a * a;
    dot += a * e;
  }
  const double en = sqrt(e2), an = sqrt(a2);
  l2_rel[h] = en < 1e-12 ? sqrt(diff2) : sqrt(diff2) / en;
  cos_sim[h] = (an < 1e-12 && en < 1e-12) ? 1.0
               : ((an < 1e-12 || en < 1e-12) ? 0.0 : dot / (an * en));
}

__global__ void k_full_runs(uint32_t n_q, uint32_t n, ckv_runs runs, uint32_t* __restrict__ nt) {
  const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= n_q) return;
  runs.row[size_t(h) * runs.run_cap] = 0;
  runs.off[size_t(h) * (runs.run_cap + 1)] = 0;
  runs.off[size_t(h) * (runs.run_cap + 1) + 1] = n;
  runs.count[h] = 1;
  nt[h] = n;
}

}  // namespace
}  // namespace ckvb

using namespace ckvb;

extern "C" {

int ckv_exact_topb(ckv_ctx* ctx, uint32_t n_q, uint32_t group, uint32_t n, uint32_t p_cap,
                   const float* q, const uint16_t* keys, uint32_t budget, uint32_t* ids,
                   uint32_t ids_cap) {
  if (!ctx || !q || !keys || !ids) { set_error("ckv_exact_topb: NULL argument"); return CKV_EINVAL; }
  const uint32_t Bn = std::min(budget, n);
  if (group < 1 || n > p_cap || ids_cap < Bn || n > 49152) {
    set_error("ckv_exact_topb: need group >= 1, n <= p_cap, ids_cap >= min(B, n), n <= 49152");
    return CKV_EINVAL;
  }
  if (n_q == 0 || n == 0 || Bn == 0) return CKV_OK;
  void* sk = nullptr;
  void* si = nullptr;
  CKV_TRY(ctx_scratch(ctx, 27, size_t(n_q) * n * 8, false, &sk));
  CKV_TRY(ctx_scratch(ctx, 28, size_t(n_q) * n * 4, false, &si));
  uint32_t n2 = 1;
  while (n2 < Bn) n2 <<= 1;
  const size_t smem = std::max<size_t>(size_t(n) * 4, size_t(n2) * 4);
  CKV_CUDA_TRY(smem_optin((const void*)k_exact_topb, 200 * 1024));
  k_exact_topb<<<n_q, MT_THREADS, smem, ctx->stream>>>(
      group, n, p_cap, q, keys, budget, ids, ids_cap, static_cast<unsigned long long*>(sk),
      static_cast<uint32_t*>(si));
  CKV_LAUNCH_CHECK("k_exact_topb");
  ctx->launches++;
  return CKV_OK;
}

int ckv_recall(ckv_ctx* ctx, uint32_t n_q, const uint32_t* sel, uint32_t sel_cap,
               const uint32_t* n_sel, const uint32_t* truth, uint32_t truth_cap, uint32_t n_truth,
               double* recall) {
  if (!ctx || !sel || !n_sel || !truth || !recall) { set_error("ckv_recall: NULL argument"); return CKV_EINVAL; }
  if (n_truth == 0) { set_error("recall_rate: truth set must be non-empty"); return CKV_EINVAL; }
  if (n_q == 0) return CKV_OK;
  k_recall<<<n_q, 256, 0, ctx->stream>>>(n_q, sel, sel_cap, n_sel, truth, truth_cap, n_truth,
                                         recall);
  CKV_LAUNCH_CHECK("k_recall");
  ctx->launches++;
  return CKV_OK;
}

int ckv_output_error(ckv_ctx* ctx, uint32_t n_q, const float* approx, const float* exact,
                     double* l2_rel, double* cos_sim) {
  if (!ctx || !approx || !exact || !l2_rel || !cos_sim) { set_error("ckv_output_error: NULL argument"); return CKV_EINVAL; }
  if (n_q == 0) return CKV_OK;
  k_output_error<<<(n_q + 127) / 128, 128, 0, ctx->stream>>>(n_q, approx, exact, l2_rel, cos_sim);
  CKV_LAUNCH_CHECK("k_output_error");
  ctx->launches++;
  return CKV_OK;
}

int ckv_full_runs(ckv_ctx* ctx, uint32_t n_q, uint32_t n, const ckv_runs* runs,
                  uint32_t* n_tokens) {
  if (!ctx || !runs || !runs->row || !n_tokens || runs->run_cap < 1) {
    set_error("ckv_full_runs: bad argument");
    return CKV_EINVAL;
  }
  if (n_q == 0) return CKV_OK;
  k_full_runs<<<(n_q + 127) / 128, 128, 0, ctx->stream>>>(n_q, n, *runs, n_tokens);
  CKV_LAUNCH_CHECK("k_full_runs");
  ctx->launches++;
  return CKV_OK;
}

}  // extern "C"

// ckv_page.cu — the page-select baseline on the GPU (
// selection.hpp:136-194 page_select, the Quest-style comparison point for
// ClusterKV's cluster selection).
//
//   k_page_reps    per (unit, page): the elementwise max / min of the page's
//                  keys (std::max / std::min semantics), once per prefill.
//   k_page_select  one CTA per q head: every page's score with the exact f64
//                  sequential chain (dot_f64 of q and the max representative,
//                  or sum_j max(q_j max_j, q_j min_j) for PageRepr::MaxMin),
//                  the top n_sel = min(n_pages, B / page_size) pages by
//                  (score desc, id asc) through a 64-bit radix select, their
//                  ids ascending, emitted as runs of a position-ordered KV
//                  store (adjacent pages merge), which ckv_attend consumes.
// Bit-exact against the reference's selection (tests/test_gpu_page.py).
#include "ckv_internal.cuh"

namespace ckvb {
namespace {

constexpr int PG_THREADS = 256;

__global__ void __launch_bounds__(256)
k_page_reps(const uint16_t* __restrict__ keys, uint32_t p_cap, uint32_t n, uint32_t page_size,
            uint32_t pages_cap, float* __restrict__ rmax, float* __restrict__ rmin) {
  const uint32_t u = blockIdx.y;
  const uint32_t p = blockIdx.x * (blockDim.x >> 5) + warp_id();
  const uint32_t n_pages = (n + page_size - 1) / page_size;
  if (p >= n_pages) return;
  const int lane = lane_id();
  const uint32_t b = p * page_size, e = min(n, b + page_size);
  const uint2* kb = reinterpret_cast<const uint2*>(keys + size_t(u) * p_cap * D) + lane;
  uint2 v = __ldg(kb + size_t(b) * (D / 4));
  float mx[4] = {__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u),
                 __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u)};
  float mn[4] = {mx[0], mx[1], mx[2], mx[3]};
  for (uint32_t i = b + 1; i < e; ++i) {
    v = __ldg(kb + size_t(i) * (D / 4));
    const float x[4] = {__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u),
                        __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u)};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mx[k] = mx[k] < x[k] ? x[k] : mx[k];  // std::max(max_rep, row)
      mn[k] = x[k] < mn[k] ? x[k] : mn[k];  // std::min(min_rep, row)
    }
  }
  const size_t o = (size_t(u) * pages_cap + p) * D;
  reinterpret_cast<float4*>(rmax + o)[lane] = make_float4(mx[0], mx[1], mx[2], mx[3]);
  if (rmin) reinterpret_cast<float4*>(rmin + o)[lane] = make_float4(mn[0], mn[1], mn[2], mn[3]);
}

__device__ __forceinline__ unsigned long long pkey(double s) {
  return isnan(s) ? 0ull : dkey(s);  // NaN ranks last (never on finite keys)
}

__global__ void __launch_bounds__(PG_THREADS)
k_page_select(ckv_page_desc d, const float* __restrict__ q, const float* __restrict__ rmax,
              const float* __restrict__ rmin, const double* __restrict__ scores, ckv_runs runs,
              uint32_t* __restrict__ token_ids, uint32_t* __restrict__ n_tokens) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const uint32_t n_pages = (d.n + d.page_size - 1) / d.page_size;
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smraw);  // [n_pages]
  uint32_t* sel = reinterpret_cast<uint32_t*>(key + n_pages);               // [n_sel pow2]
  __shared__ uint32_t s_hist[256], s_bin, s_above, s_n, s_nt, s_nrun;
  __shared__ float qs[D];
  const uint32_t h = blockIdx.x, unit = h / d.group;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t n_sel = min(n_pages, d.budget / d.page_size);
  if (tid < D) qs[tid] = q[size_t(h) * D + tid];
  __syncthreads();
  // ---- scores (exact: products of floats are exact in f64, summed in j order)
  const float* rx = rmax + size_t(unit) * d.pages_cap * D;
  const float* rn = rmin ? rmin + size_t(unit) * d.pages_cap * D : nullptr;
  for (uint32_t p = tid; p < n_pages && scores; p += PG_THREADS)  // precomputed (Max)
    key[p] = pkey(scores[size_t(h) * n_pages + p]);
  for (uint32_t p = tid; p < n_pages && !scores; p += PG_THREADS) {
    const float4* mx = reinterpret_cast<const float4*>(rx + size_t(p) * D);
    double s = 0.0;
    if (!d.maxmin) {
#pragma unroll 4
      for (int j4 = 0; j4 < D / 4; ++j4) {
        const float4 m = __ldg(mx + j4);
        s = __fma_rn(double(qs[4 * j4 + 0]), double(m.x), s);
        s = __fma_rn(double(qs[4 * j4 + 1]), double(m.y), s);
        s = __fma_rn(double(qs[4 * j4 + 2]), double(m.z), s);
        s = __fma_rn(double(qs[4 * j4 + 3]), double(m.w), s);
      }
    } else {
      const float4* mn = reinterpret_cast<const float4*>(rn + size_t(p) * D);
#pragma unroll 2
      for (int j4 = 0; j4 < D / 4; ++j4) {
        const float4 a = __ldg(mx + j4), c = __ldg(mn + j4);
        const float av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double x = double(qs[4 * j4 + k]) * double(av[k]);
          const double y = double(qs[4 * j4 + k]) * double(cv[k]);
          s += x < y ? y : x;  // std::max(q max, q min), then the running sum
        }
      }
    }
    key[p] = pkey(s);
  }
  __syncthreads();
  // ---- top n_sel by (score desc, id asc): count radix select on the keys
  unsigned long long prefix_k = 0ull;
  uint32_t above = 0;
  if (n_sel > 0 && n_sel < n_pages) {
    s_hist[tid] = 0u;
    __syncthreads();
    for (int pass = 0; pass < 8; ++pass) {
      const int sh = 56 - 8 * pass;
      const unsigned long long hm = pass == 0 ? 0ull : (~0ull << (sh + 8));
      for (uint32_t p = tid; p < n_pages; p += PG_THREADS)
        if (((key[p] ^ prefix_k) & hm) == 0ull) atomicAdd(&s_hist[(key[p] >> sh) & 255u], 1u);
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
          if (found < 0 && run + v[k] >= n_sel) { found = 255 - 8 * lane - k; above_sel = run; }
          run += v[k];
        }
        const unsigned f = __ballot_sync(0xffffffffu, found >= 0);
        const int src = __ffs(f) - 1;
        if (lane == src) { s_bin = uint32_t(found); s_above = above_sel; }
      }
      __syncthreads();
      prefix_k |= (unsigned long long)s_bin << sh;
      above = s_above;
    }
  }
  // the selected set: keys above the cutoff, then the cutoff's ties in id order
  if (tid == 0) { s_n = 0; s_nt = 0; }
  __syncthreads();
  uint32_t* ties = sel + 4096;  // scratch past the selection (see smem sizing)
  if (n_sel >= n_pages) {
    for (uint32_t p = tid; p < n_pages; p += PG_THREADS) sel[p] = p;
    if (tid == 0) s_n = n_pages;
  } else if (n_sel > 0) {
    for (uint32_t p = tid; p < n_pages; p += PG_THREADS) {
      if (key[p] > prefix_k) sel[atomicAdd(&s_n, 1u)] = p;
      else if (key[p] == prefix_k) ties[atomicAdd(&s_nt, 1u)] = p;
    }
    __syncthreads();
    if (tid == 0) {  // ascending ids among the ties, up to n_sel in total
      uint32_t n = s_n;
      while (n < n_sel) {
        uint32_t best = 0xffffffffu, bi = 0;
        for (uint32_t i = 0; i < s_nt; ++i)
          if (ties[i] < best) { best = ties[i]; bi = i; }
        ties[bi] = 0xffffffffu;
        sel[n++] = best;
      }
      s_n = n;
    }
  }
  __syncthreads();
  const uint32_t ns = s_n;
  // ascending page ids (block bitonic over the padded selection)
  uint32_t n2 = 1;
  while (n2 < ns) n2 <<= 1;
  for (uint32_t i = ns + tid; i < n2; i += PG_THREADS) sel[i] = 0xffffffffu;
  __syncthreads();
  for (uint32_t k = 2; k <= n2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = tid; i < n2; i += PG_THREADS) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint32_t a = sel[i], b = sel[ixj];
          if (((i & k) == 0) == (a > b)) { sel[i] = b; sel[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
  // runs: adjacent pages merge; entry offsets follow the ascending ids
  if (tid == 0) {
    uint32_t* rr = runs.row + size_t(h) * runs.run_cap;
    uint32_t* ro = runs.off + size_t(h) * (runs.run_cap + 1);
    uint32_t nr = 0, off = 0;
    for (uint32_t i = 0; i < ns; ++i) {
      const uint32_t b = sel[i] * d.page_size, e = min(d.n, b + d.page_size);
      if (nr > 0 && rr[nr - 1] + (off - ro[nr - 1]) == b) {
        off += e - b;
        continue;
      }
      rr[nr] = b;
      ro[nr] = off;
      off += e - b;
      ++nr;
    }
    ro[nr] = off;
    runs.count[h] = nr;
    n_tokens[h] = off;
    s_nrun = off;
  }
  __syncthreads();
  if (token_ids) {
    uint32_t* out = token_ids + size_t(h) * d.sel_cap;
    for (uint32_t i = 0; i < ns; ++i) {  // pages in ascending order, a row each per thread
      const uint32_t b = sel[i] * d.page_size, e = min(d.n, b + d.page_size);
      const uint32_t base = i * d.page_size;  // all pages before a partial one are full
      for (uint32_t r = b + tid; r < e; r += PG_THREADS) out[base + (r - b)] = r;
    }
  }
}

}  // namespace
}  // namespace ckvb

using namespace ckvb;

extern "C" {

int ckv_page_reps(ckv_ctx* ctx, uint32_t n_units, uint32_t n, uint32_t p_cap, uint32_t page_size,
                  uint32_t pages_cap, const uint16_t* keys, float* rep_max, float* rep_min) {
  if (!ctx || !keys || !rep_max) { set_error("ckv_page_reps: NULL argument"); return CKV_EINVAL; }
  if (page_size < 1) { set_error("page_select: page_size must be >= 1"); return CKV_EINVAL; }
  const uint32_t n_pages = (n + page_size - 1) / page_size;
  if (n > p_cap || n_pages > pages_cap) {
    set_error("ckv_page_reps: need n <= p_cap and n_pages <= pages_cap");
    return CKV_EINVAL;
  }
  if (n_units == 0 || n == 0) return CKV_OK;
  k_page_reps<<<dim3((n_pages + 7) / 8, n_units), 256, 0, ctx->stream>>>(
      keys, p_cap, n, page_size, pages_cap, rep_max, rep_min);
  CKV_LAUNCH_CHECK("k_page_reps");
  ctx->launches++;
  return CKV_OK;
}

int ckv_page_select(ckv_ctx* ctx, const ckv_page_desc* d, const float* q, const float* rep_max,
                    const float* rep_min, const ckv_runs* runs, uint32_t* token_ids,
                    uint32_t* n_tokens) {
  if (!ctx || !d || !q || !rep_max || !runs || !runs->row || !n_tokens || (d->maxmin && !rep_min)) {
    set_error("ckv_page_select: NULL argument");
    return CKV_EINVAL;
  }
  if (d->page_size < 1) { set_error("page_select: page_size must be >= 1"); return CKV_EINVAL; }
  const uint32_t n_pages = (d->n + d->page_size - 1) / d->page_size;
  const uint32_t n_sel = std::min(n_pages, d->budget / d->page_size);
  if (n_pages > 4096 || n_pages > d->pages_cap || runs->run_cap < n_sel + 1 ||
      (token_ids && d->sel_cap < n_sel * d->page_size)) {
    set_error("ckv_page_select: need n_pages <= 4096 and pages_cap, run_cap > n_sel, "
              "sel_cap >= n_sel * page_size");
    return CKV_EINVAL;
  }
  if (d->n_q == 0) return CKV_OK;
  // keys [n_pages] u64 + selection [4096] + tie scratch [n_pages] u32
  const size_t smem = size_t(n_pages) * 8 + 4096 * 4 + size_t(n_pages) * 4;
  CKV_CUDA_TRY(smem_optin((const void*)k_page_select, 96 * 1024));
  // PageRepr::Max scores are dot_f64(q, max_rep): the register-blocked exact
  // scorer of the sharded path (all G heads of a unit per centroid-row read)
  double* sc = nullptr;
  if (!d->maxmin && (d->group == 1 || d->group == 2 || d->group == 4 || d->group == 8)) {
    void* p = nullptr;
    CKV_TRY(ctx_scratch(ctx, 23, size_t(d->n_q) * n_pages * 8, false, &p));
    sc = static_cast<double*>(p);
    CKV_TRY(ckv_score_range(ctx, d->n_q / d->group, d->group, q, rep_max, d->pages_cap, n_pages,
                            0, n_pages, sc));
  }
  k_page_select<<<d->n_q, PG_THREADS, smem, ctx->stream>>>(*d, q, rep_max, rep_min, sc, *runs,
                                                            token_ids, n_tokens);
  CKV_LAUNCH_CHECK("k_page_select");
  ctx->launches++;
  return CKV_OK;
}

}  // extern "C"

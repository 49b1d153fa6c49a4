// ckv_attend.cu — K7: sparse decode attention over the gathered KV
// (attention.hpp:20-69 attention_over / approx_attention), split-K
// flash-decode with a log-sum-exp merge.
//
// Grid (q head, split).  Each CTA owns a contiguous slice of the q head's
// row list (I_T mapped to KV-store rows) and streams it through a
// STAGES-deep shared-memory ring of 32-row tiles with cp.async (16 B per
// request, L1 bypass).  The whole slice's row ids are staged in smem first,
// so every tile's K/V requests issue back to back without waiting on an id
// load; with the cluster-major store (ckv_session_prefill) the rows of a
// selected cluster are consecutive, so the requests are long contiguous runs.
// Per tile, a half-warp owns one row (16 lanes x 8 bf16 dims): dot product
// (fp32 FMA + 4 shuffles), then an online-softmax update of that half-warp's
// running (m, l, acc[8]).  The eight half-warp states merge in smem, and the
// last CTA of a q head (atomic ticket) merges the split partials in a fixed
// order, so results do not depend on scheduling.
//
// Numerics: fp32 logits / exp2 / sums; the reference uses f64.  Tolerance-
// checked against the oracle (tests/test_gpu_attend.py).
#include "ckv_internal.cuh"

namespace ckvb {

constexpr int AT_THREADS = 128;  // 4 warps = 8 half-warps
constexpr int AT_TILE = 32;      // rows per pipeline stage
constexpr int AT_STAGES = 4;
constexpr int AT_MAX_ROWS = 2048;  // rows per CTA slice (ids staged in smem)
constexpr int PART = 2 + D;        // partial: m (log2 domain), l, acc[128]

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;  // src-size 0 zero-fills
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ float dot8(const uint4 k, const float* qv) {
  float s = 0.f;
  s = fmaf(__uint_as_float(k.x << 16), qv[0], s);
  s = fmaf(__uint_as_float(k.x & 0xffff0000u), qv[1], s);
  s = fmaf(__uint_as_float(k.y << 16), qv[2], s);
  s = fmaf(__uint_as_float(k.y & 0xffff0000u), qv[3], s);
  s = fmaf(__uint_as_float(k.z << 16), qv[4], s);
  s = fmaf(__uint_as_float(k.z & 0xffff0000u), qv[5], s);
  s = fmaf(__uint_as_float(k.w << 16), qv[6], s);
  s = fmaf(__uint_as_float(k.w & 0xffff0000u), qv[7], s);
  return s;
}

__device__ __forceinline__ void axpy8(float p, const uint4 v, float* acc) {
  acc[0] = fmaf(p, __uint_as_float(v.x << 16), acc[0]);
  acc[1] = fmaf(p, __uint_as_float(v.x & 0xffff0000u), acc[1]);
  acc[2] = fmaf(p, __uint_as_float(v.y << 16), acc[2]);
  acc[3] = fmaf(p, __uint_as_float(v.y & 0xffff0000u), acc[3]);
  acc[4] = fmaf(p, __uint_as_float(v.z << 16), acc[4]);
  acc[5] = fmaf(p, __uint_as_float(v.z & 0xffff0000u), acc[5]);
  acc[6] = fmaf(p, __uint_as_float(v.w << 16), acc[6]);
  acc[7] = fmaf(p, __uint_as_float(v.w & 0xffff0000u), acc[7]);
}

struct AttSmem {
  uint4 k[AT_STAGES][AT_TILE][16];  // 16 KB
  uint4 v[AT_STAGES][AT_TILE][16];  // 16 KB
  uint32_t ids[AT_MAX_ROWS];        // 8 KB
  float hm[8], hl[8];
  float hacc[8][D];
  uint32_t last;
};

__global__ void __launch_bounds__(AT_THREADS, 4)
k_attend(ckv_attend_desc desc, uint32_t splits, const float* __restrict__ q,
         const uint16_t* __restrict__ K, const uint16_t* __restrict__ V,
         const uint32_t* __restrict__ rows, const uint32_t* __restrict__ n_tokens,
         float* __restrict__ out, float* __restrict__ logits_ws, float* __restrict__ part,
         uint32_t* __restrict__ tickets, float* __restrict__ weights) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  AttSmem& sm = *reinterpret_cast<AttSmem*>(sm_raw);
  const uint32_t h = blockIdx.x, split = blockIdx.y;
  const uint32_t nt = n_tokens[h];
  // balanced slices: split s covers [nt*s/S, nt*(s+1)/S)
  const uint32_t r0 = uint32_t((uint64_t(nt) * split) / splits);
  const uint32_t r1 = uint32_t((uint64_t(nt) * (split + 1)) / splits);
  const uint32_t nr = r1 - r0;
  const int t = threadIdx.x;
  const uint32_t unit = h / desc.group;
  const uint16_t* Ku = K + size_t(unit) * desc.p_cap * D;
  const uint16_t* Vu = V + size_t(unit) * desc.p_cap * D;

  const uint32_t* rl = rows + size_t(h) * desc.sel_cap + r0;
  for (uint32_t i = t; i < nr; i += AT_THREADS) sm.ids[i] = __ldg(rl + i);
  __syncthreads();

  const uint32_t n_tiles = (nr + AT_TILE - 1) / AT_TILE;
  auto issue = [&](uint32_t tile) {
    const int st = tile % AT_STAGES;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = t + AT_THREADS * k;  // 0..511: row e/16, 16-B column e%16
      const int r = e >> 4, c = e & 15;
      const uint32_t gr = tile * AT_TILE + r;
      const bool ok = gr < nr;
      const size_t row = ok ? sm.ids[gr] : 0;
      cp_async16(&sm.k[st][r][c], reinterpret_cast<const uint4*>(Ku + row * D) + c, ok);
      cp_async16(&sm.v[st][r][c], reinterpret_cast<const uint4*>(Vu + row * D) + c, ok);
    }
  };
#pragma unroll
  for (int s = 0; s < AT_STAGES - 1; ++s) {
    if (uint32_t(s) < n_tiles) issue(s);
    cp_async_commit();
  }

  const int hw = t >> 4;  // half-warp 0..7
  const int hl = t & 15;  // dims [8*hl, 8*hl+8)
  const float qscale = 1.4426950408889634f * rsqrtf(float(D));  // exp -> exp2
  float qv[8];
  {
    const float4* qp = reinterpret_cast<const float4*>(q + size_t(h) * D + 8 * hl);
    const float4 a = __ldg(qp), b = __ldg(qp + 1);
    qv[0] = a.x * qscale; qv[1] = a.y * qscale; qv[2] = a.z * qscale; qv[3] = a.w * qscale;
    qv[4] = b.x * qscale; qv[5] = b.y * qscale; qv[6] = b.z * qscale; qv[7] = b.w * qscale;
  }
  float m = -INFINITY, l = 0.f;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float* lw = logits_ws ? logits_ws + size_t(h) * desc.sel_cap + r0 : nullptr;

  for (uint32_t tile = 0; tile < n_tiles; ++tile) {
    cp_async_wait<AT_STAGES - 2>();
    __syncthreads();  // tile's bytes visible to all; the stage refilled below is free
    if (tile + AT_STAGES - 1 < n_tiles) issue(tile + AT_STAGES - 1);
    cp_async_commit();
    const int st = tile % AT_STAGES;
    // this half-warp's 4 rows of the tile: hw, hw+8, hw+16, hw+24
    float s[4];
    uint4 vv[4];
    float tmax = -INFINITY;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = hw + 8 * k;
      const uint4 kk = sm.k[st][r][hl];
      vv[k] = sm.v[st][r][hl];
      float x = dot8(kk, qv);
      x += __shfl_xor_sync(0xffffffffu, x, 8);
      x += __shfl_xor_sync(0xffffffffu, x, 4);
      x += __shfl_xor_sync(0xffffffffu, x, 2);
      x += __shfl_xor_sync(0xffffffffu, x, 1);
      const bool ok = tile * AT_TILE + r < nr;
      s[k] = ok ? x : -INFINITY;
      if (lw && ok && hl == 0) lw[tile * AT_TILE + r] = x;
      tmax = fmaxf(tmax, s[k]);
    }
    const float mn = fmaxf(m, tmax);
    if (mn != -INFINITY) {
      const float sc = exp2f(m - mn);  // m = -inf -> 0
      l *= sc;
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] *= sc;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float p = exp2f(s[k] - mn);
        l += p;
        axpy8(p, vv[k], acc);
      }
      m = mn;
    }
  }
  cp_async_wait<0>();

  // merge the 8 half-warp states of this CTA
  if (hl == 0) { sm.hm[hw] = m; sm.hl[hw] = l; }
#pragma unroll
  for (int i = 0; i < 8; ++i) sm.hacc[hw][8 * hl + i] = acc[i];
  __syncthreads();
  float M = sm.hm[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) M = fmaxf(M, sm.hm[i]);
  float* pp = part + (size_t(h) * splits + split) * PART;
  {
    float a = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float w = sm.hm[i] == -INFINITY ? 0.f : exp2f(sm.hm[i] - M);
      a += sm.hacc[i][t] * w;
    }
    pp[2 + t] = a;  // AT_THREADS == D
  }
  if (t == 0) {
    float ls = 0.f;
    for (int i = 0; i < 8; ++i) ls += sm.hm[i] == -INFINITY ? 0.f : sm.hl[i] * exp2f(sm.hm[i] - M);
    pp[0] = M;
    pp[1] = ls;
  }
  // ---- the last CTA of this q head merges the split partials ----------------
  __threadfence();
  __syncthreads();
  if (t == 0) sm.last = (atomicAdd(&tickets[h], 1u) == splits - 1);
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  const float* pb = part + size_t(h) * splits * PART;
  float MM = -INFINITY;
  for (uint32_t c = 0; c < splits; ++c) MM = fmaxf(MM, __ldcg(pb + c * PART));
  float L = 0.f, o = 0.f;
  for (uint32_t c = 0; c < splits; ++c) {
    const float mc = __ldcg(pb + c * PART);
    const float w = mc == -INFINITY ? 0.f : exp2f(mc - MM);
    L += __ldcg(pb + c * PART + 1) * w;
    o += __ldcg(pb + c * PART + 2 + t) * w;
  }
  const float invL = 1.f / L;
  out[size_t(h) * D + t] = o * invL;
  if (weights) {
    const float* lg = logits_ws + size_t(h) * desc.sel_cap;
    float* wo = weights + size_t(h) * desc.sel_cap;
    for (uint32_t i = t; i < nt; i += AT_THREADS) wo[i] = exp2f(__ldcg(lg + i) - MM) * invL;
  }
  if (t == 0) tickets[h] = 0;  // re-arm for the next launch
}

uint32_t attend_splits(const ckv_attend_desc& d) {
  // aim for >= ~4 CTAs per SM worth of work, slices of <= AT_MAX_ROWS rows
  uint32_t s = 1;
  const uint32_t want = uint32_t(num_sms()) * 8;
  while (d.n_q * s < want && s < 16 && d.max_tokens / (2 * s) >= 256) s *= 2;
  while ((d.max_tokens + s - 1) / s > AT_MAX_ROWS) ++s;
  return s;
}

int launch_attend(cudaStream_t st, const ckv_attend_desc& desc, const float* q,
                  const uint16_t* K, const uint16_t* V, const uint32_t* rows,
                  const uint32_t* n_tokens, float* out, float* weights, float* logits_ws,
                  float* part, uint32_t* tickets) {
  if (desc.n_q == 0 || desc.max_tokens == 0) return CKV_OK;
  const uint32_t splits = attend_splits(desc);
  const size_t smem = sizeof(AttSmem);
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    CKV_CUDA_TRY(cudaFuncSetAttribute(k_attend, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem)));
    attr_dev = dev;
  }
  dim3 grid(desc.n_q, splits);
  k_attend<<<grid, AT_THREADS, smem, st>>>(desc, splits, q, K, V, rows, n_tokens, out,
                                           weights ? logits_ws : nullptr, part, tickets,
                                           weights);
  CKV_LAUNCH_CHECK("k_attend");
  return CKV_OK;
}

size_t attend_part_floats(uint32_t n_q, uint32_t max_tokens) {
  ckv_attend_desc d{};
  d.n_q = n_q;
  d.max_tokens = max_tokens;
  return size_t(n_q) * attend_splits(d) * PART;
}

}  // namespace ckvb

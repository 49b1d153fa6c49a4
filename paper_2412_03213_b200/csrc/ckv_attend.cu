// ckv_attend.cu — K7: sparse decode attention over the gathered KV
// (attention.hpp:20-69 attention_over / approx_attention), split-K
// flash-decode with a log-sum-exp merge.
//
// Grid (q head, 128-row chunk of I_T).  256 threads: a half-warp owns one
// I_T row per step, each lane 16 B (8 bf16 dims) of it, so every K / V row
// (256 B each) is one fully-coalesced 256 B request.  All 8 K rows and 8 V
// rows a thread needs are issued before any is consumed (16 x 128-bit
// loads in flight per thread, 64 KB per CTA) — the kernel is HBM-bound and
// latency hiding is the whole game.  The last CTA to finish a q head
// (atomic ticket) merges the chunk partials in a fixed order, so the result
// does not depend on scheduling.
//
// Numerics: logits, softmax and the weighted sum in f32 with exp2; the
// reference uses f64 (attention.hpp:28-47).  Tolerance-checked.
#include "ckv_internal.cuh"

namespace ckvb {

constexpr int ATT_ROWS = 128;     // rows per CTA
constexpr int ATT_THREADS = 256;  // 16 half-warps x 8 rows each

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
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

// partial layout per (q, chunk): [0]=m (log2 domain), [1]=l, [2..129]=acc
constexpr int PART = 2 + D;

__global__ void __launch_bounds__(ATT_THREADS, 2)
k_attend(ckv_attend_desc desc, const float* __restrict__ q, const uint16_t* __restrict__ K,
         const uint16_t* __restrict__ V, const uint32_t* __restrict__ token_ids,
         const uint32_t* __restrict__ n_tokens, float* __restrict__ out,
         float* __restrict__ logits_ws, float* __restrict__ part,
         uint32_t* __restrict__ tickets, float* __restrict__ weights) {
  const uint32_t h = blockIdx.x, chunk = blockIdx.y;
  const uint32_t nt = n_tokens[h];
  const uint32_t n_chunks = (nt + ATT_ROWS - 1) / ATT_ROWS;
  if (chunk >= n_chunks) return;
  const uint32_t unit = h / desc.group;
  const int t = threadIdx.x;
  const int hl = t & 15;        // lane within half-warp: dims [8*hl, 8*hl+8)
  const int rg = t >> 4;        // row group 0..15
  const uint32_t r0 = chunk * ATT_ROWS;

  // q pre-scaled by log2(e)/sqrt(d) so exp(x) becomes exp2
  const float qscale = 1.4426950408889634f * rsqrtf(float(D));
  float qv[8];
  {
    const float4* qp = reinterpret_cast<const float4*>(q + size_t(h) * D + 8 * hl);
    float4 a = __ldg(qp), b = __ldg(qp + 1);
    qv[0] = a.x * qscale; qv[1] = a.y * qscale; qv[2] = a.z * qscale; qv[3] = a.w * qscale;
    qv[4] = b.x * qscale; qv[5] = b.y * qscale; qv[6] = b.z * qscale; qv[7] = b.w * qscale;
  }
  const uint32_t* ids = token_ids + size_t(h) * desc.sel_cap;
  const uint16_t* Ku = K + size_t(unit) * desc.p_cap * D;
  const uint16_t* Vu = V + size_t(unit) * desc.p_cap * D;

  uint4 kr[8], vr[8];
  bool ok[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t r = r0 + rg + 16 * k;
    ok[k] = r < nt;
    const uint32_t id = ok[k] ? __ldg(ids + r) : 0u;
    const uint4* kp = reinterpret_cast<const uint4*>(Ku + size_t(id) * D) + hl;
    const uint4* vp = reinterpret_cast<const uint4*>(Vu + size_t(id) * D) + hl;
    kr[k] = ok[k] ? ld_stream(kp) : make_uint4(0, 0, 0, 0);
    vr[k] = ok[k] ? ld_stream(vp) : make_uint4(0, 0, 0, 0);
  }
  float lg[8];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float s = dot8(kr[k], qv);
    s += __shfl_xor_sync(0xffffffffu, s, 8);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    lg[k] = ok[k] ? s : -INFINITY;
    m = fmaxf(m, lg[k]);
  }
  if (logits_ws && hl == 0) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (ok[k]) logits_ws[size_t(h) * desc.sel_cap + r0 + rg + 16 * k] = lg[k];
  }
  // chunk max across the 16 row groups
  __shared__ float s_m[16];
  __shared__ float s_l[16];
  __shared__ float s_acc[16][D + 4];
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
  if ((t & 31) == 0) s_m[t >> 5] = m;
  __syncthreads();
  float M = s_m[0];
#pragma unroll
  for (int i = 1; i < ATT_THREADS / 32; ++i) M = fmaxf(M, s_m[i]);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float l = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float p = ok[k] ? exp2f(lg[k] - M) : 0.f;
    l += p;
    axpy8(p, vr[k], acc);
  }
  // reduce over the 16 row groups
#pragma unroll
  for (int i = 0; i < 8; ++i) s_acc[rg][8 * hl + i] = acc[i];
  if (hl == 0) s_l[rg] = l;
  __syncthreads();
  float* pp = part + (size_t(h) * gridDim.y + chunk) * PART;
  if (t < D) {
    float a = 0.f;
#pragma unroll
    for (int g = 0; g < 16; ++g) a += s_acc[g][t];
    pp[2 + t] = a;
  }
  if (t == 0) {
    float ls = 0.f;
#pragma unroll
    for (int g = 0; g < 16; ++g) ls += s_l[g];
    pp[0] = M;
    pp[1] = ls;
  }
  // ---- last CTA of this q head merges the partials ------------------------
  __shared__ uint32_t s_last;
  __threadfence();
  __syncthreads();
  if (t == 0) s_last = (atomicAdd(&tickets[h], 1u) == n_chunks - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* pb = part + size_t(h) * gridDim.y * PART;
  float MM = -INFINITY;
  for (uint32_t c = 0; c < n_chunks; ++c) MM = fmaxf(MM, __ldcg(pb + c * PART));
  float L = 0.f;
  for (uint32_t c = 0; c < n_chunks; ++c)
    L += __ldcg(pb + c * PART + 1) * exp2f(__ldcg(pb + c * PART) - MM);
  const float invL = 1.f / L;
  if (t < D) {
    float o = 0.f;
    for (uint32_t c = 0; c < n_chunks; ++c)
      o += __ldcg(pb + c * PART + 2 + t) * exp2f(__ldcg(pb + c * PART) - MM);
    out[size_t(h) * D + t] = o * invL;
  }
  if (weights) {
    const float* lw = logits_ws + size_t(h) * desc.sel_cap;
    float* wo = weights + size_t(h) * desc.sel_cap;
    for (uint32_t i = t; i < nt; i += blockDim.x) wo[i] = exp2f(__ldcg(lw + i) - MM) * invL;
  }
  if (t == 0) tickets[h] = 0;  // re-arm for the next launch
}

int launch_attend(cudaStream_t st, const ckv_attend_desc& desc, const float* q,
                  const uint16_t* K, const uint16_t* V, const uint32_t* token_ids,
                  const uint32_t* n_tokens, float* out, float* weights, float* logits_ws,
                  float* part, uint32_t* tickets) {
  const uint32_t chunks = (desc.max_tokens + ATT_ROWS - 1) / ATT_ROWS;
  if (chunks == 0 || desc.n_q == 0) return CKV_OK;
  dim3 grid(desc.n_q, chunks);
  k_attend<<<grid, ATT_THREADS, 0, st>>>(desc, q, K, V, token_ids, n_tokens, out,
                                         weights ? logits_ws : nullptr, part, tickets, weights);
  CKV_LAUNCH_CHECK("k_attend");
  return CKV_OK;
}

size_t attend_part_floats(uint32_t n_q, uint32_t max_tokens) {
  return size_t(n_q) * ((max_tokens + ATT_ROWS - 1) / ATT_ROWS) * PART;
}

}  // namespace ckvb

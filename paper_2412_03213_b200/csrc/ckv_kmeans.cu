// ckv_kmeans.cu — K1-K4: batched cosine k-means (clustering.hpp:157-263).
//
// All active units advance in lock step, one assignment pass per host loop
// iteration; per-unit convergence masks the finished ones.  Per iteration:
//   update   : centroid = float(f64 sum / count) over the members in the
//              counting-sort order (position-ascending per cluster, exactly
//              the reference's accumulation order, clustering.hpp:207-216),
//              fused with normalize() of the next assignment's directions
//   assign   : tensor-core candidate filter + exact f64 re-score
//              (ckv_assign_tc.cu), or the exact CUDA-core pass below
//   index    : counting sort -> counts, member lists, changed-vs-previous
//   repair   : empty-cluster repair (clustering.hpp:128-153), rare
//   control  : convergence / max_iters bookkeeping, one 4-byte read-back
// Every integer result (labels, iterations, converged, repair iterations)
// and every centroid bit equals the reference for identical inputs.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "ckv_internal.cuh"
#include "ckv_kmeans_dev.cuh"

namespace ckvb {

// ---------------------------------------------------------------------------
// validation: kmeans_cosine's input checks (clustering.hpp:166-172)
// flags[u]: bit0 = some non-finite value, bit1 = some row with norm >= 1e-12,
// bit2 = some non-zero element (k_validate_scan: a streaming pass; only a
// unit whose non-zero elements are all tiny needs the per-row f64 norms of
// k_validate_rows).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_scan_keys(const uint16_t* __restrict__ keys, uint64_t key_stride, uint32_t n,
            int32_t* __restrict__ flags, float* __restrict__ knorm, uint16_t* __restrict__ k16,
            uint32_t n_pad, uint32_t* __restrict__ kerr) {
  // one pass over the keys: validation flags (if flags) and the tensor-core
  // key operands (if knorm): the fp16 copy h(k) (k16), the band scale |k| +
  // |k - h(k)| (knorm) and the unit's max |k - h(k)| (kerr, float bits; zero
  // for keys inside fp16's normal range, where bf16 -> fp16 is exact).
  // A warp takes 16 rows, a half-warp one row per step (16 lanes x 16 B),
  // all 8 loads in flight.
  const uint32_t u = blockIdx.y;
  const int lane = lane_id(), half = lane >> 4, hl = lane & 15;
  const uint32_t r0 = (blockIdx.x * (blockDim.x >> 5) + warp_id()) * 16;
  const uint16_t* base = keys + u * key_stride;
  // one element >= 1e-12 already gives its row norm >= 1e-12 (float threshold
  // rounded up so the decision is never looser than the f64 comparison)
  const float big = __uint_as_float(__float_as_uint(1e-12f) + 1u);
  uint4 q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t r = r0 + 2 * i + half;
    q[i] = r < n ? __ldg(reinterpret_cast<const uint4*>(base + size_t(r) * D) + hl)
                 : make_uint4(0, 0, 0, 0);
  }
  int f = 0;
  float emax = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t w[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
    float ss = 0.f, es = 0.f;
    uint32_t hw[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t hk = 0u;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t b = h ? (w[k] >> 16) : (w[k] & 0xffffu);
        const float x = __uint_as_float(b << 16);
        ss = fmaf(x, x, ss);
        if ((b & 0x7f80u) == 0x7f80u) f |= 1;
        if (b & 0x7fffu) f |= 4;
        if (fabsf(x) >= big) f |= 2;
        const uint16_t hb = f32_to_f16_tc(x);
        const float d = x - f16_to_f32(hb);  // exact (both are f32 values)
        es = fmaf(d, d, es);
        hk |= uint32_t(hb) << (16 * h);
      }
      hw[k] = hk;
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
      es += __shfl_xor_sync(0xffffffffu, es, o);
    }
    const uint32_t r = r0 + 2 * i + half;
    if (knorm && r < n) {
      reinterpret_cast<uint4*>(k16 + (size_t(u) * n_pad + r) * D)[hl] =
          make_uint4(hw[0], hw[1], hw[2], hw[3]);
      const float e = es > 0.f ? sqrtf(es) * 1.0001f : 0.f;  // rounding margin
      if (hl == 0) knorm[size_t(u) * n + r] = (sqrtf(ss) + e) * 1.0001f;
      emax = fmaxf(emax, e);
    }
  }
  if (knorm) {
    emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, 16));
    if (lane == 0 && emax > 0.f) atomicMax(kerr + u, __float_as_uint(emax));
  }
  if (flags) {
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane == 0 && f) atomicOr(&flags[u], f);
  }
}

__global__ void k_validate_rows(const uint16_t* __restrict__ keys, uint64_t key_stride,
                                uint32_t n, int32_t* __restrict__ flags) {
  const uint32_t u = blockIdx.y;
  if ((flags[u] & 6) != 4) return;  // decided by the scan
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  int f = 0;
  if (i < n) {
    const uint16_t* row = keys + u * key_stride + size_t(i) * D;
    double s = 0.0;
    for (int j = 0; j < D; ++j) {
      float x = bf16_to_f32(row[j]);
      s = __fma_rn(double(x), double(x), s);
    }
    if (sqrt(s) >= 1e-12) f |= 2;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (lane_id() == 0 && f) atomicOr(&flags[u], f);
}

// centroids[u][c] = keys[u][init_rows[u][c]]  (clustering.hpp:195-198)
__global__ void k_init_centroids(const uint16_t* __restrict__ keys, uint64_t key_stride,
                                 const uint32_t* __restrict__ init_rows, uint32_t C,
                                 uint32_t c_stride, float* __restrict__ cents) {
  const uint32_t u = blockIdx.y, c = blockIdx.x;
  const uint32_t r = init_rows[size_t(u) * C + c];
  const uint16_t* src = keys + u * key_stride + size_t(r) * D;
  float* dst = cents + (size_t(u) * c_stride + c) * D;
  for (int j = threadIdx.x; j < D; j += blockDim.x) dst[j] = bf16_to_f32(src[j]);
}

// normalize() (common.hpp:141-147) of every centroid -> f32 dirs (exact),
// fp16 dirs (tensor-core B operand), f64 norms (for cosine_distance).
// One warp per centroid: the row is loaded coalesced (lane L holds dims
// 4L..4L+3) and staged in shared memory, where lane 0 runs the norm's
// sequential f64 chain (the contract's order); every lane then divides and
// stores its four dims (coalesced 16-B / 8-B stores).
__global__ void __launch_bounds__(256)
k_dirs(const float* __restrict__ cents, uint32_t C, uint32_t c_stride, uint32_t c_pad,
       float* __restrict__ dirs, uint16_t* __restrict__ dirs16, double* __restrict__ cnorm,
       float* __restrict__ deps, const int32_t* __restrict__ active) {
  const uint32_t u = blockIdx.y;
  if (active && !active[u]) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t c = blockIdx.x * 8 + uint32_t(w);
  if (c >= c_pad) return;
  float4* dr = reinterpret_cast<float4*>(dirs + (size_t(u) * c_pad + c) * D) + lane;
  uint2* db = reinterpret_cast<uint2*>(dirs16 + (size_t(u) * c_pad + c) * D) + lane;
  if (c >= C) {  // padding columns of the MMA operand
    *dr = make_float4(0.f, 0.f, 0.f, 0.f);
    *db = make_uint2(0u, 0u);
    if (lane == 0) deps[size_t(u) * c_pad + c] = 0.f;
    return;
  }
  __shared__ float row[8][D];
  const float4 x = reinterpret_cast<const float4*>(cents + (size_t(u) * c_stride + c) * D)[lane];
  reinterpret_cast<float4*>(row[w])[lane] = x;
  __syncwarp();
  double nrm = 0.0;
  if (lane == 0) {
    nrm = sqrt(dot_seq_ff(row[w], row[w]));
    cnorm[size_t(u) * c_pad + c] = nrm;
  }
  nrm = __shfl_sync(0xffffffffu, nrm, 0);
  const float xs[4] = {x.x, x.y, x.z, x.w};
  float y[4];
  uint16_t h[4];
  double e2 = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    y[i] = nrm > 0.0 ? float(double(xs[i]) / nrm) : xs[i];
    h[i] = f32_to_f16_tc(y[i]);
    const double e = double(y[i]) - double(f16_to_f32(h[i]));
    e2 += e * e;
  }
  *dr = make_float4(y[0], y[1], y[2], y[3]);
  *db = make_uint2(uint32_t(h[0]) | uint32_t(h[1]) << 16, uint32_t(h[2]) | uint32_t(h[3]) << 16);
  e2 = warp_sum(e2);  // any order: the 1.0001 margin covers the rounding of the sum
  if (lane == 0) deps[size_t(u) * c_pad + c] = float(sqrt(e2)) * 1.0001f;
}

// ---------------------------------------------------------------------------
// exact assignment on CUDA cores (AssignScorer::assign, clustering.hpp:104-115)
// 128 keys per CTA, keys transposed in smem, one sequential f64 chain per
// (key, centroid).  Used for small problems (decode batches) and as the
// reference path the tensor-core filter is tested against.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128)
k_assign_exact(const uint16_t* __restrict__ keys, uint64_t key_stride, uint32_t n, uint32_t C,
               uint32_t c_pad, const float* __restrict__ dirs, int32_t* __restrict__ labels,
               uint32_t label_stride, const int32_t* __restrict__ active) {
  const uint32_t u = blockIdx.y;
  if (active && !active[u]) return;
  __shared__ uint16_t ks[D][130];
  const uint32_t i0 = blockIdx.x * 128;
  const uint16_t* kb = keys + u * key_stride;
  for (uint32_t e = threadIdx.x; e < 128u * D; e += 128) {
    uint32_t r = e / D, j = e % D;
    ks[j][r] = (i0 + r < n) ? kb[size_t(i0 + r) * D + j] : uint16_t(0);
  }
  __syncthreads();
  const uint32_t i = i0 + threadIdx.x;
  if (i >= n) return;
  const float* dr = dirs + size_t(u) * c_pad * D;
  uint32_t best = 0;
  double best_s = -INFINITY;
  for (uint32_t c = 0; c < C; ++c) {
    const float* dc = dr + size_t(c) * D;
    double s = 0.0;
#pragma unroll 16
    for (int j = 0; j < D; ++j) s = __fma_rn(double(bf16_to_f32(ks[j][threadIdx.x])), double(__ldg(dc + j)), s);
    if (s > best_s) { best_s = s; best = c; }
  }
  labels[size_t(u) * label_stride + i] = int32_t(best);
}

// ---------------------------------------------------------------------------
// update: per (unit, cluster) one warp; lane owns dims [4*lane, 4*lane+4).
// f64 sums over the members in sorted (= position) order, then
// float(sum / count), then the next pass's dirs (normalize, fused).
// ---------------------------------------------------------------------------
#ifndef CKV_UPD_MINB
#define CKV_UPD_MINB 4  // 64 registers: 2x the resident warps of the latency-bound tail (measured 634 vs 872 us per all-dirty pass)
#endif
__global__ void __launch_bounds__(256, CKV_UPD_MINB)
k_update(const uint16_t* __restrict__ keys, uint64_t key_stride, uint32_t C, uint32_t c_stride,
         uint32_t c_pad, uint32_t label_stride, const uint32_t* __restrict__ sizes,
         const uint32_t* __restrict__ starts, const uint32_t* __restrict__ sorted_ids,
         float* __restrict__ cents, float* __restrict__ dirs, uint16_t* __restrict__ dirs16,
         double* __restrict__ cnorm, float* __restrict__ deps, const int32_t* __restrict__ active,
         const uint8_t* __restrict__ dirty, double* __restrict__ sums_out,
         const double* __restrict__ sums_in) {
  const uint32_t u = blockIdx.y;
  if (active && !active[u]) return;
  const uint32_t c = blockIdx.x * (blockDim.x >> 5) + warp_id();
  const int lane = lane_id();
  if (c >= c_pad) return;
  // same members as the centroid's last computation -> the same f64 sums,
  // centroid, direction, norm and band: nothing to do
  if (dirty && (c >= C || !dirty[size_t(u) * c_stride + c])) return;
  float* dr = dirs + (size_t(u) * c_pad + c) * D;
  uint16_t* db = dirs16 + (size_t(u) * c_pad + c) * D;
  if (c >= C) {
    for (int j = lane; j < D; j += 32) { dr[j] = 0.f; db[j] = 0; }
    if (lane == 0) deps[size_t(u) * c_pad + c] = 0.f;
    return;
  }
  const uint32_t cnt = sizes[size_t(u) * c_stride + c];
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  if (sums_in) {  // incremental pass: the member sums were updated by k_update_delta
    const double2* sp = reinterpret_cast<const double2*>(sums_in + (size_t(u) * c_stride + c) * D) + 2 * lane;
    const double2 x = sp[0], y = sp[1];
    finish_centroid(x.x, x.y, y.x, y.y, double(cnt), cents + (size_t(u) * c_stride + c) * D, dr, db,
                    cnorm + size_t(u) * c_pad + c, deps + size_t(u) * c_pad + c);
    return;
  }
  const uint32_t beg = starts[size_t(u) * (c_stride + 1) + c];
  const uint32_t* ids = sorted_ids + size_t(u) * label_stride + beg;
  const uint2* kb = reinterpret_cast<const uint2*>(keys + u * key_stride) + lane;
  // member ids 32 at a time (one coalesced load), rows 16 in flight; the
  // f64 adds stay in member (= position) order, as update_centroids sums.
  for (uint32_t m0 = 0; m0 < cnt; m0 += 32) {
    const uint32_t nb = min(32u, cnt - m0);
    const uint32_t myid = uint32_t(lane) < nb ? __ldg(ids + m0 + lane) : 0u;
    for (uint32_t k0 = 0; k0 < nb; k0 += 16) {
      uint2 v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t id = __shfl_sync(0xffffffffu, myid, (k0 + k) & 31);
        v[k] = k0 + k < nb ? __ldg(kb + size_t(id) * (D / 4)) : make_uint2(0, 0);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k0 + k < nb) {
          a0 += double(__uint_as_float(v[k].x << 16));
          a1 += double(__uint_as_float(v[k].x & 0xffff0000u));
          a2 += double(__uint_as_float(v[k].y << 16));
          a3 += double(__uint_as_float(v[k].y & 0xffff0000u));
        }
      }
    }
  }
  if (sums_out) {
    double2* sp = reinterpret_cast<double2*>(sums_out + (size_t(u) * c_stride + c) * D) + 2 * lane;
    sp[0] = make_double2(a0, a1);
    sp[1] = make_double2(a2, a3);
  }
  finish_centroid(a0, a1, a2, a3, double(cnt), cents + (size_t(u) * c_stride + c) * D, dr, db,
                  cnorm + size_t(u) * c_pad + c, deps + size_t(u) * c_pad + c);
}

// ---------------------------------------------------------------------------
// incremental update (passes >= 2): only the keys whose label changed since
// the last update move their bf16 values between the persisted f64 member
// sums (subtract from the old cluster, add to the new).  Sums of bf16 values
// in f64 are exact in any order, and so are these differences,
// so the sums -- hence the centroids k_update finishes from them -- equal the
// position-ordered recomputation bit for bit, at a cost proportional to the
// moved keys instead of every member of every dirty cluster.
// One warp per 32 consecutive keys; lane L adds dims 4L..4L+3 of each moved key.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_update_delta(const uint16_t* __restrict__ keys, uint64_t key_stride, uint32_t n,
               uint32_t c_stride, uint32_t label_stride, const int32_t* __restrict__ now,
               const int32_t* __restrict__ before, const int32_t* __restrict__ active,
               double* __restrict__ sums) {
  const uint32_t u = blockIdx.y;
  if (active && !active[u]) return;
  const int lane = lane_id();
  const uint32_t i0 = (blockIdx.x * (blockDim.x >> 5) + warp_id()) * 32;
  if (i0 >= n) return;
  const uint32_t i = i0 + lane;
  const int32_t ln = i < n ? now[size_t(u) * label_stride + i] : -1;
  const int32_t lb = i < n ? before[size_t(u) * label_stride + i] : -1;
  unsigned moved = __ballot_sync(0xffffffffu, ln != lb);
  const uint2* kb = reinterpret_cast<const uint2*>(keys + u * key_stride) + lane;
  double* su = sums + size_t(u) * c_stride * D + 4 * lane;
  while (moved) {
    const int src = __ffs(moved) - 1;
    moved &= moved - 1;
    const int32_t cn = __shfl_sync(0xffffffffu, ln, src), cb = __shfl_sync(0xffffffffu, lb, src);
    const uint2 v = __ldg(kb + size_t(i0 + src) * (D / 4));
    const double x0 = double(__uint_as_float(v.x << 16)), x1 = double(__uint_as_float(v.x & 0xffff0000u));
    const double x2 = double(__uint_as_float(v.y << 16)), x3 = double(__uint_as_float(v.y & 0xffff0000u));
    if (cn >= 0) {
      double* d = su + size_t(cn) * D;
      atomicAdd(d, x0); atomicAdd(d + 1, x1); atomicAdd(d + 2, x2); atomicAdd(d + 3, x3);
    }
    if (cb >= 0) {
      double* d = su + size_t(cb) * D;
      atomicAdd(d, -x0); atomicAdd(d + 1, -x1); atomicAdd(d + 2, -x2); atomicAdd(d + 3, -x3);
    }
  }
}

// ---------------------------------------------------------------------------
// empty-cluster repair (clustering.hpp:128-153) — one CTA per unit that has
// an empty cluster; sequential over empty ids as the reference is.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_repair(const uint16_t* __restrict__ keys, uint64_t key_stride, uint32_t n, uint32_t C,
         uint32_t c_stride, uint32_t c_pad, int32_t* __restrict__ labels, uint32_t label_stride,
         uint32_t* __restrict__ sizes, const float* __restrict__ cents,
         const double* __restrict__ cnorm, const int32_t* __restrict__ need,
         uint32_t* __restrict__ repair_count) {
  const uint32_t u = blockIdx.x;
  if (!need[u]) return;
  uint32_t* counts = sizes + size_t(u) * c_stride;
  int32_t* lab = labels + size_t(u) * label_stride;
  const uint16_t* kb = keys + u * key_stride;
  __shared__ uint32_t s_cnt[8];
  __shared__ uint32_t s_idx[8];
  __shared__ double s_d[8];
  __shared__ uint32_t s_largest;
  uint32_t repairs = 0;
  for (uint32_t c = 0; c < C; ++c) {
    __syncthreads();
    if (counts[c] > 0) continue;
    // largest = first maximum of counts
    uint32_t bc = 0, bi = 0xffffffffu;
    for (uint32_t k = threadIdx.x; k < C; k += blockDim.x) {
      uint32_t v = counts[k];
      if (v > bc || (v == bc && k < bi)) { bc = v; bi = k; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      uint32_t oc = __shfl_xor_sync(0xffffffffu, bc, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oc > bc || (oc == bc && oi < bi)) { bc = oc; bi = oi; }
    }
    if (lane_id() == 0) { s_cnt[warp_id()] = bc; s_idx[warp_id()] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t b = s_cnt[0], ix = s_idx[0];
      for (int w = 1; w < int(blockDim.x >> 5); ++w)
        if (s_cnt[w] > b || (s_cnt[w] == b && s_idx[w] < ix)) { b = s_cnt[w]; ix = s_idx[w]; }
      s_largest = ix;
      s_cnt[0] = b;
    }
    __syncthreads();
    const uint32_t largest = s_largest;
    if (s_cnt[0] <= 1) continue;
    // victim = first member of `largest` with the maximum cosine distance
    const float* cl = cents + (size_t(u) * c_stride + largest) * D;
    const double nb = cnorm[size_t(u) * c_pad + largest];
    double bd = -1.0;
    uint32_t bv = 0xffffffffu;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      if (uint32_t(lab[i]) != largest) continue;
      double dd = cosine_distance_dev(kb + size_t(i) * D, cl, nb);
      if (dd > bd) { bd = dd; bv = i; }  // i increases per thread: first max kept
    }
    for (int o = 16; o > 0; o >>= 1) {
      double od = __shfl_xor_sync(0xffffffffu, bd, o);
      uint32_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
      if (od > bd || (od == bd && ov < bv)) { bd = od; bv = ov; }
    }
    __syncthreads();
    if (lane_id() == 0) { s_d[warp_id()] = bd; s_idx[warp_id()] = bv; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = s_d[0];
      uint32_t v = s_idx[0];
      for (int w = 1; w < int(blockDim.x >> 5); ++w)
        if (s_d[w] > b || (s_d[w] == b && s_idx[w] < v)) { b = s_d[w]; v = s_idx[w]; }
      if (v == 0xffffffffu) v = 0;  // no member beat worst = -1 (NaN): reference keeps 0
      lab[v] = int32_t(c);
      counts[largest]--;
      counts[c]++;
    }
    repairs++;
  }
  if (threadIdx.x == 0) repair_count[u] = repairs;
}

// objective (clustering.hpp:118-124) — diagnostic; f64 sum, any order
__global__ void k_objective(const uint16_t* __restrict__ keys, uint64_t key_stride, uint32_t n,
                            uint32_t c_stride, uint32_t c_pad, const int32_t* __restrict__ labels,
                            uint32_t label_stride, const float* __restrict__ cents,
                            const double* __restrict__ cnorm, double* __restrict__ obj,
                            const int32_t* __restrict__ active) {
  const uint32_t u = blockIdx.y;
  if (active && !active[u]) return;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (i < n) {
    uint32_t l = uint32_t(labels[size_t(u) * label_stride + i]);
    v = cosine_distance_dev(keys + u * key_stride + size_t(i) * D,
                            cents + (size_t(u) * c_stride + l) * D, cnorm[size_t(u) * c_pad + l]);
  }
  v = warp_sum(v);
  if (lane_id() == 0) atomicAdd(&obj[u], v);
}

// convergence bookkeeping after pass t (t = 0 is the initial assignment)
__global__ void k_control(uint32_t n_units, uint32_t t, uint32_t max_iters,
                          int32_t* __restrict__ active, const int32_t* __restrict__ changed,
                          int32_t* __restrict__ converged, uint32_t* __restrict__ iters,
                          int32_t* __restrict__ any_empty, uint32_t* __restrict__ repair_count,
                          uint32_t* __restrict__ repair_log, double* __restrict__ obj,
                          double* __restrict__ obj_log, int32_t* __restrict__ n_active) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  int still = 0;
  if (u < n_units && active[u]) {
    repair_log[size_t(u) * (max_iters + 1) + t] = repair_count[u];
    obj_log[size_t(u) * (max_iters + 1) + t] = obj[u];
    repair_count[u] = 0;
    obj[u] = 0.0;
    any_empty[u] = 0;
    if (t >= 1 && !changed[u]) {
      converged[u] = 1;
      iters[u] = t;
      active[u] = 0;
    } else if (t == max_iters) {
      iters[u] = t;
      active[u] = 0;
    } else {
      still = 1;
    }
  }
  still = __reduce_add_sync(0xffffffffu, still);
  if (lane_id() == 0 && still) atomicAdd(n_active, still);
}

__global__ void k_copy_labels(const int32_t* __restrict__ src, int32_t* __restrict__ dst,
                              uint32_t n, uint32_t stride, const uint32_t* __restrict__ iters,
                              int parity_wanted) {
  const uint32_t u = blockIdx.y;
  if (int(iters[u] & 1u) != parity_wanted) return;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[size_t(u) * stride + i] = src[size_t(u) * stride + i];
}

// tensor-core assignment (ckv_assign_tc.cu); returns CKV_EINVAL if the shape
// is unsupported so the caller falls back to the exact path
int assign_tc(cudaStream_t st, const uint16_t* keys, uint64_t key_stride, uint32_t n,
              uint32_t C, uint32_t c_pad, uint32_t n_units, const uint16_t* dirs16,
              const float* deps,
              const float* dirs, int32_t* labels, uint32_t label_stride, const int32_t* active,
              void* scratch, size_t scratch_bytes, uint64_t* launches,
              const uint16_t* k16p = nullptr, const uint32_t* perm = nullptr);
int launch_permute_keys(cudaStream_t st, const uint16_t* k16, uint32_t n, uint32_t n_pad,
                        const uint32_t* sorted, uint32_t label_stride, uint32_t n_units,
                        const int32_t* active, uint16_t* k16p, uint32_t* perm);

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
namespace {
// a view of one of the context's grow-only scratch slots
struct DevBuf {
  void* p = nullptr;
  template <typename T> T* as() { return static_cast<T*>(p); }
};
int dalloc(ckv_ctx* ctx, int slot, DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (ctx->scratch_cap[slot] < bytes) {
    if (ctx->scratch[slot]) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->scratch[slot]);
      ctx->scratch[slot] = nullptr;
      ctx->scratch_cap[slot] = 0;
    }
    cudaError_t e = cudaMalloc(&ctx->scratch[slot], bytes);
    if (e != cudaSuccess) {
      ctx->scratch[slot] = nullptr;
      set_error(std::string("kmeans: device allocation failed: ") + cudaGetErrorString(e));
      return CKV_ENOMEM;
    }
    ctx->scratch_cap[slot] = bytes;
  }
  b.p = ctx->scratch[slot];
  return CKV_OK;
}
}  // namespace

static int kmeans_run_units(ckv_ctx* ctx, const KMeansArgs& a, ckv_kmeans_info* info_host,
                            double* objective_host, uint32_t* repair_host);

// the two-stream overlap (kmeans_run) for calls of at least this many units;
// CKV_KM_OVERLAP=0 turns it off
constexpr uint32_t kOverlapMinUnits = 16;
static bool overlap_on() {
  static const bool v = !(getenv("CKV_KM_OVERLAP") && atoi(getenv("CKV_KM_OVERLAP")) == 0);
  return v;
}

// Units are independent, so a call whose scratch (dominated by the fp16 key
// copy of the tensor-core path, ~n * 256 B per unit) would not fit next to
// the caller's data runs its units in batches, each a complete k-means run.
int kmeans_run(ckv_ctx* ctx, const KMeansArgs& a, ckv_kmeans_info* info_host,
               double* objective_host, uint32_t* repair_host) {
  const uint32_t U = a.n_units;
  const size_t per_unit = assign_tc_scratch_bytes(1, a.n, a.C) + size_t(a.label_stride) * 16 +
                          size_t(a.c_stride) * D * 24;
  // the budget is at least 16 GiB: only a call that needs more asks the
  // driver for the free memory (cudaMemGetInfo measured 5-9 ms on some calls,
  // the prefill's largest source of call-to-call jitter)
  const size_t floor_b = size_t(16) << 30;
  size_t free_b = 0, total_b = 0;
  if (size_t(U) * per_unit > floor_b) {
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 0;
    trace_mark("memgetinfo");
  }
  const size_t budget = std::max<size_t>(floor_b, free_b / 10 * 6);
  const uint32_t ub = uint32_t(std::max<size_t>(1, std::min<size_t>(U, budget / per_unit)));
  const size_t MI1 = size_t(a.max_iters) + 1;
  if (ub >= U && U >= kOverlapMinUnits && overlap_on()) {
    // two halves, each a complete k-means run on its own context / stream
    // from its own host thread; the GPU interleaves them (units are
    // independent, so every result is the one-stream result)
    if (!ctx->aux) {
      ckv_ctx* x = nullptr;
      CKV_TRY(ckv_ctx_create(ctx->device, nullptr, &x));
      if (cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking) != cudaSuccess) {
        ckv_ctx_destroy(x);
        set_error("kmeans: aux stream creation failed");
        return CKV_ECUDA;
      }
      x->own_stream = true;
      ctx->aux = x;
    }
    ckv_ctx* x = ctx->aux;
    // the two fork / join events, destroyed on every path out
    struct Events {
      cudaEvent_t in = nullptr, out = nullptr;
      ~Events() {
        if (in) cudaEventDestroy(in);
        if (out) cudaEventDestroy(out);
      }
    } ev;
    CKV_CUDA_TRY(cudaEventCreateWithFlags(&ev.in, cudaEventDisableTiming));
    CKV_CUDA_TRY(cudaEventCreateWithFlags(&ev.out, cudaEventDisableTiming));
    CKV_CUDA_TRY(cudaEventRecord(ev.in, ctx->stream));  // the caller's inputs are ready
    CKV_CUDA_TRY(cudaStreamWaitEvent(x->stream, ev.in, 0));
    const uint32_t u0 = U / 2;
    KMeansArgs b = a;
    b.n_units = U - u0;
    b.keys = a.keys + size_t(u0) * a.key_stride;
    b.init_rows = a.init_rows + size_t(u0) * a.C;
    b.centroids = a.centroids + size_t(u0) * a.c_stride * D;
    b.labels = a.labels + size_t(u0) * a.label_stride;
    KMeansArgs f = a;
    f.n_units = u0;
    int rc2 = CKV_OK;
    std::string err2;
    auto second = [&] {
      cudaSetDevice(x->device);
      rc2 = kmeans_run_units(x, b, info_host ? info_host + u0 : nullptr,
                             objective_host ? objective_host + u0 * MI1 : nullptr,
                             repair_host ? repair_host + u0 * MI1 : nullptr);
      if (rc2 != CKV_OK) err2 = ckv_last_error();
    };
    std::thread th;
    try {
      th = std::thread(second);
    } catch (...) {  // no thread to be had: the halves run one after the other
    }
    const int rc1 = kmeans_run_units(ctx, f, info_host, objective_host, repair_host);
    if (th.joinable()) th.join(); else second();
    cudaEventRecord(ev.out, x->stream);
    cudaStreamWaitEvent(ctx->stream, ev.out, 0);  // the caller's stream sees both halves
    if (rc1 != CKV_OK) return rc1;
    if (rc2 != CKV_OK) { set_error(err2); return rc2; }
    return CKV_OK;
  }
  if (ub >= U) return kmeans_run_units(ctx, a, info_host, objective_host, repair_host);
  for (uint32_t u0 = 0; u0 < U; u0 += ub) {
    KMeansArgs b = a;
    b.n_units = std::min(ub, U - u0);
    b.keys = a.keys + size_t(u0) * a.key_stride;
    b.init_rows = a.init_rows + size_t(u0) * a.C;
    b.centroids = a.centroids + size_t(u0) * a.c_stride * D;
    b.labels = a.labels + size_t(u0) * a.label_stride;
    CKV_TRY(kmeans_run_units(ctx, b, info_host ? info_host + u0 : nullptr,
                             objective_host ? objective_host + u0 * MI1 : nullptr,
                             repair_host ? repair_host + u0 * MI1 : nullptr));
  }
  return CKV_OK;
}

static int kmeans_run_units(ckv_ctx* ctx, const KMeansArgs& a, ckv_kmeans_info* info_host,
                            double* objective_host, uint32_t* repair_host) {
  cudaStream_t st = ctx->stream;
  const uint32_t U = a.n_units, n = a.n, C = a.C, MI = a.max_iters;
  if (U == 0) return CKV_OK;
  if (C < 1 || C > n) { set_error("kmeans: need 1 <= C <= N"); return CKV_EINVAL; }
  if (MI < 1) { set_error("ClusterConfig: max_iters must be >= 1"); return CKV_EINVAL; }
  const uint32_t c_pad = (C + 31) / 32 * 32;
  const bool want_obj = (a.flags & CKV_KM_OBJECTIVE) != 0;

  // ---- scratch ----------------------------------------------------------
  DevBuf b_flags, b_lab1, b_sizes, b_starts, b_sorted, b_dirs, b_dirs16, b_cnorm, b_deps, b_active,
      b_changed, b_conv, b_iters, b_empty, b_rep, b_replog, b_obj, b_objlog, b_nact, b_tc, b_dirty;
  const uint32_t LS = a.label_stride, CS = a.c_stride;
  CKV_TRY(dalloc(ctx, 1, b_flags, sizeof(int32_t) * U));
  CKV_TRY(dalloc(ctx, 2, b_lab1, sizeof(int32_t) * size_t(U) * LS));
  CKV_TRY(dalloc(ctx, 3, b_sizes, sizeof(uint32_t) * size_t(U) * CS));
  CKV_TRY(dalloc(ctx, 4, b_starts, sizeof(uint32_t) * size_t(U) * (CS + 1)));
  CKV_TRY(dalloc(ctx, 5, b_sorted, sizeof(uint32_t) * size_t(U) * LS));
  CKV_TRY(dalloc(ctx, 6, b_dirs, sizeof(float) * size_t(U) * c_pad * D));
  CKV_TRY(dalloc(ctx, 7, b_dirs16, sizeof(uint16_t) * size_t(U) * c_pad * D));
  CKV_TRY(dalloc(ctx, 8, b_cnorm, sizeof(double) * size_t(U) * c_pad));
  CKV_TRY(dalloc(ctx, 9, b_deps, sizeof(float) * size_t(U) * c_pad));
  CKV_TRY(dalloc(ctx, 10, b_active, sizeof(int32_t) * U));
  CKV_TRY(dalloc(ctx, 11, b_changed, sizeof(int32_t) * U));
  CKV_TRY(dalloc(ctx, 12, b_conv, sizeof(int32_t) * U));
  CKV_TRY(dalloc(ctx, 13, b_iters, sizeof(uint32_t) * U));
  CKV_TRY(dalloc(ctx, 14, b_empty, sizeof(int32_t) * U));
  CKV_TRY(dalloc(ctx, 15, b_rep, sizeof(uint32_t) * U));
  CKV_TRY(dalloc(ctx, 16, b_replog, sizeof(uint32_t) * size_t(U) * (MI + 1)));
  CKV_TRY(dalloc(ctx, 17, b_obj, sizeof(double) * U));
  CKV_TRY(dalloc(ctx, 18, b_objlog, sizeof(double) * size_t(U) * (MI + 1)));
  CKV_TRY(dalloc(ctx, 19, b_nact, sizeof(int32_t)));
  CKV_TRY(dalloc(ctx, 21, b_dirty, size_t(U) * CS));
  // persisted f64 member sums of the last update (incremental passes)
  DevBuf b_sums;
  CKV_TRY(dalloc(ctx, 38, b_sums, sizeof(double) * size_t(U) * CS * D));

  const bool use_tc = !(a.flags & CKV_KM_EXACT_ONLY) && assign_tc_supported(n, C);
  size_t tc_bytes = use_tc ? assign_tc_scratch_bytes(U, n, C) : 0;
  // the tensor-core key operands (fp16 copy, band norms, conversion error),
  // filled by k_scan_keys
  TcKeyPrep prep{};
  if (use_tc) {
    CKV_TRY(dalloc(ctx, 20, b_tc, tc_bytes));
    prep = assign_tc_keyprep(b_tc.p, U, n);
    CKV_CUDA_TRY(cudaMemsetAsync(prep.kerr, 0, sizeof(uint32_t) * U, st));
  }
  float* knorm = prep.knorm;

  // [0, U) validation flags, [U] the active-unit count the loop tests,
  // [U + 1 + s] the lagged read-back slots
  if (!ctx->h_flags || ctx->h_flags_cap < U + 3) {
    if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
    CKV_CUDA_TRY(cudaMallocHost(&ctx->h_flags, sizeof(int32_t) * (U + 3)));
    ctx->h_flags_cap = U + 3;
  }
  int32_t* hf = ctx->h_flags;

  // ---- validation (clustering.hpp:166-172) -------------------------------
  if (!(a.flags & CKV_KM_NO_VALIDATE)) {
    CKV_CUDA_TRY(cudaMemsetAsync(b_flags.p, 0, sizeof(int32_t) * U, st));
    k_scan_keys<<<dim3((n + 127) / 128, U), 256, 0, st>>>(a.keys, a.key_stride, n,
                                                          b_flags.as<int32_t>(), knorm, prep.k16,
                                                          prep.n_pad, prep.kerr);
    CKV_LAUNCH_CHECK("k_scan_keys");
    knorm = nullptr;  // done
    k_validate_rows<<<dim3((n + 255) / 256, U), 256, 0, st>>>(a.keys, a.key_stride, n,
                                                              b_flags.as<int32_t>());
    CKV_LAUNCH_CHECK("k_validate_rows");
    ctx->launches += 2;
    CKV_CUDA_TRY(cudaMemcpyAsync(hf, b_flags.p, sizeof(int32_t) * U, cudaMemcpyDeviceToHost, st));
    trace_mark("validation queued");
    CKV_CUDA_TRY(cudaStreamSynchronize(st));
    trace_mark("validation synced");
    for (uint32_t u = 0; u < U; ++u)
      if (hf[u] & 1) { set_error("kmeans: keys must be finite"); return CKV_EINVAL; }
    for (uint32_t u = 0; u < U; ++u)
      if (!(hf[u] & 2)) {
        set_error("kmeans: degenerate input, all keys zero-norm");
        return CKV_EINVAL;
      }
  }
  if (knorm) {  // validation skipped: the norms still need their pass
    k_scan_keys<<<dim3((n + 127) / 128, U), 256, 0, st>>>(a.keys, a.key_stride, n, nullptr,
                                                          knorm, prep.k16, prep.n_pad, prep.kerr);
    CKV_LAUNCH_CHECK("k_scan_keys");
    ctx->launches++;
  }

  int32_t* lab[2] = {a.labels, b_lab1.as<int32_t>()};
  float* dirs = b_dirs.as<float>();
  uint16_t* dirs16 = b_dirs16.as<uint16_t>();
  double* cnorm = b_cnorm.as<double>();
  float* deps = b_deps.as<float>();
  int32_t* active = b_active.as<int32_t>();

  // active = 1, others = 0
  {
    std::vector<int32_t> ones(U, 1);
    CKV_CUDA_TRY(cudaMemcpyAsync(active, ones.data(), sizeof(int32_t) * U,
                                 cudaMemcpyHostToDevice, st));
    CKV_CUDA_TRY(cudaMemsetAsync(b_conv.p, 0, sizeof(int32_t) * U, st));
    CKV_CUDA_TRY(cudaMemsetAsync(b_iters.p, 0, sizeof(uint32_t) * U, st));
    CKV_CUDA_TRY(cudaMemsetAsync(b_empty.p, 0, sizeof(int32_t) * U, st));
    CKV_CUDA_TRY(cudaMemsetAsync(b_rep.p, 0, sizeof(uint32_t) * U, st));
    CKV_CUDA_TRY(cudaMemsetAsync(b_obj.p, 0, sizeof(double) * U, st));
    CKV_CUDA_TRY(cudaMemsetAsync(b_changed.p, 0, sizeof(int32_t) * U, st));
    CKV_CUDA_TRY(cudaStreamSynchronize(st));  // `ones` leaves scope
    trace_mark("active set");
  }

  // ---- init (clustering.hpp:174-198) --------------------------------------
  k_init_centroids<<<dim3(C, U), 128, 0, st>>>(a.keys, a.key_stride, a.init_rows, C, CS,
                                                a.centroids);
  CKV_LAUNCH_CHECK("k_init_centroids");
  k_dirs<<<dim3((c_pad + 7) / 8, U), 256, 0, st>>>(a.centroids, C, CS, c_pad, dirs, dirs16,
                                                    cnorm, deps, active);
  CKV_LAUNCH_CHECK("k_dirs");
  ctx->launches += 2;

  // CKV_KM_PERM_AT=t (experiment, off by default): from pass t on the fp16
  // operand is cluster-major (k_permute_keys, built once from that pass's
  // index) so the rows of a tile share their clusters and the epilogue's
  // warp-uniform block skip could apply; labels keep their positions.
  // Measured at config B: 15% fewer epilogue instructions but 8% slower
  // (the per-row perm / knorm gathers and scattered label writes; on these
  // keys the ~50 centroids of a key's true centre are near-ties spread over
  // many blocks, so few blocks are skipped).
  const uint16_t* k16p = nullptr;
  const uint32_t* perm = nullptr;
  static const uint32_t perm_at = getenv("CKV_KM_PERM_AT")
                                      ? uint32_t(atoi(getenv("CKV_KM_PERM_AT"))) : 0u;
  auto assign = [&](int32_t* out) -> int {
    if (use_tc)
      return assign_tc(st, a.keys, a.key_stride, n, C, c_pad, U, dirs16, deps, dirs, out, LS, active,
                       b_tc.p, tc_bytes, &ctx->launches, k16p, perm);
    k_assign_exact<<<dim3((n + 127) / 128, U), 128, 0, st>>>(a.keys, a.key_stride, n, C, c_pad,
                                                            dirs, out, LS, active);
    CKV_LAUNCH_CHECK("k_assign_exact");
    ctx->launches++;
    return CKV_OK;
  };

  // the member lists (sorted ids) feed only a full k_update (and the opt-in
  // MCR / permutation): once the next update is incremental the index pass
  // skips its stable scatter, the costliest part of k_index
  static const uint32_t incr_from_ = getenv("CKV_KM_INCR_FROM")
                                         ? uint32_t(atoi(getenv("CKV_KM_INCR_FROM"))) : 5u;
  auto count_repair = [&](int32_t* cur, const int32_t* prev, bool need_sorted) -> int {
    uint32_t* srt = need_sorted ? b_sorted.as<uint32_t>() : nullptr;
    CKV_TRY(launch_index(st, U, cur, n, LS, CS, nullptr, C, b_sizes.as<uint32_t>(),
                         b_starts.as<uint32_t>(), srt, prev,
                         b_changed.as<int32_t>(), active, b_empty.as<int32_t>(),
                         prev ? b_dirty.as<uint8_t>() : nullptr));
    k_repair<<<U, 256, 0, st>>>(a.keys, a.key_stride, n, C, CS, c_pad, cur, LS,
                                b_sizes.as<uint32_t>(), a.centroids, cnorm,
                                b_empty.as<int32_t>(), b_rep.as<uint32_t>());
    CKV_LAUNCH_CHECK("k_repair");
    // re-sort (and re-compare) the units that were repaired
    CKV_TRY(launch_index(st, U, cur, n, LS, CS, nullptr, C, b_sizes.as<uint32_t>(),
                         b_starts.as<uint32_t>(), srt, prev,
                         b_changed.as<int32_t>(), b_empty.as<int32_t>(), nullptr,
                         prev ? b_dirty.as<uint8_t>() : nullptr));
    ctx->launches += 3;
    if (want_obj) {
      k_objective<<<dim3((n + 255) / 256, U), 256, 0, st>>>(a.keys, a.key_stride, n, CS, c_pad,
                                                             cur, LS, a.centroids, cnorm,
                                                             b_obj.as<double>(), active);
      CKV_LAUNCH_CHECK("k_objective");
      ctx->launches++;
    }
    return CKV_OK;
  };

  // lagged read-back (CKV_KM_LAG=0 turns it off): the active count of a
  // read-back pass is copied behind an event and only waited for at the next
  // read-back pass, so the launch queue never drains on the host round trip;
  // the passes queued past the last convergence are no-ops, as above
  static const bool lag = !(getenv("CKV_KM_LAG") && atoi(getenv("CKV_KM_LAG")) == 0);
  cudaEvent_t ev_rb[2] = {nullptr, nullptr};
  int pend = -1, rb_next = 0;
  auto control_lagged = [&](uint32_t t) -> int {
    CKV_CUDA_TRY(cudaMemsetAsync(b_nact.p, 0, sizeof(int32_t), st));
    k_control<<<(U + 127) / 128, 128, 0, st>>>(
        U, t, MI, active, b_changed.as<int32_t>(), b_conv.as<int32_t>(), b_iters.as<uint32_t>(),
        b_empty.as<int32_t>(), b_rep.as<uint32_t>(), b_replog.as<uint32_t>(), b_obj.as<double>(),
        b_objlog.as<double>(), b_nact.as<int32_t>());
    CKV_LAUNCH_CHECK("k_control");
    ctx->launches++;
    const int sl = rb_next;
    rb_next ^= 1;
    if (!ev_rb[sl]) CKV_CUDA_TRY(cudaEventCreateWithFlags(&ev_rb[sl], cudaEventDisableTiming));
    CKV_CUDA_TRY(cudaMemcpyAsync(&hf[U + 1 + sl], b_nact.p, sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, st));
    CKV_CUDA_TRY(cudaEventRecord(ev_rb[sl], st));
    if (pend >= 0) {  // the previous read-back decides whether to go on
      CKV_CUDA_TRY(cudaEventSynchronize(ev_rb[pend]));
      hf[U] = hf[U + 1 + pend];
      trace_mark("lagged control, active units", long(hf[U]));
    }
    pend = sl;
    return CKV_OK;
  };
  auto control = [&](uint32_t t, int32_t* n_active_host, bool read_back) -> int {
    CKV_CUDA_TRY(cudaMemsetAsync(b_nact.p, 0, sizeof(int32_t), st));
    k_control<<<(U + 127) / 128, 128, 0, st>>>(
        U, t, MI, active, b_changed.as<int32_t>(), b_conv.as<int32_t>(), b_iters.as<uint32_t>(),
        b_empty.as<int32_t>(), b_rep.as<uint32_t>(), b_replog.as<uint32_t>(), b_obj.as<double>(),
        b_objlog.as<double>(), b_nact.as<int32_t>());
    CKV_LAUNCH_CHECK("k_control");
    ctx->launches++;
    if (!read_back) return CKV_OK;
    CKV_CUDA_TRY(cudaMemcpyAsync(n_active_host, b_nact.p, sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, st));
    trace_mark("control queued, pass", long(t));
    CKV_CUDA_TRY(cudaStreamSynchronize(st));
    trace_mark("control synced, active units", long(*n_active_host));
    return CKV_OK;
  };

  // pass 0: initial assignment, count, repair, objective
  CKV_TRY(assign(lab[0]));
  CKV_TRY(count_repair(lab[0], nullptr, true));
  CKV_TRY(control(0, &hf[U], true));

  // CKV_DEBUG_KMEANS=1: per-phase device times of each pass on stderr
  static const bool dbg = getenv("CKV_DEBUG_KMEANS") != nullptr;
  cudaEvent_t dev_[5];
  if (dbg) for (auto& e : dev_) cudaEventCreate(&e);
  for (uint32_t t = 1; t <= MI && hf[U] > 0; ++t) {
    int32_t* prev = lab[(t - 1) & 1];
    int32_t* cur = lab[t & 1];
    if (dbg) cudaEventRecord(dev_[0], st);
    // update from the previous labels (sizes/starts/sorted hold its sort)
    // the first passes (most keys move) recompute the dirty clusters from
    // their members and keep the f64 sums; from pass KM_INCR_FROM on (a few
    // percent of the keys move) only the moved keys update the sums and the
    // dirty clusters are finished from them (measured at config B: the
    // atomic delta costs 2.7 / 1.1 / 0.6 ms in passes 2-4 against ~0.6 ms of
    // recomputation, and 0.4 -> 0.03 ms afterwards).  CKV_KM_INCR_FROM=N
    // overrides (a large N: always the full recomputation).
    static const uint32_t incr_from = getenv("CKV_KM_INCR_FROM")
                                          ? uint32_t(atoi(getenv("CKV_KM_INCR_FROM"))) : 5u;
    const bool incr = t >= std::max(2u, incr_from);
    if (incr) {
      k_update_delta<<<dim3((n + 255) / 256, U), 256, 0, st>>>(
          a.keys, a.key_stride, n, CS, LS, prev, cur, active, b_sums.as<double>());
      CKV_LAUNCH_CHECK("k_update_delta");
      ctx->launches++;
    }
    k_update<<<dim3((c_pad + 7) / 8, U), 256, 0, st>>>(
        a.keys, a.key_stride, C, CS, c_pad, LS, b_sizes.as<uint32_t>(), b_starts.as<uint32_t>(),
        b_sorted.as<uint32_t>(), a.centroids, dirs, dirs16, cnorm, deps, active,
        t == 1 ? nullptr : b_dirty.as<uint8_t>(), incr ? nullptr : b_sums.as<double>(),
        incr ? b_sums.as<double>() : nullptr);
    CKV_LAUNCH_CHECK("k_update");
    ctx->launches++;
    if (dbg) cudaEventRecord(dev_[1], st);
    // passes >= 2: only the clusters recomputed by this update moved, so the
    // moved-cluster reduced assignment applies (exact; ckv_assign_tc.cu);
    // bounded by its permuted-key staging (<= 8 GB)
    const bool mcr = use_tc && t >= 2 && mcr_enabled() &&
                     size_t(U) * ((n + 127) / 128 * 128) * D * 2 <= (size_t(8) << 30);
    if (mcr)
      CKV_TRY(assign_mcr(ctx, a.keys, a.key_stride, n, C, c_pad, U, CS, dirs16, deps, dirs,
                         prev, cur, LS, active, b_dirty.as<uint8_t>(), b_sorted.as<uint32_t>(),
                         b_tc.p, tc_bytes));
    else
      CKV_TRY(assign(cur));
    if (dbg) cudaEventRecord(dev_[2], st);
    CKV_TRY(count_repair(cur, prev, t + 1 < std::max(2u, incr_from_) || mcr_enabled() ||
                                        (perm_at && t == perm_at)));
    if (dbg) cudaEventRecord(dev_[3], st);
    const int32_t active_before = hf[U];
    // the host reads the active count back only every KM_SYNC passes: the
    // passes queued after the last unit converged are no-ops (every kernel
    // skips inactive units), and the launch queue stays ahead of the GPU
    // instead of draining on a host round trip per pass
    constexpr uint32_t KM_SYNC = 4;
    if (lag && !dbg && t % KM_SYNC == 0 && t < MI)
      CKV_TRY(control_lagged(t));
    else
      CKV_TRY(control(t, &hf[U], dbg || t % KM_SYNC == 0 || t == MI));
    if (use_tc && perm_at && t == perm_at && !mcr_enabled() && !k16p) {
      // b_sorted holds the index of this pass's labels (count_repair)
      DevBuf b_k16p, b_perm;
      if (dalloc(ctx, 39, b_k16p, size_t(U) * prep.n_pad * D * 2) == CKV_OK &&
          dalloc(ctx, 40, b_perm, size_t(U) * prep.n_pad * 4) == CKV_OK) {
        CKV_TRY(launch_permute_keys(st, prep.k16, n, prep.n_pad, b_sorted.as<uint32_t>(), LS, U,
                                    active, b_k16p.as<uint16_t>(), b_perm.as<uint32_t>()));
        ctx->launches++;
        k16p = b_k16p.as<uint16_t>();
        perm = b_perm.as<uint32_t>();
      } else {
        cudaGetLastError();  // no room for the copy: stay in position order
      }
    }
    if (dbg) {
      cudaEventRecord(dev_[4], st);
      cudaEventSynchronize(dev_[4]);
      float x[4];
      for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&x[k], dev_[k], dev_[k + 1]);
      fprintf(stderr, "[kmeans dbg] pass %u active %d: update %.3f assign %.3f index+repair %.3f "
              "control %.3f ms\n", t, active_before, x[0], x[1], x[2], x[3]);
    }
  }
  if (dbg) for (auto& e : dev_) cudaEventDestroy(e);
  for (auto& e : ev_rb)
    if (e) cudaEventDestroy(e);

  // final labels live in lab[iterations_used & 1]; lab[0] is the output
  k_copy_labels<<<dim3(32, U), 256, 0, st>>>(lab[1], lab[0], n, LS, b_iters.as<uint32_t>(), 1);
  CKV_LAUNCH_CHECK("k_copy_labels");
  ctx->launches++;

  // ---- results -----------------------------------------------------------
  std::vector<uint32_t> iters(U), reps(size_t(U) * (MI + 1));
  std::vector<int32_t> conv(U);
  std::vector<double> objs(size_t(U) * (MI + 1));
  CKV_CUDA_TRY(cudaMemcpyAsync(iters.data(), b_iters.p, sizeof(uint32_t) * U,
                               cudaMemcpyDeviceToHost, st));
  CKV_CUDA_TRY(cudaMemcpyAsync(conv.data(), b_conv.p, sizeof(int32_t) * U,
                               cudaMemcpyDeviceToHost, st));
  CKV_CUDA_TRY(cudaMemcpyAsync(reps.data(), b_replog.p, sizeof(uint32_t) * reps.size(),
                               cudaMemcpyDeviceToHost, st));
  if (want_obj)
    CKV_CUDA_TRY(cudaMemcpyAsync(objs.data(), b_objlog.p, sizeof(double) * objs.size(),
                                 cudaMemcpyDeviceToHost, st));
  CKV_CUDA_TRY(cudaStreamSynchronize(st));
  trace_mark("results synced");
  for (uint32_t u = 0; u < U; ++u) {
    uint32_t it = iters[u];
    uint32_t nrep = 0;
    for (uint32_t t = 0; t <= it; ++t) {
      if (reps[size_t(u) * (MI + 1) + t] > 0) {
        if (repair_host) repair_host[size_t(u) * (MI + 1) + nrep] = t;
        nrep++;
      }
      if (objective_host && want_obj)
        objective_host[size_t(u) * (MI + 1) + t] = objs[size_t(u) * (MI + 1) + t];
    }
    if (info_host) {
      info_host[u].iterations_used = it;
      info_host[u].converged = conv[u];
      info_host[u].n_repair = nrep;
      info_host[u].n_objective = want_obj ? it + 1 : 0;
    }
  }
  return CKV_OK;
}

}  // namespace ckvb

// ---------------------------------------------------------------------------
// launch wrappers for the sequence-sharded driver (ckv_kmshard.cu): the same
// kernels on one shard's keys
// ---------------------------------------------------------------------------
namespace ckvb {

int launch_scan_keys(cudaStream_t st, const uint16_t* keys, uint64_t key_stride, uint32_t n,
                     uint32_t n_units, int32_t* flags, const TcKeyPrep* prep) {
  if (n == 0 || n_units == 0) return CKV_OK;
  if (prep) CKV_CUDA_TRY(cudaMemsetAsync(prep->kerr, 0, sizeof(uint32_t) * n_units, st));
  k_scan_keys<<<dim3((n + 127) / 128, n_units), 256, 0, st>>>(
      keys, key_stride, n, flags, prep ? prep->knorm : nullptr, prep ? prep->k16 : nullptr,
      prep ? prep->n_pad : 0u, prep ? prep->kerr : nullptr);
  CKV_LAUNCH_CHECK("k_scan_keys");
  if (flags) {
    k_validate_rows<<<dim3((n + 255) / 256, n_units), 256, 0, st>>>(keys, key_stride, n, flags);
    CKV_LAUNCH_CHECK("k_validate_rows");
  }
  return CKV_OK;
}

int launch_assign(cudaStream_t st, bool use_tc, const uint16_t* keys, uint64_t key_stride,
                  uint32_t n, uint32_t C, uint32_t c_pad, uint32_t n_units,
                  const uint16_t* dirs16, const float* deps, const float* dirs, int32_t* labels,
                  uint32_t label_stride, const int32_t* active, void* tc_scratch,
                  size_t tc_bytes, uint64_t* launches) {
  if (n == 0 || n_units == 0) return CKV_OK;
  if (use_tc)
    return assign_tc(st, keys, key_stride, n, C, c_pad, n_units, dirs16, deps, dirs, labels,
                     label_stride, active, tc_scratch, tc_bytes, launches);
  k_assign_exact<<<dim3((n + 127) / 128, n_units), 128, 0, st>>>(keys, key_stride, n, C, c_pad,
                                                                 dirs, labels, label_stride,
                                                                 active);
  CKV_LAUNCH_CHECK("k_assign_exact");
  ++*launches;
  return CKV_OK;
}

int launch_objective(cudaStream_t st, const uint16_t* keys, uint64_t key_stride, uint32_t n,
                     uint32_t n_units, uint32_t c_stride, uint32_t c_pad, const int32_t* labels,
                     uint32_t label_stride, const float* cents, const double* cnorm, double* obj,
                     const int32_t* active) {
  if (n == 0 || n_units == 0) return CKV_OK;
  k_objective<<<dim3((n + 255) / 256, n_units), 256, 0, st>>>(keys, key_stride, n, c_stride,
                                                               c_pad, labels, label_stride, cents,
                                                               cnorm, obj, active);
  CKV_LAUNCH_CHECK("k_objective");
  return CKV_OK;
}

}  // namespace ckvb

// ---------------------------------------------------------------------------
// K4 fused: cluster_decode_batch's whole kmeans_cosine (clustering.hpp:160-263
// on one decode batch, 310-332) in ONE launch, one CTA per unit, everything
// in shared memory: no per-iteration host round trip (the generic driver
// above pays ~2 launches + a sync per pass, ~3.5 ms per event at config D).
// Same numerics as the generic path, so the same bits: normalize() and
// float(sum / count) through finish_centroid, exact sequential f64
// assignment with strict '>', f64 member sums in position order, the
// reference's repair, convergence on label equality after repair.
// ---------------------------------------------------------------------------
namespace ckvb {

constexpr int KS_THREADS = 512;
constexpr int KS_WARPS = KS_THREADS / 32;
constexpr uint32_t KS_MAX_ROWS = 512;  // one batch row per thread
constexpr uint32_t KS_MAX_C = 32;
constexpr uint32_t KS_CS = D + 1;      // centroid row stride (floats): conflict-free chains

// row stride (u16) of the transposed key stage: even, with an odd word
// stride, so both access patterns are conflict-free — the assignment's lanes
// read consecutive rows of one dim, the update's lanes consecutive dims of
// one row
__host__ __device__ inline uint32_t ks_row_stride(uint32_t rows) {
  uint32_t rs = (rows + 1) & ~1u;
  return ((rs / 2) & 1u) ? rs : rs + 2;
}

__host__ __device__ inline size_t ks_smem_bytes(uint32_t rows, uint32_t C) {
  const size_t C4 = (C + 3) & ~3u;
  return C4 * D * 8 + C4 * 8 + C4 * KS_CS * 4 + (2 * C4 + 4) * 4 + size_t(KS_WARPS) * C4 * 4 +
         2 * size_t(KS_MAX_ROWS) * 4 + KS_MAX_ROWS * 2 + size_t(D) * ks_row_stride(rows) * 2;
}

// centroids cent[c] (c < C) -> f64 norms (sequential chain, common.hpp:141-147)
// and the next assignment's directions dir = float(x / |x|), kept in f64 in
// the [C/4][D][4] layout the assignment loop reads with two 16-B loads
__device__ __forceinline__ void ks_finish(uint32_t C, const float* cent, double* cnorm,
                                          double* dird) {
  const int tid = threadIdx.x;
  __syncthreads();
  if (tid < int(C)) {
    const float* x = cent + tid * KS_CS;
    double s = 0.0;
#pragma unroll 16
    for (int j = 0; j < D; ++j) s = __fma_rn(double(x[j]), double(x[j]), s);
    cnorm[tid] = sqrt(s);
  }
  __syncthreads();
  for (uint32_t e = tid; e < C * D; e += KS_THREADS) {
    const uint32_t c = e / D, j = e % D;
    const double nrm = cnorm[c];
    const float x = cent[c * KS_CS + j];
    const float dv = nrm > 0.0 ? float(double(x) / nrm) : x;
    dird[((c >> 2) * D + j) * 4 + (c & 3)] = double(dv);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// K4 fused: cluster_decode_batch's whole kmeans_cosine (clustering.hpp:160-263
// on one decode batch, 310-332) in ONE launch, one CTA per unit, one batch
// row per thread, everything in shared memory: no per-iteration launch or
// host round trip.  Numerics are the reference's, bit for bit:
//   assignment   a sequential f64 chain per (key, c) (common.hpp:86-90),
//                four clusters interleaved, strict '>' in id order;
//   counts       warp ballots (no atomics);
//   repair       clustering.hpp:128-153, sequential over empty ids;
//   update       f64 member sums in POSITION order (members listed per
//                cluster by __match_any ranks), float(sum / count);
//   directions   normalize(): sequential f64 norm chain, float(x / |x|).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(KS_THREADS, 2)
k_kmeans_small(const uint16_t* __restrict__ keys, uint64_t key_stride, uint32_t rows,
               uint32_t C, uint32_t max_iters, const uint32_t* __restrict__ init_rows,
               float* __restrict__ out_cents, uint32_t c_cap, int32_t* __restrict__ out_labels,
               uint32_t label_stride, uint32_t* __restrict__ n_clusters,
               uint32_t* __restrict__ iters_out, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char ks_raw[];
  const uint32_t u = blockIdx.x;
  const int tid = threadIdx.x, lane = lane_id(), wid = warp_id();
  const uint32_t C4 = (C + 3) & ~3u, RS = ks_row_stride(rows);
  double* dird = reinterpret_cast<double*>(ks_raw);                     // [C4/4][D][4]
  double* cnorm = dird + C4 * D;                                        // [C4]
  float* cent = reinterpret_cast<float*>(cnorm + C4);                   // [C4][KS_CS]
  uint32_t* cnt = reinterpret_cast<uint32_t*>(cent + C4 * KS_CS);       // [C4]
  uint32_t* cbase = cnt + C4;                                           // [C4 + 4]
  uint32_t* wcnt = cbase + C4 + 4;                                      // [KS_WARPS][C4]
  int32_t* lab0 = reinterpret_cast<int32_t*>(wcnt + KS_WARPS * C4);     // [KS_MAX_ROWS]
  int32_t* lab1 = lab0 + KS_MAX_ROWS;                                   // [KS_MAX_ROWS]
  uint16_t* mem = reinterpret_cast<uint16_t*>(lab1 + KS_MAX_ROWS);      // [KS_MAX_ROWS]
  uint16_t* kt = mem + KS_MAX_ROWS;                                     // [D][RS]
  __shared__ uint32_t s_largest, s_lcnt;
  __shared__ double s_wd[KS_WARPS];
  __shared__ uint32_t s_wi[KS_WARPS];
  const uint16_t* kb = keys + u * key_stride;

  // stage the batch transposed, 16-B loads four rounds deep, and run
  // kmeans_cosine's input checks (clustering.hpp:166-172)
  int bad = 0, nonzero = 0;
  const uint4* kb4 = reinterpret_cast<const uint4*>(kb);
  const uint32_t n4 = rows * (D / 8);
  for (uint32_t v0 = tid; v0 < n4; v0 += 4 * KS_THREADS) {
    uint4 x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t v = v0 + k * KS_THREADS;
      x[k] = v < n4 ? __ldg(kb4 + v) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t v = v0 + k * KS_THREADS;
      if (v < n4) {
        const uint32_t r = v / (D / 8), j0 = (v % (D / 8)) * 8;
        const uint32_t w[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint16_t b = uint16_t(w[i >> 1] >> (16 * (i & 1)));
          kt[(j0 + i) * RS + r] = b;
          if ((b & 0x7f80u) == 0x7f80u) bad = 1;
        }
      }
    }
  }
  for (uint32_t e = tid; e < C4 * D; e += KS_THREADS) dird[e] = 0.0;  // padding clusters
  __syncthreads();
  if (tid < int(rows)) {
    double s = 0.0;
#pragma unroll 8
    for (int j = 0; j < D; ++j) {
      const double x = double(bf16_to_f32(kt[j * RS + tid]));
      s = __fma_rn(x, x, s);
    }
    if (sqrt(s) >= 1e-12) nonzero = 1;
  }
  bad = __syncthreads_or(bad);
  nonzero = __syncthreads_or(nonzero);
  if (bad || !nonzero) {
    if (tid == 0) status[u] = bad ? 1 : 2;
    return;
  }
  // init: centroid c = key row init_rows[c] (clustering.hpp:194-198)
  for (uint32_t e = tid; e < C * D; e += KS_THREADS) {
    const uint32_t c = e / D, j = e % D;
    cent[c * KS_CS + j] = bf16_to_f32(kt[j * RS + init_rows[size_t(u) * C + c]]);
  }
  ks_finish(C, cent, cnorm, dird);

  int32_t* lab[2] = {lab0, lab1};
  uint32_t it = 0;
  int converged = 0;
  for (uint32_t t = 0;; ++t) {
    int32_t* cur = lab[t & 1];
    const int32_t* prev = lab[(t & 1) ^ 1];
    // ---- assign (AssignScorer::assign, clustering.hpp:104-115) -------------
    int32_t my = -1;
    if (tid < int(rows)) {
      uint32_t best = 0;
      double bs = -INFINITY;
      for (uint32_t c0 = 0; c0 < C; c0 += 4) {
        const double2* d2 = reinterpret_cast<const double2*>(dird + size_t(c0 >> 2) * D * 4);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll 8
        for (int j = 0; j < D; ++j) {
          const double x = double(bf16_to_f32(kt[j * RS + tid]));
          const double2 a = d2[2 * j], b = d2[2 * j + 1];
          s0 = __fma_rn(x, a.x, s0);
          s1 = __fma_rn(x, a.y, s1);
          s2 = __fma_rn(x, b.x, s2);
          s3 = __fma_rn(x, b.y, s3);
        }
        if (s0 > bs) { bs = s0; best = c0; }
        if (c0 + 1 < C && s1 > bs) { bs = s1; best = c0 + 1; }
        if (c0 + 2 < C && s2 > bs) { bs = s2; best = c0 + 2; }
        if (c0 + 3 < C && s3 > bs) { bs = s3; best = c0 + 3; }
      }
      my = int32_t(best);
      cur[tid] = my;
    }
    // ---- counts: one ballot per (warp, cluster) --------------------------
    for (uint32_t c = 0; c < C; ++c) {
      const unsigned m = __ballot_sync(0xffffffffu, my == int32_t(c));
      if (lane == 0) wcnt[wid * C4 + c] = __popc(m);
    }
    __syncthreads();
    if (tid < int(C)) {
      uint32_t sum = 0;
      for (int w = 0; w < KS_WARPS; ++w) sum += wcnt[w * C4 + tid];
      cnt[tid] = sum;
    }
    __syncthreads();
    // ---- repair_empty_clusters (clustering.hpp:128-153), sequential ids ---
    bool repaired = false;
    for (uint32_t c = 0; c < C; ++c) {
      if (cnt[c] > 0) continue;  // uniform: cnt is shared and stable here
      if (tid == 0) {
        uint32_t l = 0;
        for (uint32_t k = 1; k < C; ++k) if (cnt[k] > cnt[l]) l = k;
        s_largest = l;
        s_lcnt = cnt[l];
      }
      __syncthreads();
      const uint32_t largest = s_largest;
      if (s_lcnt > 1) {
        repaired = true;
        double bd = -1.0;
        uint32_t bv = 0xffffffffu;
        if (tid < int(rows) && uint32_t(cur[tid]) == largest) {
          double na = 0.0, dd = 0.0;
          for (int j = 0; j < D; ++j) {
            const double x = double(bf16_to_f32(kt[j * RS + tid]));
            na = __fma_rn(x, x, na);
            dd = __fma_rn(x, double(cent[largest * KS_CS + j]), dd);
          }
          na = sqrt(na);
          const double nb = cnorm[largest];
          double dist = 1.0;
          if (!(na < 1e-12 || nb < 1e-12)) {
            dist = 1.0 - dd / (na * nb);
            dist = dist < 0.0 ? 0.0 : (dist > 2.0 ? 2.0 : dist);
          }
          bd = dist;
          bv = tid;
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double od = __shfl_xor_sync(0xffffffffu, bd, o);
          const uint32_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
          if (od > bd || (od == bd && ov < bv)) { bd = od; bv = ov; }
        }
        if (lane == 0) { s_wd[wid] = bd; s_wi[wid] = bv; }
        __syncthreads();
        if (tid == 0) {
          double b = s_wd[0];
          uint32_t v = s_wi[0];
          for (int w = 1; w < KS_WARPS; ++w)
            if (s_wd[w] > b || (s_wd[w] == b && s_wi[w] < v)) { b = s_wd[w]; v = s_wi[w]; }
          v = v == 0xffffffffu ? 0u : v;  // no member beat -1: the victim stays 0
          cur[v] = int32_t(c);
          cnt[largest]--;
          cnt[c]++;
        }
      }
      __syncthreads();
    }
    if (repaired && tid < int(rows)) my = cur[tid];
    // ---- convergence: next == labels (after repair) ------------------------
    if (t > 0) {
      const int ch = __syncthreads_or(tid < int(rows) && my != prev[tid]);
      if (!ch) { converged = 1; it = t; break; }
      if (t == max_iters) { it = t; break; }
    } else {
      __syncthreads();  // every repair-loop read of cnt[] before it is rewritten below
    }
    // ---- update_centroids (clustering.hpp:205-218) --------------------------
    // members of each cluster in position order: per-warp counts, their
    // exclusive scan over warps, then each row's rank among its warp's
    // same-cluster lanes
    if (repaired) {
      for (uint32_t c = 0; c < C; ++c) {
        const unsigned m = __ballot_sync(0xffffffffu, my == int32_t(c));
        if (lane == 0) wcnt[wid * C4 + c] = __popc(m);
      }
      __syncthreads();
    }
    if (tid < int(C)) {
      uint32_t sum = 0;
      for (int w = 0; w < KS_WARPS; ++w) {
        const uint32_t x = wcnt[w * C4 + tid];
        wcnt[w * C4 + tid] = sum;
        sum += x;
      }
      cnt[tid] = sum;
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t b = 0;
      for (uint32_t c = 0; c < C; ++c) { cbase[c] = b; b += cnt[c]; }
      cbase[C] = b;
    }
    __syncthreads();
    {
      const unsigned same = __match_any_sync(0xffffffffu, my);
      if (my >= 0) {
        const uint32_t rank = __popc(same & ((1u << lane) - 1u));
        mem[cbase[my] + wcnt[wid * C4 + my] + rank] = uint16_t(tid);
      }
    }
    __syncthreads();
    for (uint32_t e = tid; e < C * D; e += KS_THREADS) {
      const uint32_t c = e / D, j = e % D;
      const uint32_t i0 = cbase[c], i1 = cbase[c + 1];
      const uint16_t* col = kt + j * RS;
      double a = 0.0;
      uint32_t i = i0;
      for (; i + 4 <= i1; i += 4) {
        const float x0 = bf16_to_f32(col[mem[i]]), x1 = bf16_to_f32(col[mem[i + 1]]);
        const float x2 = bf16_to_f32(col[mem[i + 2]]), x3 = bf16_to_f32(col[mem[i + 3]]);
        a += double(x0);
        a += double(x1);
        a += double(x2);
        a += double(x3);
      }
      for (; i < i1; ++i) a += double(bf16_to_f32(col[mem[i]]));
      cent[c * KS_CS + j] = float(a / double(i1 - i0));
    }
    ks_finish(C, cent, cnorm, dird);
  }
  // final labels = the last assignment (equal to the previous one when
  // converged); append (cluster_decode_batch: fresh ids from n_clusters)
  const int32_t* fin = lab[it & 1];
  const uint32_t base = n_clusters[u];
  for (uint32_t e = tid; e < C * D; e += KS_THREADS)
    out_cents[(size_t(u) * c_cap + base) * D + e] = cent[(e / D) * KS_CS + e % D];
  for (uint32_t r = tid; r < rows; r += KS_THREADS)
    out_labels[size_t(u) * label_stride + r] = fin[r] + int32_t(base);
  __syncthreads();
  if (tid == 0) {
    n_clusters[u] = base + C;
    iters_out[u] = it | (converged ? 0x80000000u : 0u);
    status[u] = 0;
  }
}

bool kmeans_small_supported(uint32_t rows, uint32_t C) {
  return rows >= 1 && rows <= KS_MAX_ROWS && C >= 1 && C <= KS_MAX_C;
}

int launch_kmeans_small(cudaStream_t st, const uint16_t* keys, uint64_t key_stride,
                        uint32_t n_units, uint32_t rows, uint32_t C, uint32_t max_iters,
                        const uint32_t* init_rows, float* cents, uint32_t c_cap,
                        int32_t* labels, uint32_t label_stride, uint32_t* n_clusters,
                        uint32_t* iters, int32_t* status) {
  const size_t smem = ks_smem_bytes(rows, C);
  CKV_CUDA_TRY(smem_optin((const void*)k_kmeans_small, 200 * 1024));
  k_kmeans_small<<<n_units, KS_THREADS, smem, st>>>(keys, key_stride, rows, C, max_iters,
                                                     init_rows, cents, c_cap, labels,
                                                     label_stride, n_clusters, iters, status);
  CKV_LAUNCH_CHECK("k_kmeans_small");
  return CKV_OK;
}

}  // namespace ckvb

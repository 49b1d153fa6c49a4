// ckv_kmeans_dev.cuh — device pieces of the cosine k-means shared by the
// single-GPU driver (ckv_kmeans.cu) and the sequence-sharded one
// (ckv_kmshard.cu), so both produce the same bits.
#pragma once
#include "ckv_common.cuh"

namespace ckvb {

// cosine_distance (clustering.hpp:59-65) of a bf16 key and an f32 centroid
// whose f64 norm nb is precomputed.
__device__ __forceinline__ double cosine_distance_dev(const uint16_t* k, const float* c,
                                                      double nb) {
  double na = sqrt(dot_seq_bb(k, k));
  if (na < 1e-12 || nb < 1e-12) return 1.0;
  double dd = 1.0 - dot_seq_bf(k, c) / (na * nb);
  return dd < 0.0 ? 0.0 : (dd > 2.0 ? 2.0 : dd);
}

// The end of update_centroids for one (unit, cluster) by one warp, lane L
// holding dims 4L..4L+3 of the f64 member sum: centroid = float(sum / count)
// (clustering.hpp:214-217), then the next pass's AssignScorer direction
// normalize(centroid) (common.hpp:141-147; sequential f64 norm chain), its
// fp16 copy h(dir) (the tensor-core B operand), the f64 norm (cosine_distance)
// and |dir - h(dir)| (the tensor-core error band).
__device__ __forceinline__ void finish_centroid(double a0, double a1, double a2, double a3,
                                                double count, float* __restrict__ ct,
                                                float* __restrict__ dr,
                                                uint16_t* __restrict__ db,
                                                double* __restrict__ cnorm_out,
                                                float* __restrict__ deps_out) {
  const int lane = lane_id();
  float x0 = float(a0 / count), x1 = float(a1 / count), x2 = float(a2 / count),
        x3 = float(a3 / count);
  reinterpret_cast<float4*>(ct)[lane] = make_float4(x0, x1, x2, x3);
  // sequential norm chain over j = 0..127 (lane L holds j = 4L..4L+3): the
  // values are staged once in shared memory as f64 and every lane walks them
  // with broadcast 16-B loads (64 LDS per warp instead of 256 shuffles)
  __shared__ __align__(16) double fc_stage[8][D];  // callers run <= 8 warps per block
  double* stg = fc_stage[warp_id()];
  reinterpret_cast<double2*>(stg)[2 * lane] = make_double2(double(x0), double(x1));
  reinterpret_cast<double2*>(stg)[2 * lane + 1] = make_double2(double(x2), double(x3));
  __syncwarp();
  double s = 0.0;
#pragma unroll 16
  for (int j = 0; j < D / 2; ++j) {
    const double2 y = reinterpret_cast<const double2*>(stg)[j];
    s = __fma_rn(y.x, y.x, s);
    s = __fma_rn(y.y, y.y, s);
  }
  __syncwarp();  // the stage is free for the warp's next call
  const double nrm = sqrt(s);
  if (lane == 0) *cnorm_out = nrm;
  float d0 = nrm > 0.0 ? float(double(x0) / nrm) : x0;
  float d1 = nrm > 0.0 ? float(double(x1) / nrm) : x1;
  float d2 = nrm > 0.0 ? float(double(x2) / nrm) : x2;
  float d3 = nrm > 0.0 ? float(double(x3) / nrm) : x3;
  reinterpret_cast<float4*>(dr)[lane] = make_float4(d0, d1, d2, d3);
  uint2 pk;
  const uint16_t h0 = f32_to_f16_tc(d0), h1 = f32_to_f16_tc(d1), h2 = f32_to_f16_tc(d2),
                 h3 = f32_to_f16_tc(d3);
  pk.x = uint32_t(h0) | (uint32_t(h1) << 16);
  pk.y = uint32_t(h2) | (uint32_t(h3) << 16);
  reinterpret_cast<uint2*>(db)[lane] = pk;
  // |dir - h(dir)|: the per-centroid error the tensor-core band uses
  const double e0 = double(d0) - double(f16_to_f32(h0));
  const double e1 = double(d1) - double(f16_to_f32(h1));
  const double e2 = double(d2) - double(f16_to_f32(h2));
  const double e3 = double(d3) - double(f16_to_f32(h3));
  const double ee = warp_sum(e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3);
  if (lane == 0) *deps_out = float(sqrt(ee)) * 1.0001f;
}

}  // namespace ckvb

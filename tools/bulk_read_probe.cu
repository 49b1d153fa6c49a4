// Read-bandwidth probe (tools only, not product): what a one-pass HBM read
// stream reaches on this B200, to place k_attend's memory pipeline (95.4 us
// for 515 MB at config B) against a ceiling.
//   (a) plain 16-B loads (ld.global.nc.L1::no_allocate), grid-stride, U in flight
//   (b) cp.async.bulk global->shared, S-byte pieces, NS-stage ring per CTA,
//       no consumer work (the stage is re-armed as soon as it lands)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulk_read_probe tools/bulk_read_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int U>
__global__ void k_ld(const uint4* __restrict__ a, size_t n16, unsigned long long* sink) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(a + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void k_bulk(const char* __restrict__ a, size_t bytes, uint32_t piece, int ns,
                       int hint, unsigned long long* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < ns; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  size_t npieces = bytes / piece;
  uint32_t phase[16] = {0};
  size_t it = 0;
  for (size_t p = blockIdx.x; p < npieces; p += gridDim.x, ++it) {
    int s = (int)(it % ns);
    if (it >= (size_t)ns) {  // wait for the stage's previous copy
      uint32_t b = su32(&bar[s]);
      asm volatile(
          "{ .reg .pred q; W: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W; }" ::"r"(b),
          "r"(phase[s]) : "memory");
      phase[s] ^= 1;
    }
    uint32_t b = su32(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(piece) : "memory");
    if (hint)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              su32(sm + (size_t)s * piece)),
          "l"(a + p * piece), "r"(piece), "r"(b), "l"(pol) : "memory");
    else
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(sm + (size_t)s * piece)),
                   "l"(a + p * piece), "r"(piece), "r"(b) : "memory");
  }
  for (int s = 0; s < ns && (size_t)s < it; ++s) {
    uint32_t b = su32(&bar[s]);
    asm volatile(
        "{ .reg .pred q; W2: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W2; }" ::"r"(b),
        "r"(phase[s]) : "memory");
  }
  if (sm[0] == 123 && sm[1] == 45) atomicAdd(sink, 1ull);
}

int main() {
  const size_t bytes = 512ull << 20;  // ~ k_attend's 515 MB per launch
  char* a;
  unsigned long long* sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(a, 1, bytes);
  char* flush;
  cudaMalloc(&flush, 256ull << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  auto timeit = [&](auto launch) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaMemsetAsync(flush, r, 256ull << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    return best;
  };
  for (int bpsm : {2, 4, 8}) {
    float ms = timeit([&] { k_ld<4><<<sms * bpsm, 256>>>((const uint4*)a, bytes / 16, sink); });
    printf("ld.v4 U=4 %d blk/SM x256: %.1f us  %.0f GB/s\n", bpsm, ms * 1e3, bytes / ms / 1e6);
    ms = timeit([&] { k_ld<8><<<sms * bpsm, 256>>>((const uint4*)a, bytes / 16, sink); });
    printf("ld.v4 U=8 %d blk/SM x256: %.1f us  %.0f GB/s\n", bpsm, ms * 1e3, bytes / ms / 1e6);
  }
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (uint32_t piece : {8192u, 16384u, 32768u}) {
    for (int ns : {2, 3, 4, 6}) {
      for (int cps : {1, 2, 3, 4}) {
        size_t smem = (size_t)piece * ns;
        if (smem * cps > 220 * 1024) continue;
        for (int hint : {0, 1}) {
          float ms = timeit([&] { k_bulk<<<sms * cps, 32, smem>>>(a, bytes, piece, ns, hint, sink); });
          printf("bulk piece=%5u ns=%d cta/SM=%d hint=%d inflight/SM=%4zu KB: %.1f us  %.0f GB/s\n", piece,
                 ns, cps, hint, smem * cps / 1024, ms * 1e3, bytes / ms / 1e6);
        }
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

// PCIe read probe for the zero-copy session step: 256 CTAs each read 2 KB
// (one kv unit's 4 q rows, f32) from mapped pinned host memory, by
// (a) float4 loads per lane, (b) one cp.async.bulk per CTA into shared
// memory, (c) a copy-engine cudaMemcpyAsync of the whole 512 KB, and the
// 256 x 512 B k/v rows by (a) / (b).  Event-timed, median of 50.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pcie_probe tools/pcie_probe.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void k_ld(const float4* __restrict__ src, float4* dst, int per_cta) {
  const int n = per_cta / 16;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    dst[size_t(blockIdx.x) * n + i] = __ldg(src + size_t(blockIdx.x) * n + i);
}

__global__ void k_bulk(const char* __restrict__ src, char* dst, int per_cta) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned sb = unsigned(__cvta_generic_to_shared(&bar));
  const unsigned sd = unsigned(__cvta_generic_to_shared(sm));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sb), "r"(per_cta) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sd), "l"(src + size_t(blockIdx.x) * per_cta), "r"(per_cta), "r"(sb) : "memory");
  }
  __syncthreads();
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(sb) : "memory");
  const int n = per_cta / 16;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    reinterpret_cast<float4*>(dst)[size_t(blockIdx.x) * n + i] = reinterpret_cast<float4*>(sm)[i];
}

template <typename F>
static float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> t;
  for (int r = 0; r < 60; ++r) {
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r >= 10) t.push_back(ms * 1000.f);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int main() {
  const int ctas = 256;
  char* h; char* d;
  cudaHostAlloc(&h, 1 << 22, cudaHostAllocMapped);
  cudaMalloc(&d, 1 << 22);
  for (int per : {2048, 512}) {
    const size_t tot = size_t(ctas) * per;
    float a = timeit([&] { k_ld<<<ctas, 128>>>((const float4*)h, (float4*)d, per); });
    float b = timeit([&] { k_bulk<<<ctas, 128, per>>>(h, d, per); });
    float c = timeit([&] { cudaMemcpyAsync(d, h, tot, cudaMemcpyHostToDevice); });
    float e = timeit([&] { k_ld<<<ctas, 128>>>((const float4*)d, (float4*)(d + (1 << 21)), per); });
    printf("%d x %d B: ld %.1f us (%.1f GB/s)  bulk %.1f us (%.1f GB/s)  memcpy %.1f us (%.1f GB/s)  "
           "device-ld %.1f us\n", ctas, per, a, tot / a / 1e3, b, tot / b / 1e3, c, tot / c / 1e3, e);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

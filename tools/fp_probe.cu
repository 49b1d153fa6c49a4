// Microbenchmark: DFMA / FFMA latency and throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T, int CHAINS>
__global__ void chains(T* out, int iters, T a, T b) {
  T acc[CHAINS];
  for (int c = 0; c < CHAINS; ++c) acc[c] = T(threadIdx.x + c);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  T s = 0;
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename T, int CHAINS>
void run(const char* name, int blocks, int threads, int iters) {
  T* out;
  cudaMalloc(&out, sizeof(T) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  chains<T, CHAINS><<<blocks, threads>>>(out, iters, T(0.999), T(0.001));
  cudaEventRecord(e0);
  chains<T, CHAINS><<<blocks, threads>>>(out, iters, T(0.999), T(0.001));
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fmas = double(blocks) * threads * iters * CHAINS;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-28s blocks=%5d thr=%4d: %8.3f ms  %8.2f TFMA/s  per-chain-step %.1f cycles\n", name,
         blocks, threads, ms, fmas / ms / 1e9, ms * 1e-3 * clk * 1e3 / iters);
  cudaFree(out);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<double, 1>("f64 latency (1 warp)", 1, 32, 100000);
  run<float, 1>("f32 latency (1 warp)", 1, 32, 100000);
  run<double, 8>("f64 throughput", sms * 8, 256, 20000);
  run<float, 8>("f32 throughput", sms * 8, 256, 20000);
  return 0;
}

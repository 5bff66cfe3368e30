// FP64 FMA throughput microbenchmark ("confirm the FMA rate with a
// microbenchmark before quoting FP64 pipe %").  Every thread runs 16 independent DFMA chains;
// grid = 8 CTAs of 256 threads per SM.  Prints one JSON line: measured FP64 TFLOP/s (2 flops per
// FMA), the SM count and the SM clock the driver reports.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak scripts/fp64_peak.cu
#include <cuda_runtime.h>
#include <cstdio>

constexpr int kChains = 16;
constexpr int kIters = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 1234.5) out[0] = s;  // keeps the chains alive
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  const int grid = 8 * sms, block = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dfma<<<grid, block>>>(out, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<grid, block>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fmas = static_cast<double>(grid) * block * kIters * kChains;
  const double tflops = 2.0 * fmas / (best * 1e-3) / 1e12;
  std::printf("{\"fp64_tflops\": %.2f, \"fma_per_clk_per_sm_at_max_clock\": %.1f, \"sms\": %d, "
              "\"sm_max_mhz\": %.0f, \"best_ms\": %.4f, \"how\": \"%d CTAs x %d threads x %d chains x %d DFMA, "
              "best of 10, CUDA events\"}\n",
              tflops, fmas / (best * 1e-3) / (sms * clk_khz * 1e3), sms, clk_khz / 1e3, best, grid, block, kChains,
              kIters);
  cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? 0 : 1;
}

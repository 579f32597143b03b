// fp64 FMA peak of this B200 (SURVEY.md §8d asks for the fp64 fraction beside
// the HBM one; MEASURED_PEAKS.json has no fp64 figure). Each thread runs 8
// independent DFMA chains (enough ILP to hide the pipe latency), 148 x 8 CTAs
// of 256 threads; best of 10 timed launches with CUDA events.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void dfma_chains(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;  // keeps the chains live
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_chains<<<blocks, threads>>>(out, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    dfma_chains<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * kChains * kIters * double(blocks) * threads;
  const double tf = flops / (best * 1e-3) / 1e12;
  const double per_clk = flops / 2 / (best * 1e-3) / (sms * (clk * 1e3));
  std::printf("{\"fp64_tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, \"clock_mhz_attr\": %.0f, "
              "\"dfma_per_clk_per_sm_at_attr_clock\": %.1f, \"how\": \"%d CTAs x %d threads x %d chains x %d DFMA, "
              "best of 10, CUDA events\", \"error\": \"%s\"}\n",
              tf, best, sms, clk / 1e3, per_clk, blocks, threads, kChains, kIters,
              cudaGetErrorString(cudaGetLastError()));
  return 0;
}

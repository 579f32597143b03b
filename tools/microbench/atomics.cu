// Microbenchmark: shared-memory fp64 accumulation options on sm_100a, and
// global fp64 RED with scattered vs sector-coalesced lanes. Informs the
// scatter design. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ACC = 6144;
constexpr int OPS = 4096;

__device__ __forceinline__ unsigned hash(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; return x ^ (x >> 16); }

template <int MODE>
__global__ void smem_acc(double* out, int spread) {
  __shared__ double acc[ACC];
  for (int i = threadIdx.x; i < ACC; i += blockDim.x) acc[i] = 0.0;
  __syncthreads();
  unsigned s = hash(blockIdx.x * 1024 + threadIdx.x);
  double v = 1.0 + threadIdx.x;
  for (int k = 0; k < OPS; ++k) {
    s = hash(s + k);
    // spread: random slot; otherwise lanes of a warp hit a 64-slot window (row-like locality)
    const int idx = spread ? (s % ACC) : ((threadIdx.x / 32) * 64 + (s & 63)) % ACC;
    if (MODE == 0) atomicAdd(&acc[idx], v);                       // fp64 CAS loop
    if (MODE == 1) acc[idx] += v;                                  // plain RMW (racy, throughput only)
    if (MODE == 2) atomicAdd((unsigned long long*)&acc[idx], 3ull); // native 64-bit int add
  }
  __syncthreads();
  double t = 0;
  for (int i = threadIdx.x; i < ACC; i += blockDim.x) t += acc[i];
  if (t == 12345.0) out[0] = t;
}

template <int MODE>
__global__ void global_red(double* vals, long long n, int per_thread) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  unsigned s = hash((unsigned)tid);
  for (int k = 0; k < per_thread; ++k) {
    s = hash(s + k);
    long long idx;
    if (MODE == 0) idx = (long long)(s % (unsigned)(n / 8)) * 8 + (lane & 7);          // scattered (1 lane per random 64B)
    else idx = (long long)(__shfl_sync(0xffffffffu, s, lane / 10 * 10) % (unsigned)(n / 64)) * 64 + lane % 10 * 3 % 38; // 10-lane groups in one ~300B row
    if (MODE == 0 || lane < 30) atomicAdd(vals + idx, 1.0);
  }
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 2 * 4;
  const char* names[] = {"smem fp64 atomicAdd (CAS)", "smem plain RMW (LDS+DADD+STS)", "smem u64 atomicAdd"};
  for (int spread = 1; spread >= 0; --spread)
    for (int mode = 0; mode < 3; ++mode) {
      auto k = mode == 0 ? smem_acc<0> : mode == 1 ? smem_acc<1> : smem_acc<2>;
      k<<<grid, 256>>>(out, spread);
      cudaEventRecord(a);
      k<<<grid, 256>>>(out, spread);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)grid * 256 * OPS;
      printf("%-34s %-8s %8.3f ms  %7.1f Gop/s  %6.2f lane-ops/clk/SM\n", names[mode], spread ? "random" : "window", ms,
             ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.9e9);
    }
  const long long n = 500000000LL;  // 4 GB of doubles
  double* vals;
  cudaMalloc(&vals, n * 8);
  cudaMemset(vals, 0, n * 8);
  for (int mode = 0; mode < 2; ++mode) {
    auto k = mode == 0 ? global_red<0> : global_red<1>;
    const int per = 64;
    k<<<sms * 16, 256>>>(vals, n, per);
    cudaEventRecord(a);
    k<<<sms * 16, 256>>>(vals, n, per);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)sms * 16 * 256 * per * (mode == 0 ? 1.0 : 30.0 / 32.0);
    printf("global RED.F64 %-24s %8.3f ms  %7.1f Gop/s\n", mode == 0 ? "scattered lanes" : "10-lane row groups", ms, ops / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

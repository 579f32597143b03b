// Downstream consumer of the assembled system: CSR
// SpMV and the reference's unpreconditioned conjugate gradients on the device
// (replaces linalg::matvec(EllMatrix) linalg.cpp:35-49 and cg_solve
// linalg.cpp:61-96, OpenMP on the host). fp64 throughout; reductions are
// two-pass (per-block partials, one final block) so results are bitwise
// reproducible run to run.
#include <cmath>
#include <cstdint>

#include "kernels.hpp"

namespace ffb::kernels {

namespace {

constexpr int kThreads = 256;

// one warp per row: lanes stride the row, shuffle reduction
__global__ void spmv_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ a, const double* __restrict__ x, double* __restrict__ y,
                            int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + (threadIdx.x >> 5); r < n; r += warps) {
    const int64_t b = rp[r], e = rp[r + 1];
    double s = 0.0;
    for (int64_t k = b + lane; k < e; k += 32) s += __ldg(a + k) * __ldg(x + ci[k]);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[r] = s;
  }
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  __syncthreads();
  return t;
}

// partial[blockIdx] = sum over the block's grid-stride share of a[i] * b[i]
__global__ void dot_partial(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                            double* __restrict__ partial) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s += a[i] * b[i];
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void dot_final(const double* __restrict__ partial, int n, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) *out = t;
}

// x += alpha p; r -= alpha ap
__global__ void cg_update_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ ap, double alpha, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    x[i] += alpha * p[i];
    r[i] -= alpha * ap[i];
  }
}

// p = r + beta p
__global__ void cg_update_p(double* __restrict__ p, const double* __restrict__ r, double beta, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = r[i] + beta * p[i];
}

int grid(int64_t n, int sm_count) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  const int64_t cap = static_cast<int64_t>(sm_count) * 8;
  return static_cast<int>(g < 1 ? 1 : (g < cap ? g : cap));
}

}  // namespace

cudaError_t spmv(const int64_t* rp, const int32_t* ci, const double* a, const double* x, double* y, int64_t n,
                 int sm_count, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = (n + kThreads / 32 - 1) / (kThreads / 32);
  const int64_t cap = static_cast<int64_t>(sm_count) * 16;
  spmv_kernel<<<static_cast<int>(blocks < cap ? blocks : cap), kThreads, 0, s>>>(rp, ci, a, x, y, n);
  return cudaGetLastError();
}

cudaError_t cg_solve(const int64_t* rp, const int32_t* ci, const double* a, const double* b, double* x, int64_t n,
                     double tol, int max_iter, int sm_count, cudaStream_t s, CgStats* st) {
  *st = CgStats{};
  const int g = grid(n, sm_count);
  double *r = nullptr, *p = nullptr, *ap = nullptr, *partial = nullptr, *scal = nullptr, *hs = nullptr;
  cudaError_t err = cudaSuccess;
  auto done = [&](cudaError_t e) {
    cudaFree(r);
    cudaFree(p);
    cudaFree(ap);
    cudaFree(partial);
    cudaFree(scal);
    cudaFreeHost(hs);
    return e;
  };
  if ((err = cudaMalloc(&r, (n > 0 ? n : 1) * sizeof(double))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&p, (n > 0 ? n : 1) * sizeof(double))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&ap, (n > 0 ? n : 1) * sizeof(double))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&partial, g * sizeof(double))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&scal, 2 * sizeof(double))) != cudaSuccess) return done(err);
  if ((err = cudaMallocHost(&hs, 2 * sizeof(double))) != cudaSuccess) return done(err);
  auto dot = [&](const double* u, const double* v, double* out) -> double {
    dot_partial<<<g, kThreads, 0, s>>>(u, v, n, partial);
    dot_final<<<1, kThreads, 0, s>>>(partial, g, scal);
    cudaMemcpyAsync(out, scal, sizeof(double), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return *out;
  };
  // linalg.cpp:61-96: x = 0, r = b, p = r
  cudaMemsetAsync(x, 0, n * sizeof(double), s);
  cudaMemcpyAsync(r, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  cudaMemcpyAsync(p, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  double rr = dot(r, r, hs);
  const double bnorm = std::sqrt(dot(b, b, hs));
  if ((err = cudaGetLastError()) != cudaSuccess) return done(err);
  if (bnorm == 0.0) {
    st->converged = 1;
    return done(cudaSuccess);
  }
  for (int it = 0; it < max_iter; ++it) {
    if (std::sqrt(rr) <= tol * bnorm) {
      st->converged = 1;
      break;
    }
    if ((err = spmv(rp, ci, a, p, ap, n, sm_count, s)) != cudaSuccess) return done(err);
    const double pap = dot(p, ap, hs);
    const double alpha = rr / pap;
    if (!std::isfinite(alpha)) {
      st->breakdown = 1;
      return done(cudaSuccess);
    }
    cg_update_xr<<<g, kThreads, 0, s>>>(x, r, p, ap, alpha, n);
    const double rr_new = dot(r, r, hs);
    if (!std::isfinite(rr_new)) {
      st->breakdown = 2;
      return done(cudaSuccess);
    }
    const double beta = rr_new / rr;
    rr = rr_new;
    cg_update_p<<<g, kThreads, 0, s>>>(p, r, beta, n);
    st->iterations = it + 1;
  }
  st->residual = std::sqrt(rr) / bnorm;
  st->converged = st->converged || st->residual <= tol;
  if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);
  return done(cudaGetLastError());
}

}  // namespace ffb::kernels

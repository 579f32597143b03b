// Mesh validation on the device (replaces fem::Mesh::validate,
// /root/reference/proj/src/fem/fem.cpp:17-34, which flatten_mesh and
// build_sparsity call first, device.cpp:49 and :67) and the exact
// connectivity comparison behind ff_assemble's re-upload check.
//
// One thread per element evaluates the reference's checks in the reference's
// order -- vertex index range, duplicate vertices, then orientation -- plus
// the same two checks on the DOF connectivity of higher-order spaces; the
// lowest failing element wins (atomicMin), so the host reports exactly the
// element the reference's sequential loop throws for. The host rebuilds the
// message from that one element (capi.cpp: mesh_error).
#include <cstdint>

#include "kernels.hpp"

namespace ffb::kernels {

namespace {

constexpr int kThreads = 256;

int grid_for(int64_t n, int cap) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

__global__ void validate_kernel(const double* __restrict__ coords, int dim, int64_t nv,
                                const int32_t* __restrict__ vconn, const int32_t* __restrict__ dconn, int k,
                                int64_t n_dofs, int64_t ne, int orient, unsigned long long* __restrict__ bad) {
  const int nn = dim + 1;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < ne;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t v[4];
    bool ok = true;
    for (int a = 0; a < nn; ++a) {
      v[a] = vconn[t * nn + a];
      ok = ok && v[a] >= 0 && v[a] < nv;
    }
    for (int a = 0; ok && a < nn; ++a)
      for (int b = a + 1; b < nn; ++b) ok = ok && v[a] != v[b];
    if (ok && dconn) {
      for (int a = 0; ok && a < k; ++a) {
        const int32_t d = dconn[t * k + a];
        ok = d >= 0 && d < n_dofs;
        for (int b = 0; ok && b < a; ++b) ok = dconn[t * k + b] != d;
      }
    }
    if (ok && orient) {
      // fem.cpp:9-15 (signed area) and its tetrahedral analogue, same
      // operation order as the host Mesh::signed_area / signed_volume
      double meas;
      if (dim == 2) {
        const double ax = coords[2 * v[0]], ay = coords[2 * v[0] + 1];
        const double bx = coords[2 * v[1]], by = coords[2 * v[1] + 1];
        const double cx = coords[2 * v[2]], cy = coords[2 * v[2] + 1];
        meas = 0.5 * ((bx - ax) * (cy - ay) - (cx - ax) * (by - ay));
      } else {
        double m[3][3];
        for (int c = 0; c < 3; ++c)
          for (int r = 0; r < 3; ++r) m[r][c] = coords[3 * v[c + 1] + r] - coords[3 * v[0] + r];
        const double det = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                           m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                           m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
        meas = det / 6.0;
      }
      ok = meas > 0.0;
    }
    if (!ok) atomicMin(bad, static_cast<unsigned long long>(t));
  }
}

// dst := src; *diff |= (dst != src) anywhere (exact, element by element)
__global__ void copy_compare_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n,
                                    unsigned long long* __restrict__ diff) {
  bool d = false;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t x = src[t];
    if (dst[t] != x) {
      d = true;
      dst[t] = x;
    }
  }
  if (__any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) atomicOr(diff, 1ull);
}

// *diff |= 1 when src and dst differ anywhere (exact; dst is not written)
__global__ void compare_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t n,
                               unsigned long long* __restrict__ diff) {
  bool d = false;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d |= src[t] != dst[t];
  if (__any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) atomicOr(diff, 1ull);
}

}  // namespace

cudaError_t compare(const int32_t* d_src, const int32_t* d_dst, int64_t n, unsigned long long* d_diff, int sm_count,
                    cudaStream_t s) {
  if (n > 0) compare_kernel<<<grid_for(n, sm_count * 8), kThreads, 0, s>>>(d_src, d_dst, n, d_diff);
  return cudaGetLastError();
}

cudaError_t validate_mesh(const double* d_coords, int dim, int64_t nv, const int32_t* d_vconn, const int32_t* d_dconn,
                          int k, int64_t n_dofs, int64_t ne, bool orient, unsigned long long* d_bad, int sm_count,
                          cudaStream_t s) {
  cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), s);
  if (ne > 0)
    validate_kernel<<<grid_for(ne, sm_count * 8), kThreads, 0, s>>>(d_coords, dim, nv, d_vconn, d_dconn, k, n_dofs, ne,
                                                                    orient ? 1 : 0, d_bad);
  return cudaGetLastError();
}

cudaError_t copy_compare(const int32_t* d_src, int32_t* d_dst, int64_t n, unsigned long long* d_diff, int sm_count,
                         cudaStream_t s) {
  if (n > 0) copy_compare_kernel<<<grid_for(n, sm_count * 8), kThreads, 0, s>>>(d_src, d_dst, n, d_diff);
  return cudaGetLastError();
}

}  // namespace ffb::kernels

// K1 -- GPU CSR sparsity builder (replaces device::build_sparsity,
// /root/reference/proj/src/device/device.cpp:66-88, std::set per row on one
// core) and K0 -- the zero-fill of values/rhs that precedes the atomic
// scatter. Compiled offline by nvcc for sm_100a.
//
// Pattern rules kept bit-exact with the reference: every row contains its
// diagonal (device.cpp:70) and the columns of every element it shares, sorted
// ascending and unique. Construction: one 64-bit key ((row-row_begin) << 32 |
// col) per owned off-diagonal element DOF pair plus one diagonal key per row
// -> CUB radix sort -> unique -> row boundaries. The element slot plan
// (position of column dof[b] inside row dof[a], stored as u8/u16 per local
// entry) is derived from the finished pattern with one binary search per
// entry; it is what lets the numeric kernel scatter without any search.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <unordered_map>
#include <vector>

#include "kernels.hpp"

namespace ffb::kernels {

namespace {

constexpr int kThreads = 256;

__global__ void pair_keys(const int32_t* __restrict__ dconn, int64_t ne, int k, int64_t rb, int64_t re,
                          uint64_t* __restrict__ keys) {
  const int64_t n_rows = re - rb;
  const int per = k * (k - 1);
  const uint64_t invalid = static_cast<uint64_t>(n_rows) << 32;  // sorts after every owned key
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < ne * per;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = t / per;
    const int p = static_cast<int>(t - e * per);
    const int a = p / (k - 1);
    int b = p - a * (k - 1);
    b += (b >= a);  // skip b == a (the diagonal is added explicitly)
    const int32_t* d = dconn + e * k;
    const int64_t row = d[a];
    const int64_t col = d[b];
    keys[t] = (row >= rb && row < re) ? (static_cast<uint64_t>(row - rb) << 32) | static_cast<uint32_t>(col) : invalid;
  }
}

__global__ void diagonal_keys(int64_t rb, int64_t n_rows, uint64_t* __restrict__ keys) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    keys[r] = (static_cast<uint64_t>(r) << 32) | static_cast<uint32_t>(r + rb);
}

// unique sorted keys -> row_ptr (row starts) and col_idx
__global__ void split_keys(const uint64_t* __restrict__ keys, const int64_t* __restrict__ n_unique, int64_t n_rows,
                           int64_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx) {
  const int64_t n = *n_unique;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = keys[t];
    const int64_t row = static_cast<int64_t>(key >> 32);
    if (row >= n_rows) continue;  // the single trailing "invalid" key
    col_idx[t] = static_cast<int32_t>(key & 0xffffffffu);
    const int64_t prev = t == 0 ? -1 : static_cast<int64_t>(keys[t - 1] >> 32);
    for (int64_t r = prev + 1; r <= row; ++r) row_ptr[r] = t;  // empty rows impossible (diagonal)
    if (t == n - 1 || static_cast<int64_t>(keys[t + 1] >> 32) >= n_rows) row_ptr[n_rows] = t + 1;
  }
}

__global__ void row_max(const int64_t* __restrict__ row_ptr, int64_t n_rows, int* __restrict__ out) {
  int m = 0;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = max(m, static_cast<int>(row_ptr[r + 1] - row_ptr[r]));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

template <typename SlotT>
__global__ void element_slots(const int32_t* __restrict__ dconn, int64_t ne, int k, int64_t rb, int64_t re,
                              const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                              SlotT* __restrict__ slots, unsigned long long* __restrict__ bad_row) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < ne * k;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = t / k;
    const int a = static_cast<int>(t - e * k);
    const int32_t* d = dconn + e * k;
    const int64_t row = d[a];
    SlotT* out = slots + t * k;
    if (row < rb || row >= re) {
      for (int b = 0; b < k; ++b) out[b] = 0;
      continue;
    }
    const int64_t begin = row_ptr[row - rb], end = row_ptr[row - rb + 1];
    for (int b = 0; b < k; ++b) {
      const int32_t col = d[b];
      int64_t lo = begin, hi = end;  // lower_bound, device.cpp:276-284
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (col_idx[mid] < col)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo >= end || col_idx[lo] != col) {
        atomicMin(bad_row, static_cast<unsigned long long>(row));
        out[b] = 0;
      } else {
        out[b] = static_cast<SlotT>(lo - begin);
      }
    }
  }
}

__global__ void zero_kernel(double* __restrict__ a, int64_t na, double* __restrict__ b, int64_t nb,
                            unsigned long long* __restrict__ status) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (tid < 2 && status) status[tid] = ~0ull;
  // 32-byte stores (two double2) per thread and iteration
  const bool aligned = (reinterpret_cast<uintptr_t>(a) & 15) == 0;
  const int64_t n2 = aligned ? na / 2 : 0;
  double2* a2 = reinterpret_cast<double2*>(a);
  const double2 z = make_double2(0.0, 0.0);
  for (int64_t i = tid; i < n2; i += stride) a2[i] = z;
  for (int64_t i = 2 * n2 + tid; i < na; i += stride) a[i] = 0.0;
  for (int64_t i = tid; i < nb; i += stride) b[i] = 0.0;
}


// ---- row-gather plan ---------------------------------------------------------
//
// The row-gather kernel (assemble_template.inc: ff_gather_rows) gives every
// owned CSR row to one lane. This plan (built once per (pattern, mesh)):
//  1. lists the incidences (e, i) of every row (element e has the row's DOF at
//     local index i) and sorts them by (i, slot bytes, e);
//  2. hashes that (i, slot bytes) sequence into a row signature and orders the
//     rows by (window of consecutive Morton ranks of the DOF points,
//     signature), so that warps of 32
//     rows step in lock-step through identical incidence sequences (on a
//     structured mesh the 32 lanes then read the same slot pattern and their
//     shared-memory row accumulators never collide on a bank);
//  3. per warp item and local index i, the lock-step count = max over lanes;
//  4. the records [step][32]: element id + the k slot bytes of (e, i).

__global__ void inc_count(const int32_t* __restrict__ dconn, int64_t nk, int64_t rb, int64_t n_rows,
                          int32_t* __restrict__ cnt) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nk;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = static_cast<int64_t>(dconn[t]) - rb;
    if (r >= 0 && r < n_rows) atomicAdd(cnt + r, 1);
  }
}

__global__ void inc_fill(const int32_t* __restrict__ dconn, int64_t nk, int64_t rb, int64_t n_rows,
                         int64_t* __restrict__ cursor, int32_t* __restrict__ inc) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nk;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = static_cast<int64_t>(dconn[t]) - rb;
    if (r >= 0 && r < n_rows) inc[atomicAdd(reinterpret_cast<unsigned long long*>(cursor + r), 1ull)] =
        static_cast<int32_t>(t);
  }
}

// (i, slot bytes, e) order of two incidences t = e*k + i
__device__ __forceinline__ bool inc_less(int32_t a, int32_t b, int k, const uint8_t* __restrict__ slots) {
  const int ia = a % k, ib = b % k;
  if (ia != ib) return ia < ib;
  const uint8_t* sa = slots + static_cast<int64_t>(a) * k;
  const uint8_t* sb = slots + static_cast<int64_t>(b) * k;
  for (int j = 0; j < k; ++j)
    if (sa[j] != sb[j]) return sa[j] < sb[j];
  return a < b;
}

__global__ void inc_sort_sign(const int64_t* __restrict__ inc_ptr, int64_t n_rows, int k,
                              const uint8_t* __restrict__ slots, int32_t* __restrict__ inc, uint64_t* __restrict__ sig) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = inc_ptr[r], e = inc_ptr[r + 1];
    for (int64_t p = b + 1; p < e; ++p) {  // insertion sort (rows hold a few dozen incidences)
      const int32_t x = inc[p];
      int64_t q = p - 1;
      while (q >= b && inc_less(x, inc[q], k, slots)) {
        inc[q + 1] = inc[q];
        --q;
      }
      inc[q + 1] = x;
    }
    uint64_t h = 1469598103934665603ull;  // FNV-1a over (i, slot bytes) of the sorted list
    for (int64_t p = b; p < e; ++p) {
      const int32_t t = inc[p];
      h = (h ^ static_cast<uint64_t>(t % k + 1)) * 1099511628211ull;
      const uint8_t* sl = slots + static_cast<int64_t>(t) * k;
      for (int j = 0; j < k; ++j) h = (h ^ sl[j]) * 1099511628211ull;
    }
    sig[r] = h;
  }
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {  // 21 bits -> every third bit
  x &= 0x1fffffull;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}
__device__ __forceinline__ uint64_t spread2(uint64_t x) {  // 31 bits -> every other bit
  x &= 0x7fffffffull;
  x = (x | x << 16) & 0x0000ffff0000ffffull;
  x = (x | x << 8) & 0x00ff00ff00ff00ffull;
  x = (x | x << 4) & 0x0f0f0f0f0f0f0f0full;
  x = (x | x << 2) & 0x3333333333333333ull;
  x = (x | x << 1) & 0x5555555555555555ull;
  return x;
}

// Morton code of every owned DOF's point (vertex, or edge midpoint for the
// P2 local DOFs dim+1.. in fem.cpp's edge order), quantised over the mesh
// bounding box. Several elements write the same row with the same value.
__global__ void dof_morton(const double* __restrict__ coords, const int32_t* __restrict__ vconn,
                           const int32_t* __restrict__ dconn, int64_t ne, int k, int dim, int64_t rb, int64_t n_rows,
                           double lx, double ly, double lz, double sx, double sy, double sz,
                           uint64_t* __restrict__ code) {
  const int e3[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  const int e2[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  const int nv = dim + 1;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < ne * k;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = static_cast<int64_t>(dconn[t]) - rb;
    if (r < 0 || r >= n_rows) continue;
    const int64_t e = t / k;
    const int a = static_cast<int>(t - e * k);
    double p[3] = {0.0, 0.0, 0.0};
    if (a < nv) {
      const int64_t v = vconn[e * nv + a];
      for (int c = 0; c < dim; ++c) p[c] = coords[v * dim + c];
    } else {
      const int q = a - nv;
      const int64_t v0 = vconn[e * nv + (dim == 3 ? e3[q][0] : e2[q][0])];
      const int64_t v1 = vconn[e * nv + (dim == 3 ? e3[q][1] : e2[q][1])];
      for (int c = 0; c < dim; ++c) p[c] = 0.5 * (coords[v0 * dim + c] + coords[v1 * dim + c]);
    }
    const double lo[3] = {lx, ly, lz}, sc[3] = {sx, sy, sz};
    uint64_t qv[3] = {0, 0, 0};
    const double qmax = dim == 3 ? 2097151.0 : 2147483647.0;
    for (int c = 0; c < dim; ++c) qv[c] = static_cast<uint64_t>(fmin(fmax((p[c] - lo[c]) * sc[c], 0.0), qmax));
    code[r] = dim == 3 ? (spread3(qv[0]) | spread3(qv[1]) << 1 | spread3(qv[2]) << 2)
                       : (spread2(qv[0]) | spread2(qv[1]) << 1);
  }
}

// Morton code of every element's vertex centroid (element data order of the
// gather: elements used by the same rows are neighbours in memory)
__global__ void elem_morton(const double* __restrict__ coords, const int32_t* __restrict__ vconn, int64_t ne, int dim,
                            double lx, double ly, double lz, double sx, double sy, double sz,
                            uint64_t* __restrict__ code, int32_t* __restrict__ ids) {
  const int nv = dim + 1;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double p[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < nv; ++a) {
      const int64_t v = vconn[e * nv + a];
      for (int c = 0; c < dim; ++c) p[c] += coords[v * dim + c];
    }
    const double lo[3] = {lx, ly, lz}, sc[3] = {sx, sy, sz};
    uint64_t qv[3] = {0, 0, 0};
    const double qmax = dim == 3 ? 2097151.0 : 2147483647.0;
    for (int c = 0; c < dim; ++c) qv[c] = static_cast<uint64_t>(fmin(fmax((p[c] / nv - lo[c]) * sc[c], 0.0), qmax));
    code[e] = dim == 3 ? (spread3(qv[0]) | spread3(qv[1]) << 1 | spread3(qv[2]) << 2)
                       : (spread2(qv[0]) | spread2(qv[1]) << 1);
    ids[e] = static_cast<int32_t>(e);
  }
}

__global__ void invert_perm(const int32_t* __restrict__ order, int64_t n, int32_t* __restrict__ rank) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    rank[order[t]] = static_cast<int32_t>(t);
}

__global__ void iota_rows(int64_t n_rows, int32_t* __restrict__ rows) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    rows[r] = static_cast<int32_t>(r);
}

// rows in Morton order -> key (window of `window` consecutive Morton ranks, signature)
__global__ void row_order_keys(const uint64_t* __restrict__ sig, const int32_t* __restrict__ morton_order, int64_t n_rows,
                               int window, uint64_t* __restrict__ keys, int32_t* __restrict__ rows) {
  for (int64_t pos = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; pos < n_rows;
       pos += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t r = morton_order[pos];
    keys[pos] = (static_cast<uint64_t>(pos / window) << 40) | (sig[r] >> 24);
    rows[pos] = r;
  }
}

__global__ void item_steps(const int32_t* __restrict__ order, int64_t n_rows, int64_t n_items, int k,
                           const int64_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc,
                           const int64_t* __restrict__ row_ptr, int32_t* __restrict__ warp_rows,
                           int32_t* __restrict__ warp_steps, int64_t* __restrict__ item_total,
                           int32_t* __restrict__ item_len) {
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < n_items;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int mx[32];
    int ml = 0;
    for (int i = 0; i < k; ++i) mx[i] = 0;
    for (int l = 0; l < 32; ++l) {
      const int64_t pos = w * 32 + l;
      const int32_t row = pos < n_rows ? order[pos] : -1;
      warp_rows[pos] = row;
      if (row < 0) continue;
      ml = max(ml, static_cast<int>(row_ptr[row + 1] - row_ptr[row]));
      int64_t p = inc_ptr[row];
      const int64_t e = inc_ptr[row + 1];
      for (int i = 0; i < k; ++i) {
        int c = 0;
        while (p < e && inc[p] % k == i) {
          ++c;
          ++p;
        }
        mx[i] = max(mx[i], c);
      }
    }
    int64_t tot = 0;
    for (int i = 0; i < k; ++i) {
      warp_steps[w * k + i] = mx[i];
      tot += mx[i];
    }
    item_total[w] = tot;
    item_len[w] = ml;
  }
}

// class id of every row: binary search of its signature among the class
// signatures (sorted); representative row = the lowest row of the class
__global__ void row_class(const uint64_t* __restrict__ sig, int64_t n_rows, const uint64_t* __restrict__ csig,
                          const int32_t* __restrict__ cid, int n_cls, int32_t* __restrict__ cls,
                          int32_t* __restrict__ reps) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t h = sig[r];
    int lo = 0, hi = n_cls;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (csig[mid] < h)
        lo = mid + 1;
      else
        hi = mid;
    }
    const int c = lo < n_cls && csig[lo] == h ? cid[lo] : -1;
    cls[r] = c;
    if (c >= 0) atomicMin(reps + c, static_cast<int32_t>(r));
  }
}

// class templates of the representative rows: [c][2 + kMaxSteps*(1+k)] ints:
// len, steps, then per step the local index and the k slot bytes
constexpr int kMaxClassSteps = 64;
__global__ void class_templates(const int32_t* __restrict__ reps, int n_cls, const int64_t* __restrict__ inc_ptr,
                                const int32_t* __restrict__ inc, const uint8_t* __restrict__ slots, int k,
                                const int64_t* __restrict__ row_ptr, int32_t* __restrict__ out) {
  const int stride = 2 + kMaxClassSteps * (1 + k);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cls; c += gridDim.x * blockDim.x) {
    const int32_t r = reps[c];
    int32_t* o = out + static_cast<int64_t>(c) * stride;
    const int64_t b = inc_ptr[r];
    const int n = static_cast<int>(inc_ptr[r + 1] - b);
    o[0] = static_cast<int32_t>(row_ptr[r + 1] - row_ptr[r]);
    o[1] = n;
    for (int q = 0; q < n && q < kMaxClassSteps; ++q) {
      const int32_t t = inc[b + q];
      o[2 + q * (1 + k)] = t % k;
      for (int j = 0; j < k; ++j) o[3 + q * (1 + k) + j] = slots[static_cast<int64_t>(t) * k + j];
    }
  }
}

// demotes rows whose incidences differ from their class template (hash collisions)
__global__ void class_verify(int32_t* __restrict__ cls, int64_t n_rows, const int32_t* __restrict__ tmpl, int k,
                             const int64_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc,
                             const uint8_t* __restrict__ slots, const int64_t* __restrict__ row_ptr) {
  const int stride = 2 + kMaxClassSteps * (1 + k);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = cls[r];
    if (c < 0) continue;
    const int32_t* o = tmpl + static_cast<int64_t>(c) * stride;
    const int64_t b = inc_ptr[r];
    const int n = static_cast<int>(inc_ptr[r + 1] - b);
    bool ok = o[0] == static_cast<int32_t>(row_ptr[r + 1] - row_ptr[r]) && o[1] == n && n <= kMaxClassSteps;
    for (int q = 0; ok && q < n; ++q) {
      const int32_t t = inc[b + q];
      ok = o[2 + q * (1 + k)] == t % k;
      for (int j = 0; ok && j < k; ++j) ok = o[3 + q * (1 + k) + j] == slots[static_cast<int64_t>(t) * k + j];
    }
    if (!ok) cls[r] = -1;
  }
}

// class item records: [steps][32] element ids of each item (incidence order)
// out[t][c] = in[order[t]][c] for c < cols (row stride in_stride)
__global__ void gather_rows_i32(const int32_t* __restrict__ in, int in_stride, int cols,
                                const int32_t* __restrict__ order, int64_t n, int32_t* __restrict__ out) {
  for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; f < n * cols;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = f / cols;
    out[f] = in[static_cast<int64_t>(order[t]) * in_stride + f % cols];
  }
}

// records of the class items in the class's processing order: step t of
// item w holds the element of incidence perm[class][t] of the lane's row
__global__ void fill_class_records(const int32_t* __restrict__ erank, const int32_t* __restrict__ citem_class,
                                   const int32_t* __restrict__ citem_rows,
                                   const int64_t* __restrict__ citem_rec, int64_t n_citems,
                                   const int32_t* __restrict__ cls_steps, const int32_t* __restrict__ perm,
                                   const int64_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc, int k,
                                   int32_t* __restrict__ crec) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n_citems * 32;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = t / 32;
    const int lane = static_cast<int>(t % 32);
    const int32_t row = citem_rows[t];
    const int c = citem_class[w];
    const int n = cls_steps[c];
    const int64_t base = citem_rec[w] * 32 + lane;
    const int64_t p = row >= 0 ? inc_ptr[row] : 0;
    for (int q = 0; q < n; ++q)
      crec[base + q * 32] = row >= 0 ? erank[inc[p + perm[c * kMaxClassSteps + q]] / k] : -1;
  }
}

// [steps][32] records per item (prefix irec) -> the first `pre` steps of item
// w at the computable position (w * pre + t) * 32, the rest after all of them
// at (n_items * pre + irec2[w] + t - pre) * 32
__global__ void relayout_records(const int32_t* __restrict__ src, const int64_t* __restrict__ irec,
                                 const int64_t* __restrict__ irec2, int64_t n_items, int pre,
                                 int32_t* __restrict__ dst) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n_items * 32;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = t / 32;
    const int lane = static_cast<int>(t % 32);
    const int64_t n = irec[w + 1] - irec[w];
    for (int64_t q = 0; q < n; ++q) {
      const int32_t v = src[(irec[w] + q) * 32 + lane];
      if (q < pre)
        dst[(w * pre + q) * 32 + lane] = v;
      else
        dst[(n_items * pre + irec2[w] + q - pre) * 32 + lane] = v;
    }
  }
}


// First touch of every element by the class records (crec position p, in
// item, step, lane order): records ordered by first touch put the elements of
// the 32 lanes of one step side by side, so a warp's record load touches a few
// consecutive lines instead of 32 scattered ones.
__global__ void first_touch(const int32_t* __restrict__ crec, int64_t n, const int32_t* __restrict__ eorder,
                            unsigned long long* __restrict__ first) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t r = crec[p];
    if (r >= 0) atomicMin(first + eorder[r], static_cast<unsigned long long>(p));
  }
}

// sort key of every element: first touch, else (rows of generic items only)
// after every touched element in the previous (Morton) record order
__global__ void touch_keys(const unsigned long long* __restrict__ first, const int32_t* __restrict__ erank, int64_t ne,
                           int64_t n_crec, uint64_t* __restrict__ keys, int32_t* __restrict__ ids) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    keys[e] = first[e] != ~0ull ? first[e] : static_cast<uint64_t>(n_crec) + static_cast<uint64_t>(erank[e]);
    ids[e] = static_cast<int32_t>(e);
  }
}

// record ranks of the old order -> ranks of the new one
__global__ void remap_ranks(int32_t* __restrict__ crec, int64_t n, const int32_t* __restrict__ eorder_old,
                            const int32_t* __restrict__ erank_new) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t r = crec[p];
    if (r >= 0) crec[p] = erank_new[eorder_old[r]];
  }
}

template <int K>
__global__ void fill_records(const int32_t* __restrict__ erank, const int32_t* __restrict__ warp_rows,
                             const int32_t* __restrict__ warp_steps,
                             const int64_t* __restrict__ warp_rec, int64_t n_items, const int64_t* __restrict__ inc_ptr,
                             const int32_t* __restrict__ inc, const uint8_t* __restrict__ slots, void* __restrict__ rec) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n_items * 32;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = t / 32;
    const int lane = static_cast<int>(t % 32);
    const int32_t row = warp_rows[t];
    int64_t p = row >= 0 ? inc_ptr[row] : 0;
    const int64_t pe = row >= 0 ? inc_ptr[row + 1] : 0;
    int64_t step = warp_rec[w];
    for (int i = 0; i < K; ++i) {
      const int n = warp_steps[w * K + i];
      for (int s = 0; s < n; ++s, ++step) {
        uint32_t word[4] = {0xffffffffu, 0u, 0u, 0u};
        if (p < pe && inc[p] % K == i) {
          const int32_t x = inc[p++];
          word[0] = static_cast<uint32_t>(erank[x / K]);
          const uint8_t* sl = slots + static_cast<int64_t>(x) * K;
          for (int j = 0; j < K; ++j) word[1 + j / 4] |= static_cast<uint32_t>(sl[j]) << (8 * (j & 3));
        }
        if (K <= 4)
          reinterpret_cast<uint2*>(rec)[step * 32 + lane] = make_uint2(word[0], word[1]);
        else
          reinterpret_cast<uint4*>(rec)[step * 32 + lane] = make_uint4(word[0], word[1], word[2], word[3]);
      }
    }
  }
}

int grid_for(int64_t n, int sm_blocks) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return static_cast<int>(g < sm_blocks ? (g < 1 ? 1 : g) : sm_blocks);
}

}  // namespace

cudaError_t build_pattern(const int32_t* d_dconn, int64_t ne, int k, int64_t rb, int64_t re, int sm_count,
                          cudaStream_t s, int64_t** row_ptr, int32_t** col_idx, int64_t* nnz, int* max_row_len) {
  const int64_t n_rows = re - rb;
  const int64_t n_pair = ne * k * (k - 1);
  const int64_t n_keys = n_pair + n_rows;
  const int cap = sm_count * 16;
  uint64_t *keys = nullptr, *sorted = nullptr;
  int64_t* d_count = nullptr;
  void* temp = nullptr;
  int* d_max = nullptr;
  cudaError_t err = cudaSuccess;
  auto fail = [&](cudaError_t e) {
    cudaFree(keys);
    cudaFree(sorted);
    cudaFree(temp);
    cudaFree(d_count);
    cudaFree(d_max);
    return e;
  };
  if ((err = cudaMalloc(&keys, n_keys * sizeof(uint64_t))) != cudaSuccess) return fail(err);
  if ((err = cudaMalloc(&sorted, n_keys * sizeof(uint64_t))) != cudaSuccess) return fail(err);
  if ((err = cudaMalloc(&d_count, sizeof(int64_t))) != cudaSuccess) return fail(err);
  if ((err = cudaMalloc(&d_max, sizeof(int))) != cudaSuccess) return fail(err);
  if (n_pair > 0) pair_keys<<<grid_for(n_pair, cap), kThreads, 0, s>>>(d_dconn, ne, k, rb, re, keys);
  diagonal_keys<<<grid_for(n_rows, cap), kThreads, 0, s>>>(rb, n_rows, keys + n_pair);
  int end_bit = 32;
  while ((static_cast<int64_t>(1) << (end_bit - 32)) <= n_rows) ++end_bit;  // row field incl. the invalid row
  size_t t_sort = 0, t_uniq = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, t_sort, keys, sorted, n_keys, 0, end_bit, s);
  cub::DeviceSelect::Unique(nullptr, t_uniq, sorted, keys, d_count, n_keys, s);
  if ((err = cudaMalloc(&temp, t_sort > t_uniq ? t_sort : t_uniq)) != cudaSuccess) return fail(err);
  if ((err = cub::DeviceRadixSort::SortKeys(temp, t_sort, keys, sorted, n_keys, 0, end_bit, s)) != cudaSuccess)
    return fail(err);
  if ((err = cub::DeviceSelect::Unique(temp, t_uniq, sorted, keys, d_count, n_keys, s)) != cudaSuccess) return fail(err);
  int64_t n_unique = 0;
  if ((err = cudaMemcpyAsync(&n_unique, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return fail(err);
  if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return fail(err);
  // the trailing invalid key (if any pair was not owned) is not a column
  int64_t last = 0;
  if ((err = cudaMemcpy(&last, keys + (n_unique - 1), sizeof(int64_t), cudaMemcpyDeviceToHost)) != cudaSuccess)
    return fail(err);
  const int64_t n_cols = (static_cast<uint64_t>(last) >> 32) >= static_cast<uint64_t>(n_rows) ? n_unique - 1 : n_unique;
  if ((err = cudaMalloc(row_ptr, (n_rows + 1) * sizeof(int64_t))) != cudaSuccess) return fail(err);
  if ((err = cudaMalloc(col_idx, (n_cols > 0 ? n_cols : 1) * sizeof(int32_t))) != cudaSuccess) {
    cudaFree(*row_ptr);
    return fail(err);
  }
  split_keys<<<grid_for(n_unique, cap), kThreads, 0, s>>>(keys, d_count, n_rows, *row_ptr, *col_idx);
  cudaMemsetAsync(d_max, 0, sizeof(int), s);
  row_max<<<grid_for(n_rows, cap), kThreads, 0, s>>>(*row_ptr, n_rows, d_max);
  int mx = 0;
  cudaMemcpyAsync(&mx, d_max, sizeof(int), cudaMemcpyDeviceToHost, s);
  if ((err = cudaStreamSynchronize(s)) != cudaSuccess) {
    cudaFree(*row_ptr);
    cudaFree(*col_idx);
    return fail(err);
  }
  *nnz = n_cols;
  *max_row_len = mx;
  return fail(cudaGetLastError());
}


cudaError_t build_gather_plan(const double* d_coords, const int32_t* d_vconn, int dim, const double* bbox,
                              const int32_t* d_dconn, int64_t ne, int k, int64_t rb, int64_t n_rows,
                              const int64_t* d_row_ptr, const uint8_t* d_slots, int window, int sm_count,
                              cudaStream_t s, GatherPlan* out, int min_class_rows, int max_classes,
                              bool use_eorder, bool split_long, const ClassOrderFn* step_order,
                              double class_frac, int row_lanes) {
  if (k > 12) return cudaErrorInvalidValue;
  if (ne * k >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  // FF_PLAN_TIMING=1: phase times of the plan build on stderr
  const bool timing = std::getenv("FF_PLAN_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* name) {
    if (!timing) return;
    cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[plan] %-24s %8.1f ms\n", name, std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  const int cap = sm_count * 16;
  const int64_t nk = ne * k;
  int32_t* cnt = nullptr;
  int64_t *inc_ptr = nullptr, *cursor = nullptr, *item_total = nullptr;
  int32_t *inc = nullptr, *rows = nullptr, *order = nullptr;
  uint64_t *sig = nullptr, *keys = nullptr, *keys2 = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  cudaError_t err = cudaSuccess;
  auto done = [&](cudaError_t e) {
    cudaFree(cnt);
    cudaFree(inc_ptr);
    cudaFree(cursor);
    cudaFree(item_total);
    cudaFree(inc);
    cudaFree(rows);
    cudaFree(order);
    cudaFree(sig);
    cudaFree(keys);
    cudaFree(keys2);
    cudaFree(temp);
    return e;
  };
  auto need_temp = [&](size_t b) -> cudaError_t {
    if (b <= temp_bytes) return cudaSuccess;
    cudaFree(temp);
    temp = nullptr;
    temp_bytes = b;
    return cudaMalloc(&temp, b);
  };
  const int64_t nr1 = n_rows + 1;
  if ((err = cudaMalloc(&cnt, nr1 * sizeof(int32_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&inc_ptr, nr1 * sizeof(int64_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&cursor, nr1 * sizeof(int64_t))) != cudaSuccess) return done(err);
  cudaMemsetAsync(cnt, 0, nr1 * sizeof(int32_t), s);
  if (nk > 0) inc_count<<<grid_for(nk, cap), kThreads, 0, s>>>(d_dconn, nk, rb, n_rows, cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, inc_ptr, nr1, s);
  if ((err = need_temp(tb)) != cudaSuccess) return done(err);
  if ((err = cub::DeviceScan::ExclusiveSum(temp, tb, cnt, inc_ptr, nr1, s)) != cudaSuccess) return done(err);
  int64_t n_inc = 0;
  cudaMemcpyAsync(&n_inc, inc_ptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&inc, (n_inc > 0 ? n_inc : 1) * sizeof(int32_t))) != cudaSuccess) return done(err);
  cudaMemcpyAsync(cursor, inc_ptr, nr1 * sizeof(int64_t), cudaMemcpyDeviceToDevice, s);
  if (nk > 0) inc_fill<<<grid_for(nk, cap), kThreads, 0, s>>>(d_dconn, nk, rb, n_rows, cursor, inc);
  if ((err = cudaMalloc(&sig, nr1 * sizeof(uint64_t))) != cudaSuccess) return done(err);
  if (n_rows > 0) inc_sort_sign<<<grid_for(n_rows, cap), kThreads, 0, s>>>(inc_ptr, n_rows, k, d_slots, inc, sig);
  // rows in Morton order of their DOF points (3D-compact windows keep the
  // element data of a window hot in L2), then by (window, signature);
  // radix sorts are stable, so ties keep the previous order
  if ((err = cudaMalloc(&keys, nr1 * sizeof(uint64_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&keys2, nr1 * sizeof(uint64_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&rows, nr1 * sizeof(int32_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&order, nr1 * sizeof(int32_t))) != cudaSuccess) return done(err);
  if (n_rows > 0) {
    double sc[3] = {0.0, 0.0, 0.0};
    const double qmax = dim == 3 ? 2097151.0 : 2147483647.0;
    for (int c = 0; c < dim; ++c) {
      const double ext = bbox[3 + c] - bbox[c];
      sc[c] = ext > 0 ? qmax / ext : 0.0;
    }
    cudaMemsetAsync(keys, 0, nr1 * sizeof(uint64_t), s);
    dof_morton<<<grid_for(nk, cap), kThreads, 0, s>>>(d_coords, d_vconn, d_dconn, ne, k, dim, rb, n_rows, bbox[0],
                                                     bbox[1], bbox[2], sc[0], sc[1], sc[2], keys);
    iota_rows<<<grid_for(n_rows, cap), kThreads, 0, s>>>(n_rows, rows);
  }
  // element order of the gather's per-element records (K2a writes record t
  // for element eorder[t]): Morton order of the element centroids, or the
  // identity when use_eorder is false
  if ((err = cudaMalloc(&out->eorder, std::max<int64_t>(ne, 1) * sizeof(int32_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&out->erank, std::max<int64_t>(ne, 1) * sizeof(int32_t))) != cudaSuccess) return done(err);
  if (ne > 0) {
    uint64_t *ek = nullptr, *ek2 = nullptr;
    int32_t* eid = nullptr;
    if ((err = cudaMalloc(&ek, ne * sizeof(uint64_t))) != cudaSuccess) return done(err);
    if ((err = cudaMalloc(&ek2, ne * sizeof(uint64_t))) != cudaSuccess) return cudaFree(ek), done(err);
    if ((err = cudaMalloc(&eid, ne * sizeof(int32_t))) != cudaSuccess) return cudaFree(ek), cudaFree(ek2), done(err);
    double sc[3] = {0.0, 0.0, 0.0};
    const double qmax = dim == 3 ? 2097151.0 : 2147483647.0;
    for (int c = 0; c < dim; ++c) {
      const double ext = bbox[3 + c] - bbox[c];
      sc[c] = ext > 0 ? qmax / ext : 0.0;
    }
    elem_morton<<<grid_for(ne, cap), kThreads, 0, s>>>(d_coords, d_vconn, ne, dim, bbox[0], bbox[1], bbox[2], sc[0],
                                                      sc[1], sc[2], ek, eid);
    if (!use_eorder) cudaMemsetAsync(ek, 0, ne * sizeof(uint64_t), s);  // stable sort of equal keys: identity
    size_t te = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, te, ek, ek2, eid, out->eorder, ne, 0, 64, s);
    if ((err = need_temp(te)) != cudaSuccess) return cudaFree(ek), cudaFree(ek2), cudaFree(eid), done(err);
    err = cub::DeviceRadixSort::SortPairs(temp, te, ek, ek2, eid, out->eorder, ne, 0, 64, s);
    if (err == cudaSuccess) invert_perm<<<grid_for(ne, cap), kThreads, 0, s>>>(out->eorder, ne, out->erank);
    // vertex ids in record order for K2a (P1: the DOF ids are the vertices)
    if (err == cudaSuccess) err = cudaMalloc(&out->vconn_m, ne * (dim + 1) * sizeof(int32_t));
    if (err == cudaSuccess)
      gather_rows_i32<<<grid_for(ne * (dim + 1), cap), kThreads, 0, s>>>(k == dim + 1 ? d_dconn : d_vconn,
                                                                        k == dim + 1 ? k : dim + 1, dim + 1,
                                                                        out->eorder, ne, out->vconn_m);
    if (err == cudaSuccess) err = cudaStreamSynchronize(s);
    cudaFree(ek);
    cudaFree(ek2);
    cudaFree(eid);
    if (err != cudaSuccess) return done(err);
  }
  phase("incidences+morton");
  tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, rows, order, n_rows, 0, 64, s);
  if ((err = need_temp(tb)) != cudaSuccess) return done(err);
  if ((err = cub::DeviceRadixSort::SortPairs(temp, tb, keys, keys2, rows, order, n_rows, 0, 64, s)) != cudaSuccess)
    return done(err);
  phase("row sort");
  // ---- row classes (signature counts on the host, verified on the device)
  std::vector<int32_t> cls_h(n_rows, -1);
  {
    // signature counts on the device: sort + run-length encode; the host sees
    // only the distinct signatures
    std::vector<uint64_t> usig;
    std::vector<int32_t> ucnt;
    if (n_rows > 0) {
      uint64_t *ssorted = nullptr, *uniq = nullptr;
      int32_t *counts = nullptr, *nruns = nullptr;
      auto sfree = [&]() {
        cudaFree(ssorted);
        cudaFree(uniq);
        cudaFree(counts);
        cudaFree(nruns);
      };
      if ((err = cudaMalloc(&ssorted, n_rows * sizeof(uint64_t))) != cudaSuccess) return sfree(), done(err);
      if ((err = cudaMalloc(&uniq, n_rows * sizeof(uint64_t))) != cudaSuccess) return sfree(), done(err);
      if ((err = cudaMalloc(&counts, n_rows * sizeof(int32_t))) != cudaSuccess) return sfree(), done(err);
      if ((err = cudaMalloc(&nruns, sizeof(int32_t))) != cudaSuccess) return sfree(), done(err);
      size_t t1 = 0, t2 = 0;
      cub::DeviceRadixSort::SortKeys(nullptr, t1, sig, ssorted, static_cast<int>(n_rows), 0, 64, s);
      cub::DeviceRunLengthEncode::Encode(nullptr, t2, ssorted, uniq, counts, nruns, static_cast<int>(n_rows), s);
      if ((err = need_temp(std::max(t1, t2))) != cudaSuccess) return sfree(), done(err);
      err = cub::DeviceRadixSort::SortKeys(temp, t1, sig, ssorted, static_cast<int>(n_rows), 0, 64, s);
      if (err == cudaSuccess)
        err = cub::DeviceRunLengthEncode::Encode(temp, t2, ssorted, uniq, counts, nruns, static_cast<int>(n_rows), s);
      int32_t nr = 0;
      if (err == cudaSuccess) err = cudaMemcpyAsync(&nr, nruns, sizeof nr, cudaMemcpyDeviceToHost, s);
      if (err == cudaSuccess) err = cudaStreamSynchronize(s);
      if (err == cudaSuccess) {
        usig.resize(nr);
        ucnt.resize(nr);
        cudaMemcpyAsync(usig.data(), uniq, nr * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(ucnt.data(), counts, nr * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        err = cudaStreamSynchronize(s);
      }
      sfree();
      if (err != cudaSuccess) return done(err);
    }
    if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);
    // classes worth a specialised kernel: >= min_class_rows rows and >= 0.05 %
    // of the block (the mesh boundary's classes included: with one item per
    // warp they are as cheap as interior rows, while the generic gather costs
    // ~3x per row -- NS 2.00 -> 1.89 ms, C3 0.88 -> 0.82 against 0.5 %);
    // ordered by row count, then signature
    // (vector forms too since their per-block record quantities: config 5
    // 49.6 ms with 32 classes vs 51.0 with 8 at 0.5 %)
    const char* frac_env = std::getenv("FF_CLASS_FRAC");  // tuning knob
    const double frac = frac_env ? std::atof(frac_env) : class_frac;
    const int64_t min_rows = std::max<int64_t>(min_class_rows, static_cast<int64_t>(frac * n_rows));
    std::vector<std::pair<int64_t, uint64_t>> big;
    for (size_t u = 0; u < usig.size(); ++u)
      if (ucnt[u] >= min_rows) big.push_back({ucnt[u], usig[u]});
    std::sort(big.begin(), big.end(), [](const auto& a, const auto& b) {
      return a.first != b.first ? a.first > b.first : a.second < b.second;
    });
    if (static_cast<int>(big.size()) > max_classes) big.resize(max_classes);
    const int n_cls = static_cast<int>(big.size());
    out->classes.clear();
    if (n_cls > 0) {
      const int stride = 2 + kMaxClassSteps * (1 + k);
      int32_t *d_reps = nullptr, *d_tmpl = nullptr, *d_cls = nullptr;
      auto cleanup = [&]() {
        cudaFree(d_reps);
        cudaFree(d_tmpl);
        cudaFree(d_cls);
      };
      if ((err = cudaMalloc(&d_reps, n_cls * sizeof(int32_t))) != cudaSuccess) return cleanup(), done(err);
      if ((err = cudaMalloc(&d_tmpl, static_cast<size_t>(n_cls) * stride * sizeof(int32_t))) != cudaSuccess)
        return cleanup(), done(err);
      if ((err = cudaMalloc(&d_cls, n_rows * sizeof(int32_t))) != cudaSuccess) return cleanup(), done(err);
      {
        // class signatures sorted (for the per-row binary search) with their ids
        std::vector<std::pair<uint64_t, int32_t>> by_sig;
        for (int c = 0; c < n_cls; ++c) by_sig.push_back({big[c].second, c});
        std::sort(by_sig.begin(), by_sig.end());
        std::vector<uint64_t> csig(n_cls);
        std::vector<int32_t> cidv(n_cls);
        for (int c = 0; c < n_cls; ++c) csig[c] = by_sig[c].first, cidv[c] = by_sig[c].second;
        uint64_t* d_csig = nullptr;
        int32_t* d_cid = nullptr;
        if ((err = cudaMalloc(&d_csig, n_cls * sizeof(uint64_t))) != cudaSuccess) return cleanup(), done(err);
        if ((err = cudaMalloc(&d_cid, n_cls * sizeof(int32_t))) != cudaSuccess)
          return cudaFree(d_csig), cleanup(), done(err);
        cudaMemcpyAsync(d_csig, csig.data(), n_cls * sizeof(uint64_t), cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(d_cid, cidv.data(), n_cls * sizeof(int32_t), cudaMemcpyHostToDevice, s);
        cudaMemsetAsync(d_reps, 0x7f, n_cls * sizeof(int32_t), s);
        row_class<<<grid_for(n_rows, cap), kThreads, 0, s>>>(sig, n_rows, d_csig, d_cid, n_cls, d_cls, d_reps);
        err = cudaStreamSynchronize(s);
        cudaFree(d_csig);
        cudaFree(d_cid);
        if (err != cudaSuccess) return cleanup(), done(err);
      }
      cudaMemsetAsync(d_tmpl, 0, static_cast<size_t>(n_cls) * stride * sizeof(int32_t), s);
      class_templates<<<1, 64, 0, s>>>(d_reps, n_cls, inc_ptr, inc, d_slots, k, d_row_ptr, d_tmpl);
      class_verify<<<grid_for(n_rows, cap), kThreads, 0, s>>>(d_cls, n_rows, d_tmpl, k, inc_ptr, inc, d_slots,
                                                             d_row_ptr);
      std::vector<int32_t> tmpl(static_cast<size_t>(n_cls) * stride);
      cudaMemcpyAsync(tmpl.data(), d_tmpl, tmpl.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(cls_h.data(), d_cls, n_rows * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return cleanup(), done(err);
      cleanup();
      for (int c = 0; c < n_cls; ++c) {
        const int32_t* o = tmpl.data() + static_cast<size_t>(c) * stride;
        GatherPlan::Class cl;
        cl.len = o[0];
        cl.steps = o[1];
        if (cl.steps > kMaxClassSteps) cl.steps = -1;  // never matches: rows stay generic
        for (int q = 0; q < std::max(cl.steps, 0); ++q) {
          cl.local.push_back(o[2 + q * (1 + k)]);
          for (int j = 0; j < k; ++j) cl.slots.push_back(static_cast<uint8_t>(o[3 + q * (1 + k) + j]));
        }
        // processing order of the class kernel (code generator's choice):
        // records are laid out in it
        if (step_order && cl.steps > 0) cl.order = (*step_order)(cl);
        if (static_cast<int>(cl.order.size()) != std::max(cl.steps, 0)) {
          cl.order.resize(std::max(cl.steps, 0));
          for (int q = 0; q < std::max(cl.steps, 0); ++q) cl.order[q] = q;
        }
        out->classes.push_back(std::move(cl));
      }
    }
    phase("class detection");
    // class items: each class's rows in Morton order, 32 per item; items
    // interleaved by the Morton position of their first row
    // class rows in row (DOF) order: on a lattice numbering the 32 rows of an
    // item are a line of same-class DOFs, so at every step the lanes' elements
    // are neighbours along that line (measured against the Morton order of the DOF
    // points; NS 2.49 -> 2.09 ms together with the first-touch records below)
    // rows per class item: 32, or 32 / row_lanes rows of row_lanes lanes each
    // (vector forms: the trial components of a row in neighbouring lanes)
    const int rpi = 32 / std::max(1, row_lanes);
    std::vector<std::vector<int32_t>> members(n_cls);
    std::vector<std::vector<int64_t>> first_pos(n_cls);
    for (int64_t pos = 0; pos < n_rows; ++pos) {
      const int32_t r = static_cast<int32_t>(pos);
      const int c = cls_h[r];
      if (c < 0) continue;
      if (members[c].size() % rpi == 0) first_pos[c].push_back(pos);
      members[c].push_back(r);
    }
    struct Item {
      int64_t key;
      int c;
      int64_t idx;
    };
    std::vector<Item> items;
    for (int c = 0; c < n_cls; ++c) {
      out->classes[c].rows = static_cast<int64_t>(members[c].size());
      for (size_t q = 0; q < first_pos[c].size(); ++q) items.push_back({first_pos[c][q], c, static_cast<int64_t>(q)});
    }
    // short-row classes (<= 33 entries) first, then long-row ones: two
    // specialised kernels with their own register budgets
    auto longrows = [&](const Item& it) { return split_long && out->classes[it.c].len > 33 ? 1 : 0; };
    // within each, by (Morton window of 4096 rows, class, position): the 16
    // items a CTA takes are of one class (one instruction footprint per CTA)
    const char* iw_env = std::getenv("FF_ITEM_WINDOW");  // tuning knob: rows per item window
    // 16384 rows: 2.570 ms at NS against 2.582 (4096) and 2.602 (65536), run 85
    const int64_t iwin = iw_env ? std::max(32, std::atoi(iw_env)) : 16384;
    auto win = [&](const Item& it) { return it.key / iwin; };
    std::sort(items.begin(), items.end(), [&](const Item& a, const Item& b) {
      if (longrows(a) != longrows(b)) return longrows(a) < longrows(b);
      if (win(a) != win(b)) return win(a) < win(b);
      return a.c != b.c ? a.c < b.c : a.key < b.key;
    });
    out->n_citems_short = 0;
    for (const Item& it : items) out->n_citems_short += longrows(it) ? 0 : 1;
    const int64_t nci = static_cast<int64_t>(items.size());
    std::vector<int32_t> ic(nci), ir(nci * 32, -1), cls_steps(std::max(n_cls, 1), 0);
    std::vector<int64_t> irec(nci + 1, 0);
    for (int c = 0; c < n_cls; ++c) cls_steps[c] = out->classes[c].steps;
    int64_t nrec = 0, ncr = 0;
    for (int64_t w = 0; w < nci; ++w) {
      const Item& it = items[w];
      ic[w] = it.c;
      const auto& m = members[it.c];
      for (int l = 0; l < rpi * std::max(1, row_lanes); ++l) {
        const size_t q = static_cast<size_t>(it.idx) * rpi + l / std::max(1, row_lanes);
        if (q < m.size()) {
          ir[w * 32 + l] = m[q];
          ncr += l % std::max(1, row_lanes) == 0;
        }
      }
      irec[w] = nrec;
      nrec += cls_steps[it.c];
    }
    irec[nci] = nrec;
    out->n_citems = nci;
    out->n_crec = nrec * 32;
    out->n_class_rows = ncr;
    if (nci > 0) {
      int32_t* d_steps = nullptr;
      if ((err = cudaMalloc(&out->citem_class, nci * sizeof(int32_t))) != cudaSuccess) return done(err);
      if ((err = cudaMalloc(&out->citem_rows, nci * 32 * sizeof(int32_t))) != cudaSuccess) return done(err);
      if ((err = cudaMalloc(&out->citem_rec, (nci + 1) * sizeof(int64_t))) != cudaSuccess) return done(err);
      // padded by 8 steps: the class kernel prefetches 8 records per item without a bound
      if ((err = cudaMalloc(&out->crec, (out->n_crec + 8 * 32) * sizeof(int32_t))) != cudaSuccess) return done(err);
      cudaMemsetAsync(out->crec + out->n_crec, 0xff, 8 * 32 * sizeof(int32_t), s);
      if ((err = cudaMalloc(&d_steps, cls_steps.size() * sizeof(int32_t))) != cudaSuccess) return done(err);
      cudaMemcpyAsync(out->citem_class, ic.data(), nci * sizeof(int32_t), cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(out->citem_rows, ir.data(), nci * 32 * sizeof(int32_t), cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(out->citem_rec, irec.data(), (nci + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(d_steps, cls_steps.data(), cls_steps.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s);
      std::vector<int32_t> perm(static_cast<size_t>(std::max(n_cls, 1)) * kMaxClassSteps, 0);
      for (int c = 0; c < n_cls; ++c)
        for (size_t t = 0; t < out->classes[c].order.size(); ++t) perm[c * kMaxClassSteps + t] = out->classes[c].order[t];
      int32_t* d_perm = nullptr;
      if ((err = cudaMalloc(&d_perm, perm.size() * sizeof(int32_t))) != cudaSuccess) return cudaFree(d_steps), done(err);
      cudaMemcpyAsync(d_perm, perm.data(), perm.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s);
      fill_class_records<<<grid_for(nci * 32, cap), kThreads, 0, s>>>(out->erank, out->citem_class, out->citem_rows,
                                                                      out->citem_rec, nci, d_steps, d_perm, inc_ptr,
                                                                      inc, k, out->crec);
      err = cudaStreamSynchronize(s);
      cudaFree(d_steps);
      cudaFree(d_perm);
      if (err != cudaSuccess) return done(err);
      // element records in first-touch order of the class records (item, step,
      // lane): the elements the 32 lanes of one step read are then stored side
      // by side, and a warp's 32-byte record loads cover 8 consecutive lines
      // instead of 32 scattered ones (the class kernel was bound by L1 tag
      // wavefronts of those scattered loads).
      if (ne > 0) {
        unsigned long long* first = nullptr;
        uint64_t *ek = nullptr, *ek2 = nullptr;
        int32_t *eid = nullptr, *eorder_new = nullptr;
        auto tfree = [&]() {
          cudaFree(first);
          cudaFree(ek);
          cudaFree(ek2);
          cudaFree(eid);
          cudaFree(eorder_new);
        };
        if ((err = cudaMalloc(&first, ne * sizeof(unsigned long long))) != cudaSuccess) return tfree(), done(err);
        if ((err = cudaMalloc(&ek, ne * sizeof(uint64_t))) != cudaSuccess) return tfree(), done(err);
        if ((err = cudaMalloc(&ek2, ne * sizeof(uint64_t))) != cudaSuccess) return tfree(), done(err);
        if ((err = cudaMalloc(&eid, ne * sizeof(int32_t))) != cudaSuccess) return tfree(), done(err);
        if ((err = cudaMalloc(&eorder_new, ne * sizeof(int32_t))) != cudaSuccess) return tfree(), done(err);
        cudaMemsetAsync(first, 0xff, ne * sizeof(unsigned long long), s);
        first_touch<<<grid_for(out->n_crec, cap), kThreads, 0, s>>>(out->crec, out->n_crec, out->eorder, first);
        touch_keys<<<grid_for(ne, cap), kThreads, 0, s>>>(first, out->erank, ne, out->n_crec, ek, eid);
        size_t te = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, te, ek, ek2, eid, eorder_new, ne, 0, 64, s);
        if ((err = need_temp(te)) != cudaSuccess) return tfree(), done(err);
        err = cub::DeviceRadixSort::SortPairs(temp, te, ek, ek2, eid, eorder_new, ne, 0, 64, s);
        if (err == cudaSuccess) {
          invert_perm<<<grid_for(ne, cap), kThreads, 0, s>>>(eorder_new, ne, out->erank);
          remap_ranks<<<grid_for(out->n_crec, cap), kThreads, 0, s>>>(out->crec, out->n_crec, out->eorder,
                                                                       out->erank);
          gather_rows_i32<<<grid_for(ne * (dim + 1), cap), kThreads, 0, s>>>(k == dim + 1 ? d_dconn : d_vconn,
                                                                            k == dim + 1 ? k : dim + 1, dim + 1,
                                                                            eorder_new, ne, out->vconn_m);
          std::swap(out->eorder, eorder_new);
          err = cudaStreamSynchronize(s);
        }
        tfree();
        if (err != cudaSuccess) return done(err);
      }
      // FF_PLAN_DUMP=<path> (analysis only): class items + element records
      if (const char* dump = std::getenv("FF_PLAN_DUMP")) {
        std::vector<int32_t> crec_h(out->n_crec);
        cudaMemcpy(crec_h.data(), out->crec, out->n_crec * sizeof(int32_t), cudaMemcpyDeviceToHost);
        if (FILE* fp = std::fopen(dump, "wb")) {
          const int64_t hdr[3] = {nci, out->n_crec, ne};
          std::fwrite(hdr, sizeof hdr, 1, fp);
          std::fwrite(ic.data(), sizeof(int32_t), nci, fp);
          std::fwrite(ir.data(), sizeof(int32_t), nci * 32, fp);
          std::fwrite(irec.data(), sizeof(int64_t), nci + 1, fp);
          std::fwrite(crec_h.data(), sizeof(int32_t), out->n_crec, fp);
          std::fclose(fp);
        }
      }
      // the first `pre` steps of every item (the class kernel's prefetch) at a
      // position computable from the item index: the warp loads them together
      // with the item header instead of after it
      int pre = kMaxClassSteps;
      for (int c = 0; c < n_cls; ++c)
        if (out->classes[c].steps > 0) pre = std::min(pre, out->classes[c].steps);
      pre = std::min(pre, 8);
      std::vector<int64_t> irec2(nci + 1, 0);
      for (int64_t w = 0; w < nci; ++w) irec2[w + 1] = irec2[w] + (irec[w + 1] - irec[w]) - pre;
      std::vector<int64_t> crec_at(nci + 1);
      for (int64_t w = 0; w <= nci; ++w) crec_at[w] = nci * pre + irec2[w];
      int32_t* crec2 = nullptr;
      int64_t* d_irec2 = nullptr;
      if ((err = cudaMalloc(&crec2, (out->n_crec + 8 * 32) * sizeof(int32_t))) != cudaSuccess) return done(err);
      if ((err = cudaMalloc(&d_irec2, (nci + 1) * sizeof(int64_t))) != cudaSuccess)
        return cudaFree(crec2), done(err);
      cudaMemsetAsync(crec2 + out->n_crec, 0xff, 8 * 32 * sizeof(int32_t), s);
      cudaMemcpyAsync(d_irec2, irec2.data(), (nci + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
      relayout_records<<<grid_for(nci * 32, cap), kThreads, 0, s>>>(out->crec, out->citem_rec, d_irec2, nci, pre,
                                                                    crec2);
      cudaMemcpyAsync(out->citem_rec, crec_at.data(), (nci + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
      err = cudaStreamSynchronize(s);
      cudaFree(d_irec2);
      if (err != cudaSuccess) return cudaFree(crec2), done(err);
      cudaFree(out->crec);
      out->crec = crec2;
      out->pre_steps = pre;
    }
  }
  phase("class items");
  // ---- generic rows: the rest, ordered by (Morton window, signature)
  if (n_rows > 0) row_order_keys<<<grid_for(n_rows, cap), kThreads, 0, s>>>(sig, order, n_rows, window, keys, rows);
  if ((err = cub::DeviceRadixSort::SortPairs(temp, tb, keys, keys2, rows, order, n_rows, 0, 64, s)) != cudaSuccess)
    return done(err);
  int64_t n_gen = n_rows;
  if (out->n_class_rows > 0) {
    std::vector<int32_t> ord(n_rows);
    cudaMemcpyAsync(ord.data(), order, n_rows * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);
    n_gen = 0;
    for (int64_t pos = 0; pos < n_rows; ++pos)
      if (cls_h[ord[pos]] < 0) ord[n_gen++] = ord[pos];
    if (n_gen > 0) cudaMemcpyAsync(order, ord.data(), n_gen * sizeof(int32_t), cudaMemcpyHostToDevice, s);
    if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);
  }
  const int64_t n_items = (n_gen + 31) / 32;
  out->n_items = n_items;
  if ((err = cudaMalloc(&out->warp_rows, (n_items > 0 ? n_items : 1) * 32 * sizeof(int32_t))) != cudaSuccess)
    return done(err);
  if ((err = cudaMalloc(&out->warp_steps, (n_items > 0 ? n_items : 1) * k * sizeof(int32_t))) != cudaSuccess)
    return done(err);
  if ((err = cudaMalloc(&out->warp_rec, (n_items + 1) * sizeof(int64_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&item_total, (n_items + 1) * sizeof(int64_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&out->item_order, (n_items > 0 ? n_items : 1) * sizeof(int32_t))) != cudaSuccess)
    return done(err);
  int32_t* item_len = cnt;  // reuse: n_items <= n_rows + 1
  cudaMemsetAsync(item_total, 0, (n_items + 1) * sizeof(int64_t), s);
  if (n_items > 0)
    item_steps<<<grid_for(n_items, cap), kThreads, 0, s>>>(order, n_gen, n_items, k, inc_ptr, inc, d_row_ptr,
                                                           out->warp_rows, out->warp_steps, item_total, item_len);
  // item order: items whose rows fit the short accumulator pitch first, then
  // the long ones (two launches, each at the occupancy its pitch allows)
  {
    std::vector<int32_t> len(n_items > 0 ? n_items : 1);
    if (n_items > 0) cudaMemcpyAsync(len.data(), item_len, n_items * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);
    int mx = 1;
    for (int64_t w = 0; w < n_items; ++w) mx = std::max(mx, len[w] | 1);
    out->pitch_long = mx;
    out->pitch_short = std::min(mx, 33);
    std::vector<int32_t> ord;
    ord.reserve(n_items);
    for (int64_t w = 0; w < n_items; ++w)
      if ((len[w] | 1) <= out->pitch_short) ord.push_back(static_cast<int32_t>(w));
    out->n_short = static_cast<int64_t>(ord.size());
    for (int64_t w = 0; w < n_items; ++w)
      if ((len[w] | 1) > out->pitch_short) ord.push_back(static_cast<int32_t>(w));
    if (n_items > 0)
      cudaMemcpyAsync(out->item_order, ord.data(), n_items * sizeof(int32_t), cudaMemcpyHostToDevice, s);
    if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);
  }
  tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, item_total, out->warp_rec, n_items + 1, s);
  if ((err = need_temp(tb)) != cudaSuccess) return done(err);
  if ((err = cub::DeviceScan::ExclusiveSum(temp, tb, item_total, out->warp_rec, n_items + 1, s)) != cudaSuccess)
    return done(err);
  int64_t total = 0;
  cudaMemcpyAsync(&total, out->warp_rec + n_items, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);
  out->n_steps = total;
  out->n_incidences = n_inc;
  out->rec_bytes = k <= 4 ? 8 : 16;
  if ((err = cudaMalloc(&out->rec, (total > 0 ? total : 1) * 32 * out->rec_bytes)) != cudaSuccess) return done(err);
  if (n_items > 0) {
    const int g = grid_for(n_items * 32, cap);
    switch (k) {
#define FF_FILL(K) \
  case K: fill_records<K><<<g, kThreads, 0, s>>>(out->erank, out->warp_rows, out->warp_steps, out->warp_rec, n_items, inc_ptr, inc, d_slots, out->rec); break;
      FF_FILL(1) FF_FILL(2) FF_FILL(3) FF_FILL(4) FF_FILL(5) FF_FILL(6) FF_FILL(7) FF_FILL(8) FF_FILL(9) FF_FILL(10)
      FF_FILL(11) FF_FILL(12)
#undef FF_FILL
      default: return done(cudaErrorInvalidValue);
    }
  }
  if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);

  phase("generic items");
  return done(cudaGetLastError());
}

__global__ void expand_block_kernel(const int64_t* __restrict__ rp_s, const int32_t* __restrict__ ci_s, int64_t n_rows,
                                    int bs, int64_t* __restrict__ rp_v, int32_t* __restrict__ ci_v) {
  for (int64_t n = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; n < n_rows;
       n += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = rp_s[n], len = rp_s[n + 1] - b;
    for (int c = 0; c < bs; ++c) {
      const int64_t o = static_cast<int64_t>(bs) * bs * b + static_cast<int64_t>(c) * bs * len;
      rp_v[bs * n + c] = o;
      for (int64_t t = 0; t < len; ++t)
        for (int d = 0; d < bs; ++d) ci_v[o + t * bs + d] = bs * ci_s[b + t] + d;
    }
    if (n == n_rows - 1) rp_v[bs * n_rows] = static_cast<int64_t>(bs) * bs * rp_s[n_rows];
  }
}

cudaError_t expand_block_pattern(const int64_t* rp_s, const int32_t* ci_s, int64_t n_rows, int bs, int64_t* rp_v,
                                 int32_t* ci_v, int sm_count, cudaStream_t s) {
  if (n_rows == 0) return cudaMemsetAsync(rp_v, 0, sizeof(int64_t), s);
  expand_block_kernel<<<grid_for(n_rows, sm_count * 8), kThreads, 0, s>>>(rp_s, ci_s, n_rows, bs, rp_v, ci_v);
  return cudaGetLastError();
}

void free_gather_plan(GatherPlan* p) {
  cudaFree(p->eorder);
  cudaFree(p->erank);
  cudaFree(p->citem_class);
  cudaFree(p->citem_rows);
  cudaFree(p->vconn_m);
  cudaFree(p->citem_rec);
  cudaFree(p->crec);
  cudaFree(p->item_order);
  cudaFree(p->warp_rows);
  cudaFree(p->warp_steps);
  cudaFree(p->warp_rec);
  cudaFree(p->rec);
  *p = GatherPlan{};
}

cudaError_t build_slots(const int32_t* d_dconn, int64_t ne, int k, int64_t rb, int64_t re, const int64_t* row_ptr,
                        const int32_t* col_idx, int slot_bytes, void* d_slots, unsigned long long* d_bad_row,
                        int sm_count, cudaStream_t s) {
  const int g = grid_for(ne * k, sm_count * 16);
  if (slot_bytes == 1)
    element_slots<uint8_t><<<g, kThreads, 0, s>>>(d_dconn, ne, k, rb, re, row_ptr, col_idx,
                                                  static_cast<uint8_t*>(d_slots), d_bad_row);
  else
    element_slots<uint16_t><<<g, kThreads, 0, s>>>(d_dconn, ne, k, rb, re, row_ptr, col_idx,
                                                   static_cast<uint16_t*>(d_slots), d_bad_row);
  return cudaGetLastError();
}

cudaError_t zero_fill(double* a, int64_t na, double* b, int64_t nb, unsigned long long* status, int sm_count,
                      cudaStream_t s) {
  zero_kernel<<<sm_count * 8, kThreads, 0, s>>>(a, na, b, nb, status);
  return cudaGetLastError();
}

}  // namespace ffb::kernels

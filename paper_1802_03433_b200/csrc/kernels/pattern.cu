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
#include <cub/device/device_select.cuh>

#include <cstdint>

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


// ---- row-tile plan ---------------------------------------------------------

__global__ void row_tile_map(const int64_t* __restrict__ tile_row, int64_t n_tiles, int64_t n_rows,
                             int32_t* __restrict__ row_tile) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = n_tiles;  // last t with tile_row[t] <= r
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (tile_row[mid] <= r)
        lo = mid;
      else
        hi = mid;
    }
    row_tile[r] = static_cast<int32_t>(lo);
  }
}

__global__ void visit_keys(const int32_t* __restrict__ dconn, int64_t ne, int k, int64_t rb, int64_t n_rows,
                           const int32_t* __restrict__ row_tile, int64_t n_tiles, uint64_t* __restrict__ keys) {
  const uint64_t invalid = static_cast<uint64_t>(n_tiles) << 32;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < ne * k;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = t / k;
    const int64_t row = static_cast<int64_t>(dconn[t]) - rb;
    keys[t] = (row >= 0 && row < n_rows) ? (static_cast<uint64_t>(row_tile[row]) << 32) | static_cast<uint32_t>(e)
                                         : invalid;
  }
}

__global__ void split_visits(const uint64_t* __restrict__ keys, const int64_t* __restrict__ n_unique, int64_t n_tiles,
                             int64_t* __restrict__ tile_vptr, int32_t* __restrict__ visit_elem) {
  const int64_t n = *n_unique;
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t tile = static_cast<int64_t>(keys[v] >> 32);
    if (tile >= n_tiles) continue;
    visit_elem[v] = static_cast<int32_t>(keys[v] & 0xffffffffu);
    const int64_t prev = v == 0 ? -1 : static_cast<int64_t>(keys[v - 1] >> 32);
    for (int64_t t = prev + 1; t <= tile; ++t) tile_vptr[t] = v;
    if (v == n - 1 || static_cast<int64_t>(keys[v + 1] >> 32) >= n_tiles)
      for (int64_t t = tile + 1; t <= n_tiles; ++t) tile_vptr[t] = v + 1;
  }
}

// one thread per tile: staging offsets and chunk starts (bit 15)
__global__ void chunk_visits(const int32_t* __restrict__ dconn, int k, int64_t rb, const int64_t* __restrict__ tile_row,
                             const int64_t* __restrict__ tile_vptr, const int32_t* __restrict__ visit_elem,
                             int64_t n_tiles, int stage_cap, int chunk_cap, uint16_t* __restrict__ visit_stage) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n_tiles;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t lo = rb + tile_row[t], hi = rb + tile_row[t + 1];
    int stage = 0, count = 0;
    for (int64_t v = tile_vptr[t]; v < tile_vptr[t + 1]; ++v) {
      const int32_t* d = dconn + static_cast<int64_t>(visit_elem[v]) * k;
      int own = 0;
      for (int a = 0; a < k; ++a) own += d[a] >= lo && d[a] < hi;
      bool start = count == 0;
      if (count == chunk_cap || stage + own > stage_cap) {
        stage = 0;
        count = 0;
        start = true;
      }
      visit_stage[v] = static_cast<uint16_t>(stage | (start ? 0x8000 : 0));
      stage += own;
      ++count;
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


cudaError_t build_rowtile_plan(const int32_t* d_dconn, int64_t ne, int k, int64_t rb, int64_t n_rows,
                               const int64_t* d_tile_row, int64_t n_tiles, int stage_cap, int chunk_cap, int sm_count,
                               cudaStream_t s, int64_t** tile_vptr, int32_t** visit_elem, uint16_t** visit_stage,
                               int64_t* n_visits) {
  const int cap = sm_count * 16;
  const int64_t n_keys = ne * k;
  int32_t* row_tile = nullptr;
  uint64_t *keys = nullptr, *sorted = nullptr;
  int64_t* d_count = nullptr;
  void* temp = nullptr;
  cudaError_t err = cudaSuccess;
  auto done = [&](cudaError_t e) {
    cudaFree(row_tile);
    cudaFree(keys);
    cudaFree(sorted);
    cudaFree(d_count);
    cudaFree(temp);
    return e;
  };
  if ((err = cudaMalloc(&row_tile, (n_rows > 0 ? n_rows : 1) * sizeof(int32_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&keys, (n_keys > 0 ? n_keys : 1) * sizeof(uint64_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&sorted, (n_keys > 0 ? n_keys : 1) * sizeof(uint64_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(&d_count, sizeof(int64_t))) != cudaSuccess) return done(err);
  row_tile_map<<<grid_for(n_rows, cap), kThreads, 0, s>>>(d_tile_row, n_tiles, n_rows, row_tile);
  visit_keys<<<grid_for(n_keys, cap), kThreads, 0, s>>>(d_dconn, ne, k, rb, n_rows, row_tile, n_tiles, keys);
  int end_bit = 32;
  while ((static_cast<int64_t>(1) << (end_bit - 32)) <= n_tiles) ++end_bit;
  size_t t_sort = 0, t_uniq = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, t_sort, keys, sorted, n_keys, 0, end_bit, s);
  cub::DeviceSelect::Unique(nullptr, t_uniq, sorted, keys, d_count, n_keys, s);
  if ((err = cudaMalloc(&temp, t_sort > t_uniq ? t_sort : t_uniq)) != cudaSuccess) return done(err);
  if ((err = cub::DeviceRadixSort::SortKeys(temp, t_sort, keys, sorted, n_keys, 0, end_bit, s)) != cudaSuccess)
    return done(err);
  if ((err = cub::DeviceSelect::Unique(temp, t_uniq, sorted, keys, d_count, n_keys, s)) != cudaSuccess) return done(err);
  int64_t n_unique = 0;
  cudaMemcpyAsync(&n_unique, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(tile_vptr, (n_tiles + 1) * sizeof(int64_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(visit_elem, (n_unique > 0 ? n_unique : 1) * sizeof(int32_t))) != cudaSuccess) return done(err);
  if ((err = cudaMalloc(visit_stage, (n_unique > 0 ? n_unique : 1) * sizeof(uint16_t))) != cudaSuccess) return done(err);
  cudaMemsetAsync(*tile_vptr, 0, (n_tiles + 1) * sizeof(int64_t), s);
  split_visits<<<grid_for(n_unique, cap), kThreads, 0, s>>>(keys, d_count, n_tiles, *tile_vptr, *visit_elem);
  chunk_visits<<<grid_for(n_tiles, cap), 64, 0, s>>>(d_dconn, k, rb, d_tile_row, *tile_vptr, *visit_elem, n_tiles,
                                                     stage_cap, chunk_cap, *visit_stage);
  int64_t last_key = 0;
  if (n_unique > 0) cudaMemcpyAsync(&last_key, keys + (n_unique - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return done(err);
  *n_visits = n_unique - ((static_cast<uint64_t>(last_key) >> 32) >= static_cast<uint64_t>(n_tiles) ? 1 : 0);
  return done(cudaGetLastError());
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

// Host launchers of the offline-compiled (nvcc, sm_100a) kernels.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <vector>

#include <cstdint>

namespace ffb::kernels {

// K1: CSR pattern of rows [rb, re) from device DOF connectivity [ne][k].
// Allocates *row_ptr (n_rows+1, int64) and *col_idx (nnz, int32) with cudaMalloc.
cudaError_t build_pattern(const int32_t* d_dconn, int64_t ne, int k, int64_t rb, int64_t re, int sm_count,
                          cudaStream_t s, int64_t** row_ptr, int32_t** col_idx, int64_t* nnz, int* max_row_len);

// Element slot plan [ne][k][k] (u8 or u16): position of dof[b] in row dof[a].
cudaError_t build_slots(const int32_t* d_dconn, int64_t ne, int k, int64_t rb, int64_t re, const int64_t* row_ptr,
                        const int32_t* col_idx, int slot_bytes, void* d_slots, unsigned long long* d_bad_row,
                        int sm_count, cudaStream_t s);

// Row-gather plan (one CSR row per lane, 32 rows per warp item, lock-step
// records [step][32] of (element id, k slot bytes); see pattern.cu).
struct GatherPlan {
  int64_t n_items = 0, n_steps = 0, n_incidences = 0;
  int rec_bytes = 0;                 // 8 (k <= 4) or 16 (k <= 12)
  int32_t* warp_rows = nullptr;      // [n_items][32] local row or -1
  int32_t* warp_steps = nullptr;     // [n_items][k]
  int64_t* warp_rec = nullptr;       // [n_items + 1] first record step of each item
  void* rec = nullptr;               // [n_steps][32] records
  int32_t* item_order = nullptr;     // [n_items]: the n_short short-pitch items, then the long ones
  int64_t n_short = 0;
  int pitch_short = 1, pitch_long = 1;  // odd accumulator pitches (longest row of the class, | 1)
  // Row classes: rows whose sorted incidence sequence (local index + slot
  // bytes of every incidence) and length are identical. Frequent classes
  // get a specialised NVRTC kernel with the slots as compile-time register
  // indices; the rows above (the generic items) are the others.
  struct Class {
    int len = 0, steps = 0;
    std::vector<int> local;         // [steps] local index i of each step
    std::vector<uint8_t> slots;     // [steps][k]
    std::vector<int> order;         // processing order of the steps (records are laid out in it)
    int64_t rows = 0;
  };
  std::vector<Class> classes;
  int64_t n_citems = 0, n_citems_short = 0, n_crec = 0, n_class_rows = 0;
  int32_t* citem_class = nullptr;   // [n_citems]
  int32_t* citem_rows = nullptr;    // [n_citems][32] local row of each lane or -1 (row_lanes lanes per row)
  int32_t* vconn_m = nullptr;       // [E][dim+1] vertex ids in record (Morton) order, read by K2a
  // element ids of the class items, in each class's processing order: item
  // w's first pre_steps steps at crec[(w * pre_steps + t) * 32 + lane], its
  // other steps from crec[citem_rec[w] * 32]
  int64_t* citem_rec = nullptr;     // [n_citems + 1]
  int32_t* crec = nullptr;          // [n_crec (+ 8 steps of padding)] element records (-1: idle lane)
  int pre_steps = 0;
  // element order of the per-element records: record t belongs to element
  // eorder[t]; records (rec, crec) hold erank[e]
  int32_t* eorder = nullptr;
  int32_t* erank = nullptr;
};
// bbox: {min x, min y, min z, max x, max y, max z} of the mesh coordinates.
// Processing order of a row class's steps (the code generator's choice; the
// records of its items are laid out in that order).
using ClassOrderFn = std::function<std::vector<int>(const GatherPlan::Class&)>;
cudaError_t build_gather_plan(const double* d_coords, const int32_t* d_vconn, int dim, const double* bbox,
                              const int32_t* d_dconn, int64_t ne, int k, int64_t rb, int64_t n_rows,
                              const int64_t* d_row_ptr, const uint8_t* d_slots, int window, int sm_count,
                              cudaStream_t s, GatherPlan* out, int min_class_rows = 128, int max_classes = 64,
                              bool use_eorder = true, bool split_long = true,
                              const ClassOrderFn* step_order = nullptr, double class_frac = 0.0005,
                              int row_lanes = 1);
void free_gather_plan(GatherPlan* p);

// fem::Mesh::validate (fem.cpp:17-34) on the device: *d_bad = the lowest
// element with a vertex id outside [0, nv), duplicate vertices, a DOF id
// outside [0, n_dofs) or duplicate DOFs (d_dconn may be null), or -- when
// `orient` -- a non-positive signed area / volume; ~0 when every element passes.
cudaError_t validate_mesh(const double* d_coords, int dim, int64_t nv, const int32_t* d_vconn, const int32_t* d_dconn,
                          int k, int64_t n_dofs, int64_t ne, bool orient, unsigned long long* d_bad, int sm_count,
                          cudaStream_t s);
// *d_diff |= 1 when d_src and d_dst differ anywhere (exact; nothing written).
cudaError_t compare(const int32_t* d_src, const int32_t* d_dst, int64_t n, unsigned long long* d_diff, int sm_count,
                    cudaStream_t s);
// d_dst := d_src (n int32); *d_diff |= 1 when any value changed (exact).
cudaError_t copy_compare(const int32_t* d_src, int32_t* d_dst, int64_t n, unsigned long long* d_diff, int sm_count,
                         cudaStream_t s);


// Block expansion of a scalar CSR: row bs*n + c holds columns bs*m + d of every
// scalar column m of row n (d = 0..bs-1), sorted. rp_v [bs*n_rows + 1].
cudaError_t expand_block_pattern(const int64_t* rp_s, const int32_t* ci_s, int64_t n_rows, int bs, int64_t* rp_v,
                                 int32_t* ci_v, int sm_count, cudaStream_t s);

// Downstream consumer (linalg.cu): y = A x (warp per row) and the reference's
// unpreconditioned CG (linalg.cpp:61-96) with deterministic reductions.
struct CgStats {
  int iterations = 0;
  double residual = 0.0;
  int converged = 0;
  int breakdown = 0;  // 1: non-finite step, 2: non-finite residual
};
cudaError_t spmv(const int64_t* rp, const int32_t* ci, const double* a, const double* x, double* y, int64_t n,
                 int sm_count, cudaStream_t s);
cudaError_t cg_solve(const int64_t* rp, const int32_t* ci, const double* a, const double* b, double* x, int64_t n,
                     double tol, int max_iter, int sm_count, cudaStream_t s, CgStats* st);

// K0: values[0:na] = 0, rhs[0:nb] = 0, status[0:2] = ~0 (one launch).
cudaError_t zero_fill(double* a, int64_t na, double* b, int64_t nb, unsigned long long* status, int sm_count,
                      cudaStream_t s);

}  // namespace ffb::kernels

// femforge-b200 runtime internals: NVRTC compilation with a CUBIN cache,
// error types, and the C-ABI handle structures.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "femforge/codegen.hpp"
#include "femforge/fem.hpp"
#include "../kernels/kernels.hpp"

namespace ffb {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);

struct CompiledModule {
  std::string cubin;
  std::string log;
  int registers = 0;
  int shared_bytes = 0;
  double ms = 0.0;
};

// NVRTC -> sm_100a CUBIN. Cached in memory by (source, options); optionally
// on disk under $FF_CUBIN_CACHE. Throws Error(FF_E_NVRTC) with the log.
CompiledModule nvrtc_compile(const std::string& source, const std::string& name);

}  // namespace ffb

struct ff_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;             // second stream: concurrent gather launches
  cudaStream_t upload = nullptr;           // ff_assemble: connectivity upload + compare
  cudaEvent_t fork = nullptr, join = nullptr;
  unsigned long long* d_status = nullptr;  // [bad_elem, bad_row, scratch, vconn diff, dconn diff]
  unsigned long long* h_status = nullptr;  // pinned mirror (4: [bad_elem, bad_row, vconn diff, dconn diff])
  int scatter = 2;                          // FF_SCATTER_*_MODE (default: row gather)
  int64_t class_min_rows = 128;             // gather row classes (0: off)
};

struct ff_form {
  ff_ctx* ctx = nullptr;
  std::uint64_t id = 0;             // process-unique (graph replay keys)
  int dim = 2, degree = 1, n_local = 3, block = 256;
  int ncomp = 1;                    // components of a vector (blocked) form
  femforge::codegen::ElementPlan plan;
  bool raw = false;                 // ff_compile route (caller source)
  femforge::fem::InstantiatedForm inst;
  femforge::codegen::LaunchParams params;
  int quad_rule = 0;
  double compile_ms = 0.0;
  // one module per slot width (1: u8 plans, 2: u16 plans)
  std::string source[3];
  ffb::CompiledModule module[3];
  cudaLibrary_t lib[3] = {nullptr, nullptr, nullptr};
  cudaKernel_t kernel[3] = {nullptr, nullptr, nullptr};          // ff_assemble_atomic
  cudaKernel_t kernel_ginv[3] = {nullptr, nullptr, nullptr};     // ff_gather_invariants
  cudaKernel_t kernel_grows[3] = {nullptr, nullptr, nullptr};    // ff_gather_rows
};

struct ff_mesh {
  ff_ctx* ctx = nullptr;
  int dim = 2;
  int k = 3;  // (scalar) DOFs per element
  int bs = 1; // components per node: global DOF bs * node + c
  int64_t nv = 0, ne = 0, n_dofs = 0;
  double* coords = nullptr;
  int32_t* vconn = nullptr;
  int32_t* dconn = nullptr;  // == vconn for P1
  std::uint64_t generation = 0;      // process-wide unique per connectivity (plan keys)
  int32_t* stage = nullptr;          // ff_assemble upload staging of vconn (exact re-upload compare)
  int32_t* stage_d = nullptr;        // ... of dconn (P2: uploaded concurrently with vconn's compare)
};

struct ff_pattern {
  ff_ctx* ctx = nullptr;
  // rows [rb, re) and nnz of the SCALAR pattern; a blocked pattern (bs > 1)
  // is its bs x bs expansion: bs*(re-rb) rows, bs^2*nnz entries
  int64_t rb = 0, re = 0, nnz = 0;
  int bs = 1;
  int64_t* vrow_ptr = nullptr;  // expanded CSR on the device (blocked; built on demand)
  int32_t* vcol_idx = nullptr;
  int max_row_len = 0;
  int k = 0;
  int64_t ne = 0;
  int64_t* row_ptr = nullptr;
  int32_t* col_idx = nullptr;
  // element slot plan for one mesh
  const ff_mesh* plan_mesh = nullptr;
  std::uint64_t plan_generation = ~0ull;
  void* slots = nullptr;
  int slot_bytes = 1;
  // row-gather plan for plan_mesh, and the per-element invariant buffers
  std::uint64_t gather_generation = ~0ull;
  // CUDA graph of the last device assembly (ff_assemble_device replays it when
  // every pointer and plan it captured is unchanged)
  std::vector<std::uint64_t> graph_key, graph_warm_key;
  cudaGraphExec_t graph_exec = nullptr;
  int64_t gather_class_min = -1;            // class_min_rows the plan was built with
  const ff_mesh* gather_mesh = nullptr;
  ffb::kernels::GatherPlan gather;
  double gather_ms = 0.0;
  // class-specialised gather kernels for (form source, plan)
  std::string class_key;
  cudaLibrary_t class_lib = nullptr;
  cudaKernel_t class_kernel[2] = {nullptr, nullptr};  // short rows, long rows
  int class_smem[2] = {0, 0};                           // their dynamic shared memory
  double class_compile_ms = 0.0;
  double* ginv = nullptr;   // [ne][nkp]
  double* bvec = nullptr;   // [ne][k]
  std::size_t ginv_cap = 0, bvec_cap = 0;
  // FF_SCATTER_AUTO_MODE: the measured choice for (form id, slot-plan generation)
  std::uint64_t auto_form = 0, auto_generation = ~0ull;
  int auto_mode = 0;
  double auto_ms[2] = {-1.0, -1.0};  // gather, atomic
  // device scratch of the host-buffer (end-to-end) entry point
  double* e2e_values = nullptr;
  double* e2e_rhs = nullptr;
};

// femforge-b200 C++ assembly API: the reference's device layer
// (/root/reference/proj/include/femforge/device/device.hpp:13-159) with the
// simulated GPU replaced by the real one. Thin RAII wrappers over the C ABI
// (include/femforge_b200.h); error codes are rethrown as the reference's
// exception types and messages.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "femforge/codegen.hpp"
#include "femforge/fem.hpp"

struct ff_ctx;
struct ff_form;
struct ff_mesh;
struct ff_pattern;

namespace femforge::device {

class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// One CUDA device + stream (the reference runs everything on the host).
class Engine {
 public:
  explicit Engine(int device = 0);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  ff_ctx* handle() const { return ctx_; }
  void synchronize() const;
  static Engine& default_engine();

 private:
  ff_ctx* ctx_ = nullptr;
};

// device.hpp:81-89: elems_per_block / mode / workers / seed are accepted for
// API parity; the GPU kernel's block is `block_size` threads (one element
// each) and the atomic scatter makes every launch "parallel mode".
enum class ExecMode { Deterministic, Parallel };
struct LaunchConfig {
  int elems_per_block = 4;
  ExecMode mode = ExecMode::Deterministic;
  int workers = 1;
  std::uint64_t seed = 0;
  int block_size = 256;
  int quad_rule = 0;
  codegen::Strategy strategy = codegen::Strategy::Auto;
  void validate() const;  // DeviceError on launch-limit violations
};

// The runtime-compiled element kernel: the FormEvaluator plug-in of the
// reference (device.hpp:97-126), NVRTC-compiled for sm_100a.
class CompiledKernel {
 public:
  CompiledKernel(const fem::WeakForm& wf, const LaunchConfig& cfg = {}, Engine& eng = Engine::default_engine());
  ~CompiledKernel();
  CompiledKernel(const CompiledKernel&) = delete;
  CompiledKernel& operator=(const CompiledKernel&) = delete;
  ff_form* handle() const { return form_; }
  std::string source() const;
  int registers() const;

 private:
  ff_form* form_ = nullptr;
};

// Device-resident mesh: coordinates, vertex connectivity and DOF map (the
// reference's flattened DeviceArrays, device.hpp:54-63, without the per-element
// coordinate copies).
class DeviceArrays {
 public:
  DeviceArrays(const fem::Mesh& m, const fem::DofMap& dofs, Engine& eng = Engine::default_engine());
  ~DeviceArrays();
  DeviceArrays(const DeviceArrays&) = delete;
  DeviceArrays& operator=(const DeviceArrays&) = delete;
  ff_mesh* handle() const { return mesh_; }
  std::int64_t n_dofs() const { return n_dofs_; }
  int element_count() const { return n_elems_; }

 private:
  ff_mesh* mesh_ = nullptr;
  std::int64_t n_dofs_ = 0;
  int n_elems_ = 0;
};
std::unique_ptr<DeviceArrays> flatten_mesh(const fem::Mesh& m, int degree = 1);

// Sorted unique rows with the diagonal (device.hpp:65-74). CSR on the device;
// host copies (CSR + the reference's ELL view) on request.
class SparsityPattern {
 public:
  SparsityPattern(const DeviceArrays& d, std::int64_t row_begin = 0, std::int64_t row_end = -1,
                  Engine& eng = Engine::default_engine());
  ~SparsityPattern();
  SparsityPattern(const SparsityPattern&) = delete;
  SparsityPattern& operator=(const SparsityPattern&) = delete;
  ff_pattern* handle() const { return pat_; }
  std::int64_t n = 0;       // rows in the block
  std::int64_t nnz = 0;
  int max_nz = 0;           // longest row
  std::int64_t row_begin = 0;
  std::vector<std::int64_t> row_ptr() const;
  std::vector<std::int32_t> col_idx() const;
  std::vector<int> row_len() const;   // ELL view
  std::vector<int> row_cols() const;  // n x max_nz, -1 padded

 private:
  ff_pattern* pat_ = nullptr;
};
std::unique_ptr<SparsityPattern> build_sparsity(const DeviceArrays& d);

struct CsrMatrix {
  std::int64_t n = 0;
  std::vector<std::int64_t> row_ptr;
  std::vector<std::int32_t> col_idx;
  std::vector<double> values;
};

struct CsrSystem {
  CsrMatrix a;
  std::vector<double> b;
};

// ELL result of the reference layout (linalg.hpp:26-42 + device.hpp:136-139).
struct EllMatrix {
  int n = 0;
  int max_nz = 0;
  std::vector<double> values;
  std::vector<int> columns;
};
struct EllSystem {
  EllMatrix a;
  std::vector<double> b;
};

// device.hpp:143-153 equivalents (host results).
CsrSystem assemble_csr(const CompiledKernel& k, const DeviceArrays& d, SparsityPattern& sp);
EllSystem assemble_sparse(const CompiledKernel& k, const DeviceArrays& d, SparsityPattern& sp,
                          const LaunchConfig& cfg = {});

// One call: weak form + mesh -> CSR + RHS (the north-star assemble()).
CsrSystem assemble(const fem::WeakForm& wf, const fem::Mesh& m, const LaunchConfig& cfg = {});

}  // namespace femforge::device

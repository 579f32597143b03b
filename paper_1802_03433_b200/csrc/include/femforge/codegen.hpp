// femforge-b200 code generation: symbolic integrands -> SSA register IR ->
// CUDA C++ for NVRTC (sm_100a).
//
// API parity with /root/reference/proj/include/femforge/codegen/kernel.hpp:13-78
// (Op, Instr, CodegenError, KernelProgram{run,disassemble}, lower,
// CompiledForm, compile_form, LaunchParams, emit_source). Differences, by
// design: emit_source renders the REAL kernel that NVRTC compiles (the
// reference's template is inspection-only), and the element body
// comes from a quadrature compiler (plan_element) instead of one __device__
// function per entry and quadrature point.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "femforge/fem.hpp"
#include "femforge/symbolic.hpp"

namespace femforge::codegen {

using symbolic::Expr;
using symbolic::SymbolTable;

enum class Op : std::uint8_t { LoadArg, LoadConst, Add, Sub, Mul, Div, Neg, PowInt, Sin, Cos, Sqrt };

struct Instr {
  Op op;
  int a = -1;
  int b = -1;
  std::int64_t imm = 0;
};

class CodegenError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// Flat SSA program: instruction k writes register k (kernel.hpp:43-54).
struct KernelProgram {
  std::vector<Instr> code;
  std::vector<double> consts;
  int arity = 0;
  int result = 0;

  double run(std::span<const double> args) const;
  double run(std::span<const double> args, std::vector<double>& scratch) const;
  std::string disassemble() const;
};

KernelProgram lower(const Expr& e, const SymbolTable& args);

// Several outputs lowered into one SSA program with common-subexpression
// elimination across all of them (the reference lowers entries separately,
// kernel.cpp:277-283, so det J is recomputed per entry).
struct MultiProgram {
  std::vector<Instr> code;
  std::vector<double> consts;
  std::vector<std::string> arg_names;
  std::vector<int> results;
  void run(std::span<const double> args, std::span<double> out) const;
};
MultiProgram lower_many(const std::vector<Expr>& outputs, const SymbolTable& args);

struct CompiledForm {
  std::vector<KernelProgram> bilinear;  // n_local^2
  std::vector<KernelProgram> linear;    // n_local
  int n_quad = 3;
  int n_local = 3;
  int dim = 2;
};

CompiledForm compile_form(const fem::InstantiatedForm& f);

// ---------------------------------------------------------------------------
// GPU element code

enum class Strategy : int {
  Auto = 0,
  // Quadrature summed at compile time: every entry becomes a constant-weight
  // combination of per-element geometric invariants (reference-tensor form).
  // Requires integrands polynomial in the reference coordinates.
  ReferenceTensor = 1,
  // Integrand evaluated at each quadrature point in registers, weighted sum
  // in ascending q (device.cpp:176-192 order); always applicable.
  Pointwise = 2,
};

struct ElementPlan {
  int dim = 2;
  int degree = 1;
  int n_local = 3;
  int n_quad = 3;
  Strategy strategy = Strategy::ReferenceTensor;
  std::string body;        // CUDA statements; emits FF_EMIT_A(i,j,v) / FF_EMIT_B(i,v)
  std::string prelude;     // namespace-scope declarations the body uses (quadrature tables)
  int n_invariants = 0;    // ReferenceTensor: merged geometric invariants
  int n_unique_entries = 0;
  std::int64_t flops = 0;  // fp64 operations per element after CSE (estimate)
  // Row-gather split (ReferenceTensor only): the invariants the bilinear
  // entries read (stored per element by the invariants kernel, body lines
  // FF_KINV(q, ff_tT)), and per local row i the static code computing
  // v[j] = K_ij from g[q] (ff_row<i> specialisations).
  int n_kinv = 0;
  std::string row_code;
  std::int64_t row_flops = 0;  // fp64 operations of all n_local rows
  // Vector forms (block-uniform record): component block (c, d)'s entries
  // are one linear map of its n_bq quantities at record offset
  // block_q[c * ncomp + d] (ff_vrow<a> in row_code, ff_block_q, FF_NBQ).
  int n_bq = 0;
  std::vector<int> block_q;
  // load-vector entries that are identically zero (the record skips them)
  std::vector<char> b_zero;
};
// Element-record slot of load-vector entry i in the SoA part (entries
// below n_bpad ride in the invariants' chunk padding; -1: zero, not stored)
// and the number of stored SoA entries.
std::vector<int> record_bslots(const ElementPlan& plan, int n_local, int ncomp, int* n_soa = nullptr);

ElementPlan plan_element(const fem::InstantiatedForm& f, const fem::QuadratureRule& rule,
                         Strategy strategy = Strategy::Auto);

// Scatter variants of the assembly template.
enum class Scatter : int {
  Auto = 0,
  Atomic = 1,     // element-parallel, fp64 RED into CSR slots (K0 zero-fill first)
  Gather = 3,     // row per lane: element invariants + lock-step row gather
};

struct LaunchParams {
  int n_quad = 3;           // informational (taken from the rule)
  int n_local = 3;          // informational (taken from the form)
  int elems_per_block = 4;  // reference knob; maps to the CUDA block size (x32 threads)
  int max_nz = 7;           // informational (ELL width of the reference layout)
  int quad_rule = 0;        // 0: default rule for (dim, degree)
  Strategy strategy = Strategy::Auto;
  Scatter scatter = Scatter::Atomic;
  int block_size = 256;     // threads per CTA of the element kernel
  int slot_bytes = 1;       // 1 or 2: width of the element slot plan entries
};

int default_quad_rule(int dim, int degree);

// Renders the complete NVRTC translation unit (template + element body).
// Byte-deterministic for identical inputs; throws CodegenError on bad params.
std::string emit_source(const fem::InstantiatedForm& f, const LaunchParams& cfg);
std::string emit_source(const fem::InstantiatedForm& f, const LaunchParams& cfg, ElementPlan* plan_out);

// Row classes of a gather plan (rows with identical incidence sequences):
// the specialised gather kernels keep a class's row in registers, indexed by
// the compile-time slots.
struct RowClass {
  int len = 0;                       // row length (CSR entries)
  int steps = 0;                     // incidences
  std::vector<int> local;            // [steps] local index i of each incidence
  std::vector<std::uint8_t> slots;   // [steps][n_local] slot of column dof[j] in the row
  std::vector<int> order;            // processing order of the steps (empty: class_step_order)
};
// Incidence order of a class that keeps few row slots open at once.
std::vector<int> class_step_order(const RowClass& k, int n_local);

// Whether the plan's kernels include the row gather (K2a + generic K2b).
int record_pair_tail(int n_local);
bool gather_capable(const ElementPlan& plan, int n_local, int ncomp, int block_size);

// Incidence order of a row class that minimises the number of row slots whose
// register accumulators are open at once (deterministic).
std::vector<int> class_step_order(const RowClass& k, int n_local);
// Staging-row pitch of class kernel `kernel` (0: _s, 1: _l; odd, >= its
// longest class row).
// Vector forms (bs > 1) stage whole rows in one kernel: the longest row, odd.
int class_stage_pitch(const std::vector<RowClass>& classes, int kernel, bool fused, int bs = 1);
// Vector forms: row pitch of the CSR-order staging tile (32 / bs rows + a
// spare row per warp): >= bs * longest row, = bs (mod 16).
int vector_stage_pitch(const std::vector<RowClass>& classes, int bs, int kernel = 0, bool fused = true);
// Dynamic shared memory of class kernel `kernel` (4 warps).
inline int class_shared_bytes(const std::vector<RowClass>& classes, int kernel, bool fused, int warps = 4,
                              int bs = 1) {
  if (bs > 1)
    return warps * (((32 / bs + 1) * vector_stage_pitch(classes, bs, kernel, fused) + 1) & ~1) * 8 + warps * 32 * 8;
  return warps * 32 * class_stage_pitch(classes, kernel, fused, bs) * 8 + warps * 32 * 8;
}

// NVRTC translation unit with ff_gather_classes_s (classes of rows <= 33
// entries) and ff_gather_classes_l (longer rows). Needs a gather-capable
// plan (plan.n_kinv > 0). Byte-deterministic.
// pre: the item's first `pre` record ids come from the plan's computable
// prefix block (GatherPlan::pre_steps; every class has >= pre steps).
std::string emit_class_source(const ElementPlan& plan, int n_local, const std::vector<RowClass>& classes,
                              bool fused = false, int bs = 1, int pre = 1);

// Shortest round-trip double literal valid in C/CUDA source.
std::string double_literal(double v);

}  // namespace femforge::codegen

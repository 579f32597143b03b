// C++ host-API suites (run by tests/test_capi.py::test_cpp_host_suites).
//
// Mirrors the reference's own C++ tests for the path:
//  * test_codegen.cpp:102-123  IR VM (KernelProgram::run) vs the tree
//    evaluator on 1,200 random argument vectors of the demo form, <= 1e-12;
//  * test_codegen.cpp:89-100   the compiled stiffness entry integrates to K00 = 1;
//  * test_fem.cpp / SURVEY App. B  reference-element KATs (2D and 3D P1);
//  * fem.cpp:17-34             Mesh::validate wording and check order;
//  * test_device.cpp:176-260   the C++ device API (device.hpp facade over the
//    C ABI) against a host assembly that runs the reference's algorithm with
//    the IR VM (per element, per entry, ascending-q sum of w*f, binary-search
//    scatter, device.cpp:147-205 and :265-305). Needs a GPU, else skipped.
#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <random>
#include <set>

#include "check.hpp"
#include "femforge/codegen.hpp"
#include "femforge/device.hpp"
#include "femforge/fem.hpp"
#include "femforge/meshgen.hpp"
#include "femforge/symbolic.hpp"
#include "femforge_b200.h"

using namespace femforge;
using symbolic::Expr;
using symbolic::integer;
using symbolic::parse;
using symbolic::sym;

namespace {

fem::WeakForm demo_weak_form() {
  Expr x = sym("x"), y = sym("y");
  fem::Mat2 sigma{integer(1), -x - y, x + y, integer(1)};
  return fem::helmholtz_form(sigma, integer(1), parse("-2*(x^2+y^2)+36"));
}

std::map<std::string, double> to_map(const symbolic::SymbolTable& t, std::span<const double> a) {
  std::map<std::string, double> m;
  for (int i = 0; i < t.size(); ++i) m[t.names()[i]] = a[i];
  return m;
}

double rel(double a, double b) { return std::abs(a - b) / std::max(1.0, std::abs(b)); }

bool have_gpu() {
  int n = 0;
  return ff_device_count(&n) == FF_OK && n > 0;
}

}  // namespace

TEST_CASE("IR VM: semantic preservation against the tree evaluator (2D demo form)") {
  fem::InstantiatedForm f = fem::instantiate(demo_weak_form());
  const symbolic::SymbolTable& args = fem::kernel_args();
  std::mt19937 rng(2024);
  std::uniform_real_distribution<double> coord(-1.0, 1.0);
  std::vector<Expr> corpus(f.bilinear.begin(), f.bilinear.end());
  corpus.insert(corpus.end(), f.linear.begin(), f.linear.end());
  int checked = 0;
  for (const Expr& e : corpus) {
    codegen::KernelProgram p = codegen::lower(e, args);
    for (std::size_t k = 0; k < p.code.size(); ++k) {  // SSA: operands precede their use
      CHECK(p.code[k].a < static_cast<int>(k));
      CHECK(p.code[k].b < static_cast<int>(k));
    }
    for (int t = 0; t < 100; ++t) {
      std::array<double, 8> a;
      for (double& v : a) v = coord(rng);
      const double vm = p.run(a), tree = symbolic::eval(e, to_map(args, a));
      CHECK(std::abs(vm - tree) <= 1e-12 * std::max(1.0, std::abs(tree)));
      ++checked;
    }
  }
  CHECK(checked == 1200);
  CHECK_THROWS_AS(codegen::lower(sym("xi"), args).run(std::vector<double>{1.0}), codegen::CodegenError);
}

TEST_CASE("IR VM: 3D P2 variable-coefficient form, VM == tree and lower_many == lower") {
  fem::Mesh cube = meshgen::kuhn_cube_mesh(1);
  Expr x = sym("x"), y = sym("y"), z = sym("z");
  fem::Mat3 sigma{integer(1) + x * y * z, integer(0), integer(0), integer(0), integer(1) + x * y * z, integer(0),
                  integer(0), integer(0), integer(1) + x * y * z};
  fem::WeakForm wf = fem::convection_form(sigma, integer(1) + x * x, {integer(1), x, -y}, parse("x*y+z"));
  wf.space = fem::function_space(cube, 2);
  fem::InstantiatedForm f = fem::instantiate(wf);
  CHECK(f.n_local == 10 && f.bilinear.size() == 100 && f.linear.size() == 10);
  const symbolic::SymbolTable& args = fem::kernel_args(3);
  std::vector<Expr> outs(f.bilinear.begin(), f.bilinear.end());
  outs.insert(outs.end(), f.linear.begin(), f.linear.end());
  codegen::MultiProgram mp = codegen::lower_many(outs, args);
  std::mt19937 rng(7);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::vector<double> many(outs.size());
  for (int t = 0; t < 5; ++t) {
    std::vector<double> a(args.size());
    for (double& v : a) v = u(rng);
    mp.run(a, many);
    const auto env = to_map(args, a);
    for (std::size_t k = 0; k < outs.size(); k += 7) {
      const double one = codegen::lower(outs[k], args).run(a);
      CHECK(one == many[k]);  // cross-root CSE keeps every operation: bit-identical
      CHECK(rel(one, symbolic::eval(outs[k], env)) <= 1e-12);
    }
  }
}

TEST_CASE("compiled stiffness entry integrates to the derived K00 (test_codegen.cpp:89-100)") {
  fem::WeakForm wf = fem::helmholtz_form(fem::Mat2{integer(1), integer(0), integer(0), integer(1)}, integer(0),
                                         integer(0));
  codegen::CompiledForm cf = codegen::compile_form(fem::instantiate(wf));
  fem::QuadratureRule q = fem::quadrature_rule();
  double acc = 0.0;
  for (int k = 0; k < q.size(); ++k) {
    std::array<double, 8> a{q.points[k][0], q.points[k][1], 0, 0, 1, 0, 0, 1};
    acc += q.weights[k] * cf.bilinear[0].run(a);
  }
  CHECK(std::abs(acc - 1.0) <= 1e-14);
}

TEST_CASE("3D P1 reference tet: K, M and load through the VM (SURVEY App. B)") {
  fem::Mesh cube = meshgen::kuhn_cube_mesh(1);
  fem::WeakForm wf = fem::helmholtz_form(
      fem::Mat3{integer(1), integer(0), integer(0), integer(0), integer(1), integer(0), integer(0), integer(0), integer(1)},
      integer(1), integer(1));
  wf.space = fem::function_space(cube, 1);
  codegen::CompiledForm cf = codegen::compile_form(fem::instantiate(wf));
  fem::QuadratureRule q = fem::quadrature_rule(3, 4);
  const double K6[4][4] = {{3, -1, -1, -1}, {-1, 1, 0, 0}, {-1, 0, 1, 0}, {-1, 0, 0, 1}};
  const double M120[4][4] = {{2, 1, 1, 1}, {1, 2, 1, 1}, {1, 1, 2, 1}, {1, 1, 1, 2}};
  for (int i = 0; i < 4; ++i) {
    double l = 0.0;
    for (int j = 0; j < 4; ++j) {
      double acc = 0.0;
      for (int k = 0; k < q.size(); ++k) {
        std::array<double, 15> a{q.points[k][0], q.points[k][1], q.points[k][2], 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1};
        acc += q.weights[k] * cf.bilinear[i * 4 + j].run(a);
        if (j == 0) l += q.weights[k] * cf.linear[i].run(a);
      }
      CHECK(std::abs(acc - (K6[i][j] / 6.0 + M120[i][j] / 120.0)) <= 1e-14);
    }
    CHECK(std::abs(l - 1.0 / 24.0) <= 1e-15);
  }
}

TEST_CASE("Mesh::validate: wording and check order (fem.cpp:17-34)") {
  fem::Mesh m = meshgen::unit_square_mesh(2);
  m.validate();
  fem::Mesh a = m;
  a.elements[3].nodes[1] = 99;
  auto msg = [](const fem::Mesh& mm) {
    try {
      mm.validate();
    } catch (const fem::MeshError& e) {
      return std::string(e.what());
    }
    return std::string();
  };
  CHECK(msg(a) == "element 3: node index 99 out of range");
  fem::Mesh b = m;
  b.elements[2].nodes[2] = b.elements[2].nodes[0];
  CHECK(msg(b) == "element 2: duplicate node indices");
  fem::Mesh c = m;
  std::swap(c.elements[5].nodes[1], c.elements[5].nodes[2]);
  CHECK(msg(c) == "element 5: non-positive signed area");
  fem::Mesh t = meshgen::kuhn_cube_mesh(2);
  t.validate();
  std::swap(t.elements[7].nodes[0], t.elements[7].nodes[3]);
  CHECK(msg(t) == "element 7: non-positive signed volume");
}

namespace {

// The reference algorithm on the host, evaluator = the IR VM (CompiledForm):
// det mode, element order, ascending q, binary search in the sorted row.
void host_assemble(const codegen::CompiledForm& cf, const fem::Mesh& m, const std::vector<std::int64_t>& rp,
                   const std::vector<std::int32_t>& ci, std::vector<double>& vals, std::vector<double>& rhs) {
  const fem::QuadratureRule q = fem::quadrature_rule();
  vals.assign(ci.size(), 0.0);
  rhs.assign(rp.size() - 1, 0.0);
  for (const fem::Element& e : m.elements) {
    double la[9] = {0}, lb[3] = {0};
    for (int k = 0; k < q.size(); ++k) {
      std::array<double, 8> a{q.points[k][0], q.points[k][1]};
      for (int v = 0; v < 3; ++v) a[2 + 2 * v] = m.nodes[e.nodes[v]].x, a[3 + 2 * v] = m.nodes[e.nodes[v]].y;
      for (int t = 0; t < 9; ++t) la[t] += q.weights[k] * cf.bilinear[t].run(a);
      for (int t = 0; t < 3; ++t) lb[t] += q.weights[k] * cf.linear[t].run(a);
    }
    for (int i = 0; i < 3; ++i) {
      const int r = e.nodes[i];
      for (int j = 0; j < 3; ++j) {
        const auto b = ci.begin() + rp[r], end = ci.begin() + rp[r + 1];
        vals[std::lower_bound(b, end, e.nodes[j]) - ci.begin()] += la[i * 3 + j];
      }
      rhs[r] += lb[i];
    }
  }
}

double normwise(const std::vector<double>& got, const std::vector<double>& want) {
  double d = 0.0, s = 0.0;
  for (std::size_t i = 0; i < want.size(); ++i) d = std::max(d, std::abs(got[i] - want[i])), s = std::max(s, std::abs(want[i]));
  return d / (s > 0 ? s : 1.0);
}

}  // namespace

TEST_CASE("device facade: assemble() == the reference algorithm on the host (2D demo form, n=16)") {
  if (!have_gpu()) SKIP("no CUDA device");
  fem::Mesh m = meshgen::unit_square_mesh(16);
  fem::WeakForm wf = demo_weak_form();
  wf.space = fem::function_space(m, 1);
  device::CsrSystem gpu = device::assemble(wf, m);
  // sparsity: build_sparsity's std::set rows (device.cpp:66-88)
  std::vector<std::set<int>> rows(m.node_count());
  for (int i = 0; i < m.node_count(); ++i) rows[i].insert(i);
  for (const auto& e : m.elements)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) rows[e.nodes[a]].insert(e.nodes[b]);
  std::vector<std::int64_t> rp{0};
  std::vector<std::int32_t> ci;
  for (const auto& r : rows) {
    ci.insert(ci.end(), r.begin(), r.end());
    rp.push_back(static_cast<std::int64_t>(ci.size()));
  }
  CHECK(gpu.a.row_ptr == rp);
  CHECK(gpu.a.col_idx == ci);
  std::vector<double> vals, rhs;
  host_assemble(codegen::compile_form(fem::instantiate(wf)), m, rp, ci, vals, rhs);
  CHECK(normwise(gpu.a.values, vals) <= 1e-12);
  CHECK(normwise(gpu.b, rhs) <= 1e-12);
}

TEST_CASE("device facade: ELL view, launch limits and errors with the reference's types") {
  if (!have_gpu()) SKIP("no CUDA device");
  fem::Mesh m = meshgen::unit_square_mesh(8);
  fem::WeakForm wf = demo_weak_form();
  wf.space = fem::function_space(m, 1);
  device::CompiledKernel k(wf);
  auto d = device::flatten_mesh(m, 1);
  auto sp = device::build_sparsity(*d);
  device::EllSystem ell = device::assemble_sparse(k, *d, *sp);
  device::CsrSystem csr = device::assemble_csr(k, *d, *sp);
  CHECK(ell.a.n == sp->n && ell.a.max_nz == sp->max_nz);
  const auto rl = sp->row_len();
  for (int i = 0; i < ell.a.n; ++i)
    for (int s = 0; s < ell.a.max_nz; ++s) {
      const double v = ell.a.values[static_cast<std::size_t>(i) * ell.a.max_nz + s];
      CHECK(s < rl[i] ? v == csr.a.values[csr.a.row_ptr[i] + s] : v == 0.0);
    }
  device::LaunchConfig big;
  big.elems_per_block = 64;  // 3*9*64 > 1024 threads (device.cpp:90-97)
  CHECK_THROWS_AS(big.validate(), device::DeviceError);
  fem::Mesh bad = m;
  std::swap(bad.elements[4].nodes[1], bad.elements[4].nodes[2]);
  CHECK_THROWS_AS(device::flatten_mesh(bad, 1), fem::MeshError);
}

int main() { return ffcheck::run_all(); }

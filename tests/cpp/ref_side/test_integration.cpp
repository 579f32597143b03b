// tests/cpp/ref_side/test_integration.cpp -- the drop-in, compiled the way a
// reference maintainer would build it: the UNMODIFIED reference library
// (oracle/_ref/obj, from /root/reference/proj/src) + the binding of
// INTEGRATION.md §2 (device_b200.cpp) + libfemforge_b200.so.
//
// On the 2D n=64 unit-square mesh, for the reference's demo Helmholtz form
// (test_device.cpp:38-42) and for Poisson, the GPU overload
// assemble_sparse_b200(wf, mesh, sp) must return the same EllSystem as the
// reference's own assemble_sparse(CompiledEvaluator, flatten_mesh,
// build_sparsity, det mode) (device.hpp:143-153): identical ELL columns,
// values and RHS within 1e-12 normwise (acceptance.cpp:58-67). Exit 0 = pass.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>

#include "femforge/codegen/kernel.hpp"
#include "femforge/device/device.hpp"
#include "femforge/fem/fem.hpp"
#include "femforge/meshgen/meshgen.hpp"
#include "femforge/symbolic/expr.hpp"

namespace femforge::device {
EllSystem assemble_sparse_b200(const fem::WeakForm& wf, const fem::Mesh& mesh, const SparsityPattern& sp,
                               int device = 0);
}

using namespace femforge;

namespace {

double normwise(const std::vector<double>& got, const std::vector<double>& want) {
  double d = 0.0, s = 0.0;
  for (std::size_t i = 0; i < want.size(); ++i) {
    d = std::max(d, std::abs(got[i] - want[i]));
    s = std::max(s, std::abs(want[i]));
  }
  return d / (s > 0 ? s : 1.0);
}

bool check(const char* name, const fem::WeakForm& wf, const fem::Mesh& mesh) {
  const device::SparsityPattern sp = device::build_sparsity(mesh);
  const device::DeviceArrays arrays = device::flatten_mesh(mesh);
  const device::EllSystem ref =
      device::assemble_sparse(codegen::compile_form(fem::instantiate(wf)), arrays, sp, device::LaunchConfig{});
  const device::EllSystem gpu = device::assemble_sparse_b200(wf, mesh, sp);
  const bool cols = gpu.a.n == ref.a.n && gpu.a.max_nz == ref.a.max_nz && gpu.a.columns == ref.a.columns;
  const double ea = normwise(gpu.a.values, ref.a.values), eb = normwise(gpu.b, ref.b);
  const bool ok = cols && gpu.b.size() == ref.b.size() && ea <= 1e-12 && eb <= 1e-12;
  std::printf("%s: n=%d max_nz=%d columns %s, values err %.3e, rhs err %.3e -> %s\n", name, ref.a.n, ref.a.max_nz,
              cols ? "identical" : "DIFFER", ea, eb, ok ? "ok" : "FAIL");
  return ok;
}

}  // namespace

int main() {
  try {
    using symbolic::integer;
    using symbolic::sym;
    const fem::Mesh mesh = meshgen::unit_square_mesh(64);
    const symbolic::Expr x = sym("x"), y = sym("y");
    const symbolic::Expr f = symbolic::parse("-2*(x^2+y^2)+36");
    const fem::WeakForm demo = fem::helmholtz_form(fem::Mat2{integer(1), -x - y, x + y, integer(1)}, integer(1), f);
    const fem::WeakForm poisson = fem::helmholtz_form(fem::Mat2{integer(1), integer(0), integer(0), integer(1)},
                                                      integer(0), f);
    bool ok = check("demo Helmholtz", demo, mesh);
    ok = check("Poisson", poisson, mesh) && ok;
    std::printf(ok ? "integration ok\n" : "integration FAILED\n");
    return ok ? 0 : 1;
  } catch (const std::exception& e) {
    std::printf("integration error: %s\n", e.what());
    return 2;
  }
}

// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" driver around the UNMODIFIED reference library
// (/root/reference/proj/src, compiled by oracle/Makefile into oracle/_ref/).
// It is used (a) to generate the committed golden fixtures under tests/golden/
// and (b) as the CPU baseline arm of bench.py (`--impl reference`).
//
// 2D P1 (the only configuration the reference implements) runs the
// reference's own pipeline end to end:
//   fem::helmholtz_form / WeakForm{parse(...)}  (fem.cpp:99-107)
//   fem::instantiate                            (fem.cpp:122-158)
//   codegen::compile_form                       (kernel.cpp:277-283)
//   device::flatten_mesh / build_sparsity       (device.cpp:48-88)
//   device::assemble_sparse(CompiledEvaluator)  (device.cpp:265-305)
// and converts the ELL result to CSR (row_len prefix sum, linalg.hpp:26-42).
//
// 3D P1/P2 has no reference implementation. Here the harness
// drives the reference's own symbolic engine (symbolic::diff/substitute/mul,
// expr.cpp) and IR compiler/interpreter (codegen::lower, KernelProgram::run,
// kernel.cpp:22-46, 111-283) through a line-by-line 3D restatement of
// fem::instantiate (fem.cpp:122-158) and of the device loop
// (device.cpp:147-205 entry/quadrature order; device.cpp:265-305 binary
// search scatter; device.cpp:66-88 pattern rules).
#include <omp.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "femforge/codegen/kernel.hpp"
#include "femforge/device/device.hpp"
#include "femforge/fem/fem.hpp"
#include "femforge/linalg/linalg.hpp"
#include "femforge/symbolic/expr.hpp"

using namespace femforge;
using symbolic::Expr;

namespace {

thread_local std::string g_err;

struct QuadRule3 {
  std::vector<std::array<double, 3>> p;
  std::vector<double> w;
};

// Tet rules shared by convention with the product and the C oracle
// (SURVEY.md Appendix C).
QuadRule3 tet_rule(int id) {
  QuadRule3 r;
  auto add = [&](double a, double b, double c, double w) {
    r.p.push_back({a, b, c});
    r.w.push_back(w);
  };
  auto perm4 = [&](double a, double w) {  // (a,a,a) with 4th barycentric 1-3a
    double b = 1.0 - 3.0 * a;
    add(a, a, a, w);
    add(b, a, a, w);
    add(a, b, a, w);
    add(a, a, b, w);
  };
  auto perm6 = [&](double a, double w) {  // two barycentrics a, two 1/2-a
    double b = 0.5 - a;
    add(a, a, b, w);
    add(a, b, a, w);
    add(b, a, a, w);
    add(a, b, b, w);
    add(b, a, b, w);
    add(b, b, a, w);
  };
  switch (id) {
    case 1:
      add(0.25, 0.25, 0.25, 1.0 / 6.0);
      break;
    case 4: {
      const double a = 0.1381966011250105151795413165634361882280;  // (5-sqrt5)/20
      const double b = 0.5854101966249684544613760503096914353161;  // (5+3sqrt5)/20
      add(a, a, a, 1.0 / 24.0);
      add(b, a, a, 1.0 / 24.0);
      add(a, b, a, 1.0 / 24.0);
      add(a, a, b, 1.0 / 24.0);
      break;
    }
    case 11:
      add(0.25, 0.25, 0.25, -74.0 / 5625.0);
      perm4(1.0 / 14.0, 343.0 / 45000.0);
      perm6(0.1005964238332007950038978525383593769, 56.0 / 2250.0);
      break;
    case 14:
      perm4(0.09273525031089122640232391373703060, 0.01224884051939365825728503424772125);
      perm4(0.31088591926330060979734573376345783, 0.01878132095300264179986427538888106);
      perm6(0.04550370412564964949188052627933944, 0.00709100346284691107301157135337624);
      break;
    default:
      break;
  }
  return r;
}

struct Harness {
  int dim = 2, degree = 1, nloc = 3, nvert = 3;
  std::int64_t n_dofs = 0, n_elems = 0;
  // 2D reference objects
  fem::Mesh mesh2;
  std::unique_ptr<device::CompiledEvaluator> eval2;
  device::DeviceArrays arrays2;
  device::SparsityPattern sp2;
  // 3D restatement state
  std::vector<double> coords;      // [nv][3]
  std::vector<std::int32_t> vconn; // [ne][4]
  std::vector<std::int32_t> dconn; // [ne][nloc]
  std::vector<codegen::KernelProgram> bil, lin;
  QuadRule3 quad;
  std::vector<std::int64_t> row_ptr;
  std::vector<std::int32_t> col_idx;
  // CSR the scatter searches: the vectors above, or a caller-owned pattern
  // (ffref_create3_on_pattern: full-size meshes whose std::set build would
  // not fit the bench's time budget; the pattern is outside the timed
  // region, acceptance.cpp:295-296)
  const std::int64_t* rp = nullptr;
  const std::int32_t* ci = nullptr;
};

// fem.cpp:68-71 generalised: Lagrange basis on the reference tet; P2 local
// order is vertices 0-3 then edges (0,1),(0,2),(0,3),(1,2),(1,3),(2,3).
std::vector<Expr> tet_basis(int degree, const Expr& xi, const Expr& eta, const Expr& zeta) {
  Expr one = symbolic::integer(1);
  std::array<Expr, 4> l{one - xi - eta - zeta, xi, eta, zeta};
  std::vector<Expr> phi;
  if (degree == 1) {
    for (auto& e : l) phi.push_back(e);
    return phi;
  }
  for (int i = 0; i < 4; ++i) phi.push_back(l[i] * (symbolic::integer(2) * l[i] - one));
  const int edges[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  for (auto& ed : edges) phi.push_back(symbolic::integer(4) * l[ed[0]] * l[ed[1]]);
  return phi;
}

// 3D restatement of fem::instantiate (fem.cpp:122-158): u->phi_j, v->phi_i,
// grad -> J^{-T} grad_ref (cofactor/det), x -> affine map, times det J.
void instantiate3(Harness& h, const Expr& bilinear, const Expr& linear) {
  using symbolic::sym;
  Expr xi = sym("xi"), eta = sym("eta"), zeta = sym("zeta");
  Expr X[4][3];
  const char* cn[3] = {"x", "y", "z"};
  for (int v = 0; v < 4; ++v)
    for (int c = 0; c < 3; ++c) X[v][c] = sym(std::string(cn[c]) + std::to_string(v));
  Expr J[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) J[r][c] = X[c + 1][r] - X[0][r];
  Expr det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
             J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
             J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  // cofactor matrix C: J^{-T} = C / det
  Expr C[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      int r1 = (r + 1) % 3, r2 = (r + 2) % 3, c1 = (c + 1) % 3, c2 = (c + 2) % 3;
      C[r][c] = J[r1][c1] * J[r2][c2] - J[r1][c2] * J[r2][c1];
    }
  Expr xyz[3];
  for (int r = 0; r < 3; ++r) xyz[r] = X[0][r] + J[r][0] * xi + J[r][1] * eta + J[r][2] * zeta;
  std::vector<Expr> phi = tet_basis(h.degree, xi, eta, zeta);
  const int n = static_cast<int>(phi.size());
  std::vector<std::array<Expr, 3>> g(n);
  Expr ref[3] = {xi, eta, zeta};
  for (int i = 0; i < n; ++i) {
    Expr d[3];
    for (int c = 0; c < 3; ++c) d[c] = symbolic::diff(phi[i], ref[c]);
    for (int r = 0; r < 3; ++r) g[i][r] = (C[r][0] * d[0] + C[r][1] * d[1] + C[r][2] * d[2]) / det;
  }
  Expr u = sym("u"), v = sym("v");
  Expr ux = sym("u_x"), uy = sym("u_y"), uz = sym("u_z");
  Expr vx = sym("v_x"), vy = sym("v_y"), vz = sym("v_z");
  Expr sx = sym("x"), sy = sym("y"), sz = sym("z");
  symbolic::SymbolTable args;
  for (const char* a : {"xi", "eta", "zeta"}) args.add(a);
  for (int vtx = 0; vtx < 4; ++vtx)
    for (int c = 0; c < 3; ++c) args.add(std::string(cn[c]) + std::to_string(vtx));
  h.bil.clear();
  h.lin.clear();
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      Expr e = symbolic::substitute(
          bilinear, {{u, phi[j]}, {ux, g[j][0]}, {uy, g[j][1]}, {uz, g[j][2]}, {v, phi[i]},
                     {vx, g[i][0]}, {vy, g[i][1]}, {vz, g[i][2]}, {sx, xyz[0]}, {sy, xyz[1]},
                     {sz, xyz[2]}});
      h.bil.push_back(codegen::lower(e * det, args));
    }
    Expr l = symbolic::substitute(linear, {{v, phi[i]}, {sx, xyz[0]}, {sy, xyz[1]}, {sz, xyz[2]}});
    h.lin.push_back(codegen::lower(l * det, args));
  }
}

// device.cpp:66-88 restated on DOF connectivity: sorted, unique, diagonal
// always present.
void pattern3(Harness& h) {
  std::vector<std::set<int>> rows(h.n_dofs);
  for (std::int64_t i = 0; i < h.n_dofs; ++i) rows[i].insert(static_cast<int>(i));
  for (std::int64_t e = 0; e < h.n_elems; ++e) {
    const std::int32_t* d = &h.dconn[e * h.nloc];
    for (int a = 0; a < h.nloc; ++a)
      for (int b = 0; b < h.nloc; ++b) rows[d[a]].insert(d[b]);
  }
  h.row_ptr.assign(h.n_dofs + 1, 0);
  for (std::int64_t i = 0; i < h.n_dofs; ++i) h.row_ptr[i + 1] = h.row_ptr[i] + rows[i].size();
  h.col_idx.resize(h.row_ptr.back());
  for (std::int64_t i = 0; i < h.n_dofs; ++i) {
    std::int64_t k = h.row_ptr[i];
    for (int c : rows[i]) h.col_idx[k++] = c;
  }
}

inline std::int64_t find_slot(const Harness& h, int i, int j) {
  // binary search exactly as device.cpp:274-288
  std::int64_t lo = h.rp[i], hi = h.rp[i + 1];
  while (lo < hi) {
    std::int64_t mid = (lo + hi) / 2;
    if (h.ci[mid] < j)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo >= h.rp[i + 1] || h.ci[lo] != j) return -1;
  return lo;
}

// One element of the 3D device loop: IR-VM entries summed in ascending-q
// order (device.cpp:147-205), binary-search scatter (device.cpp:265-305),
// plain adds (det) or device::atomic_add (par, device.cpp:14-19).
void element3(const Harness& h, std::int64_t e, double* values, double* rhs, bool par) {
  thread_local std::vector<double> scratch;
  const int nq = static_cast<int>(h.quad.w.size());
  const int n = h.nloc;
  const std::int32_t* vc = &h.vconn[4 * e];
  const std::int32_t* dc = &h.dconn[n * e];
  std::array<double, 15> a{};
  for (int v = 0; v < 4; ++v)
    for (int c = 0; c < 3; ++c) a[3 + 3 * v + c] = h.coords[3 * vc[v] + c];
  double jm[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) jm[r][c] = a[3 + 3 * (c + 1) + r] - a[3 + r];
  double det = jm[0][0] * (jm[1][1] * jm[2][2] - jm[1][2] * jm[2][1]) -
               jm[0][1] * (jm[1][0] * jm[2][2] - jm[1][2] * jm[2][0]) +
               jm[0][2] * (jm[1][0] * jm[2][1] - jm[1][1] * jm[2][0]);
  if (std::abs(det) <= 1e-14)  // device.cpp:128, 180-186
    throw std::runtime_error("degenerate element " + std::to_string(e) + " (|det J| <= 1e-14)");
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int q = 0; q < nq; ++q) {
        a[0] = h.quad.p[q][0];
        a[1] = h.quad.p[q][1];
        a[2] = h.quad.p[q][2];
        acc += h.quad.w[q] * h.bil[i * n + j].run(a, scratch);
      }
      std::int64_t s = find_slot(h, dc[i], dc[j]);
      if (s < 0)
        throw std::runtime_error("column " + std::to_string(dc[j]) + " not present in sparsity row " +
                                 std::to_string(dc[i]));
      if (par)
        device::atomic_add(values[s], acc);
      else
        values[s] += acc;
    }
    double acc = 0.0;
    for (int q = 0; q < nq; ++q) {
      a[0] = h.quad.p[q][0];
      a[1] = h.quad.p[q][1];
      a[2] = h.quad.p[q][2];
      acc += h.quad.w[q] * h.lin[i].run(a, scratch);
    }
    if (par)
      device::atomic_add(rhs[dc[i]], acc);
    else
      rhs[dc[i]] += acc;
  }
}

// Elements first, first+stride, ... (count of them) of the 3D loop: in order
// (det mode) or OpenMP dynamic chunks with atomic adds (par mode).
void run3(const Harness& h, std::int64_t first, std::int64_t stride, std::int64_t count, double* values, double* rhs,
          int workers) {
  const bool par = workers > 1;
  if (!par) {
    for (std::int64_t i = 0; i < count; ++i) element3(h, first + i * stride, values, rhs, false);
    return;
  }
  std::string err;
#pragma omp parallel for schedule(dynamic, 64) num_threads(workers)
  for (std::int64_t i = 0; i < count; ++i) {
    try {
      element3(h, first + i * stride, values, rhs, true);
    } catch (const std::exception& ex) {
#pragma omp critical(ffref_err)
      if (err.empty()) err = ex.what();
    }
  }
  if (!err.empty()) throw std::runtime_error(err);
}

Harness* create(int dim, int degree, const double* coords, std::int64_t nv, const std::int32_t* vconn,
                const std::int32_t* dconn, std::int64_t ne, std::int64_t n_dofs, const char* bilinear,
                const char* linear, int quad_id, const std::int64_t* ext_row_ptr, const std::int32_t* ext_col_idx) {
  try {
    auto h = std::make_unique<Harness>();
    h->dim = dim;
    h->degree = degree;
    h->n_elems = ne;
    h->n_dofs = n_dofs;
    Expr bl = symbolic::parse(bilinear);
    Expr li = symbolic::parse(linear);
    if (dim == 2) {
      if (degree != 1) throw std::runtime_error("reference supports 2D P1 only");
      h->nloc = 3;
      h->mesh2.nodes.resize(nv);
      for (std::int64_t k = 0; k < nv; ++k) h->mesh2.nodes[k] = {coords[2 * k], coords[2 * k + 1]};
      h->mesh2.elements.resize(ne);
      for (std::int64_t e = 0; e < ne; ++e)
        h->mesh2.elements[e].nodes = {vconn[3 * e], vconn[3 * e + 1], vconn[3 * e + 2]};
      fem::WeakForm wf;
      wf.bilinear = bl;
      wf.linear = li;
      fem::InstantiatedForm inst = fem::instantiate(wf);
      h->eval2 = std::make_unique<device::CompiledEvaluator>(codegen::compile_form(inst));
      h->arrays2 = device::flatten_mesh(h->mesh2);
      h->sp2 = device::build_sparsity(h->mesh2);
      // ELL -> CSR (lossless re-index)
      h->row_ptr.assign(h->sp2.n + 1, 0);
      for (int i = 0; i < h->sp2.n; ++i) h->row_ptr[i + 1] = h->row_ptr[i] + h->sp2.row_len[i];
      h->col_idx.resize(h->row_ptr.back());
      for (int i = 0; i < h->sp2.n; ++i)
        for (int k = 0; k < h->sp2.row_len[i]; ++k)
          h->col_idx[h->row_ptr[i] + k] = h->sp2.row_cols[static_cast<std::size_t>(i) * h->sp2.max_nz + k];
      h->rp = h->row_ptr.data();
      h->ci = h->col_idx.data();
      return h.release();
    }
    if (dim != 3 || (degree != 1 && degree != 2)) throw std::runtime_error("unsupported dim/degree");
    h->nloc = degree == 1 ? 4 : 10;
    h->coords.assign(coords, coords + 3 * nv);
    h->vconn.assign(vconn, vconn + 4 * ne);
    h->dconn.assign(dconn, dconn + h->nloc * ne);
    h->quad = tet_rule(quad_id);
    if (h->quad.w.empty()) throw std::runtime_error("unknown tet rule");
    instantiate3(*h, bl, li);
    if (ext_row_ptr) {  // caller-owned pattern (ffref_create3_on_pattern)
      h->rp = ext_row_ptr;
      h->ci = ext_col_idx;
      h->row_ptr.assign(1, ext_row_ptr[n_dofs]);  // ffref_nnz
      return h.release();
    }
    pattern3(*h);
    h->rp = h->row_ptr.data();
    h->ci = h->col_idx.data();
    return h.release();
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return nullptr;
  }
}

}  // namespace

extern "C" {

const char* ffref_last_error() { return g_err.c_str(); }

// Create a harness. coords: [nv][dim]; vconn: [ne][dim+1]; dconn: [ne][nloc]
// (for P1, dconn == vconn). bilinear/linear: weak-form text over the reserved
// symbols (u, u_x, u_y[, u_z], v, v_x, v_y[, v_z], x, y[, z]).
// quad_id: 3D rule id (1, 4, 11, 14); ignored in 2D (reference rule, fem.cpp:43-48).
void* ffref_create(int dim, int degree, const double* coords, std::int64_t nv,
                   const std::int32_t* vconn, const std::int32_t* dconn, std::int64_t ne,
                   std::int64_t n_dofs, const char* bilinear, const char* linear, int quad_id) {
  return create(dim, degree, coords, nv, vconn, dconn, ne, n_dofs, bilinear, linear, quad_id, nullptr, nullptr);
}


// 3D harness over a caller-owned CSR (row_ptr [n_dofs+1], col_idx; must stay
// alive with the harness): full-size meshes (Kuhn 128^3 P2: 485M nnz) whose
// std::set pattern build (pattern3) would take minutes and tens of GB. The
// pattern is built outside the timed region either way (acceptance.cpp:295-296).
void* ffref_create3_on_pattern(int degree, const double* coords, std::int64_t nv, const std::int32_t* vconn,
                               const std::int32_t* dconn, std::int64_t ne, std::int64_t n_dofs,
                               const char* bilinear, const char* linear, int quad_id,
                               const std::int64_t* row_ptr, const std::int32_t* col_idx) {
  if (!row_ptr || !col_idx) {
    g_err = "ffref_create3_on_pattern: null pattern";
    return nullptr;
  }
  return create(3, degree, coords, nv, vconn, dconn, ne, n_dofs, bilinear, linear, quad_id, row_ptr, col_idx);
}

// Timing sample of the 3D parallel loop: elements first, first+stride, ...
// (count of them), accumulated into values/rhs WITHOUT the zero fill (the
// caller zeroes once). Used by bench.py's reference arm on the full mesh:
// the stride spreads the sample over the whole CSR, like the full pass.
int ffref_assemble_sample(void* p, int workers, std::int64_t first, std::int64_t stride, std::int64_t count,
                          double* values, double* rhs) {
  auto* h = static_cast<Harness*>(p);
  try {
    if (h->dim != 3) throw std::runtime_error("ffref_assemble_sample: 3D harness only");
    if (first < 0 || stride < 1 || count < 0 || (count > 0 && first + (count - 1) * stride >= h->n_elems))
      throw std::runtime_error("ffref_assemble_sample: element range outside the mesh");
    run3(*h, first, stride, count, values, rhs, workers);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

void ffref_destroy(void* p) { delete static_cast<Harness*>(p); }

std::int64_t ffref_nnz(void* p) { return static_cast<Harness*>(p)->row_ptr.back(); }

void ffref_pattern(void* p, std::int64_t* row_ptr, std::int32_t* col_idx) {
  auto* h = static_cast<Harness*>(p);
  std::memcpy(row_ptr, h->row_ptr.data(), h->row_ptr.size() * sizeof(std::int64_t));
  std::memcpy(col_idx, h->col_idx.data(), h->col_idx.size() * sizeof(std::int32_t));
}

// Numeric assembly. workers <= 1: deterministic mode (fixed order); otherwise
// the reference's parallel mode (2D: device.cpp:222-237 via LaunchConfig;
// 3D: OpenMP over elements + device::atomic_add, device.cpp:14-19).
// elem_limit > 0 assembles only the first elem_limit elements (bounded CPU
// baseline samples). Returns 0 on success, -1 on error (message in
// ffref_last_error).
int ffref_assemble(void* p, int workers, std::int64_t elem_limit, double* values, double* rhs) {
  auto* h = static_cast<Harness*>(p);
  try {
    const std::int64_t nnz = h->row_ptr.back();
    if (h->dim == 2) {
      device::LaunchConfig cfg;
      if (workers > 1) {
        cfg.mode = device::ExecMode::Parallel;
        cfg.workers = workers;
      }
      device::DeviceArrays arr = h->arrays2;
      if (elem_limit > 0 && elem_limit < h->n_elems) {
        arr.x.resize(3 * elem_limit);
        arr.y.resize(3 * elem_limit);
        arr.g_idx.resize(3 * elem_limit);
      }
      device::EllSystem sys = device::assemble_sparse(*h->eval2, arr, h->sp2, cfg);
      for (int i = 0; i < h->sp2.n; ++i) {
        for (int k = 0; k < h->sp2.row_len[i]; ++k)
          values[h->row_ptr[i] + k] = sys.a.values[static_cast<std::size_t>(i) * h->sp2.max_nz + k];
        rhs[i] = sys.b[i];
      }
      return 0;
    }
    std::fill(values, values + nnz, 0.0);
    std::fill(rhs, rhs + h->n_dofs, 0.0);
    const std::int64_t ne = elem_limit > 0 ? std::min(elem_limit, h->n_elems) : h->n_elems;
    run3(*h, 0, 1, ne, values, rhs, workers);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// Reference emit_source for the demo form (kernel.cpp:409-449); used to pin
// the golden file through this build.
int ffref_emit_demo_source(char* buf, std::int64_t cap) {
  using symbolic::integer;
  using symbolic::sym;
  Expr x = sym("x"), y = sym("y");
  fem::Mat2 sigma{integer(1), -x - y, x + y, integer(1)};
  auto form = fem::instantiate(fem::helmholtz_form(sigma, integer(1), symbolic::parse("-2*(x^2+y^2)+36")));
  std::string s = codegen::emit_source(form, codegen::LaunchParams{});
  if (static_cast<std::int64_t>(s.size()) + 1 > cap) return -static_cast<int>(s.size() + 1);
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

int ffref_max_threads() { return omp_get_max_threads(); }

#ifndef FFREF_FLAGS
#define FFREF_FLAGS "unknown"
#endif
// Compiler and flags the reference library was built with (bench.py prints
// them with the CPU baseline).
const char* ffref_build_info() { return "g++ " __VERSION__ " " FFREF_FLAGS; }

// The reference's own export (linalg::export_matrix(EllMatrix) / export_vector,
// linalg.cpp:148-210) of a 2D system given as CSR values over the harness's
// pattern. fmt 0: MatrixMarket, 1: CSV. Returns 0 / -1.
int ffref_export(void* p, const double* values, const double* rhs, const char* mpath, const char* vpath, int fmt) {
  auto* h = static_cast<Harness*>(p);
  try {
    if (h->dim != 2) throw std::runtime_error("export parity uses the 2D reference pipeline");
    linalg::EllMatrix a(h->sp2.n, h->sp2.max_nz);
    a.columns = h->sp2.row_cols;
    for (int i = 0; i < h->sp2.n; ++i)
      for (int k = 0; k < h->sp2.row_len[i]; ++k)
        a.values[static_cast<std::size_t>(i) * h->sp2.max_nz + k] = values[h->row_ptr[i] + k];
    const auto f = fmt == 0 ? linalg::ExportFormat::MatrixMarket : linalg::ExportFormat::Csv;
    linalg::export_matrix(a, mpath, f);
    linalg::export_vector(linalg::Vector(rhs, rhs + h->sp2.n), vpath, f);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// The reference's cg_solve (linalg.cpp:61-96) on the same 2D system.
int ffref_cg(void* p, const double* values, const double* rhs, double tol, int max_iter, double* x, int* iters,
             double* residual) {
  auto* h = static_cast<Harness*>(p);
  try {
    linalg::EllMatrix a(h->sp2.n, h->sp2.max_nz);
    a.columns = h->sp2.row_cols;
    for (int i = 0; i < h->sp2.n; ++i)
      for (int k = 0; k < h->sp2.row_len[i]; ++k)
        a.values[static_cast<std::size_t>(i) * h->sp2.max_nz + k] = values[h->row_ptr[i] + k];
    linalg::CgResult r = linalg::cg_solve(a, linalg::Vector(rhs, rhs + h->sp2.n), tol, max_iter);
    std::memcpy(x, r.x.data(), r.x.size() * sizeof(double));
    *iters = r.iterations;
    *residual = r.residual;
    return r.converged ? 0 : 1;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

}  // extern "C"

// femforge-b200 fem layer: meshes, Lagrange spaces, quadrature, weak forms
// and their instantiation into per-entry element integrands.
//
// API parity with /root/reference/proj/include/femforge/fem/fem.hpp:10-114
// (Mesh, FunctionSpace, FormSymbols, WeakForm, QuadratureRule,
// quadrature_rule, kernel_args, reference_shape_functions, affine_map,
// InstantiatedForm, instantiate, grad/dot/matvec, helmholtz_form), generalised
// from 2D P1 triangles to {2D,3D} x {P1,P2} (BASELINE.json configs 1-4).
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "femforge/symbolic.hpp"

namespace femforge::fem {

using symbolic::Expr;

struct Point {
  double x = 0.0;
  double y = 0.0;
  double z = 0.0;  // unused in 2D
};

// Simplex: 3 nodes (triangle) or 4 nodes (tetrahedron, last slot used).
struct Element {
  std::array<int, 4> nodes{};
};

class MeshError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// Simplicial mesh with positively oriented elements (fem.hpp:27-39).
struct Mesh {
  int dim = 2;
  std::vector<Point> nodes;
  std::vector<Element> elements;

  int node_count() const { return static_cast<int>(nodes.size()); }
  int element_count() const { return static_cast<int>(elements.size()); }
  int nodes_per_element() const { return dim + 1; }

  double signed_area(int element) const;    // 2D (fem.cpp:9-15)
  double signed_volume(int element) const;  // 3D
  // Throws MeshError on out-of-range indices, duplicate nodes within an
  // element, or non-positive measure (fem.cpp:17-34).
  void validate() const;

  // Flat views used at the C-ABI: coords [nv][dim], connectivity [ne][dim+1].
  std::vector<double> coords_flat() const;
  std::vector<std::int32_t> conn_flat() const;
};

// Element -> global DOF map of a scalar Lagrange space.
struct DofMap {
  int n_local = 3;
  std::int64_t n_dofs = 0;
  std::vector<std::int32_t> dofs;  // [ne][n_local]
};

struct FunctionSpace {
  const Mesh* mesh = nullptr;
  Expr x, y, z;  // coordinate symbols
  std::string family = "Lagrange";
  int degree = 1;
  int n_local = 3;
  int dim = 0;    // 0: taken from mesh (or 2 when there is no mesh)
  DofMap dofmap;  // empty -> built on demand by lagrange_dofs()
};

// P1: DOFs are mesh nodes. P2: nodes first, then edges numbered in
// ascending (min,max) order; local order vertices, then edges
// (0,1),(0,2),(0,3),(1,2),(1,3),(2,3) [(0,1),(0,2),(1,2) in 2D].
DofMap lagrange_dofs(const Mesh& m, int degree);
FunctionSpace function_space(const Mesh& m, int degree);
int local_dofs(int dim, int degree);

// Reserved symbols (fem.hpp:49-55, extended by z, u_z, v_z).
struct FormSymbols {
  Expr u, u_x, u_y, u_z;
  Expr v, v_x, v_y, v_z;
  Expr x, y, z;
};
const FormSymbols& form_symbols();

struct WeakForm {
  Expr bilinear;  // over {u, u_x, u_y, u_z, v, v_x, v_y, v_z, x, y, z}
  Expr linear;    // over {v, x, y, z}
  FunctionSpace space;
};

class FormError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct QuadratureRule {
  int dim = 2;
  std::vector<std::array<double, 3>> points;  // reference coordinates
  std::vector<double> weights;
  int id = 3;
  int size() const { return static_cast<int>(points.size()); }
};

// The reference's 3-point rule exact for total degree <= 2 (fem.cpp:43-48).
QuadratureRule quadrature_rule();
// dim 2: id 1 (centroid) or 3 (reference rule); dim 3: id 1, 4, 11, 14
// (SURVEY.md Appendix C). Throws FormError for unknown rules.
QuadratureRule quadrature_rule(int dim, int id);

// Kernel argument slots of the reference semantics: (xi, eta, x0, y0, x1, y1,
// x2, y2) in 2D (fem.cpp:50-57); (xi, eta, zeta, x0, y0, z0, ..., x3, y3, z3)
// in 3D.
constexpr int kNumKernelArgs = 8;
const symbolic::SymbolTable& kernel_args();
const symbolic::SymbolTable& kernel_args(int dim);
const Expr& arg_xi();
const Expr& arg_eta();
const Expr& arg_zeta();

// Lagrange basis on the reference simplex (fem.cpp:68-71 generalised).
std::vector<Expr> reference_shape_functions(int dim, int degree);
std::array<Expr, 3> reference_shape_functions();  // 2D P1, reference API

struct AffineMap {
  Expr x, y;
  Expr j00, j01, j10, j11;
  Expr det;
};
AffineMap affine_map();  // 2D, fem.cpp:73-87

// Per-entry integrands, det J included, weight applied at evaluation
// (fem.hpp:92-98). `bilinear`/`linear` follow the reference semantics
// (entries over kernel_args(dim)). `geo_bilinear`/`geo_linear` are the same
// integrands over the reference coordinates and the per-element geometry
// symbols (see geometry_symbols()); they are what the GPU code generator
// consumes.
struct InstantiatedForm {
  int dim = 2;
  int degree = 1;
  int n_local = 3;  // DOFs per element (ncomp x scalar DOFs for vector spaces)
  int ncomp = 1;    // components of a vector space; local DOF index = a * ncomp + c
  std::vector<Expr> bilinear;  // n_local x n_local, row-major (test i, trial j)
  std::vector<Expr> linear;    // n_local
  std::vector<Expr> geo_bilinear;
  std::vector<Expr> geo_linear;
  // scalar forms: the weak form itself (over u, u_x.., v, v_x.., x, y, z),
  // for the per-point bilinear planner; null for blocked forms
  Expr form_bilinear, form_linear;
};

// Geometry symbols of the GPU element prologue: gJrc (Jacobian dx_r/dxi_c),
// gdet (det J), gGrc (J^{-T}), gXr (vertex 0 coordinates).
struct GeometrySymbols {
  Expr J[3][3];
  Expr G[3][3];
  Expr det;
  Expr X[3];
};
const GeometrySymbols& geometry_symbols();

InstantiatedForm instantiate(const WeakForm& wf);

// Vector-valued (ncomp-component) Lagrange forms as blocks of scalar forms:
// a(u, v) = sum_{c,d} a_cd(u_d, v_c), l(v) = sum_c l_c(v_c), each block a
// scalar WeakForm over the reserved symbols (u*, v* = the scalar basis of
// the trial / test component). blocks is row-major [c][d] (ncomp^2 forms;
// their `linear` parts are ignored), linear has ncomp forms (their `bilinear`
// parts are ignored). The result has node-major local DOFs a * ncomp + c and
// global DOFs ncomp * node + c (3x3 blocks for elasticity, BASELINE config 5).
InstantiatedForm instantiate_blocked(const std::vector<WeakForm>& blocks, const std::vector<WeakForm>& linear,
                                     int ncomp);

// Isotropic linear elasticity, lambda div u div v + mu sum_cd d_d u_c (d_d v_c
// + d_c v_d), body force f: the block forms for instantiate_blocked.
void elasticity_blocks(int dim, const Expr& lambda, const Expr& mu, const std::vector<Expr>& f,
                       std::vector<WeakForm>& blocks, std::vector<WeakForm>& linear);

using Vec2 = std::array<Expr, 2>;
using Mat2 = std::array<Expr, 4>;
using Vec3 = std::array<Expr, 3>;
using Mat3 = std::array<Expr, 9>;

Vec2 grad(const Expr& e, const Expr& x, const Expr& y);
Vec3 grad(const Expr& e, const Expr& x, const Expr& y, const Expr& z);
Expr dot(const Vec2& a, const Vec2& b);
Expr dot(const Vec3& a, const Vec3& b);
Vec2 matvec(const Mat2& m, const Vec2& v);
Vec3 matvec(const Mat3& m, const Vec3& v);

// (grad v, sigma grad u) + lambda (v, u) = (v, f)  (fem.cpp:99-107)
WeakForm helmholtz_form(const Mat2& sigma, const Expr& lambda, const Expr& f);
WeakForm helmholtz_form(const Mat3& sigma, const Expr& lambda, const Expr& f);
// 3D with convection: + (beta . grad u) v   (BASELINE.json config 4)
WeakForm convection_form(const Mat3& sigma, const Expr& lambda, const Vec3& beta, const Expr& f);

}  // namespace femforge::fem

// femforge-b200 fem layer (see fem.hpp).
#include "femforge/fem.hpp"

#include <algorithm>
#include <cmath>
#include <set>
#include <utility>

namespace femforge::fem {

using namespace symbolic;

// ---------------------------------------------------------------------------
// meshes (fem.cpp:9-34 generalised to tetrahedra)

double Mesh::signed_area(int k) const {
  const auto& e = elements[k].nodes;
  const Point &a = nodes[e[0]], &b = nodes[e[1]], &c = nodes[e[2]];
  return 0.5 * ((b.x - a.x) * (c.y - a.y) - (c.x - a.x) * (b.y - a.y));
}

double Mesh::signed_volume(int k) const {
  const auto& e = elements[k].nodes;
  const Point& o = nodes[e[0]];
  double m[3][3];
  for (int v = 0; v < 3; ++v) {
    const Point& p = nodes[e[v + 1]];
    m[0][v] = p.x - o.x;
    m[1][v] = p.y - o.y;
    m[2][v] = p.z - o.z;
  }
  const double det = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                     m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                     m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
  return det / 6.0;
}

void Mesh::validate() const {
  if (dim != 2 && dim != 3) throw MeshError("mesh dimension must be 2 or 3");
  const int n = node_count();
  const int k = nodes_per_element();
  for (int t = 0; t < element_count(); ++t) {
    const auto& e = elements[t].nodes;
    for (int a = 0; a < k; ++a)
      if (e[a] < 0 || e[a] >= n)
        throw MeshError("element " + std::to_string(t) + ": node index " + std::to_string(e[a]) + " out of range");
    for (int a = 0; a < k; ++a)
      for (int b = a + 1; b < k; ++b)
        if (e[a] == e[b]) throw MeshError("element " + std::to_string(t) + ": duplicate node indices");
    const double meas = dim == 2 ? signed_area(t) : signed_volume(t);
    if (meas <= 0.0)
      throw MeshError("element " + std::to_string(t) + (dim == 2 ? ": non-positive signed area" : ": non-positive signed volume"));
  }
}

std::vector<double> Mesh::coords_flat() const {
  std::vector<double> c;
  c.reserve(nodes.size() * dim);
  for (const Point& p : nodes) {
    c.push_back(p.x);
    c.push_back(p.y);
    if (dim == 3) c.push_back(p.z);
  }
  return c;
}

std::vector<std::int32_t> Mesh::conn_flat() const {
  std::vector<std::int32_t> c;
  const int k = nodes_per_element();
  c.reserve(elements.size() * k);
  for (const Element& e : elements)
    for (int a = 0; a < k; ++a) c.push_back(e.nodes[a]);
  return c;
}

int local_dofs(int dim, int degree) {
  if (degree == 1) return dim + 1;
  if (degree == 2) return dim == 2 ? 6 : 10;
  throw FormError("only Lagrange degree 1 and 2 are supported");
}

namespace {

const int kEdges3[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
const int kEdges2[3][2] = {{0, 1}, {0, 2}, {1, 2}};

}  // namespace

DofMap lagrange_dofs(const Mesh& m, int degree) {
  DofMap d;
  d.n_local = local_dofs(m.dim, degree);
  const int nv = m.nodes_per_element();
  const std::int64_t ne = m.element_count();
  d.dofs.resize(ne * d.n_local);
  if (degree == 1) {
    for (std::int64_t e = 0; e < ne; ++e)
      for (int a = 0; a < nv; ++a) d.dofs[e * nv + a] = m.elements[e].nodes[a];
    d.n_dofs = m.node_count();
    return d;
  }
  const int n_edges = m.dim == 3 ? 6 : 3;
  const auto& edges = m.dim == 3 ? kEdges3 : kEdges2;
  std::vector<std::pair<int, int>> all;
  all.reserve(ne * n_edges);
  for (std::int64_t e = 0; e < ne; ++e)
    for (int q = 0; q < n_edges; ++q) {
      int a = m.elements[e].nodes[edges[q][0]], b = m.elements[e].nodes[edges[q][1]];
      all.emplace_back(std::min(a, b), std::max(a, b));
    }
  std::vector<std::pair<int, int>> uniq = all;
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  for (std::int64_t e = 0; e < ne; ++e) {
    for (int a = 0; a < nv; ++a) d.dofs[e * d.n_local + a] = m.elements[e].nodes[a];
    for (int q = 0; q < n_edges; ++q) {
      auto it = std::lower_bound(uniq.begin(), uniq.end(), all[e * n_edges + q]);
      d.dofs[e * d.n_local + nv + q] = m.node_count() + static_cast<int>(it - uniq.begin());
    }
  }
  d.n_dofs = m.node_count() + static_cast<std::int64_t>(uniq.size());
  return d;
}

FunctionSpace function_space(const Mesh& m, int degree) {
  FunctionSpace s;
  s.mesh = &m;
  s.x = sym("x");
  s.y = sym("y");
  s.z = sym("z");
  s.degree = degree;
  s.dim = m.dim;
  s.n_local = local_dofs(m.dim, degree);
  s.dofmap = lagrange_dofs(m, degree);
  return s;
}

const FormSymbols& form_symbols() {
  static const FormSymbols fs{sym("u"), sym("u_x"), sym("u_y"), sym("u_z"), sym("v"), sym("v_x"),
                              sym("v_y"), sym("v_z"), sym("x"), sym("y"), sym("z")};
  return fs;
}

// ---------------------------------------------------------------------------
// quadrature

QuadratureRule quadrature_rule() { return quadrature_rule(2, 3); }

QuadratureRule quadrature_rule(int dim, int id) {
  QuadratureRule r;
  r.dim = dim;
  r.id = id;
  auto put = [&](double a, double b, double c, double w) {
    r.points.push_back({a, b, c});
    r.weights.push_back(w);
  };
  if (dim == 2) {
    if (id == 3) {  // fem.cpp:45-46
      put(1.0 / 6.0, 1.0 / 6.0, 0, 1.0 / 6.0);
      put(2.0 / 3.0, 1.0 / 6.0, 0, 1.0 / 6.0);
      put(1.0 / 6.0, 2.0 / 3.0, 0, 1.0 / 6.0);
    } else if (id == 1) {
      put(1.0 / 3.0, 1.0 / 3.0, 0, 0.5);
    } else {
      throw FormError("unknown triangle quadrature rule " + std::to_string(id));
    }
    return r;
  }
  // Tet rules; constants derived at 40 digits by
  // tools/quad_rules.py. Orbits: (a,a,a) over 4 vertices, (a,a,1/2-a,1/2-a)
  // over 6 edges.
  auto orbit4 = [&](double a, double w) {
    const double t = 1.0 - 3.0 * a;
    put(a, a, a, w);
    put(t, a, a, w);
    put(a, t, a, w);
    put(a, a, t, w);
  };
  auto orbit6 = [&](double a, double w) {
    const double t = 0.5 - a;
    put(a, a, t, w);
    put(a, t, a, w);
    put(t, a, a, w);
    put(a, t, t, w);
    put(t, a, t, w);
    put(t, t, a, w);
  };
  switch (id) {
    case 1:
      put(0.25, 0.25, 0.25, 1.0 / 6.0);
      break;
    case 4: {  // degree 2: a = (5-sqrt5)/20, b = (5+3sqrt5)/20, w = 1/24
      const double a = 0.1381966011250105151795413165634361882280;
      const double b = 0.5854101966249684544613760503096914353161;
      put(a, a, a, 1.0 / 24.0);
      put(b, a, a, 1.0 / 24.0);
      put(a, b, a, 1.0 / 24.0);
      put(a, a, b, 1.0 / 24.0);
      break;
    }
    case 11:  // Keast degree 4 (one negative weight)
      put(0.25, 0.25, 0.25, -74.0 / 5625.0);
      orbit4(1.0 / 14.0, 343.0 / 45000.0);
      orbit6(0.1005964238332007950038978525383593769, 56.0 / 2250.0);
      break;
    case 14:  // positive degree 5
      orbit4(0.09273525031089122640232391373703060, 0.01224884051939365825728503424772125);
      orbit4(0.31088591926330060979734573376345783, 0.01878132095300264179986427538888106);
      orbit6(0.04550370412564964949188052627933944, 0.00709100346284691107301157135337624);
      break;
    default:
      throw FormError("unknown tetrahedron quadrature rule " + std::to_string(id));
  }
  return r;
}

// ---------------------------------------------------------------------------
// reference element

const SymbolTable& kernel_args() { return kernel_args(2); }

const SymbolTable& kernel_args(int dim) {
  static const SymbolTable t2 = [] {
    SymbolTable t;
    for (const char* n : {"xi", "eta", "x0", "y0", "x1", "y1", "x2", "y2"}) t.add(n);
    return t;
  }();
  static const SymbolTable t3 = [] {
    SymbolTable t;
    for (const char* n : {"xi", "eta", "zeta"}) t.add(n);
    for (int v = 0; v < 4; ++v)
      for (const char* c : {"x", "y", "z"}) t.add(std::string(c) + std::to_string(v));
    return t;
  }();
  if (dim == 3) return t3;
  return t2;
}

const Expr& arg_xi() {
  static const Expr e = sym("xi");
  return e;
}
const Expr& arg_eta() {
  static const Expr e = sym("eta");
  return e;
}
const Expr& arg_zeta() {
  static const Expr e = sym("zeta");
  return e;
}

std::vector<Expr> reference_shape_functions(int dim, int degree) {
  const Expr one = integer(1);
  std::vector<Expr> lam;  // barycentric coordinates
  if (dim == 2) {
    lam = {one - arg_xi() - arg_eta(), arg_xi(), arg_eta()};
  } else {
    lam = {one - arg_xi() - arg_eta() - arg_zeta(), arg_xi(), arg_eta(), arg_zeta()};
  }
  if (degree == 1) return lam;
  if (degree != 2) throw FormError("only Lagrange degree 1 and 2 are supported");
  std::vector<Expr> phi;
  for (const Expr& l : lam) phi.push_back(l * (integer(2) * l - one));
  const int n_edges = dim == 3 ? 6 : 3;
  for (int q = 0; q < n_edges; ++q) {
    const int a = dim == 3 ? kEdges3[q][0] : kEdges2[q][0];
    const int b = dim == 3 ? kEdges3[q][1] : kEdges2[q][1];
    phi.push_back(integer(4) * lam[a] * lam[b]);
  }
  return phi;
}

std::array<Expr, 3> reference_shape_functions() {
  auto v = reference_shape_functions(2, 1);
  return {v[0], v[1], v[2]};
}

AffineMap affine_map() {
  const Expr xi = arg_xi(), eta = arg_eta();
  const Expr x0 = sym("x0"), y0 = sym("y0"), x1 = sym("x1"), y1 = sym("y1"), x2 = sym("x2"), y2 = sym("y2");
  AffineMap m;
  m.j00 = x1 - x0;
  m.j01 = x2 - x0;
  m.j10 = y1 - y0;
  m.j11 = y2 - y0;
  m.x = x0 + m.j00 * xi + m.j01 * eta;
  m.y = y0 + m.j10 * xi + m.j11 * eta;
  m.det = m.j00 * m.j11 - m.j01 * m.j10;
  return m;
}

const GeometrySymbols& geometry_symbols() {
  static const GeometrySymbols g = [] {
    GeometrySymbols s;
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) {
        s.J[r][c] = sym("gJ" + std::to_string(r) + std::to_string(c));
        s.G[r][c] = sym("gG" + std::to_string(r) + std::to_string(c));
      }
      s.X[r] = sym("gX" + std::to_string(r));
    }
    s.det = sym("gdet");
    return s;
  }();
  return g;
}

// ---------------------------------------------------------------------------
// weak forms

Vec2 grad(const Expr& e, const Expr& x, const Expr& y) { return {diff(e, x), diff(e, y)}; }
Vec3 grad(const Expr& e, const Expr& x, const Expr& y, const Expr& z) { return {diff(e, x), diff(e, y), diff(e, z)}; }
Expr dot(const Vec2& a, const Vec2& b) { return a[0] * b[0] + a[1] * b[1]; }
Expr dot(const Vec3& a, const Vec3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
Vec2 matvec(const Mat2& m, const Vec2& v) { return {m[0] * v[0] + m[1] * v[1], m[2] * v[0] + m[3] * v[1]}; }
Vec3 matvec(const Mat3& m, const Vec3& v) {
  return {m[0] * v[0] + m[1] * v[1] + m[2] * v[2], m[3] * v[0] + m[4] * v[1] + m[5] * v[2],
          m[6] * v[0] + m[7] * v[1] + m[8] * v[2]};
}

WeakForm helmholtz_form(const Mat2& sigma, const Expr& lambda, const Expr& f) {
  const FormSymbols& s = form_symbols();
  WeakForm wf;
  wf.bilinear = dot(Vec2{s.v_x, s.v_y}, matvec(sigma, Vec2{s.u_x, s.u_y})) + lambda * s.v * s.u;
  wf.linear = f * s.v;
  wf.space.dim = 2;
  return wf;
}

WeakForm helmholtz_form(const Mat3& sigma, const Expr& lambda, const Expr& f) {
  const FormSymbols& s = form_symbols();
  WeakForm wf;
  wf.bilinear = dot(Vec3{s.v_x, s.v_y, s.v_z}, matvec(sigma, Vec3{s.u_x, s.u_y, s.u_z})) + lambda * s.v * s.u;
  wf.linear = f * s.v;
  wf.space.dim = 3;
  wf.space.n_local = 4;
  return wf;
}

WeakForm convection_form(const Mat3& sigma, const Expr& lambda, const Vec3& beta, const Expr& f) {
  const FormSymbols& s = form_symbols();
  WeakForm wf = helmholtz_form(sigma, lambda, f);
  wf.bilinear = wf.bilinear + dot(beta, Vec3{s.u_x, s.u_y, s.u_z}) * s.v;
  return wf;
}

namespace {

void require_reserved(const Expr& e, const std::set<std::string>& allowed, const char* which) {
  for (const std::string& n : free_symbols(e))
    if (!allowed.count(n))
      throw FormError(std::string(which) + " integrand references symbol '" + n + "' outside the reserved set");
}

// Shared instantiation: u -> phi_j, v -> phi_i, grad -> J^{-T} grad_ref,
// (x, y, z) -> affine map, entry *= det J  (fem.cpp:122-158). The geometry is
// supplied as expressions: either over vertex coordinates (reference
// semantics) or over the per-element geometry symbols (GPU semantics).
struct GeometryExprs {
  Expr x[3];        // physical point
  Expr g[10][3];    // physical basis gradients
  Expr det;
};

void fill_entries(int dim, const std::vector<Expr>& phi, const GeometryExprs& geo, const WeakForm& wf,
                  std::vector<Expr>& bil, std::vector<Expr>& lin) {
  const FormSymbols& s = form_symbols();
  const int n = static_cast<int>(phi.size());
  bil.assign(n * n, Expr());
  lin.assign(n, Expr());
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      std::vector<std::pair<Expr, Expr>> b{{s.u, phi[j]}, {s.u_x, geo.g[j][0]}, {s.u_y, geo.g[j][1]},
                                           {s.v, phi[i]}, {s.v_x, geo.g[i][0]}, {s.v_y, geo.g[i][1]},
                                           {s.x, geo.x[0]}, {s.y, geo.x[1]}};
      if (dim == 3) {
        b.push_back({s.u_z, geo.g[j][2]});
        b.push_back({s.v_z, geo.g[i][2]});
        b.push_back({s.z, geo.x[2]});
      }
      bil[i * n + j] = substitute(wf.bilinear, b) * geo.det;
    }
    std::vector<std::pair<Expr, Expr>> b{{s.v, phi[i]}, {s.x, geo.x[0]}, {s.y, geo.x[1]}};
    if (dim == 3) b.push_back({s.z, geo.x[2]});
    lin[i] = substitute(wf.linear, b) * geo.det;
  }
}

}  // namespace

InstantiatedForm instantiate(const WeakForm& wf) {
  int dim = wf.space.dim > 0 ? wf.space.dim : (wf.space.mesh ? wf.space.mesh->dim : 2);
  if (dim != 2 && dim != 3) throw FormError("form dimension must be 2 or 3");
  const int degree = wf.space.degree;
  if (dim == 2) {
    require_reserved(wf.bilinear, {"u", "u_x", "u_y", "v", "v_x", "v_y", "x", "y"}, "bilinear");
    require_reserved(wf.linear, {"v", "x", "y"}, "linear");
  } else {
    require_reserved(wf.bilinear, {"u", "u_x", "u_y", "u_z", "v", "v_x", "v_y", "v_z", "x", "y", "z"}, "bilinear");
    require_reserved(wf.linear, {"v", "x", "y", "z"}, "linear");
  }
  InstantiatedForm out;
  out.dim = dim;
  out.degree = degree;
  const std::vector<Expr> phi = reference_shape_functions(dim, degree);
  const int n = static_cast<int>(phi.size());
  out.n_local = n;
  const Expr ref[3] = {arg_xi(), arg_eta(), arg_zeta()};
  std::vector<std::array<Expr, 3>> dref(n);
  for (int a = 0; a < n; ++a)
    for (int c = 0; c < dim; ++c) dref[a][c] = diff(phi[a], ref[c]);

  // (1) reference semantics over vertex coordinates
  {
    Expr X[4][3];
    const char* cn[3] = {"x", "y", "z"};
    for (int v = 0; v <= dim; ++v)
      for (int c = 0; c < dim; ++c) X[v][c] = sym(std::string(cn[c]) + std::to_string(v));
    Expr J[3][3], C[3][3];
    for (int r = 0; r < dim; ++r)
      for (int c = 0; c < dim; ++c) J[r][c] = X[c + 1][r] - X[0][r];
    GeometryExprs g;
    if (dim == 2) {
      g.det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      C[0][0] = J[1][1];
      C[0][1] = -J[1][0];
      C[1][0] = -J[0][1];
      C[1][1] = J[0][0];
    } else {
      g.det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
              J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          const int r1 = (r + 1) % 3, r2 = (r + 2) % 3, c1 = (c + 1) % 3, c2 = (c + 2) % 3;
          C[r][c] = J[r1][c1] * J[r2][c2] - J[r1][c2] * J[r2][c1];
        }
    }
    for (int r = 0; r < dim; ++r) {
      Expr x = X[0][r];
      for (int c = 0; c < dim; ++c) x = x + J[r][c] * ref[c];
      g.x[r] = x;
    }
    for (int a = 0; a < n; ++a)
      for (int r = 0; r < dim; ++r) {
        Expr s = integer(0);
        for (int c = 0; c < dim; ++c) s = s + C[r][c] * dref[a][c];
        g.g[a][r] = s / g.det;
      }
    fill_entries(dim, phi, g, wf, out.bilinear, out.linear);
  }
  // (2) geometry-symbol semantics for the GPU generator
  {
    const GeometrySymbols& G = geometry_symbols();
    GeometryExprs g;
    g.det = G.det;
    for (int r = 0; r < dim; ++r) {
      Expr x = G.X[r];
      for (int c = 0; c < dim; ++c) x = x + G.J[r][c] * ref[c];
      g.x[r] = x;
    }
    for (int a = 0; a < n; ++a)
      for (int r = 0; r < dim; ++r) {
        Expr s = integer(0);
        for (int c = 0; c < dim; ++c) s = s + G.G[r][c] * dref[a][c];
        g.g[a][r] = s;
      }
    fill_entries(dim, phi, g, wf, out.geo_bilinear, out.geo_linear);
  }
  out.form_bilinear = wf.bilinear;
  out.form_linear = wf.linear;
  return out;
}


InstantiatedForm instantiate_blocked(const std::vector<WeakForm>& blocks, const std::vector<WeakForm>& linear,
                                     int ncomp) {
  if (ncomp < 1 || blocks.size() != static_cast<std::size_t>(ncomp * ncomp) ||
      linear.size() != static_cast<std::size_t>(ncomp))
    throw FormError("blocked form needs ncomp^2 bilinear blocks and ncomp linear forms");
  std::vector<InstantiatedForm> bi, li;
  for (const WeakForm& w : blocks) bi.push_back(instantiate(w));
  for (const WeakForm& w : linear) li.push_back(instantiate(w));
  const int k = bi[0].n_local;
  for (const auto& f : bi)
    if (f.n_local != k || f.dim != bi[0].dim) throw FormError("blocks of a vector form must share the scalar space");
  InstantiatedForm out;
  out.dim = bi[0].dim;
  out.degree = bi[0].degree;
  out.ncomp = ncomp;
  out.n_local = k * ncomp;
  const int n = out.n_local;
  out.bilinear.resize(static_cast<std::size_t>(n) * n);
  out.geo_bilinear.resize(static_cast<std::size_t>(n) * n);
  out.linear.resize(n);
  out.geo_linear.resize(n);
  for (int a = 0; a < k; ++a)
    for (int c = 0; c < ncomp; ++c) {
      const int i = a * ncomp + c;
      out.linear[i] = li[c].linear[a];
      out.geo_linear[i] = li[c].geo_linear[a];
      for (int b = 0; b < k; ++b)
        for (int d = 0; d < ncomp; ++d) {
          const int j = b * ncomp + d;
          const InstantiatedForm& blk = bi[c * ncomp + d];
          out.bilinear[static_cast<std::size_t>(i) * n + j] = blk.bilinear[a * k + b];
          out.geo_bilinear[static_cast<std::size_t>(i) * n + j] = blk.geo_bilinear[a * k + b];
        }
    }
  return out;
}

void elasticity_blocks(int dim, const Expr& lambda, const Expr& mu, const std::vector<Expr>& f,
                       std::vector<WeakForm>& blocks, std::vector<WeakForm>& linear) {
  const FormSymbols& s = form_symbols();
  const Expr du[3] = {s.u_x, s.u_y, s.u_z}, dv[3] = {s.v_x, s.v_y, s.v_z};
  blocks.clear();
  linear.clear();
  for (int c = 0; c < dim; ++c)
    for (int d = 0; d < dim; ++d) {
      // test component c, trial component d
      Expr e = lambda * du[d] * dv[c] + mu * du[c] * dv[d];
      if (c == d) {
        std::vector<Expr> g;
        for (int q = 0; q < dim; ++q) g.push_back(du[q] * dv[q]);
        e = e + mu * symbolic::add(g);
      }
      WeakForm w;
      w.bilinear = e;
      w.linear = symbolic::integer(0);
      w.space.dim = dim;
      w.space.degree = 2;
      blocks.push_back(w);
    }
  for (int c = 0; c < dim; ++c) {
    WeakForm w;
    w.bilinear = symbolic::integer(0);
    w.linear = f[c] * s.v;
    w.space.dim = dim;
    w.space.degree = 2;
    linear.push_back(w);
  }
}

}  // namespace femforge::fem

// The quadrature compiler: instantiated integrands (over reference
// coordinates + per-element geometry symbols) -> straight-line CUDA that
// computes every local matrix / load-vector entry of one element.
//
// The reference evaluates each entry at each quadrature point through an IR
// interpreter and sums w_q * f_q in ascending q (device.cpp:176-192,
// kernel.cpp:22-46). Two equivalent GPU strategies are generated here:
//
//  * ReferenceTensor -- when an integrand is a polynomial in the reference
//    coordinates (affine simplices with polynomial coefficients), the sum
//    over quadrature points is done at compile time in extended precision:
//      K_ij = sum_q w_q f_ij(xi_q; g) = sum_t C_ij,t * m_t(g)
//    where m_t are monomials in the geometry symbols (J, J^{-T}, det J, x_0).
//    Monomials whose coefficient columns are identical across all entries are
//    merged into one invariant (e.g. det*G0l*G0m + det*G1l*G1m + det*G2l*G2m
//    for the Laplacian -> the 6 entries of det J^{-1}J^{-T}), and identical
//    entry rows (symmetry) are computed once.
//  * Pointwise -- the integrand at each quadrature point with the reference
//    coordinates folded to constants, summed with the rule weights, lowered
//    with CSE across all entries and all points (quadrature-invariant
//    subexpressions are computed once per element).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <tuple>
#include <unordered_map>

#include "femforge/codegen.hpp"

namespace femforge::codegen {

using namespace symbolic;

namespace {

using Mono = std::vector<std::pair<int, int>>;  // (atom, exponent) sorted by atom
using Poly = std::map<Mono, long double>;

Mono mono_mul(const Mono& a, const Mono& b) {
  Mono r;
  r.reserve(a.size() + b.size());
  std::size_t i = 0, j = 0;
  while (i < a.size() || j < b.size()) {
    if (j == b.size() || (i < a.size() && a[i].first < b[j].first)) {
      r.push_back(a[i++]);
    } else if (i == a.size() || b[j].first < a[i].first) {
      r.push_back(b[j++]);
    } else {
      r.push_back({a[i].first, a[i].second + b[j].second});
      ++i;
      ++j;
    }
  }
  return r;
}

Poly poly_mul(const Poly& a, const Poly& b) {
  Poly r;
  for (const auto& [ma, ca] : a)
    for (const auto& [mb, cb] : b) r[mono_mul(ma, mb)] += ca * cb;
  return r;
}

void poly_add(Poly& acc, const Poly& b, long double s = 1.0L) {
  for (const auto& [m, c] : b) acc[m] += s * c;
}

long double number_value(const Number& n) {
  return n.exact ? static_cast<long double>(n.rat.num) / static_cast<long double>(n.rat.den)
                 : static_cast<long double>(n.flt);
}

// Converts expressions into polynomials over "atoms". Atoms 0..2 are the
// reference coordinates; every other atom is a geometry symbol or an opaque
// subexpression that does not depend on the reference coordinates.
class PolyBuilder {
 public:
  PolyBuilder() {
    for (const char* n : {"xi", "eta", "zeta"}) atom_of(sym(n));
  }

  std::optional<Poly> build(const Expr& e) {
    auto m = memo_.find(e.raw());
    if (m != memo_.end()) return m->second;
    std::optional<Poly> r = convert(e);
    memo_.emplace(e.raw(), r);
    return r;
  }

  const std::vector<Expr>& atoms() const { return atoms_; }

 private:
  int atom_of(const Expr& e) {
    auto it = index_.find(e.raw());
    if (it != index_.end()) return it->second;
    index_.emplace(e.raw(), static_cast<int>(atoms_.size()));
    atoms_.push_back(e);
    return static_cast<int>(atoms_.size()) - 1;
  }
  bool has_ref(const Expr& e) { return depends_on(e, {"xi", "eta", "zeta"}); }
  Poly single(const Expr& atom) { return Poly{{Mono{{atom_of(atom), 1}}, 1.0L}}; }

  std::optional<Poly> convert(const Expr& e) {
    const auto& k = e.children();
    switch (e.kind()) {
      case Kind::Constant:
        return Poly{{Mono{}, number_value(e.node().constant)}};
      case Kind::Symbol:
        return single(e);
      case Kind::Add: {
        Poly acc;
        for (const Expr& c : k) {
          auto p = build(c);
          if (!p) return std::nullopt;
          poly_add(acc, *p);
        }
        return acc;
      }
      case Kind::Mul: {
        Poly acc{{Mono{}, 1.0L}};
        for (const Expr& c : k) {
          auto p = build(c);
          if (!p) return std::nullopt;
          acc = poly_mul(acc, *p);
        }
        return acc;
      }
      case Kind::Pow: {
        if (e.exponent() > 0) {
          auto b = build(k[0]);
          if (!b) return std::nullopt;
          Poly acc{{Mono{}, 1.0L}};
          for (std::int64_t i = 0; i < e.exponent(); ++i) acc = poly_mul(acc, *b);
          return acc;
        }
        if (has_ref(e)) return std::nullopt;
        return single(e);
      }
      case Kind::Div: {
        if (has_ref(k[1])) return std::nullopt;
        auto num = build(k[0]);
        if (!num) return std::nullopt;
        return poly_mul(*num, single(integer(1) / k[1]));
      }
      default:  // sin, cos, sqrt
        if (has_ref(e)) return std::nullopt;
        return single(e);
    }
  }

  std::vector<Expr> atoms_;
  std::unordered_map<const Node*, int> index_;
  std::unordered_map<const Node*, std::optional<Poly>> memo_;
};

// C identifier of a geometry symbol (the template declares gJrc, gGrc, gdet, gXr).
bool is_geometry_symbol(const std::string& n) {
  return n == "gdet" || (n.size() == 4 && (n[1] == 'J' || n[1] == 'G') && n[0] == 'g') ||
         (n.size() == 3 && n[0] == 'g' && n[1] == 'X');
}

// Renders an opaque atom expression as CUDA (geometry symbols are in scope).
std::string render_expr(const Expr& e);

std::string render_expr(const Expr& e) {
  const auto& k = e.children();
  switch (e.kind()) {
    case Kind::Constant: return "(" + double_literal(e.constant_value()) + ")";
    case Kind::Symbol:
      if (!is_geometry_symbol(e.name())) throw CodegenError("unbound symbol '" + e.name() + "' in element code");
      return e.name();
    case Kind::Add: {
      std::string s = "(";
      for (std::size_t i = 0; i < k.size(); ++i) s += (i ? " + " : "") + render_expr(k[i]);
      return s + ")";
    }
    case Kind::Mul: {
      std::string s = "(";
      for (std::size_t i = 0; i < k.size(); ++i) s += (i ? " * " : "") + render_expr(k[i]);
      return s + ")";
    }
    case Kind::Pow: return "ff_powi(" + render_expr(k[0]) + ", " + std::to_string(e.exponent()) + ")";
    case Kind::Div: return "(" + render_expr(k[0]) + " / " + render_expr(k[1]) + ")";
    case Kind::Sin: return "sin(" + render_expr(k[0]) + ")";
    case Kind::Cos: return "cos(" + render_expr(k[0]) + ")";
    case Kind::Sqrt: return "sqrt(" + render_expr(k[0]) + ")";
  }
  return "0.0";
}

struct Entry {
  bool linear;
  int i, j;
};

std::vector<Entry> entry_list(int n) {
  std::vector<Entry> out;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) out.push_back({false, i, j});
  for (int i = 0; i < n; ++i) out.push_back({true, i, 0});
  return out;
}

std::string emit_call(const Entry& en, const std::string& v) {
  if (en.linear) return "FF_EMIT_B(" + std::to_string(en.i) + ", " + v + ");";
  return "FF_EMIT_A(" + std::to_string(en.i) + ", " + std::to_string(en.j) + ", " + v + ");";
}

// ---------------------------------------------------------------------------
// ReferenceTensor

// Row-gather record of a vector form, block-uniform: every (test c, trial d)
// component block's entries are ONE linear map alpha of that block's own
// n_bq record quantities, entry ((a,c),(b,d)) = sum_k alpha[a,b][k] q[block_q[c,d] + k].
// alpha's columns are coefficient columns C[(a,c),(b,d)], t of the blocks'
// invariants (sparsest first, Gram-Schmidt in long double) spanning the union
// of the blocks' column spaces (elasticity: the 6 reference tensors
// A^rs_ab + A^sr_ab); every invariant column of block B is expressed through
// them (col = sum_k X_k alpha_k, checked to 1e-13), so the block's quantity
// k is sum_t X^B_kt inv_t. An elasticity diagonal block then reads 6
// quantities instead of 18 invariants, every block's entries are <= 6 terms,
// and one code path (ff_vrow<a>) serves all nine blocks: the row gather runs
// the three trial components of a row in neighbouring lanes. Blocks with equal
// quantities share them ((c, d) and (d, c) for lambda = mu); block offsets are
// even (32-byte chunks hold whole pairs). Returns false when the union basis
// exceeds 16 columns or a column is not reproduced.
struct UniformBasis {
  std::vector<std::vector<std::pair<int, double>>> qsig;   // quantity -> invariants
  std::vector<std::vector<std::pair<int, double>>> rep;    // entry -> quantities
  std::vector<std::vector<std::pair<int, double>>> alpha;  // node pair (a, b) -> basis column k
  std::vector<int> block_q;                                 // [bs * bs] quantity offsets
  int n_bq = 0;                                             // quantities per block (even)
};
bool uniform_block_basis(const std::vector<std::vector<std::pair<int, double>>>& row_sig, int n_local, int bs,
                         UniformBasis& out) {
  using V = std::vector<long double>;
  const int nn = n_local * n_local, nsc = n_local / bs, np = nsc * nsc, nb = bs * bs;
  auto dot = [](const V& x, const V& y) {
    long double s = 0.0L;
    for (std::size_t t = 0; t < x.size(); ++t) s += x[t] * y[t];
    return s;
  };
  auto norm = [&](const V& x) { return std::sqrt(dot(x, x)); };
  // coefficient column of invariant t in block B, over the node pairs (a, b)
  std::vector<std::map<int, V>> col(nb);
  for (int r = 0; r < nn; ++r) {
    const int i = r / n_local, j = r % n_local;
    const int blk = (i % bs) * bs + j % bs, u = (i / bs) * nsc + j / bs;
    for (const auto& [t, c] : row_sig[r]) {
      auto& v = col[blk][t];
      v.resize(np, 0.0L);
      v[u] = c;
    }
  }
  std::vector<std::tuple<int, int, int>> cand;  // (nonzeros, block, t)
  for (int blk = 0; blk < nb; ++blk)
    for (const auto& [t, v] : col[blk]) {
      int nz = 0;
      for (long double x : v) nz += x != 0.0L;
      cand.push_back({nz, blk, t});
    }
  std::sort(cand.begin(), cand.end());
  std::vector<V> A, U;  // basis columns, orthonormalised
  for (const auto& [nz, blk, t] : cand) {
    const V& c = col[blk][t];
    V w = c;
    for (int pass = 0; pass < 2; ++pass)
      for (const V& q : U) {
        const long double d = dot(w, q);
        for (int u = 0; u < np; ++u) w[u] -= d * q[u];
      }
    const long double nw = norm(w);
    if (nw <= 1e-11L * norm(c)) continue;
    for (auto& x : w) x /= nw;
    U.push_back(w);
    A.push_back(c);
  }
  const int k = static_cast<int>(A.size());
  if (std::getenv("FF_PLAN_DEBUG")) std::fprintf(stderr, "[plan] uniform block basis: %d columns\n", k);
  if (k == 0 || k > 16) return false;
  // normal equations of the basis (k x k), inverted once (Gauss-Jordan)
  std::vector<V> G(k, V(2 * k, 0.0L));
  for (int x = 0; x < k; ++x) {
    for (int y = 0; y < k; ++y) G[x][y] = dot(A[x], A[y]);
    G[x][k + x] = 1.0L;
  }
  for (int c = 0; c < k; ++c) {
    int pv = c;
    for (int x = c + 1; x < k; ++x)
      if (std::fabs(G[x][c]) > std::fabs(G[pv][c])) pv = x;
    std::swap(G[c], G[pv]);
    const long double d = G[c][c];
    for (auto& e : G[c]) e /= d;
    for (int x = 0; x < k; ++x) {
      if (x == c || G[x][c] == 0.0L) continue;
      const long double fct = G[x][c];
      for (int y = 0; y < 2 * k; ++y) G[x][y] -= fct * G[c][y];
    }
  }
  out = UniformBasis{};
  out.n_bq = k + (k & 1);
  out.block_q.assign(nb, 0);
  std::map<std::vector<std::vector<std::pair<int, double>>>, int> seen;
  for (int blk = 0; blk < nb; ++blk) {
    // X[t] = G^-1 A^T col_t, the block's invariant columns over the basis
    std::vector<std::vector<std::pair<int, double>>> qs(out.n_bq);
    std::map<int, V> X;
    for (const auto& [t, c] : col[blk]) {
      V rhs(k), x(k, 0.0L);
      for (int y = 0; y < k; ++y) rhs[y] = dot(A[y], c);
      for (int y = 0; y < k; ++y)
        for (int z = 0; z < k; ++z) x[y] += G[y][k + z] * rhs[z];
      V res = c;
      for (int y = 0; y < k; ++y)
        for (int u = 0; u < np; ++u) res[u] -= x[y] * A[y][u];
      if (norm(res) > 1e-13L * norm(c)) {
        if (std::getenv("FF_PLAN_DEBUG"))
          std::fprintf(stderr, "[plan] block %d invariant %d residual %Lg\n", blk, t, norm(res) / norm(c));
        return false;
      }
      X[t] = x;
    }
    for (int y = 0; y < k; ++y) {
      long double mx = 0.0L;
      for (const auto& [t, x] : X) mx = std::max(mx, std::fabs(x[y]));
      for (const auto& [t, x] : X)
        if (std::fabs(x[y]) > 1e-14L * mx) qs[y].push_back({t, static_cast<double>(x[y])});
    }
    auto [it, fresh] = seen.emplace(qs, static_cast<int>(out.qsig.size()));
    if (fresh) out.qsig.insert(out.qsig.end(), qs.begin(), qs.end());
    out.block_q[blk] = it->second;
  }
  out.alpha.assign(np, {});
  for (int u = 0; u < np; ++u)
    for (int y = 0; y < k; ++y)
      if (A[y][u] != 0.0L) out.alpha[u].push_back({y, static_cast<double>(A[y][u])});
  out.rep.assign(nn, {});
  for (int r = 0; r < nn; ++r) {
    const int i = r / n_local, j = r % n_local;
    const int blk = (i % bs) * bs + j % bs, u = (i / bs) * nsc + j / bs;
    if (row_sig[r].empty()) continue;
    for (const auto& [y, a] : out.alpha[u])
      if (!out.qsig[out.block_q[blk] + y].empty()) out.rep[r].push_back({out.block_q[blk] + y, a});
  }
  return true;
}

std::optional<ElementPlan> plan_tensor(const fem::InstantiatedForm& f, const fem::QuadratureRule& rule) {
  PolyBuilder pb;
  std::vector<Expr> integrands = f.geo_bilinear;
  integrands.insert(integrands.end(), f.geo_linear.begin(), f.geo_linear.end());
  std::vector<Poly> polys;
  for (const Expr& e : integrands) {
    auto p = pb.build(e);
    if (!p) return std::nullopt;
    polys.push_back(std::move(*p));
  }
  // quadrature moments sum_q w_q xi^a eta^b zeta^c in extended precision
  std::map<std::array<int, 3>, long double> moments;
  auto moment = [&](const std::array<int, 3>& ex) {
    auto it = moments.find(ex);
    if (it != moments.end()) return it->second;
    long double s = 0.0L;
    for (int q = 0; q < rule.size(); ++q) {
      long double t = rule.weights[q];
      for (int c = 0; c < 3; ++c)
        for (int p = 0; p < ex[c]; ++p) t *= static_cast<long double>(rule.points[q][c]);
      s += t;
    }
    moments.emplace(ex, s);
    return s;
  };
  // coefficient matrix over geometry monomials
  std::map<Mono, int> columns;
  std::vector<std::map<int, long double>> rows(polys.size());
  for (std::size_t r = 0; r < polys.size(); ++r) {
    for (const auto& [m, c] : polys[r]) {
      std::array<int, 3> ex{0, 0, 0};
      Mono geo;
      for (const auto& [a, p] : m) {
        if (a < 3)
          ex[a] = p;
        else
          geo.push_back({a, p});
      }
      auto [it, fresh] = columns.emplace(geo, static_cast<int>(columns.size()));
      rows[r][it->second] += c * moment(ex);
    }
  }
  std::vector<Mono> col_mono(columns.size());
  for (const auto& [m, k] : columns) col_mono[k] = m;
  // round to double, drop numerical zeros (relative 1e-14 of the row's largest term)
  std::vector<std::map<int, double>> C(rows.size());
  for (std::size_t r = 0; r < rows.size(); ++r) {
    long double mx = 0.0L;
    for (const auto& [k, c] : rows[r]) mx = std::max(mx, std::fabs(c));
    for (const auto& [k, c] : rows[r])
      if (std::fabs(c) > 1e-14L * mx && c != 0.0L) C[r][k] = static_cast<double>(c);
  }
  // merge columns with identical coefficient vectors
  std::map<std::vector<std::pair<int, double>>, std::vector<int>> groups;
  for (std::size_t k = 0; k < col_mono.size(); ++k) {
    std::vector<std::pair<int, double>> sig;
    for (std::size_t r = 0; r < C.size(); ++r) {
      auto it = C[r].find(static_cast<int>(k));
      if (it != C[r].end()) sig.push_back({static_cast<int>(r), it->second});
    }
    if (!sig.empty()) groups[sig].push_back(static_cast<int>(k));
  }
  // deterministic invariant order: by first member column's monomial
  std::vector<std::vector<int>> inv;
  for (auto& [sig, cols] : groups) inv.push_back(cols);
  std::sort(inv.begin(), inv.end(), [&](const std::vector<int>& a, const std::vector<int>& b) {
    return col_mono[a[0]] < col_mono[b[0]];
  });
  std::vector<int> inv_of_col(col_mono.size(), -1);
  for (std::size_t t = 0; t < inv.size(); ++t)
    for (int k : inv[t]) inv_of_col[k] = static_cast<int>(t);

  ElementPlan plan;
  plan.strategy = Strategy::ReferenceTensor;
  std::ostringstream os;
  std::int64_t flops = 0;
  // monomial products, memoised by prefix
  std::map<Mono, std::string> prod_name;
  int next_p = 0;
  const auto& atoms = pb.atoms();
  std::map<int, std::string> atom_name;
  auto atom_ref = [&](int a) -> std::string {
    auto it = atom_name.find(a);
    if (it != atom_name.end()) return it->second;
    const Expr& x = atoms[a];
    std::string s;
    if (x.is_symbol()) {
      s = render_expr(x);
    } else {
      s = "ff_a" + std::to_string(a);
      os << "  const double " << s << " = " << render_expr(x) << ";\n";
      flops += 4;
    }
    atom_name.emplace(a, s);
    return s;
  };
  auto product = [&](const Mono& m) -> std::string {
    // expand exponents into a factor list, build left-to-right with memo
    std::vector<int> factors;
    for (const auto& [a, p] : m)
      for (int t = 0; t < p; ++t) factors.push_back(a);
    Mono prefix;
    std::string cur;
    for (std::size_t i = 0; i < factors.size(); ++i) {
      prefix = mono_mul(prefix, Mono{{factors[i], 1}});
      auto it = prod_name.find(prefix);
      if (it != prod_name.end()) {
        cur = it->second;
        continue;
      }
      std::string name;
      if (i == 0) {
        name = atom_ref(factors[0]);
      } else {
        name = "ff_p" + std::to_string(next_p++);
        os << "  const double " << name << " = " << cur << " * " << atom_ref(factors[i]) << ";\n";
        ++flops;
      }
      prod_name.emplace(prefix, name);
      cur = name;
    }
    return cur.empty() ? std::string("1.0") : cur;
  };
  os << "  // " << inv.size() << " geometric invariants\n";
  for (std::size_t t = 0; t < inv.size(); ++t) {
    std::string expr;
    for (std::size_t q = 0; q < inv[t].size(); ++q) {
      expr += (q ? " + " : "") + product(col_mono[inv[t][q]]);
      if (q) ++flops;
    }
    os << "  const double ff_t" << t << " = " << expr << ";\n";
  }
  plan.n_invariants = static_cast<int>(inv.size());
  // entries: sum_t c_t * inv_t; identical rows computed once
  const std::vector<Entry> entries = entry_list(f.n_local);
  std::map<std::vector<std::pair<int, double>>, std::vector<int>> same;
  std::vector<std::vector<std::pair<int, double>>> row_sig(C.size());
  for (std::size_t r = 0; r < C.size(); ++r) {
    std::map<int, long double> by_inv;
    for (const auto& [k, c] : C[r]) by_inv[inv_of_col[k]] = c;  // merged columns share c
    for (const auto& [t, c] : by_inv) row_sig[r].push_back({t, static_cast<double>(c)});
    same[row_sig[r]].push_back(static_cast<int>(r));
  }
  // row-gather split: invariants read by the bilinear entries, in t order
  const int nn = f.n_local * f.n_local;
  // vector forms: per-block record quantities (block_basis); empty -> one
  // record quantity per invariant
  std::vector<std::vector<std::pair<int, double>>> qsig, rep;
  UniformBasis ub;
  if (f.ncomp > 1 && uniform_block_basis(row_sig, f.n_local, f.ncomp, ub)) {
    qsig = ub.qsig;
    rep = ub.rep;
    plan.n_bq = ub.n_bq;
    plan.block_q = ub.block_q;
  }
  std::map<int, int> kq;
  for (int r = 0; r < nn && qsig.empty(); ++r)
    for (const auto& [t, c] : row_sig[r]) kq.emplace(t, 0);
  if (!qsig.empty()) {
    // record quantity q = sum_t c_t inv_t (a pivot entry's expression, as the
    // element body computes that entry)
    plan.n_kinv = static_cast<int>(qsig.size());
    for (std::size_t q = 0; q < qsig.size(); ++q) {
      std::string v;
      for (std::size_t u = 0; u < qsig[q].size(); ++u) {
        const double c = qsig[q][u].second;
        const std::string t = "ff_t" + std::to_string(qsig[q][u].first);
        if (u == 0)
          v = c == 1.0 ? t : c == -1.0 ? "-" + t : double_literal(c) + " * " + t;
        else
          v += c == 1.0 ? " + " + t : c == -1.0 ? " - " + t : " + " + double_literal(c) + " * " + t;
        flops += 2;
      }
      os << "  FF_KINV(" << q << ", " << (v.empty() ? "0.0" : v) << ");\n";
    }
    std::ostringstream rc;
    std::map<double, int> coef;
    std::vector<double> coefs;
    auto cref = [&](double c) {
      auto [it, fresh] = coef.emplace(c, static_cast<int>(coefs.size()));
      if (fresh) coefs.push_back(c);
      return "ff_kc[" + std::to_string(it->second) + "]";
    };
    std::ostringstream body;
    for (int i = 0; i < f.n_local; ++i) {
      body << "template <> __device__ __forceinline__ void ff_row<" << i
           << ">(const double* __restrict__ g, double* __restrict__ v) {\n";
      for (int j = 0; j < f.n_local; ++j) {
        const auto& sig = rep[i * f.n_local + j];
        std::string v = sig.empty() ? "0.0" : "";
        for (std::size_t q = 0; q < sig.size(); ++q) {
          const double c = sig[q].second;
          const std::string t = "g[" + std::to_string(sig[q].first) + "]";
          if (q == 0)
            v = c == 1.0 ? t : c == -1.0 ? "-" + t : cref(c) + " * " + t;
          else
            v += c == 1.0 ? " + " + t : c == -1.0 ? " - " + t : " + " + cref(c) + " * " + t;
          plan.row_flops += 2;
        }
        body << "  v[" << j << "] = " << v << ";\n";
      }
      body << "}\n";
    }
    // ff_vrow<a>: v[b] = entry ((a, c), (b, d)) of any block from that
    // block's quantities g[0 .. n_bq)
    const int nsc = f.n_local / f.ncomp;
    for (int a = 0; a < nsc; ++a) {
      body << "template <> __device__ __forceinline__ void ff_vrow<" << a
           << ">(const double* __restrict__ g, double* __restrict__ v) {\n";
      for (int b = 0; b < nsc; ++b) {
        const auto& sig = ub.alpha[a * nsc + b];
        std::string v = sig.empty() ? "0.0" : "";
        for (std::size_t q = 0; q < sig.size(); ++q) {
          const double c = sig[q].second;
          const std::string t = "g[" + std::to_string(sig[q].first) + "]";
          if (q == 0)
            v = c == 1.0 ? t : c == -1.0 ? "-" + t : cref(c) + " * " + t;
          else
            v += c == 1.0 ? " + " + t : c == -1.0 ? " - " + t : " + " + cref(c) + " * " + t;
        }
        body << "  v[" << b << "] = " << v << ";\n";
      }
      body << "}\n";
    }
    rc << "__constant__ double ff_kc[" << std::max<std::size_t>(coefs.size(), 1) << "] = {";
    for (std::size_t q = 0; q < coefs.size(); ++q) rc << (q ? ", " : "") << double_literal(coefs[q]);
    if (coefs.empty()) rc << "0.0";
    rc << "};\n";
    rc << "template <int A>\n__device__ __forceinline__ void ff_vrow(const double* __restrict__ g, double* __restrict__ v);\n";
    rc << "// quantity offset of component block (c, d) in the element record\n__constant__ int ff_block_q["
       << plan.block_q.size() << "] = {";
    for (std::size_t q = 0; q < plan.block_q.size(); ++q) rc << (q ? ", " : "") << plan.block_q[q];
    rc << "};\n#define FF_NBQ " << plan.n_bq << "\n" << body.str();
    plan.row_code = rc.str();
  }
  if (qsig.empty()) {
    // vector forms: invariants ordered by the first (test, trial) component
    // block that reads them, so the row gather of one block loads a few
    // contiguous 32-byte groups of the element record
    const int bs = std::max(1, f.ncomp);
    std::map<int, int> first_block;
    for (int r = 0; r < nn; ++r) {
      const int blk = ((r / f.n_local) % bs) * bs + (r % f.n_local) % bs;
      for (const auto& [t, c] : row_sig[r]) {
        auto it = first_block.find(t);
        if (it == first_block.end() || blk < it->second) first_block[t] = blk;
      }
    }
    std::vector<std::pair<int, int>> keyed;
    for (const auto& [t, slot] : kq) keyed.push_back({first_block[t], t});
    std::sort(keyed.begin(), keyed.end());
    int q = 0;
    for (const auto& [blk, t] : keyed) kq[t] = q++;
    plan.n_kinv = static_cast<int>(kq.size());
  }
  if (qsig.empty()) {
    std::vector<std::pair<int, int>> by_q;
    for (const auto& [t, q] : kq) by_q.push_back({q, t});
    std::sort(by_q.begin(), by_q.end());
    for (const auto& [q, t] : by_q) os << "  FF_KINV(" << q << ", ff_t" << t << ");\n";
  }
  if (qsig.empty()) {
    // ff_row<i>: v[j] = K_ij with the same expression (term order, literals)
    // as the element body, so both scatters compute bit-identical entries
    // coefficients live in a __constant__ table so the fp64 FMAs read them as
    // constant-bank operands instead of materialising 64-bit immediates
    std::ostringstream rc;
    std::map<double, int> coef;
    std::vector<double> coefs;
    auto cref = [&](double c) {
      auto [it, fresh] = coef.emplace(c, static_cast<int>(coefs.size()));
      if (fresh) coefs.push_back(c);
      return "ff_kc[" + std::to_string(it->second) + "]";
    };
    std::ostringstream body;
    for (int i = 0; i < f.n_local; ++i) {
      body << "template <> __device__ __forceinline__ void ff_row<" << i
           << ">(const double* __restrict__ g, double* __restrict__ v) {\n";
      for (int j = 0; j < f.n_local; ++j) {
        const auto& sig = row_sig[i * f.n_local + j];
        std::string v = sig.empty() ? "0.0" : "";
        for (std::size_t q = 0; q < sig.size(); ++q) {
          const double c = sig[q].second;
          const std::string t = "g[" + std::to_string(kq.at(sig[q].first)) + "]";
          if (q == 0)
            v = c == 1.0 ? t : c == -1.0 ? "-" + t : cref(c) + " * " + t;
          else
            v += c == 1.0 ? " + " + t : c == -1.0 ? " - " + t : " + " + cref(c) + " * " + t;
          plan.row_flops += 2;
        }
        body << "  v[" << j << "] = " << v << ";\n";
      }
      body << "}\n";
    }
    rc << "__constant__ double ff_kc[" << std::max<std::size_t>(coefs.size(), 1) << "] = {";
    for (std::size_t q = 0; q < coefs.size(); ++q) rc << (q ? ", " : "") << double_literal(coefs[q]);
    if (coefs.empty()) rc << "0.0";
    rc << "};\n" << body.str();
    plan.row_code = rc.str();
  }
  // rows already grouped; emit in entry order of the group's first member
  std::vector<std::vector<int>> ordered;
  for (auto& [sig, members] : same) ordered.push_back(members);
  std::sort(ordered.begin(), ordered.end());
  os << "  // " << ordered.size() << " distinct entries\n";
  int vi = 0;
  for (const auto& members : ordered) {
    const auto& sig = row_sig[members[0]];
    std::string v;
    if (sig.empty()) {
      v = "0.0";
    } else {
      for (std::size_t q = 0; q < sig.size(); ++q) {
        const double c = sig[q].second;
        const std::string t = "ff_t" + std::to_string(sig[q].first);
        if (q == 0) {
          v = c == 1.0 ? t : c == -1.0 ? "-" + t : double_literal(c) + " * " + t;
        } else {
          v += c == 1.0 ? " + " + t : c == -1.0 ? " - " + t : " + " + double_literal(c) + " * " + t;
        }
        flops += 2;
      }
    }
    const std::string name = "ff_v" + std::to_string(vi++);
    os << "  { const double " << name << " = " << v << ";";
    for (int r : members) os << " " << emit_call(entries[r], name);
    os << " }\n";
  }
  plan.b_zero.assign(f.n_local, 0);
  for (int i = 0; i < f.n_local; ++i) plan.b_zero[i] = row_sig[nn + i].empty() ? 1 : 0;
  plan.n_unique_entries = static_cast<int>(ordered.size());
  plan.flops = flops;
  plan.body = os.str();
  return plan;
}

// ---------------------------------------------------------------------------
// Pointwise, bilinear structure (scalar forms)
//
// The weak form is bilinear: a(u, v) = sum_{a,b} C_ab(x) U_a V_b with
// U = (u, u_x, u_y[, u_z]) and V = (v, v_x, v_y[, v_z]), l(v) = L(x) v, the
// C_ab = d2a / dU_a dV_b and L = dl/dv found symbolically (and checked at
// random points). Per quadrature point (runtime loop, ascending q):
//   x_q = X0 + J xi_q;  W_ab = w_q det J C_ab(x_q)  (only the nonzero C_ab)
//   U_a(j): phi_j and the physical gradient G grad_ref phi_j (tables of the
//           reference basis at the points, __constant__)
//   P_b(j) = sum_a W_ab U_a(j);  K_ij += sum_b V_b(i) P_b(j);  b_i += w det L phi_i
// i.e. per point a rank-(dim+1) update of the element matrix instead of every
// entry's expanded integrand (config 4: ~10k instead of ~38k flops per
// element). Rows go in blocks of <= 5 (accumulators in registers); P is
// recomputed per block.

namespace {

bool is_zero_expr(const Expr& e) { return e.is_zero(); }

void render_program(std::ostringstream& os, const MultiProgram& p, const std::string& prefix, const std::string& indent,
                    std::int64_t& ops) {
  auto r = [&](int k) { return prefix + std::to_string(k); };
  for (std::size_t k = 0; k < p.code.size(); ++k) {
    const Instr& in = p.code[k];
    std::string rhs;
    switch (in.op) {
      case Op::LoadArg: rhs = p.arg_names[in.imm]; break;
      case Op::LoadConst: rhs = double_literal(p.consts[in.imm]); break;
      case Op::Add: rhs = r(in.a) + " + " + r(in.b); ++ops; break;
      case Op::Sub: rhs = r(in.a) + " - " + r(in.b); ++ops; break;
      case Op::Mul: rhs = r(in.a) + " * " + r(in.b); ++ops; break;
      case Op::Div: rhs = r(in.a) + " / " + r(in.b); ops += 4; break;
      case Op::Neg: rhs = "-" + r(in.a); break;
      case Op::PowInt: rhs = "ff_powi(" + r(in.a) + ", " + std::to_string(in.imm) + ")"; ops += 8; break;
      case Op::Sin: rhs = "sin(" + r(in.a) + ")"; ops += 20; break;
      case Op::Cos: rhs = "cos(" + r(in.a) + ")"; ops += 20; break;
      case Op::Sqrt: rhs = "sqrt(" + r(in.a) + ")"; ops += 4; break;
    }
    os << indent << "const double " << r(static_cast<int>(k)) << " = " << rhs << ";\n";
  }
}

}  // namespace

std::optional<ElementPlan> plan_point_bilinear(const fem::InstantiatedForm& f, const fem::QuadratureRule& rule) {
  if (f.ncomp != 1 || !f.form_bilinear.valid() || !f.form_linear.valid() || std::getenv("FF_POINT_GENERIC"))
    return std::nullopt;
  const int dim = f.dim, n = f.n_local, nq = rule.size(), nu = dim + 1;
  const char* un[4] = {"u", "u_x", "u_y", "u_z"};
  const char* vn[4] = {"v", "v_x", "v_y", "v_z"};
  const char* xn[3] = {"x", "y", "z"};
  const std::set<std::string> coords(xn, xn + dim);
  Expr C[4][4];
  bool nz[4][4] = {};
  std::vector<Expr> outs;
  int idx[4][4];
  for (int a = 0; a < nu; ++a)
    for (int b = 0; b < nu; ++b) {
      C[a][b] = diff(diff(f.form_bilinear, sym(un[a])), sym(vn[b]));
      for (const std::string& s : free_symbols(C[a][b]))
        if (!coords.count(s)) return std::nullopt;  // not bilinear in (U, V)
      nz[a][b] = !is_zero_expr(C[a][b]);
      idx[a][b] = -1;
      if (nz[a][b]) {
        idx[a][b] = static_cast<int>(outs.size());
        outs.push_back(C[a][b]);
      }
    }
  const Expr L = diff(f.form_linear, sym("v"));
  for (const std::string& s : free_symbols(L))
    if (!coords.count(s)) return std::nullopt;
  const int iL = static_cast<int>(outs.size());
  outs.push_back(L);
  // the decomposition must reproduce the form (random points; exact for
  // bilinear / linear forms up to rounding)
  {
    std::uint64_t rng = 0x2545F4914F6CDD1Dull;
    auto rnd = [&]() {
      rng = rng * 6364136223846793005ull + 1442695040888963407ull;
      return 0.25 + 0.5 * static_cast<double>(rng >> 11) / 9007199254740992.0;
    };
    for (int t = 0; t < 4; ++t) {
      std::map<std::string, double> val;
      for (int c = 0; c < 3; ++c) val[xn[c]] = rnd();
      for (int a = 0; a < 4; ++a) val[un[a]] = rnd(), val[vn[a]] = rnd();
      double ref = eval(f.form_bilinear, val), got = 0.0, scale = std::fabs(ref);
      for (int a = 0; a < nu; ++a)
        for (int b = 0; b < nu; ++b)
          if (nz[a][b]) {
            const double term = eval(C[a][b], val) * val[un[a]] * val[vn[b]];
            got += term;
            scale = std::max(scale, std::fabs(term));
          }
      if (std::fabs(got - ref) > 1e-12 * std::max(scale, 1e-300)) return std::nullopt;
      const double lref = eval(f.form_linear, val), lgot = eval(L, val) * val["v"];
      if (std::fabs(lgot - lref) > 1e-12 * std::max(std::fabs(lref), 1e-300)) return std::nullopt;
    }
  }
  bool use_u[4] = {}, use_v[4] = {};
  for (int a = 0; a < nu; ++a)
    for (int b = 0; b < nu; ++b)
      if (nz[a][b]) use_u[a] = use_v[b] = true;
  // reference basis and gradients at the points
  const std::vector<Expr> phi = fem::reference_shape_functions(dim, f.degree);
  const Expr ref[3] = {sym("xi"), sym("eta"), sym("zeta")};
  std::ostringstream pre;
  pre << "__constant__ double ff_qp[" << nq << "][3] = { ";
  for (int q = 0; q < nq; ++q)
    pre << (q ? ", " : "") << "{" << double_literal(rule.points[q][0]) << ", " << double_literal(rule.points[q][1])
        << ", " << double_literal(dim == 3 ? rule.points[q][2] : 0.0) << "}";
  pre << "};\n__constant__ double ff_qw[" << nq << "] = {";
  for (int q = 0; q < nq; ++q) pre << (q ? ", " : "") << double_literal(rule.weights[q]);
  pre << "};\n__constant__ double ff_bphi[" << nq << "][" << n << "] = {";
  std::vector<std::array<Expr, 3>> dphi(n);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < dim; ++c) dphi[i][c] = diff(phi[i], ref[c]);
  auto at = [&](int q) {
    return std::map<std::string, double>{
        {"xi", rule.points[q][0]}, {"eta", rule.points[q][1]}, {"zeta", dim == 3 ? rule.points[q][2] : 0.0}};
  };
  for (int q = 0; q < nq; ++q)
    for (int i = 0; i < n; ++i) pre << (q || i ? ", " : "") << double_literal(eval(phi[i], at(q)));
  pre << "};\n__constant__ double ff_bdphi[" << nq << "][" << n << "][" << dim << "] = {";
  for (int q = 0; q < nq; ++q)
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < dim; ++c) pre << (q || i || c ? ", " : "") << double_literal(eval(dphi[i][c], at(q)));
  pre << "};\n";

  SymbolTable args;
  for (int c = 0; c < dim; ++c) args.add(xn[c]);
  const MultiProgram prog = lower_many(outs, args);
  ElementPlan plan;
  plan.strategy = Strategy::Pointwise;
  plan.prelude = pre.str();
  std::ostringstream os;
  std::int64_t flops = 0;
  // rows per register block (FF_PROWS tuning knob; default <= 5)
  int rmax = 5;
  if (const char* v = std::getenv("FF_PROWS")) rmax = std::max(1, std::atoi(v));
  const int nblk = (n + rmax - 1) / rmax, R = (n + nblk - 1) / nblk;
  const char* refname[3] = {"xi", "eta", "zeta"};
  auto grad = [&](const std::string& base, int r) {  // (G grad_ref phi)_r from the table row `base`
    std::string e;
    for (int c = 0; c < dim; ++c)
      e += (c ? " + " : "") + std::string("gG") + std::to_string(r) + std::to_string(c) + " * " + base + "[" +
           std::to_string(c) + "]";
    return e;
  };
  os << "  // element body: bilinear point updates, " << nq << "-point rule, rows in " << nblk << " block(s)\n";
  for (int i0 = 0; i0 < n; i0 += R) {
    const int i1 = std::min(n, i0 + R);
    os << "  {  // rows [" << i0 << ", " << i1 << ")\n";
    for (int i = i0; i < i1; ++i) {
      os << "    double ff_b" << i << " = 0.0";
      for (int j = 0; j < n; ++j) os << ", ff_a" << i << "_" << j << " = 0.0";
      os << ";\n";
    }
    os << "#pragma unroll 1\n    for (int ff_q = 0; ff_q < " << nq << "; ++ff_q) {\n";
    for (int c = 0; c < dim; ++c) os << "      const double " << refname[c] << " = ff_qp[ff_q][" << c << "];\n";
    os << "      const double ff_w = ff_qw[ff_q] * gdet;\n";
    for (int r = 0; r < dim; ++r) {
      os << "      const double " << xn[r] << " = gX" << r;
      for (int c = 0; c < dim; ++c) os << " + gJ" << r << c << " * " << refname[c];
      os << ";\n";
      flops += 2 * dim;
    }
    render_program(os, prog, "ff_c", "      ", flops);
    for (int a = 0; a < nu; ++a)
      for (int b = 0; b < nu; ++b)
        if (nz[a][b]) {
          os << "      const double ff_W" << a << b << " = ff_w * ff_c" << prog.results[idx[a][b]] << ";\n";
          ++flops;
        }
    os << "      const double ff_L = ff_w * ff_c" << prog.results[iL] << ";\n";
    ++flops;
    // test side of the block's rows
    for (int i = i0; i < i1; ++i) {
      os << "      const double ff_v" << i << "_0 = ff_bphi[ff_q][" << i << "];\n";
      for (int r = 0; r < dim; ++r)
        if (use_v[r + 1]) {
          os << "      const double ff_v" << i << "_" << r + 1 << " = " << grad("ff_bdphi[ff_q][" + std::to_string(i) + "]", r)
             << ";\n";
          flops += 2 * dim;
        }
    }
    for (int j = 0; j < n; ++j) {
      os << "      {\n        const double ff_u0 = ff_bphi[ff_q][" << j << "];\n";
      for (int r = 0; r < dim; ++r)
        if (use_u[r + 1]) {
          os << "        const double ff_u" << r + 1 << " = " << grad("ff_bdphi[ff_q][" + std::to_string(j) + "]", r)
             << ";\n";
          flops += 2 * dim;
        }
      for (int b = 0; b < nu; ++b) {
        if (!use_v[b]) continue;
        std::string e;
        for (int a = 0; a < nu; ++a)
          if (nz[a][b]) {
            e += (e.empty() ? "" : " + ") + std::string("ff_W") + std::to_string(a) + std::to_string(b) + " * ff_u" +
                 std::to_string(a);
            flops += 2;
          }
        os << "        const double ff_P" << b << " = " << e << ";\n";
      }
      for (int i = i0; i < i1; ++i) {
        // K_ij += sum_b V_b(i) P_b(j) as a chain of fused multiply-adds into
        // the accumulator (one DFMA per term, no separate product sum)
        std::string e = "ff_a" + std::to_string(i) + "_" + std::to_string(j);
        for (int b = nu - 1; b >= 0; --b)
          if (use_v[b]) {
            e = "fma(ff_v" + std::to_string(i) + "_" + std::to_string(b) + ", ff_P" + std::to_string(b) + ", " + e + ")";
            flops += 2;
          }
        os << "        ff_a" << i << "_" << j << " = " << e << ";\n";
      }
      os << "      }\n";
    }
    for (int i = i0; i < i1; ++i) {
      os << "      ff_b" << i << " += ff_L * ff_v" << i << "_0;\n";
      flops += 2;
    }
    os << "    }\n";
    for (int i = i0; i < i1; ++i) {
      for (int j = 0; j < n; ++j) os << "    FF_EMIT_A(" << i << ", " << j << ", ff_a" << i << "_" << j << ");\n";
      os << "    FF_EMIT_B(" << i << ", ff_b" << i << ");\n";
    }
    os << "  }\n";
  }
  plan.n_unique_entries = n * n + n;
  plan.flops = flops * nq;  // counted once per point inside the loop body
  plan.body = os.str();
  return plan;
}

// ---------------------------------------------------------------------------
// Pointwise

ElementPlan plan_pointwise(const fem::InstantiatedForm& f, const fem::QuadratureRule& rule) {
  if (auto p = plan_point_bilinear(f, rule)) return *p;
  // A runtime quadrature loop per block of kRows element rows: the block's
  // integrands are lowered once with the reference coordinates as symbols
  // (CSE inside the block), evaluated at every point in ascending order, and
  // w_q * f_q is added to the block's accumulators (device.cpp:176-192 order).
  // Code size and the live set stay one block of accumulators plus one
  // point's subexpressions.
  std::vector<Expr> integrands = f.geo_bilinear;
  integrands.insert(integrands.end(), f.geo_linear.begin(), f.geo_linear.end());
  SymbolTable args;
  const fem::GeometrySymbols& g = fem::geometry_symbols();
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      args.add(g.J[r][c].name());
      args.add(g.G[r][c].name());
    }
  for (int r = 0; r < 3; ++r) args.add(g.X[r].name());
  args.add(g.det.name());
  const char* refname[3] = {"xi", "eta", "zeta"};
  for (int c = 0; c < f.dim; ++c) args.add(refname[c]);
  const int n = f.n_local;
  const int nq = rule.size();
  const int kRows = 2;
  ElementPlan plan;
  plan.strategy = Strategy::Pointwise;
  {
    std::ostringstream pre;
    pre << "__constant__ double ff_qp[" << nq << "][3] = { ";
    for (int q = 0; q < nq; ++q)
      pre << (q ? ", " : "") << "{" << double_literal(rule.points[q][0]) << ", " << double_literal(rule.points[q][1])
          << ", " << double_literal(f.dim == 3 ? rule.points[q][2] : 0.0) << "}";
    pre << "};\n__constant__ double ff_qw[" << nq << "] = {";
    for (int q = 0; q < nq; ++q) pre << (q ? ", " : "") << double_literal(rule.weights[q]);
    pre << "};\n";
    plan.prelude = pre.str();
  }
  std::ostringstream os;
  std::int64_t flops = 0;
  const std::vector<Entry> entries = entry_list(n);
  for (int i0 = 0; i0 < n; i0 += kRows) {
    const int i1 = std::min(n, i0 + kRows);
    std::vector<int> members;
    for (int i = i0; i < i1; ++i)
      for (int j = 0; j < n; ++j) members.push_back(i * n + j);
    for (int i = i0; i < i1; ++i) members.push_back(n * n + i);
    std::vector<Expr> sub;
    for (int r : members) sub.push_back(integrands[r]);
    MultiProgram p = lower_many(sub, args);
    auto r = [](int k) { return "ff_r" + std::to_string(k); };
    os << "  {  // element rows [" << i0 << ", " << i1 << ")\n";
    for (std::size_t m = 0; m < members.size(); ++m) os << "    double ff_acc" << m << " = 0.0;\n";
    os << "#pragma unroll 1\n    for (int ff_q = 0; ff_q < " << nq << "; ++ff_q) {\n";
    for (int c = 0; c < f.dim; ++c) os << "      const double " << refname[c] << " = ff_qp[ff_q][" << c << "];\n";
    os << "      const double ff_w = ff_qw[ff_q];\n";
    std::int64_t per_q = 0;
    for (std::size_t k = 0; k < p.code.size(); ++k) {
      const Instr& in = p.code[k];
      std::string rhs;
      switch (in.op) {
        case Op::LoadArg: rhs = p.arg_names[in.imm]; break;
        case Op::LoadConst: rhs = double_literal(p.consts[in.imm]); break;
        case Op::Add: rhs = r(in.a) + " + " + r(in.b); ++per_q; break;
        case Op::Sub: rhs = r(in.a) + " - " + r(in.b); ++per_q; break;
        case Op::Mul: rhs = r(in.a) + " * " + r(in.b); ++per_q; break;
        case Op::Div: rhs = r(in.a) + " / " + r(in.b); per_q += 4; break;
        case Op::Neg: rhs = "-" + r(in.a); break;
        case Op::PowInt: rhs = "ff_powi(" + r(in.a) + ", " + std::to_string(in.imm) + ")"; per_q += 8; break;
        case Op::Sin: rhs = "sin(" + r(in.a) + ")"; per_q += 20; break;
        case Op::Cos: rhs = "cos(" + r(in.a) + ")"; per_q += 20; break;
        case Op::Sqrt: rhs = "sqrt(" + r(in.a) + ")"; per_q += 4; break;
      }
      os << "      const double " << r(static_cast<int>(k)) << " = " << rhs << ";\n";
    }
    for (std::size_t m = 0; m < members.size(); ++m) os << "      ff_acc" << m << " += ff_w * " << r(p.results[m]) << ";\n";
    per_q += 2 * static_cast<std::int64_t>(members.size());
    flops += per_q * nq;
    os << "    }\n";
    for (std::size_t m = 0; m < members.size(); ++m)
      os << "    " << emit_call(entries[members[m]], "ff_acc" + std::to_string(m)) << "\n";
    os << "  }\n";
  }
  plan.n_unique_entries = static_cast<int>(entries.size());
  plan.flops = flops;
  plan.body = os.str();
  return plan;
}

}  // namespace

ElementPlan plan_element(const fem::InstantiatedForm& f, const fem::QuadratureRule& rule, Strategy strategy) {
  if (f.geo_bilinear.size() != static_cast<std::size_t>(f.n_local * f.n_local) ||
      f.geo_linear.size() != static_cast<std::size_t>(f.n_local))
    throw CodegenError("instantiated form has no geometry-symbol entries");
  if (rule.dim != f.dim) throw CodegenError("quadrature rule dimension does not match the form");
  ElementPlan plan;
  if (strategy == Strategy::Pointwise) {
    plan = plan_pointwise(f, rule);
  } else {
    auto t = plan_tensor(f, rule);
    if (!t) {
      if (strategy == Strategy::ReferenceTensor)
        throw CodegenError("integrand is not polynomial in the reference coordinates; use the pointwise strategy");
      plan = plan_pointwise(f, rule);
    } else if (strategy == Strategy::Auto && (t->flops > 4000 || t->n_invariants > 48)) {
      // large tensor expansions (e.g. variable coefficients): every invariant
      // is live at once, so beyond ~48 of them the body spills; the pointwise
      // quadrature loop keeps one point live. Keep the tensor form only when it
      // is both small enough for registers and cheaper.
      ElementPlan p = plan_pointwise(f, rule);
      plan = (t->n_invariants <= 48 && t->flops < p.flops) ? *t : p;
    } else {
      plan = *t;
    }
  }
  plan.dim = f.dim;
  plan.degree = f.degree;
  plan.n_local = f.n_local;
  plan.n_quad = rule.size();
  return plan;
}

}  // namespace femforge::codegen

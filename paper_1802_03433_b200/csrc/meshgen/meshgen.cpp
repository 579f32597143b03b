// femforge-b200 synthetic mesh generators (see meshgen.hpp).
#include "femforge/meshgen.hpp"

namespace femforge::meshgen {

fem::Mesh unit_square_mesh(int n) {
  if (n < 1) throw fem::MeshError("unit_square_mesh: n must be >= 1");
  fem::Mesh m;
  m.dim = 2;
  const double h = 1.0 / n;
  m.nodes.reserve(static_cast<std::size_t>(n + 1) * (n + 1));
  for (int j = 0; j <= n; ++j)
    for (int i = 0; i <= n; ++i) m.nodes.push_back({i * h, j * h, 0.0});
  m.elements.reserve(static_cast<std::size_t>(2) * n * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const int a = j * (n + 1) + i, b = a + 1, d = a + (n + 1), c = d + 1;
      m.elements.push_back({{a, b, c, 0}});
      m.elements.push_back({{a, c, d, 0}});
    }
  return m;
}

fem::Mesh kuhn_cube_mesh(int n) {
  if (n < 1) throw fem::MeshError("kuhn_cube_mesh: n must be >= 1");
  fem::Mesh m;
  m.dim = 3;
  const double h = 1.0 / n;
  const long s = n + 1;
  m.nodes.reserve(static_cast<std::size_t>(s * s * s));
  for (int k = 0; k <= n; ++k)
    for (int j = 0; j <= n; ++j)
      for (int i = 0; i <= n; ++i) m.nodes.push_back({i * h, j * h, k * h});
  static const int kPerm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  static const bool kOdd[6] = {false, true, true, false, false, true};
  auto vid = [s](const int c[3]) { return static_cast<int>(c[0] + s * (c[1] + s * c[2])); };
  m.elements.reserve(static_cast<std::size_t>(6) * n * n * n);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        for (int p = 0; p < 6; ++p) {
          int c[3] = {i, j, k};
          fem::Element e;
          e.nodes[0] = vid(c);
          ++c[kPerm[p][0]];
          e.nodes[1] = vid(c);
          ++c[kPerm[p][1]];
          e.nodes[2] = vid(c);
          ++c[kPerm[p][2]];
          e.nodes[3] = vid(c);
          if (kOdd[p]) std::swap(e.nodes[1], e.nodes[2]);
          m.elements.push_back(e);
        }
  return m;
}

fem::DofMap kuhn_p2_dofs(int n, const fem::Mesh& m) {
  static const int kEdge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  fem::DofMap d;
  d.n_local = 10;
  const long s = n + 1, L = 2L * n + 1;
  d.n_dofs = L * L * L;
  d.dofs.resize(static_cast<std::size_t>(m.element_count()) * 10);
  for (int e = 0; e < m.element_count(); ++e) {
    long I[4], J[4], K[4];
    for (int a = 0; a < 4; ++a) {
      const long v = m.elements[e].nodes[a];
      I[a] = v % s;
      J[a] = (v / s) % s;
      K[a] = v / (s * s);
      d.dofs[10L * e + a] = static_cast<std::int32_t>(2 * I[a] + L * (2 * J[a] + L * 2 * K[a]));
    }
    for (int q = 0; q < 6; ++q) {
      const int a = kEdge[q][0], b = kEdge[q][1];
      d.dofs[10L * e + 4 + q] = static_cast<std::int32_t>((I[a] + I[b]) + L * ((J[a] + J[b]) + L * (K[a] + K[b])));
    }
  }
  return d;
}

}  // namespace femforge::meshgen

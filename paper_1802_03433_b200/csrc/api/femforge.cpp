// femforge-b200 C++ assembly API over the C ABI (see device.hpp).
#include <cstring>

#include "femforge/device.hpp"
#include "femforge/symbolic.hpp"
#include "femforge_b200.h"

namespace femforge::device {

namespace {

void ok(int rc) {
  if (rc == FF_OK) return;
  const std::string msg = ff_last_error();
  switch (rc) {
    case FF_E_MESH: throw fem::MeshError(msg);
    case FF_E_FORM: throw fem::FormError(msg);
    case FF_E_SYMBOLIC: throw symbolic::SymbolicError(msg);
    default: throw DeviceError(msg);
  }
}

}  // namespace

Engine::Engine(int device) { ok(ff_init(device, &ctx_)); }
Engine::~Engine() { ff_ctx_destroy(ctx_); }
void Engine::synchronize() const { ok(ff_ctx_synchronize(ctx_)); }
Engine& Engine::default_engine() {
  static Engine* e = new Engine(0);
  return *e;
}

void LaunchConfig::validate() const {
  if (elems_per_block < 1) throw DeviceError("elems_per_block must be >= 1");
  if (3 * 9 * elems_per_block > 1024)  // the reference's simulated block limit (device.cpp:90-97)
    throw DeviceError("block exceeds the 1024-thread device limit (elems_per_block " +
                      std::to_string(elems_per_block) + ")");
  if (mode == ExecMode::Parallel && workers < 1) throw DeviceError("workers must be >= 1");
  if (block_size < 32 || block_size > 1024 || block_size % 32) throw DeviceError("block_size must be a multiple of 32 in [32, 1024]");
}

CompiledKernel::CompiledKernel(const fem::WeakForm& wf, const LaunchConfig& cfg, Engine& eng) {
  cfg.validate();
  ff_form_desc d{};
  d.dim = wf.space.dim > 0 ? wf.space.dim : (wf.space.mesh ? wf.space.mesh->dim : 2);
  d.degree = wf.space.degree;
  d.quad_rule = cfg.quad_rule;
  d.strategy = static_cast<int>(cfg.strategy);
  d.block_size = cfg.block_size;
  const std::string bil = symbolic::print(wf.bilinear), lin = symbolic::print(wf.linear);
  d.bilinear = bil.c_str();
  d.linear = lin.c_str();
  ok(ff_form_create(eng.handle(), &d, &form_));
}
CompiledKernel::~CompiledKernel() { ff_form_destroy(form_); }

std::string CompiledKernel::source() const {
  std::size_t n = 0;
  ok(ff_form_source(form_, nullptr, 0, &n));
  std::string s(n + 1, '\0');
  ok(ff_form_source(form_, s.data(), s.size(), &n));
  s.resize(n);
  return s;
}

int CompiledKernel::registers() const {
  ff_form_info i{};
  ok(ff_form_info_get(form_, &i));
  return i.registers;
}

DeviceArrays::DeviceArrays(const fem::Mesh& m, const fem::DofMap& dofs, Engine& eng) {
  m.validate();
  const auto c = m.coords_flat();
  const auto v = m.conn_flat();
  const bool p1 = dofs.n_local == m.nodes_per_element();
  ok(ff_mesh_create(eng.handle(), m.dim, c.data(), m.node_count(), v.data(), m.element_count(),
                    p1 ? nullptr : dofs.dofs.data(), dofs.n_local, dofs.n_dofs, &mesh_));
  n_dofs_ = dofs.n_dofs;
  n_elems_ = m.element_count();
}
DeviceArrays::~DeviceArrays() { ff_mesh_destroy(mesh_); }

std::unique_ptr<DeviceArrays> flatten_mesh(const fem::Mesh& m, int degree) {
  return std::make_unique<DeviceArrays>(m, fem::lagrange_dofs(m, degree));
}

SparsityPattern::SparsityPattern(const DeviceArrays& d, std::int64_t rb, std::int64_t re, Engine& eng) {
  if (re < 0) re = d.n_dofs();
  ok(ff_pattern_build(eng.handle(), d.handle(), rb, re, &pat_));
  std::int32_t mx = 0;
  ok(ff_pattern_info(pat_, &n, &nnz, &mx));
  max_nz = mx;
  row_begin = rb;
}
SparsityPattern::~SparsityPattern() { ff_pattern_destroy(pat_); }

std::vector<std::int64_t> SparsityPattern::row_ptr() const {
  std::vector<std::int64_t> r(n + 1);
  ok(ff_pattern_export(pat_, r.data(), nullptr));
  return r;
}
std::vector<std::int32_t> SparsityPattern::col_idx() const {
  std::vector<std::int32_t> c(nnz);
  ok(ff_pattern_export(pat_, nullptr, c.data()));
  return c;
}
std::vector<int> SparsityPattern::row_len() const {
  std::vector<int> len(n), cols(n * max_nz);
  ok(ff_pattern_export_ell(pat_, max_nz, len.data(), cols.data()));
  return len;
}
std::vector<int> SparsityPattern::row_cols() const {
  std::vector<int> len(n), cols(n * max_nz);
  ok(ff_pattern_export_ell(pat_, max_nz, len.data(), cols.data()));
  return cols;
}

std::unique_ptr<SparsityPattern> build_sparsity(const DeviceArrays& d) { return std::make_unique<SparsityPattern>(d); }

CsrSystem assemble_csr(const CompiledKernel& k, const DeviceArrays& d, SparsityPattern& sp) {
  CsrSystem s;
  s.a.n = sp.n;
  s.a.row_ptr = sp.row_ptr();
  s.a.col_idx = sp.col_idx();
  s.a.values.resize(sp.nnz);
  s.b.resize(sp.n);
  ff_stats st{};
  ok(ff_assemble(k.handle(), d.handle(), sp.handle(), nullptr, nullptr, nullptr, s.a.values.data(), s.b.data(), &st));
  return s;
}

EllSystem assemble_sparse(const CompiledKernel& k, const DeviceArrays& d, SparsityPattern& sp, const LaunchConfig& cfg) {
  cfg.validate();
  if (sp.n != d.n_dofs())
    throw DeviceError("sparsity pattern is for a different mesh (" + std::to_string(sp.n) + " rows vs " +
                      std::to_string(d.n_dofs()) + " nodes)");
  CsrSystem c = assemble_csr(k, d, sp);
  EllSystem e;
  e.a.n = static_cast<int>(sp.n);
  e.a.max_nz = sp.max_nz;
  e.a.values.assign(static_cast<std::size_t>(sp.n) * sp.max_nz, 0.0);
  e.a.columns.assign(static_cast<std::size_t>(sp.n) * sp.max_nz, -1);
  for (std::int64_t i = 0; i < sp.n; ++i)
    for (std::int64_t t = c.a.row_ptr[i]; t < c.a.row_ptr[i + 1]; ++t) {
      e.a.values[i * sp.max_nz + (t - c.a.row_ptr[i])] = c.a.values[t];
      e.a.columns[i * sp.max_nz + (t - c.a.row_ptr[i])] = c.a.col_idx[t];
    }
  e.b = std::move(c.b);
  return e;
}

CsrSystem assemble(const fem::WeakForm& wf, const fem::Mesh& m, const LaunchConfig& cfg) {
  fem::WeakForm w = wf;
  w.space.dim = m.dim;
  CompiledKernel k(w, cfg);
  DeviceArrays d(m, wf.space.dofmap.dofs.empty() ? fem::lagrange_dofs(m, wf.space.degree) : wf.space.dofmap);
  SparsityPattern sp(d);
  return assemble_csr(k, d, sp);
}

}  // namespace femforge::device

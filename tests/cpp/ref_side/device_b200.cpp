// tests/cpp/ref_side/device_b200.cpp -- the reference-side binding of
// INTEGRATION.md §2, verbatim (tests/test_integration_doc.py keeps the two
// identical). Compiled by oracle/Makefile against the reference's headers and
// objects plus libfemforge_b200.so into oracle/_ref/test_integration, which
// tests/test_gpu_validation.py runs on the GPU.
// src/device/device_b200.cpp  (reference side; links -lfemforge_b200)
#include "femforge/device/device.hpp"
#include "femforge_b200.h"          // from femforge-b200/include

namespace femforge::device {

static void ff_ok(int rc) {
  if (rc == FF_OK) return;
  throw DeviceError(ff_last_error());     // same type + message as device.cpp:183-185, :286-287
}

// GPU assemble_sparse: same inputs as device.hpp:143-144, plus the weak form text
// that fem::instantiate consumed (the GPU generates its own element code from it).
EllSystem assemble_sparse_b200(const fem::WeakForm& wf, const fem::Mesh& mesh,
                               const SparsityPattern& sp, int device = 0) {
  ff_ctx* ctx = nullptr;
  ff_ok(ff_init(device, &ctx));
  const std::string bil = symbolic::print(wf.bilinear), lin = symbolic::print(wf.linear);
  ff_form_desc d{/*dim*/ 2, /*degree*/ 1, /*quad_rule*/ 3, /*strategy*/ FF_STRATEGY_AUTO,
                 /*block_size*/ 0, bil.c_str(), lin.c_str()};
  ff_form* form = nullptr;
  ff_ok(ff_form_create(ctx, &d, &form));
  std::vector<double> xy;  std::vector<int32_t> conn;
  for (const auto& p : mesh.nodes) { xy.push_back(p.x); xy.push_back(p.y); }
  for (const auto& e : mesh.elements) conn.insert(conn.end(), e.nodes.begin(), e.nodes.end());
  ff_mesh* m = nullptr;
  ff_ok(ff_mesh_create(ctx, 2, xy.data(), mesh.node_count(), conn.data(), mesh.element_count(),
                       nullptr, 3, mesh.node_count(), &m));
  ff_pattern* p = nullptr;
  ff_ok(ff_pattern_build(ctx, m, 0, mesh.node_count(), &p));
  int64_t nnz = 0;  ff_ok(ff_pattern_info(p, nullptr, &nnz, nullptr));
  std::vector<double> vals(nnz), rhs(sp.n);
  ff_stats st{};
  ff_ok(ff_assemble(form, m, p, xy.data(), conn.data(), nullptr, vals.data(), rhs.data(), &st));
  // CSR (GPU) -> the reference's ELL layout (linalg.hpp:26-42): same sorted columns as sp
  std::vector<int64_t> rp(sp.n + 1);  ff_ok(ff_pattern_export(p, rp.data(), nullptr));
  EllSystem out{linalg::EllMatrix(sp.n, sp.max_nz), std::move(rhs)};
  out.a.columns = sp.row_cols;  // identical sorted rows (bit-exact pattern parity)
  for (int i = 0; i < sp.n; ++i)
    for (int64_t s = rp[i]; s < rp[i + 1]; ++s) out.a.values[i * sp.max_nz + (s - rp[i])] = vals[s];
  ff_pattern_destroy(p); ff_mesh_destroy(m); ff_form_destroy(form); ff_ctx_destroy(ctx);
  return out;
}

}  // namespace femforge::device

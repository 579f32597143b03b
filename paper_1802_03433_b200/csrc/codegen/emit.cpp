// Source emission: the hand-written assembly template with the generated
// element body spliced in (the reference's template route, kernel.cpp:
// 290-449, made executable: the output is what NVRTC compiles).
#include <string>

#include "femforge/codegen.hpp"

namespace femforge::codegen {

namespace {

const char* const kAssemblyTemplate =
#include "../kernels/assemble_template.inc"
    ;

void fill(std::string& text, const std::string& key, const std::string& value) {
  const std::string tag = "{{" + key + "}}";
  const std::size_t at = text.find(tag);
  if (at == std::string::npos) throw CodegenError("missing placeholder " + tag);
  if (text.find(tag, at + 1) != std::string::npos) throw CodegenError("duplicate placeholder " + tag);
  text.replace(at, tag.size(), value);
}

}  // namespace

int RowTileParams::smem_bytes(int n_local, int slot_bytes) const {
  return 8 * acc + 8 * stage * n_local + 8 * stage + 8 * rows + 4 * 2 * (rows + 1) + 4 * 2 * stage +
         slot_bytes * stage * n_local;
}

RowTileParams rowtile_params(int n_local, int block_size) {
  RowTileParams p;
  p.chunk = block_size;
  if (n_local >= 10) {        // 3D P2: ~28 nnz/row
    p.acc = 6144, p.rows = 256, p.stage = 384;
  } else if (n_local >= 6) {  // 2D P2
    p.acc = 6144, p.rows = 512, p.stage = 512;
  } else if (n_local >= 4) {  // 3D P1: ~15 nnz/row
    p.acc = 6144, p.rows = 512, p.stage = 768;
  } else {                    // 2D P1: ~7 nnz/row
    p.acc = 4096, p.rows = 512, p.stage = 768;
  }
  return p;
}

std::string emit_source(const fem::InstantiatedForm& f, const LaunchParams& cfg) {
  return emit_source(f, cfg, nullptr);
}

std::string emit_source(const fem::InstantiatedForm& f, const LaunchParams& cfg, ElementPlan* plan_out) {
  if (cfg.elems_per_block <= 0 || cfg.max_nz <= 0 || cfg.n_quad <= 0 || cfg.n_local <= 0)
    throw CodegenError("missing placeholder value in launch parameters");
  if (cfg.block_size < 32 || cfg.block_size > 1024 || cfg.block_size % 32 != 0)
    throw CodegenError("block_size must be a multiple of 32 in [32, 1024]");
  if (cfg.slot_bytes != 1 && cfg.slot_bytes != 2) throw CodegenError("slot_bytes must be 1 or 2");
  const int rule_id = cfg.quad_rule > 0 ? cfg.quad_rule : default_quad_rule(f.dim, f.degree);
  const fem::QuadratureRule rule = fem::quadrature_rule(f.dim, rule_id);
  ElementPlan plan = plan_element(f, rule, cfg.strategy);
  std::string text = kAssemblyTemplate;
  fill(text, "SLOT_T", cfg.slot_bytes == 1 ? "unsigned char" : "unsigned short");
  fill(text, "DIM", std::to_string(f.dim));
  fill(text, "DEGREE", std::to_string(f.degree));
  fill(text, "NLOC", std::to_string(f.n_local));
  fill(text, "BLOCK", std::to_string(cfg.block_size));
  const RowTileParams tp = rowtile_params(f.n_local, cfg.block_size);
  fill(text, "TILE_ACC", std::to_string(tp.acc));
  fill(text, "TILE_ROWS", std::to_string(tp.rows));
  fill(text, "TILE_STAGE", std::to_string(tp.stage));
  std::string body = "  // element body: " + std::string(plan.strategy == Strategy::ReferenceTensor ? "reference-tensor" : "pointwise") +
                     " strategy, " + std::to_string(plan.n_quad) + "-point rule " + std::to_string(rule_id) + ", ~" +
                     std::to_string(plan.flops) + " flops\n" + plan.body;
  fill(text, "ELEMENT_BODY", body);
  // the row gather needs a reference-tensor plan and <= 12 slot bytes per record
  const bool gather = plan.n_kinv > 0 && f.n_local <= 12 && plan.n_kinv + f.n_local <= 24;
  fill(text, "NKINV", std::to_string(gather ? plan.n_kinv : 0));
  fill(text, "ROW_CODE", gather ? plan.row_code : std::string());
  {
    std::string d =
        "__device__ __forceinline__ void ff_gather_dispatch(int i, const FfRec& r, const double (&g)[FF_NKP],\n"
        "                                                   double* __restrict__ arow) {\n  switch (i) {\n";
    for (int i = 0; i < f.n_local; ++i)
      d += "    case " + std::to_string(i) + ": ff_gather_apply<" + std::to_string(i) + ">(r, g, arow); break;\n";
    d += "    default: break;\n  }\n}\n";
    fill(text, "ROW_DISPATCH", gather ? d : std::string());
  }
  if (text.find("{{") != std::string::npos) throw CodegenError("unresolved placeholder");
  if (plan_out) *plan_out = std::move(plan);
  return text;
}

}  // namespace femforge::codegen

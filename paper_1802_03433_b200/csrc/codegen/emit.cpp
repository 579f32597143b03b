// Source emission: the hand-written assembly template with the generated
// element body spliced in (the reference's template route, kernel.cpp:
// 290-449, made executable: the output is what NVRTC compiles).
#include <cstdlib>
#include <algorithm>
#include <sstream>
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

// Invariant loads for the element-record layout (FF_NFULL / FF_GTAIL /
// FF_GSTORE macros); shared by the form module (K2a, generic gather) and the
// class-specialised module so both read what K2a wrote.
const char* const kInvariantLoad = R"(// invariants of record e into t (scalar forms: FF_NFULL chunk arrays [E][4]
// and the tail array; vector forms: rows [E][FF_GS])
__device__ __forceinline__ void ff_load_inv(const double* __restrict__ einv, ff_i64 n, ff_i64 e, double (&t)[FF_GS]) {
#if FF_BS == 1
#pragma unroll
  for (int c = 0; c < FF_NFULL; ++c)
    ff_ld4(einv + (ff_i64)c * n * 4 + e * 4, t[4 * c], t[4 * c + 1], t[4 * c + 2], t[4 * c + 3]);
#if FF_GTAIL == 4
  ff_ld4(einv + (ff_i64)FF_NFULL * n * 4 + e * 4, t[4 * FF_NFULL], t[4 * FF_NFULL + 1], t[4 * FF_NFULL + 2],
         t[4 * FF_NFULL + 3]);
#elif FF_GTAIL == 2
  ff_ld2(einv + (ff_i64)FF_NFULL * n * 4 + e * 2, t[4 * FF_NFULL], t[4 * FF_NFULL + 1]);
  t[4 * FF_NFULL + 2] = 0.0;
  t[4 * FF_NFULL + 3] = 0.0;
#endif
#else
#pragma unroll
  for (int q = 0; q < FF_GS / 4; ++q) ff_ld4(einv + e * FF_GS + 4 * q, t[4 * q], t[4 * q + 1], t[4 * q + 2], t[4 * q + 3]);
#endif
}
)";

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
  fill(text, "BS", std::to_string(f.ncomp));
  fill(text, "BLOCK", std::to_string(cfg.block_size));
  std::string body = "  // element body: " + std::string(plan.strategy == Strategy::ReferenceTensor ? "reference-tensor" : "pointwise") +
                     " strategy, " + std::to_string(plan.n_quad) + "-point rule " + std::to_string(rule_id) + ", ~" +
                     std::to_string(plan.flops) + " flops\n" + plan.body;
  fill(text, "ELEMENT_BODY", body);
  fill(text, "ELEMENT_PRELUDE", plan.prelude);
  const bool gather = gather_capable(plan, f.n_local, f.ncomp, cfg.block_size);
  fill(text, "INVARIANT_LOAD", gather ? kInvariantLoad : "");
  fill(text, "NKINV", std::to_string(gather ? plan.n_kinv : 0));
  fill(text, "PAIR_TAIL", std::to_string(record_pair_tail(f.n_local)));
  fill(text, "ROW_CODE", gather ? plan.row_code : std::string());
  {
    // load-vector entries of the element record: identically zero entries are
    // not stored (config 5, f = (0, 0, -1): 20 of 30)
    const std::vector<int> sl = record_bslots(plan, f.n_local, f.ncomp);
    std::string t = "__constant__ int ff_bslot[FF_NLOC] = {";
    std::string st;
    for (int i = 0; i < f.n_local; ++i) {
      t += (i ? ", " : "") + std::to_string(sl[i]);
      if (sl[i] >= 0)
        st += "    __stcg(bs + (ff_i64)" + std::to_string(sl[i]) + " * n_elems + t, out[FF_NKINV + " + std::to_string(i) + "]);\n";
    }
    fill(text, "BSLOT", gather ? t + "};" : std::string());
    fill(text, "BSTORE", gather ? st : std::string());
  }
  {
    std::string d =
        "__device__ __forceinline__ void ff_gather_dispatch(int i, const FfRec& r, const double (&g)[FF_NKP], int d,\n"
        "                                                   double* __restrict__ arow) {\n  switch (i) {\n";
    for (int i = 0; i < f.n_local; ++i)
      d += "    case " + std::to_string(i) + ": ff_gather_apply<" + std::to_string(i) + ">(r, g, d, arow); break;\n";
    d += "    default: break;\n  }\n}\n";
    fill(text, "ROW_DISPATCH", gather ? d : std::string());
  }
  if (text.find("{{") != std::string::npos) throw CodegenError("unresolved placeholder");
  if (const char* v = std::getenv("FF_WAGG")) text = "#define FF_WAGG " + std::to_string(std::atoi(v) != 0) + "\n" + text;
  if (std::getenv("FF_NO_BPAD")) text = "#define FF_NO_BPAD 1\n" + text;  // tuning knob (both modules)
  if (plan_out) *plan_out = std::move(plan);
  return text;
}


// Tail of a scalar element record (n_kinv % 4 invariants): a pair array
// [E][2] when it holds <= 2 values and this returns 1, else a chunk array
// [E][4]. Pairs for P1 records (eight elements per line, C2 0.81 -> 0.80 ms);
// chunks for P2 (NS 2.57 -> 2.61 ms with pairs). FF_PAIR_TAIL=0/1 overrides
// (read by both modules of a process, so K2a and the class kernels agree).
int record_pair_tail(int n_local) {
  if (const char* v = std::getenv("FF_PAIR_TAIL")) return std::atoi(v) != 0 ? 1 : 0;
  return n_local <= 4 ? 1 : 0;
}

std::vector<int> record_bslots(const ElementPlan& plan, int n_local, int ncomp, int* n_soa) {
  // FF_NBPAD of the templates: scalar records whose invariants leave a
  // 4-chunk tail carry the first load-vector entries in its padding
  const int nk = plan.n_kinv;
  const int gtail = nk % 4 == 0 ? 0 : ((nk % 4 <= 2 && record_pair_tail(n_local)) ? 2 : 4);
  const int nbpad = (ncomp == 1 && gtail == 4 && !std::getenv("FF_NO_BPAD")) ? std::min(4 - nk % 4, n_local) : 0;
  std::vector<int> slot(n_local, -1);
  int k = 0;
  for (int i = nbpad; i < n_local; ++i)
    if (static_cast<int>(plan.b_zero.size()) != n_local || !plan.b_zero[i]) slot[i] = k++;
  if (n_soa) *n_soa = k;
  return slot;
}

bool gather_capable(const ElementPlan& plan, int n_local, int ncomp, int block_size) {
  // a reference-tensor plan and <= 12 slot bytes per record (node rows for
  // vector forms)
  (void)block_size;
  return plan.n_kinv > 0 && ncomp >= 1 && n_local / ncomp <= 12 &&
         (ncomp == 1 ? plan.n_kinv + n_local <= 24 : plan.n_bq > 0 && plan.n_kinv <= 96);
}

namespace {

// Peak number of row slots "open" (first contribution added, last not yet)
// when the class's incidences are accumulated in `order`.
int peak_live(const RowClass& k, int n_local, const std::vector<int>& order) {
  std::vector<int> first(k.len, -1), last(k.len, -1);
  for (int t = 0; t < static_cast<int>(order.size()); ++t)
    for (int j = 0; j < n_local; ++j) {
      const int sl = k.slots[order[t] * n_local + j];
      if (first[sl] < 0) first[sl] = t;
      last[sl] = t;
    }
  int live = 0, peak = 0;
  for (int t = 0; t < static_cast<int>(order.size()); ++t) {
    for (int sl = 0; sl < k.len; ++sl) live += first[sl] == t;
    peak = std::max(peak, live);
    for (int sl = 0; sl < k.len; ++sl) live -= last[sl] == t;
  }
  return peak;
}

}  // namespace

// Incidence order of a class that keeps few row slots open at once: a slot's
// register is live from its first to its last contribution, then the value
// goes to the staging row. Greedy (fewest newly opened slots) from every
// start, then a fixed-seed swap search; deterministic, so the source is too.
// P2 Kuhn vertex rows (65 slots, 24 incidences): 23-26 live instead of 65.
std::vector<int> class_step_order(const RowClass& k, int n_local) {
  const int n = k.steps;
  std::vector<int> best(n);
  for (int q = 0; q < n; ++q) best[q] = q;
  if (n < 2) return best;
  int bv = peak_live(k, n_local, best);
  for (int start = 0; start < n; ++start) {
    std::vector<int> order{start};
    std::vector<char> used(n, 0), seen(k.len, 0);
    used[start] = 1;
    for (int j = 0; j < n_local; ++j) seen[k.slots[start * n_local + j]] = 1;
    while (static_cast<int>(order.size()) < n) {
      int pick = -1, pc = 1 << 30;
      for (int q = 0; q < n; ++q) {
        if (used[q]) continue;
        int c = 0;
        for (int j = 0; j < n_local; ++j) c += !seen[k.slots[q * n_local + j]];
        if (c < pc) pc = c, pick = q;
      }
      used[pick] = 1;
      order.push_back(pick);
      for (int j = 0; j < n_local; ++j) seen[k.slots[pick * n_local + j]] = 1;
    }
    const int v = peak_live(k, n_local, order);
    if (v < bv) bv = v, best = order;
  }
  uint64_t rng = 0x9e3779b97f4a7c15ull;
  const int iters = n <= 8 ? 2000 : 20000;
  for (int it = 0; it < iters; ++it) {
    rng = rng * 6364136223846793005ull + 1442695040888963407ull;
    const int a = static_cast<int>((rng >> 33) % n), b = static_cast<int>((rng >> 13) % n);
    if (a == b) continue;
    std::swap(best[a], best[b]);
    const int v = peak_live(k, n_local, best);
    if (v <= bv)
      bv = v;
    else
      std::swap(best[a], best[b]);
  }
  return best;
}

int vector_stage_pitch(const std::vector<RowClass>& classes, int bs, int kernel, bool fused) {
  int m = 1;
  for (const auto& c : classes)
    if (fused || (c.len > 33) == (kernel == 1)) m = std::max(m, bs * c.len + 1);  // + 1: TMA parity shift
  while (m % 16 != bs % 16) ++m;  // FF_SP3 = bs (mod 16): conflict-free staging stores
  return m;
}

int class_stage_pitch(const std::vector<RowClass>& classes, int kernel, bool fused, int bs) {
  int m = 1;
  if (bs > 1) {  // vector forms: whole rows staged (no chunks), one kernel
    for (const auto& c : classes) m = std::max(m, c.len);
    return m | 1;
  }
  for (const auto& c : classes)
    if (fused || (c.len > 33) == (kernel == 1)) m = std::max(m, c.len);
  // rows longer than 33 are staged in chunks of 32 in finalisation order
  return std::min(m, 33) | 1;  // odd: conflict-free lane-row stores
}

std::string emit_class_source(const ElementPlan& plan, int n_local, const std::vector<RowClass>& classes, bool fused,
                              int bs, int pre) {
  if (pre < 1 || pre > 8) throw CodegenError("class source: record prefix must be 1..8 steps");
  for (const auto& c : classes)
    if (c.steps < pre) throw CodegenError("class source: a class has fewer steps than the record prefix");
  if (plan.n_kinv <= 0) throw CodegenError("row classes need a reference-tensor plan");
  if (bs < 1 || n_local % bs) throw CodegenError("class source: bad component count");
  if (bs > 1 && plan.n_bq <= 0) throw CodegenError("class source: vector forms need a block-uniform record");
  // classes are over (node) rows with nsc slots per incidence; vector forms
  // run the three trial components of a row in neighbouring lanes (vclass_fn)
  const int nsc = n_local / bs, nb = bs * bs;
  const std::vector<int> bslot = record_bslots(plan, n_local, bs);  // load-vector record slots
  std::ostringstream os;
  const int nkp = plan.n_kinv + (plan.n_kinv & 1);
  const int erec = (plan.n_kinv + n_local + 1) & ~1;
  if (std::getenv("FF_NO_BPAD")) os << "#define FF_NO_BPAD 1\n";  // tuning knob (both modules)
  os << "#define FF_PRE " << pre << "\n";
  os << "// femforge-b200 class-specialised row gather (generated per (form, gather plan));\n"
        "// every class row stays in registers, indexed by compile-time slots.\n"
        "typedef long long ff_i64;\ntypedef int ff_i32;\n"
     << "#define FF_NLOC " << n_local << "\n#define FF_BS " << bs << "\n#define FF_NB " << nb
     << "\n#define FF_NKINV " << plan.n_kinv << "\n#define FF_NKP " << nkp
     << "\n#define FF_EREC " << erec << "\n#define FF_GS " << ((plan.n_kinv + 3) / 4) * 4 << "\n"
     << "#define FF_NFULL (FF_NKINV / 4)\n#define FF_PAIR_TAIL " << record_pair_tail(n_local) << "\n"
     << "#define FF_GTAIL (FF_NKINV % 4 == 0 ? 0 : ((FF_NKINV % 4 <= 2 && FF_PAIR_TAIL) ? 2 : 4))\n"
     << "#if FF_BS == 1\n#define FF_GSTORE (4 * FF_NFULL + FF_GTAIL)\n#else\n#define FF_GSTORE FF_GS\n#endif\n"
     << "#if FF_BS == 1 && FF_GTAIL == 4 && !defined(FF_NO_BPAD)\n"
        "#define FF_NBPAD ((4 - FF_NKINV % 4) < FF_NLOC ? (4 - FF_NKINV % 4) : FF_NLOC)\n#else\n#define FF_NBPAD 0\n#endif\n"
     << "// staging pitches of the two kernels (odd: conflict-free lane-row stores)\n"
     << "#define FF_SP_S " << class_stage_pitch(classes, 0, fused, bs) << "\n#define FF_SP_L "
     << class_stage_pitch(classes, 1, fused, bs) << "\n#define FF_SP3_S " << vector_stage_pitch(classes, bs, 0, fused)
     << "\n#define FF_SP3_L " << vector_stage_pitch(classes, bs, 1, fused)
     << "\n"
     << "// per-warp staging tiles (doubles; even: every tile starts 16-byte aligned)\n"
     << "#define FF_TILE3_S (((32 / FF_BS + 1) * FF_SP3_S + 1) & ~1)\n"
     << "#define FF_TILE3_L (((32 / FF_BS + 1) * FF_SP3_L + 1) & ~1)\n"
     << "template <int I>\n__device__ __forceinline__ void ff_row(const double* __restrict__ g, double* __restrict__ v);\n"
     << plan.row_code
     << R"(
// element records through L1: in first-touch order the lanes of a step read
// neighbouring records (2.095 -> 2.082 ms at the north star against the
// round-1 L1::no_allocate stream)
__device__ __forceinline__ void ff_ld4(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void ff_ld2(const double* p, double& a, double& b) {
  asm("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
}
__device__ __forceinline__ double ff_ld1(const double* p) { return __ldg(p); }
#if defined(FF_ABL) && (FF_ABL & 8)  // ablation (timing analysis only; results wrong)
#define ff_ld1(p) (1.0)
#endif
// record id loads (FF_ABL & 4: synthetic ids, ablation only)
__device__ __forceinline__ int ff_ldid(const ff_i32* p) {
#if defined(FF_ABL) && (FF_ABL & 4)
  return (int)(((unsigned long long)p >> 7) & 0xfffff);
#else
  return __ldcs(p);
#endif
}
)" << kInvariantLoad << R"(
// element record: invariants (ff_load_inv), load vector [FF_NLOC][E]
// (idle lanes, e < 0, only occur in rows that are never written: they read
// element 0 instead of branching)
// (sl: the entry's slot in the record's load-vector array, -1: zero entry)
__device__ __forceinline__ void ff_cload(int e, int i, int sl, const double* __restrict__ einv, ff_i64 n_elems,
                                         double (&g)[FF_NKP], double& b) {
  const ff_i64 ee = e >= 0 ? e : 0;
  double t[FF_GS];
#if defined(FF_ABL) && (FF_ABL & 2)  // ablation (timing analysis only; results wrong)
#pragma unroll
  for (int q = 0; q < FF_GS; ++q) t[q] = (double)(ee + q);
  if (ee == -7) ff_load_inv(einv, n_elems, ee, t);
#else
  ff_load_inv(einv, n_elems, ee, t);
#endif
#pragma unroll
  for (int q = 0; q < FF_NKP; ++q) g[q] = q < FF_GS ? t[q < FF_GS ? q : 0] : 0.0;
  // entries b_0 .. b_{FF_NBPAD-1} came with the invariants (chunk-tail padding)
  b = i < FF_NBPAD ? t[FF_NKINV + (i < FF_NBPAD ? i : 0)]
                   : (sl < 0 ? 0.0 : ff_ld1(einv + n_elems * FF_GSTORE + (ff_i64)sl * n_elems + ee));
}
// FF_PRE: record ids of an item loaded with its header (the plan's pre_steps)
#ifndef FF_WUNROLL
#define FF_WUNROLL 32  // write-out loop unroll (NS 2.484 vs 2.514 ms with 4, run 94)
#endif
constexpr int ff_wunroll = FF_WUNROLL;  // (#pragma unroll takes a constant expression, not a macro)
// CSR value stores of the scalar write-out: streaming (evict-first), rows are
// written whole (vector forms write their rows by TMA, ff_vwriteout)
__device__ __forceinline__ void ff_stv(double* p, double v) {
#if FF_BS == 1
  __stcs(p, v);
#else
  *p = v;
#endif
}
// staged rows -> CSR values: flat index f over 32 rows x cnt slots, so
// consecutive lanes write consecutive values of one row. Shared by every
// class (one copy, not unrolled: keeps the instruction footprint small).
__device__ __noinline__ void ff_writeout(const double* __restrict__ st, int sp, const ff_i64* __restrict__ sr,
                                         int lane, int cnt, int q0, double* __restrict__ values) {
#if defined(FF_ABL) && (FF_ABL & 1)  // ablation (timing analysis only; results wrong)
  if (lane < 0) values[0] = st[0];
  return;
#endif
  __syncwarp();
  if (lane < cnt) {
#pragma unroll ff_wunroll
    for (int m = 0; m < 32; ++m) {
      const ff_i64 rb = sr[m];
#if defined(FF_ABL) && (FF_ABL & 16)  // ablation: the same stores into a 2 MB window (no DRAM writes)
      if (rb >= 0) ff_stv(values + ((rb + FF_BS * (q0 + lane)) & 0x3FFFF), st[m * sp + lane]);
#else
      if (rb >= 0) ff_stv(values + rb + FF_BS * (q0 + lane), st[m * sp + lane]);
#endif
    }
  }
  __syncwarp();
}
// chunk of a long row staged in finalisation order: lane l of the chunk
// holds the row's slot map[l]
__device__ __noinline__ void ff_writeout_map(const double* __restrict__ st, int sp, const ff_i64* __restrict__ sr,
                                             int lane, int cnt, const unsigned char* __restrict__ map,
                                             double* __restrict__ values) {
  __syncwarp();
  if (lane < cnt) {
    const int off = __ldg(map + lane);
#pragma unroll ff_wunroll
    for (int m = 0; m < 32; ++m) {
      const ff_i64 rb = sr[m];
#if defined(FF_ABL) && (FF_ABL & 16)
      if (rb >= 0) ff_stv(values + ((rb + FF_BS * off) & 0x3FFFF), st[m * sp + lane]);
#else
      if (rb >= 0) ff_stv(values + rb + FF_BS * off, st[m * sp + lane]);
#endif
    }
  }
  __syncwarp();
}

#if FF_BS > 1
// vector forms: lane = (row lane / FF_BS, trial component d = lane % FF_BS);
// quantities of component block (c, d) at the even record offset dq:
// FF_NBQ / 2 16-byte loads (no lane-dependent shuffling of a chunk)
__device__ __forceinline__ void ff_vload(int e, int dq, int sl, const double* __restrict__ einv, ff_i64 n_elems,
                                         double (&g)[FF_NBQ], double& b) {
  const ff_i64 ee = e >= 0 ? e : 0;
  const double* p = einv + ee * FF_GS + dq;
#if defined(FF_ABL) && (FF_ABL & 2)  // ablation (timing analysis only; results wrong)
#pragma unroll
  for (int k = 0; k < FF_NBQ; ++k) g[k] = (double)(ee + k);
  if (ee == -7) ff_ld2(p, g[0], g[1]);
#else
#pragma unroll
  for (int k = 0; k < FF_NBQ; k += 2) ff_ld2(p + k, g[k], g[k + 1]);
#endif
  b = sl < 0 ? 0.0 : ff_ld1(einv + n_elems * FF_GSTORE + (ff_i64)sl * n_elems + ee);
}
// the warp's staging tile holds its rows in CSR order: row r (lanes
// FF_BS r .. FF_BS r + FF_BS - 1) at r * SP3 + parity, value FF_BS * slot + d
// (SP3 = FF_BS mod 16: the lane stores of one slot hit distinct banks; the
// parity gives staging and CSR start the same 16-byte phase). Write-out: lane
// r sends row r, the odd head / tail value by a plain store, the rest by one
// cp.async.bulk (TMA): whole rows, every sector written once (config 5: 30.0
// vs 30.45 ms with a coalesced store loop)
template <int LEN, int SP3>
__device__ __noinline__ void ff_vwriteout(const double* __restrict__ st, const ff_i64* __restrict__ sr, int lane,
                                          double* __restrict__ values) {
#if defined(FF_ABL) && (FF_ABL & 1)  // ablation (timing analysis only; results wrong)
  if (lane < 0) values[0] = st[0];
  return;
#endif
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane < 32 / FF_BS) {
    const ff_i64 rb = sr[FF_BS * lane];
    if (rb >= 0) {
      constexpr int n = FF_BS * LEN;
      const int o = lane * SP3 + (int)((rb ^ (ff_i64)(lane * SP3)) & 1);
      const double* in = st + o;
      double* out = values + rb;
      const int a = (int)(rb & 1);
      if (a) out[0] = in[0];
      const int m = (n - a) & ~1;
      if (m > 0) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(in + a);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + a), "r"(sa),
                     "r"(m * 8) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if ((n - a) & 1) out[n - 1] = in[n - 1];
      if (m > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
  __syncwarp();
}
#endif

#ifndef FF_CWARPS
#define FF_CWARPS 4  // warps per CTA
#endif

#ifndef FF_MINB_S
#define FF_MINB_S 4  // CTAs per SM the register budgets are sized for
#endif
#ifndef FF_MINB_L
#define FF_MINB_L 2
#endif
)";
  // class c with rows of <= 33 entries -> ff_gather_classes_s, else _l; fused:
  // every class in _s (rows longer than 33 entries staged in chunks)
  auto is_long = [&](int c) { return !fused && classes[c].len > 33; };
  auto class_fn = [&](int c) {
    const RowClass& k = classes[c];
    const char* sp = is_long(c) ? "FF_SP_L" : "FF_SP_S";
    const int n_local = nsc;  // slots per incidence
    // one pass over the incidences in class_step_order: each element record
    // is loaded once; a slot's register opens at its first contribution and
    // goes to the staging row after its last one
    // the plan lays the items' records out in this order (RowClass::order);
    // record position t holds template step order[t]
    const std::vector<int> order = k.order.empty() ? class_step_order(k, n_local) : k.order;
    std::vector<int> first(k.len, -1), last(k.len, -1);
    for (int t = 0; t < k.steps; ++t)
      for (int j = 0; j < n_local; ++j) {
        const int sl = k.slots[order[t] * n_local + j];
        if (first[sl] < 0) first[sl] = t;
        last[sl] = t;
      }
    // staging position of every slot: the slot index when the row fits one
    // staging row, else its finalisation rank (chunks of 32 written out as
    // soon as they are complete, lanes in ascending slot order inside a chunk)
    const bool chunked = k.len > 33;
    // fin: finalisation rank (chunk = fin / 32); pos: position inside the
    // chunk's staging row (ascending slot order)
    std::vector<int> pos(k.len), fin(k.len), slot_at(k.len);
    for (int sl = 0; sl < k.len; ++sl) pos[sl] = fin[sl] = sl;
    if (chunked) {
      std::vector<int> byfin(k.len);
      for (int sl = 0; sl < k.len; ++sl) byfin[sl] = sl;
      std::stable_sort(byfin.begin(), byfin.end(), [&](int a, int b) { return last[a] < last[b]; });
      for (int r = 0; r < k.len; ++r) fin[byfin[r]] = r;
      for (int c0 = 0; c0 < k.len; c0 += 32)
        std::sort(byfin.begin() + c0, byfin.begin() + std::min(k.len, c0 + 32));
      for (int r = 0; r < k.len; ++r) pos[byfin[r]] = r;
    }
    for (int sl = 0; sl < k.len; ++sl) slot_at[pos[sl]] = sl;
    if (chunked) {
      os << "__device__ const unsigned char ff_cmap_" << c << "[" << k.len << "] = {";
      for (int r = 0; r < k.len; ++r) os << (r ? ", " : "") << slot_at[r];
      os << "};\n";
    }
    for (int cd = 0; cd < nb; ++cd) {
    const int cc = cd / bs, dd = cd % bs;
    os << "// class " << c << " (components " << cc << ", " << dd << "): " << k.len << " entries, " << k.steps
       << " incidences, at most " << peak_live(k, n_local, order) << " open\n"
       << "__device__ __forceinline__ void ff_cls_" << c << "_" << cd
       << "(const int (&ep)[FF_PRE], const ff_i32* __restrict__ rec,\n"
          "    const double* __restrict__ einv, ff_i64 n_elems,\n"
          "    double* __restrict__ st, ff_i64* __restrict__ sr, int lane, ff_i64 rbeg, int row,\n"
          "    double* __restrict__ values, double* __restrict__ rhs) {\n"
          "  int e[" << std::max(k.steps, 1) << "];\n";
    for (int t = 0; t < k.steps; ++t) {
      if (t < pre)
        os << "  e[" << order[t] << "] = ep[" << t << "];\n";
      else
        os << "  e[" << order[t] << "] = ff_ldid(rec + " << (t - pre) * 32 << ");\n";
    }
    if (dd == 0) os << "  double bs = 0.0;\n";
    for (int sl = 0; sl < k.len; ++sl) os << (sl % 16 ? ", a" : (sl ? ";\n  double a" : "  double a")) << sl;
    os << ";\n";
    // the lane's CSR row start goes to shared memory right before the first
    // write-out that reads it (it depends on the row_ptr load, which should not
    // hold up the staging stores before it)
    bool sr_done = false;
    auto store_sr = [&](const char* indent) {
      if (sr_done) return;
      sr_done = true;
      os << indent << "sr[lane] = row >= 0 ? FF_NB * rbeg + " << static_cast<long long>(bs) * cc * k.len + dd
         << " : -1;\n";
    };
    // record loads in flight per batch (registers: depth x the record size)
    const char* dk = bs == 1 ? std::getenv("FF_SDEPTH") : std::getenv("FF_VDEPTH");
    // (scalar forms: 9 -- NS 1.857 ms against 1.905 / 1.861 / 1.868 for 8 / 7 / 10,
    // C3 0.807 vs 0.828 for 8)
    const int depth = dk ? std::max(1, std::atoi(dk)) : (bs == 1 ? 9 : 2);
    for (int t0 = 0; t0 < k.steps; t0 += depth) {
      const int t1 = std::min(k.steps, t0 + depth);
      os << "  {\n";
      for (int t = t0; t < t1; ++t) {
        const int q = order[t];
        os << "    double g" << q << "[FF_NKP], b" << q << "; ff_cload(e[" << q << "], " << k.local[q] * bs + cc
             << ", " << bslot[k.local[q] * bs + cc] << ", einv, n_elems, g" << q << ", b" << q << ");\n";
      }
      for (int t = t0; t < t1; ++t) {
        const int q = order[t];
        os << "    { double v[FF_NLOC]; ff_row<" << k.local[q] * bs + cc << ">(g" << q << ", v);";
        for (int j = 0; j < n_local; ++j) {
          const int sl = k.slots[q * n_local + j];
          os << " a" << sl << (first[sl] == t ? " = v[" : " += v[") << j * bs + dd << "];";
        }
        if (!chunked) {
          for (int j = 0; j < n_local; ++j) {
            const int sl = k.slots[q * n_local + j];
            if (last[sl] == t) os << " st[lane * " << sp << " + " << sl << "] = a" << sl << ";";
          }
        } else {
          std::vector<int> closing;  // finalisation ranks closing at step t
          for (int j = 0; j < n_local; ++j)
            if (last[k.slots[q * n_local + j]] == t) closing.push_back(fin[k.slots[q * n_local + j]]);
          std::sort(closing.begin(), closing.end());
          std::vector<int> slot_of_fin(k.len);
          for (int sl = 0; sl < k.len; ++sl) slot_of_fin[fin[sl]] = sl;
          for (int f : closing) {
            const int sl = slot_of_fin[f];
            os << " st[lane * " << sp << " + " << pos[sl] % 32 << "] = a" << sl << ";";
            if (f % 32 == 31 || f == k.len - 1) {  // chunk f / 32 complete
              os << "\n";
              store_sr("      ");
              os << "      ff_writeout_map(st, " << sp << ", sr, lane, " << f % 32 + 1 << ", ff_cmap_" << c << " + "
                 << f - f % 32 << ", values);";
            }
          }
        }
        os << " }\n";
        if (dd == 0) os << "    bs += b" << q << ";\n";
      }
      os << "  }\n";
    }
    // write-out through the staging rows (consecutive lanes = consecutive CSR
    // values of one row)
    if (!chunked) store_sr("  ");
    if (!chunked)
      for (int q0 = 0; q0 < k.len; q0 += 32)
        os << "  ff_writeout(st + " << q0 << ", " << sp << ", sr, lane, " << std::min(32, k.len - q0) << ", " << q0
           << ", values);\n";
    if (dd == 0) os << "  if (row >= 0) __stcs(rhs + FF_BS * row + " << cc << ", bs);\n";
    os << "}\n";
    }  // component pairs
  };
  // vector forms: one function per (class, test component cc); the lanes of
  // a row carry its FF_BS trial components (data: the block's quantity offset)
  auto vclass_fn = [&](int c) {
    const RowClass& k = classes[c];
    const char* sp3 = is_long(c) ? "FF_SP3_L" : "FF_SP3_S";
    const std::vector<int> order = k.order.empty() ? class_step_order(k, nsc) : k.order;
    std::vector<int> last(k.len, -1), first(k.len, -1);
    for (int t = 0; t < k.steps; ++t)
      for (int j = 0; j < nsc; ++j) {
        const int sl = k.slots[order[t] * nsc + j];
        if (first[sl] < 0) first[sl] = t;
        last[sl] = t;
      }
    for (int cc = 0; cc < bs; ++cc) {
      os << "// class " << c << " (test component " << cc << "): " << k.len << " entries, " << k.steps
         << " incidences\n"
         << "__device__ __forceinline__ void ff_cls_" << c << "_" << cc
         << "(const int (&ep)[FF_PRE], const ff_i32* __restrict__ rec, const double* __restrict__ einv, ff_i64 n_elems,\n"
            "    double* __restrict__ st, double* __restrict__ stl, ff_i64* __restrict__ sr, int lane, int dq, ff_i64 rbeg,\n"
            "    int row,\n"
            "    double* __restrict__ values, double* __restrict__ rhs) {\n"
            "  int e[" << std::max(k.steps, 1) << "];\n";
      for (int t = 0; t < k.steps; ++t) {
        if (t < pre)
          os << "  e[" << order[t] << "] = ep[" << t << "];\n";
        else
          os << "  e[" << order[t] << "] = ff_ldid(rec + " << (t - pre) * 32 << ");\n";
      }
      os << "  double bs = 0.0;\n"
         << "  // the row's staging at the parity of its CSR start (TMA write-out)\n"
         << "  stl += (int)(((FF_NB * rbeg + " << static_cast<long long>(bs) * cc * k.len
         << ") ^ (ff_i64)((lane / FF_BS) * " << sp3 << ")) & 1);\n";
      for (int sl = 0; sl < k.len; ++sl) os << (sl % 16 ? ", a" : (sl ? ";\n  double a" : "  double a")) << sl;
      os << ";\n";
      const char* dk = std::getenv("FF_VDEPTH");
      const int depth = dk ? std::max(1, std::atoi(dk)) : 4;
      for (int t0 = 0; t0 < k.steps; t0 += depth) {
        const int t1 = std::min(k.steps, t0 + depth);
        os << "  {\n";
        for (int t = t0; t < t1; ++t) {
          const int q = order[t];
          os << "    double g" << q << "[FF_NBQ], b" << q << "; ff_vload(e[" << q << "], dq, "
             << bslot[k.local[q] * bs + cc] << ", einv, n_elems, g" << q << ", b" << q << ");\n";
        }
        for (int t = t0; t < t1; ++t) {
          const int q = order[t];
          os << "    { double v[" << nsc << "]; ff_vrow<" << k.local[q] << ">(g" << q << ", v);";
          for (int j = 0; j < nsc; ++j) {
            const int sl = k.slots[q * nsc + j];
            os << " a" << sl << (first[sl] == t ? " = v[" : " += v[") << j << "];";
          }
          for (int j = 0; j < nsc; ++j) {
            const int sl = k.slots[q * nsc + j];
            if (last[sl] == t) os << " stl[" << bs * sl << "] = a" << sl << ";";
          }
          os << " }\n    bs += b" << q << ";\n";
        }
        os << "  }\n";
      }
      os << "  sr[lane] = row >= 0 ? FF_NB * rbeg + " << static_cast<long long>(bs) * cc * k.len << " : -1;\n"
         << "  ff_vwriteout<" << k.len << ", " << sp3 << ">(st, sr, lane, values);\n"
         << "  if (row >= 0 && lane % FF_BS == 0) __stcs(rhs + FF_BS * row + " << cc << ", bs);\n}\n";
    }
  };
  for (int c = 0; c < static_cast<int>(classes.size()); ++c) {
    if (bs > 1)
      vclass_fn(c);
    else
      class_fn(c);
  }

  auto kernel = [&](const char* name, bool longrows) {
    os << "// items of one launch: one item per warp, CTAs in item order;\n"
          "// items are sorted by (Morton window, class): a CTA runs one class (small\n"
          "// instruction footprint per SM) and the items in flight stay spatially\n"
          "// compact (element data reused in L1/L2)\n"
          "extern \"C\" __global__ void __launch_bounds__(32 * FF_CWARPS, "
       << (longrows ? "FF_MINB_L" : "FF_MINB_S") << ")\n" << name
       << "(const double* __restrict__ einv, ff_i64 n_elems, const ff_i64* __restrict__ row_ptr,\n"
          "    double* __restrict__ values, double* __restrict__ rhs, const ff_i32* __restrict__ citem_class,\n"
          "    const ff_i32* __restrict__ citem_rows, const ff_i64* __restrict__ citem_rec,\n"
          "    const ff_i32* __restrict__ crec, ff_i64 i0, ff_i64 i1) {\n"
          "  // dynamic shared memory: 4 staging tiles [32][FF_SP] + 4 x 32 row offsets\n"
          "  extern __shared__ double ff_dsm[];\n"
          "  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;\n"
          "  double* st = ff_dsm + wid * 32 * " << (longrows ? "FF_SP_L" : "FF_SP_S") << ";\n"
          "  ff_i64* sr = (ff_i64*)(ff_dsm + FF_CWARPS * 32 * " << (longrows ? "FF_SP_L" : "FF_SP_S") << ") + wid * 32;\n"
          "  // vector forms: FF_NB consecutive CTAs run the same items, one component\n"
          "  // pair each (one code path per CTA; the items' records shared in L2, and\n"
          "  // the pairs' stride-FF_BS writes to one CSR line meet in L2 -- slabs of\n"
          "  // 16/64/256 CTAs per pair measured 62.5/63.4/71.7 vs 62.5 ms at config 5)\n"
          "  const int cd = (int)(blockIdx.x % FF_NB);\n"
          "  const ff_i64 ff_cta = blockIdx.x / FF_NB;\n"
          "  // one class item per warp (CTAs launch in item order, so the items in\n"
          "  // flight stay contiguous): nothing carried across items -- two items per\n"
          "  // warp with a two-stage item pipeline measured 2.053 vs 2.013 ms, a\n"
          "  // persistent grid 3.2-3.6 ms at the north star\n"
          "  const ff_i64 w = i0 + ff_cta * FF_CWARPS + wid;\n"
          "  if (w >= i1) return;\n"
          "  // the item's first FF_PRE record ids sit at a position computable from the\n"
          "  // item index, so they load together with the item header (every class\n"
          "  // has >= FF_PRE steps); its other steps follow from citem_rec\n"
          "  // (the record ids first: their loads must not queue behind the first\n"
          "  // use of the header; the row start loads unpredicated for the same reason)\n"
          "  int ep[FF_PRE];\n"
          "#pragma unroll\n"
          "  for (int u = 0; u < FF_PRE; ++u) ep[u] = ff_ldid(crec + (w * FF_PRE + u) * 32 + lane);\n"
          "  const int c = __ldg(citem_class + w);\n"
          "  const int row = __ldg(citem_rows + w * 32 + lane);\n"
          "  const ff_i32* rec = crec + __ldg(citem_rec + w) * 32 + lane;\n"
          "  const ff_i64 rbeg = __ldg(row_ptr + (row >= 0 ? row : 0));\n"

          "  {\n"
          "    switch (c * FF_NB + cd) {\n";
    for (int c = 0; c < static_cast<int>(classes.size()); ++c)
      if (is_long(c) == longrows)
        for (int cd = 0; cd < nb; ++cd)
          os << "      case " << c * nb + cd << ": ff_cls_" << c << "_" << cd
             << "(ep, rec, einv, n_elems, st, sr, lane, rbeg, row, values, rhs); break;\n";
    os << "      default: break;\n    }\n"
          "  }\n}\n";
  };
  auto vkernel = [&](const char* name, bool longrows) {
    const std::string sp3 = longrows ? "FF_SP3_L" : "FF_SP3_S", tile = longrows ? "FF_TILE3_L" : "FF_TILE3_S";
    os << "// vector forms: FF_BS consecutive CTAs run the same items, one test\n"
          "// component each; lane = (row lane / FF_BS, trial component lane % FF_BS)\n"
          "extern \"C\" __global__ void __launch_bounds__(32 * FF_CWARPS, " << (longrows ? "FF_MINB_L" : "FF_MINB_S")
       << ")\n" << name
       << "(const double* __restrict__ einv, ff_i64 n_elems, const ff_i64* __restrict__ row_ptr,\n"
          "    double* __restrict__ values, double* __restrict__ rhs, const ff_i32* __restrict__ citem_class,\n"
          "    const ff_i32* __restrict__ citem_rows, const ff_i64* __restrict__ citem_rec,\n"
          "    const ff_i32* __restrict__ crec, ff_i64 i0, ff_i64 i1) {\n"
          "  extern __shared__ __align__(16) double ff_dsm[];\n"
          "  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;\n"
          "  double* st = ff_dsm + wid * " << tile << ";\n"
          "  double* stl = st + (lane / FF_BS) * " << sp3 << " + lane % FF_BS;  // idle lanes: a spare row\n"
          "  ff_i64* sr = (ff_i64*)(ff_dsm + FF_CWARPS * " << tile << ") + wid * 32;\n"
          "  const int cc = (int)(blockIdx.x % FF_BS);\n"
          "  const ff_i64 w = i0 + (ff_i64)(blockIdx.x / FF_BS) * FF_CWARPS + wid;\n"
          "  if (w >= i1) return;\n"
          "  int ep[FF_PRE];\n"
          "#pragma unroll\n"
          "  for (int u = 0; u < FF_PRE; ++u) ep[u] = ff_ldid(crec + (w * FF_PRE + u) * 32 + lane);\n"
          "  const int c = __ldg(citem_class + w);\n"
          "  const int row = __ldg(citem_rows + w * 32 + lane);\n"
          "  const ff_i32* rec = crec + __ldg(citem_rec + w) * 32 + lane;\n"
          "  const ff_i64 rbeg = __ldg(row_ptr + (row >= 0 ? row : 0));\n"
          "  const int dq = ff_block_q[cc * FF_BS + lane % FF_BS];\n"
          "  switch (c * FF_BS + cc) {\n";
    for (int c = 0; c < static_cast<int>(classes.size()); ++c)
      if (is_long(c) == longrows)
      for (int cc = 0; cc < bs; ++cc)
        os << "    case " << c * bs + cc << ": ff_cls_" << c << "_" << cc
           << "(ep, rec, einv, n_elems, st, stl, sr, lane, dq, rbeg, row, values, rhs); break;\n";
    os << "    default: break;\n  }\n}\n";
  };
  if (bs > 1) {
    vkernel("ff_gather_classes_s", false);
    vkernel("ff_gather_classes_l", true);
    return os.str();
  }
  kernel("ff_gather_classes_s", false);
  kernel("ff_gather_classes_l", true);
  return os.str();
}

}  // namespace femforge::codegen

// The C ABI (include/femforge_b200.h): handles, error translation, and the
// host orchestration of K0 (zero-fill), K1 (pattern), the slot plan and K2
// (the NVRTC element kernel with its scatter).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <string>

#include "../kernels/kernels.hpp"
#include "femforge/codegen.hpp"
#include "femforge/fem.hpp"
#include "femforge/meshgen.hpp"
#include "femforge/symbolic.hpp"
#include "femforge_b200.h"
#include "../runtime/runtime.hpp"

using namespace femforge;
using ffb::Error;

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return FF_OK;
  } catch (const Error& e) {
    g_error = e.what();
    return e.code;
  } catch (const symbolic::SymbolicError& e) {
    g_error = e.what();
    return FF_E_SYMBOLIC;
  } catch (const fem::MeshError& e) {
    g_error = e.what();
    return FF_E_MESH;
  } catch (const fem::FormError& e) {
    g_error = e.what();
    return FF_E_FORM;
  } catch (const codegen::CodegenError& e) {
    g_error = e.what();
    return FF_E_FORM;
  } catch (const std::bad_alloc&) {
    g_error = "host allocation failed";
    return FF_E_NOMEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return FF_E_ARG;
  }
}

void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(FF_E_ARG, msg);
}

void check_alloc(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) throw Error(FF_E_NOMEM, std::string(what) + ": out of device memory");
  ffb::cuda_check(e, what);
}

template <typename T>
T* device_alloc(std::size_t n, const char* what) {
  T* p = nullptr;
  check_alloc(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)), what);
  return p;
}

void bind(const ff_ctx* ctx) {
  if (ctx) ffb::cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
}

// row gather: 4 warps per CTA (FF_GATHER_THREADS), each with a [32][pitch]
// fp64 row accumulator; pitch = longest row rounded up to odd
constexpr int kGatherWarps = 4;
constexpr int kGatherSmemMax = 227 * 1024;
int gather_pitch(int max_row_len) { return max_row_len | 1; }
int gather_smem(int pitch) { return kGatherWarps * 32 * pitch * 8; }

void load_module(ff_form* f, int w) {
  if (f->kernel[w] || !f->ctx) return;
  bind(f->ctx);
  ffb::cuda_check(cudaLibraryLoadData(&f->lib[w], f->module[w].cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0),
                  "cudaLibraryLoadData");
  ffb::cuda_check(cudaLibraryGetKernel(&f->kernel[w], f->lib[w], "ff_assemble_atomic"), "cudaLibraryGetKernel");
  // whether the module holds the gather kernels: known from the template for
  // generated forms (gather_capable); probed for caller-written sources
  const bool gather_known = !f->raw;
  const bool has_gather = codegen::gather_capable(f->plan, f->n_local, f->ncomp, f->block);
  if ((gather_known ? has_gather : true) &&
      cudaLibraryGetKernel(&f->kernel_ginv[w], f->lib[w], "ff_gather_invariants") == cudaSuccess &&
      cudaLibraryGetKernel(&f->kernel_grows[w], f->lib[w], "ff_gather_rows") == cudaSuccess) {
    ffb::cuda_check(cudaKernelSetAttributeForDevice(f->kernel_grows[w], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    kGatherSmemMax, f->ctx->device),
                    "row-gather shared memory attribute");
  } else {
    cudaGetLastError();
    f->kernel_ginv[w] = f->kernel_grows[w] = nullptr;
  }
  cudaFuncAttributes attr{};
  if (cudaFuncGetAttributes(&attr, reinterpret_cast<const void*>(f->kernel[w])) == cudaSuccess) {
    f->module[w].registers = attr.numRegs;
    f->module[w].shared_bytes = static_cast<int>(attr.sharedSizeBytes);
  }
}

// Renders + compiles the template for slot width w (1 or 2).
void build_variant(ff_form* f, int w) {
  if (!f->module[w].cubin.empty()) return;
  if (f->raw) throw Error(FF_E_ARG, "raw-source forms are compiled for one slot width only");
  codegen::LaunchParams p = f->params;
  p.slot_bytes = w;
  const auto t0 = std::chrono::steady_clock::now();
  f->source[w] = codegen::emit_source(f->inst, p, &f->plan);
  f->module[w] = ffb::nvrtc_compile(f->source[w], "femforge_element.cu");
  f->compile_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  load_module(f, w);
}

void ensure_plan(ff_pattern* p, const ff_mesh* m) {
  if (p->plan_mesh == m && p->plan_generation == m->generation && p->slots) return;
  require(m->k == p->k, "mesh and sparsity pattern have different DOFs per element");
  require(p->bs == m->bs, "mesh and sparsity pattern have different components per node");
  ff_ctx* ctx = p->ctx;
  bind(ctx);
  const int w = p->max_row_len <= 256 ? 1 : 2;
  require(p->max_row_len <= 65536, "rows longer than 65536 entries are not supported");
  if (p->slots && (p->ne != m->ne || p->slot_bytes != w)) {
    cudaFree(p->slots);
    p->slots = nullptr;
  }
  if (!p->slots) p->slots = device_alloc<unsigned char>(static_cast<std::size_t>(m->ne) * m->k * m->k * w, "slot plan");
  p->ne = m->ne;
  p->slot_bytes = w;
  ffb::cuda_check(cudaMemsetAsync(ctx->d_status, 0xff, 2 * sizeof(unsigned long long), ctx->stream), "memset");
  ffb::cuda_check(ffb::kernels::build_slots(m->dconn, m->ne, m->k, p->rb, p->re, p->row_ptr, p->col_idx, w, p->slots,
                                            ctx->d_status + 1, ctx->sm_count, ctx->stream),
                  "slot plan kernel");
  unsigned long long bad = 0;
  ffb::cuda_check(cudaMemcpyAsync(&bad, ctx->d_status + 1, sizeof bad, cudaMemcpyDeviceToHost, ctx->stream), "copy");
  ffb::cuda_check(cudaStreamSynchronize(ctx->stream), "slot plan");
  p->plan_mesh = m;
  p->plan_generation = m->generation;
  if (bad != ~0ull) {
    p->plan_mesh = nullptr;
    throw Error(FF_E_PATTERN, "column not present in sparsity row " + std::to_string(bad) +
                                  " (inconsistent sparsity pattern)");
  }
}

void free_class_module(ff_pattern* p) {
  if (p->class_lib) cudaLibraryUnload(p->class_lib);
  p->class_lib = nullptr;
  p->class_kernel[0] = p->class_kernel[1] = nullptr;
  p->class_key.clear();
}

void free_gather(ff_pattern* p) {
  ffb::kernels::free_gather_plan(&p->gather);
  p->gather_generation = ~0ull;
  p->gather_mesh = nullptr;
  free_class_module(p);
}

bool vector_fused() {
  const char* v = std::getenv("FF_VSPLIT");
  return v && std::atoi(v) == 0;
}

int class_cwarps(const ff_form*) {
  const char* v = std::getenv("FF_CWARPS");
  return v ? std::max(1, std::min(8, std::atoi(v))) : 2;
}

// NVRTC-compiles the class-specialised gather kernels of (form, plan).
void ensure_class_module(ff_form* f, ff_pattern* p) {
  if (p->gather.classes.empty()) return;
  const std::string key = f->source[1] + "#" + std::to_string(p->gather_generation) + "#" +
                          std::to_string(reinterpret_cast<std::uintptr_t>(p->gather.crec));
  if (p->class_key == key && p->class_lib) return;
  free_class_module(p);
  std::vector<codegen::RowClass> rc;
  for (const auto& c : p->gather.classes) {
    codegen::RowClass r;
    r.len = c.len;
    r.steps = c.steps;
    r.local = c.local;
    r.slots = c.slots;
    r.order = c.order;  // the plan laid the records out in this order
    rc.push_back(std::move(r));
  }
  const auto t0 = std::chrono::steady_clock::now();
  // one fused kernel for every class unless FF_SPLIT_CLASSES:
  // measured 3.18 vs 3.29 ms at the north star (profiles/, run 25)
  // vector forms: long rows (> 33 node entries) in their own kernel, so the
  // short rows' staging tiles allow 16 warps/SM (config 5: 37.3 vs 42.4 ms
  // fused); FF_VSPLIT=0 fuses them
  const bool fused = f->ncomp > 1 ? vector_fused() : std::getenv("FF_SPLIT_CLASSES") == nullptr;
  std::string src = codegen::emit_class_source(f->plan, f->n_local, rc, fused, f->ncomp, p->gather.pre_steps);
  // register budget: 14 warps/SM for scalar forms (one item per warp: no
  // carried item state; NS 2.013 vs 2.038 ms at 12 warps, 2.053 with two items
  // per warp), 12 for vector forms
  if (fused && !std::getenv("FF_MINB_S"))
    src = "#define FF_MINB_S " + std::to_string((f->ncomp > 1 ? 12 : 14) / class_cwarps(f)) + "\n" + src;
  if (!fused && f->ncomp > 1) {
    // split vector kernels: 20 warps/SM for short rows (config 5 27.29 ms
    // against 28.31 / 27.80 with 16 / 24), 8 for long rows (234 registers, no
    // spills: 29.96 ms against 37.35 with 10 warps at 168 registers + spills)
    if (!std::getenv("FF_MINB_S")) src = "#define FF_MINB_S " + std::to_string(20 / class_cwarps(f)) + "\n" + src;
    if (!std::getenv("FF_MINB_L")) src = "#define FF_MINB_L " + std::to_string(8 / class_cwarps(f)) + "\n" + src;
  }
  if (!std::getenv("FF_CWARPS")) src = "#define FF_CWARPS " + std::to_string(class_cwarps(f)) + "\n" + src;
  // tuning knobs (defaults in the source): FF_MINB_S, FF_MINB_L
  for (const char* knob : {"FF_MINB_S", "FF_MINB_L", "FF_WUNROLL", "FF_CWARPS"})
    if (const char* v = std::getenv(knob))
      src = "#define " + std::string(knob) + " " + std::to_string(std::max(1, std::atoi(v))) + "\n" + src;
  // FF_ABL (analysis only, wrong results): bit 1 no write-out, 2 no invariant
  // loads, 4 synthetic record ids, 8 no load-vector loads
  if (const char* v = std::getenv("FF_ABL")) src = "#define FF_ABL " + std::to_string(std::atoi(v)) + "\n" + src;
  const ffb::CompiledModule mod = ffb::nvrtc_compile(src, "femforge_classes.cu");
  bind(p->ctx);
  ffb::cuda_check(cudaLibraryLoadData(&p->class_lib, mod.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0),
                  "cudaLibraryLoadData (classes)");
  ffb::cuda_check(cudaLibraryGetKernel(&p->class_kernel[0], p->class_lib, "ff_gather_classes_s"), "class kernel");
  ffb::cuda_check(cudaLibraryGetKernel(&p->class_kernel[1], p->class_lib, "ff_gather_classes_l"), "class kernel");
  for (int c = 0; c < 2; ++c) {
    p->class_smem[c] = codegen::class_shared_bytes(rc, c, fused, class_cwarps(f), f->ncomp);
    ffb::cuda_check(cudaKernelSetAttributeForDevice(p->class_kernel[c], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    p->class_smem[c], p->ctx->device),
                    "class kernel shared memory attribute");
  }
  p->class_compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  p->class_key = key;
}

void ensure_gather_plan(ff_pattern* p, const ff_mesh* m) {
  ensure_plan(p, m);
  const int64_t cmin = p->ctx->class_min_rows;
  if (p->gather_mesh == m && p->gather_generation == m->generation && p->gather_class_min == cmin &&
      (p->gather.rec || p->gather.crec))
    return;
  require(p->slot_bytes == 1, "row gather needs rows of <= 256 entries");
  free_gather(p);
  ff_ctx* ctx = p->ctx;
  bind(ctx);
  const auto t0 = std::chrono::steady_clock::now();
  // bounding box of the coordinates (host copy; the Morton order of the DOF
  // points only needs it to quantise)
  std::vector<double> xyz(static_cast<std::size_t>(m->nv) * m->dim);
  if (!xyz.empty())
    ffb::cuda_check(cudaMemcpy(xyz.data(), m->coords, xyz.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  double bbox[6] = {0, 0, 0, 0, 0, 0};
  for (int c = 0; c < m->dim; ++c) {
    double lo = 0, hi = 0;
    for (int64_t v = 0; v < m->nv; ++v) {
      const double x = xyz[v * m->dim + c];
      if (v == 0 || x < lo) lo = x;
      if (v == 0 || x > hi) hi = x;
    }
    bbox[c] = lo;
    bbox[3 + c] = hi;
  }
  // the code generator's step order of each class: the plan lays the class
  // items' records out in it
  const int n_local_scalar = m->k;
  const ffb::kernels::ClassOrderFn order_fn = [n_local_scalar](const ffb::kernels::GatherPlan::Class& c) {
    codegen::RowClass r;
    r.len = c.len;
    r.steps = c.steps;
    r.local = c.local;
    r.slots = c.slots;
    return codegen::class_step_order(r, n_local_scalar);
  };
  const cudaError_t e = ffb::kernels::build_gather_plan(m->coords, m->vconn, m->dim, bbox, m->dconn, m->ne, m->k, p->rb,
                                                        p->re - p->rb, p->row_ptr, static_cast<const uint8_t*>(p->slots),
                                                        4096, ctx->sm_count, ctx->stream, &p->gather,
                                                        cmin > 0 ? static_cast<int>(std::min<int64_t>(cmin, 1 << 30))
                                                                 : (1 << 30),
                                                        cmin > 0 ? 64 : 0, true,
                                                        p->bs == 1 ? std::getenv("FF_SPLIT_CLASSES") != nullptr
                                                                   : !vector_fused(),
                                                        &order_fn, 0.0005, p->bs);
  if (e != cudaSuccess) {
    ffb::kernels::free_gather_plan(&p->gather);
    check_alloc(e, "row-gather plan");
  }
  p->gather_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  p->gather_mesh = m;
  p->gather_generation = m->generation;
  p->gather_class_min = cmin;
}

// The scatter a (form, pattern, flags) assembly runs (FF_SCATTER_*_MODE).
bool gather_possible(const ff_form* f, const ff_pattern* p, int w) {
  return f->kernel_grows[w] && p->max_row_len <= 255 && gather_smem(gather_pitch(p->max_row_len)) <= kGatherSmemMax;
}

int select_scatter(const ff_form* f, const ff_pattern* p, unsigned flags, int w) {
  int mode = f->ctx ? f->ctx->scatter : FF_SCATTER_GATHER_MODE;
  if (mode == FF_SCATTER_AUTO_MODE)  // the measured choice, else the row gather where it can run
    mode = (p->auto_form == f->id && p->auto_generation == p->plan_generation && p->auto_mode)
               ? p->auto_mode
               : FF_SCATTER_GATHER_MODE;
  if (flags & FF_SCATTER_ATOMIC) mode = FF_SCATTER_ATOMIC_MODE;
  if (flags & (FF_SCATTER_GATHER | FF_GATHER_INVARIANTS_ONLY | FF_GATHER_ROWS_ONLY)) mode = FF_SCATTER_GATHER_MODE;
  if (flags & (FF_ZERO_ONLY | FF_SKIP_ZERO)) mode = FF_SCATTER_ATOMIC_MODE;
  if (mode == FF_SCATTER_GATHER_MODE && !gather_possible(f, p, w)) mode = FF_SCATTER_ATOMIC_MODE;
  return mode;
}

void launch_gather(ff_form* f, const ff_mesh* m, ff_pattern* p, double* d_values, double* d_rhs, cudaStream_t s,
                   unsigned flags, int w) {
  ff_ctx* ctx = f->ctx;
  ensure_gather_plan(p, m);
  const int gs = ((f->plan.n_kinv + 3) / 4) * 4;  // FF_GS: invariants [E][gs] + load vectors [k][E]
  const std::size_t ng = static_cast<std::size_t>(std::max<int64_t>(m->ne, 1)) * (gs + f->n_local);
  if (p->ginv_cap < ng) {
    cudaFree(p->ginv);
    p->ginv = nullptr;
    p->ginv = device_alloc<double>(ng, "element invariants");
    p->ginv_cap = ng;
  }
  unsigned long long* status = ctx->d_status;
  // K2a over records [t0, t1)
  auto launch_k2a = [&](int64_t t0, int64_t t1, cudaStream_t st) {
    if (t1 <= t0) return;
    const double* coords = m->coords;
    const int32_t* vconn = p->gather.vconn_m;  // vertex ids in record order
    const int32_t* dconn = m->dconn;
    long long ne = m->ne, a = t0, b = t1;
    double* ginv = p->ginv;
    const int32_t* eorder = p->gather.eorder;
    void* args[] = {&coords, &vconn, &dconn, &eorder, &ne, &ginv, &status, &a, &b};
    const unsigned grid = static_cast<unsigned>((t1 - t0 + f->block - 1) / f->block);
    ffb::cuda_check(cudaLaunchKernel(reinterpret_cast<const void*>(f->kernel_ginv[w]), dim3(grid), dim3(f->block),
                                     args, 0, st),
                    "K2a (element invariants) launch");
  };
  const ffb::kernels::GatherPlan& gp = p->gather;
  if (!(flags & FF_GATHER_ROWS_ONLY)) {
    ffb::cuda_check(cudaMemsetAsync(status, 0xff, 2 * sizeof(unsigned long long), s), "status reset");
    launch_k2a(0, m->ne, s);
  }
  if (flags & FF_GATHER_INVARIANTS_ONLY) return;
  auto launch_generic = [&](cudaStream_t sg) {
    // K2b for the remaining rows in two launches: short-pitch items, then long-pitch items
    // vector forms: FF_BS^2 sub-items (component pairs) per item
    const int64_t nb = static_cast<int64_t>(f->ncomp) * f->ncomp;
    const int64_t ranges[2][2] = {{0, gp.n_short * nb}, {gp.n_short * nb, gp.n_items * nb}};
    const int pitches[2] = {gp.pitch_short, gp.pitch_long};
    for (int c = 0; c < 2; ++c) {
      long long i0 = ranges[c][0], i1 = ranges[c][1];
      if (i1 <= i0) continue;
      int pitch = pitches[c];
      const int smem = gather_smem(pitch);
      require(smem <= kGatherSmemMax, "row gather: rows too long for the shared-memory accumulators");
      // a few items per warp: CTAs run in item order, so the items in flight
      // stay contiguous and their element data stays in L2; one item per warp
      // when the range would not fill the GPU (small meshes, boundary rows)
      int ipw = 4;
      if ((i1 - i0) < int64_t(ctx->sm_count) * kGatherWarps * 4 * 4) ipw = 1;
      if (const char* v = std::getenv("FF_GENERIC_IPW")) ipw = std::max(1, std::atoi(v));  // tuning knob
      const int64_t per_cta = int64_t(kGatherWarps) * ipw;
      const unsigned grid = static_cast<unsigned>((i1 - i0 + per_cta - 1) / per_cta);
      const double* ginv = p->ginv;
      long long ne_arg = m->ne;
      const int64_t* row_ptr = p->row_ptr;
      const int32_t* order = gp.item_order;
      const int32_t* wrows = gp.warp_rows;
      const int32_t* wsteps = gp.warp_steps;
      const int64_t* wrec = gp.warp_rec;
      const void* rec = gp.rec;
      void* args[] = {&ginv, &ne_arg, &row_ptr, &d_values, &d_rhs, &order, &i0, &i1, &wrows, &wsteps, &wrec, &rec,
                      &pitch, &ipw};
      ffb::cuda_check(cudaLaunchKernel(reinterpret_cast<const void*>(f->kernel_grows[w]), dim3(grid),
                                       dim3(kGatherWarps * 32), args, smem, sg),
                      "K2b (row gather) launch");
    }
  };
  // class items [a, b) with kernel c (0: short rows, 1: long rows)
  auto launch_class = [&](int c, int64_t a, int64_t b, cudaStream_t sc) {
    long long i0 = a, i1 = b;
    if (i1 <= i0) return;
    // FF_CWARPS warps x one item per CTA; vector forms: one CTA per test component
    const int cw = class_cwarps(f);
    const int64_t ctas = (i1 - i0 + cw - 1) / cw;
    const unsigned grid = static_cast<unsigned>(ctas * f->ncomp);
    const double* ginv = p->ginv;
    long long ne_arg = m->ne;
    const int64_t* row_ptr = p->row_ptr;
    const int32_t* icls = gp.citem_class;
    const int32_t* irows = gp.citem_rows;
    const int64_t* irec = gp.citem_rec;
    const int32_t* crec = gp.crec;
    void* args[] = {&ginv, &ne_arg, &row_ptr, &d_values, &d_rhs, &icls, &irows, &irec, &crec, &i0, &i1};
    ffb::cuda_check(cudaLaunchKernel(reinterpret_cast<const void*>(p->class_kernel[c]), dim3(grid), dim3(32 * cw), args,
                                     p->class_smem[c], sc),
                    "K2b (class row gather) launch");
  };
  auto fork = [&](cudaStream_t to) {
    ffb::cuda_check(cudaEventRecord(ctx->fork, s), "fork");
    ffb::cuda_check(cudaStreamWaitEvent(to, ctx->fork, 0), "fork");
  };
  auto join = [&](cudaStream_t from) {
    ffb::cuda_check(cudaEventRecord(ctx->join, from), "join");
    ffb::cuda_check(cudaStreamWaitEvent(s, ctx->join, 0), "join");
  };
  if (gp.n_citems > 0) ensure_class_module(f, p);
  const int64_t ns = gp.n_citems_short;
  // the generic rows run on the side stream, concurrently with the class
  // kernel (disjoint rows, both only read the element records): 2.861 ->
  // 2.846 ms at the north star (run 34)
  const bool generic_side = gp.n_citems > 0 && gp.n_items > 0 && !std::getenv("FF_GENERIC_SERIAL");
  if (generic_side) {
    fork(ctx->side);
    launch_generic(ctx->side);
  }
  // K2b for the row classes: specialised kernels (rows in registers); the
  // long-row kernel runs on the side stream, concurrently with the short-row
  // one (disjoint rows): the two register budgets share the SMs and the
  // element records they both read stay in L2
  if (gp.n_citems > 0) {
    const bool both = !generic_side && ns > 0 && gp.n_citems > ns && !std::getenv("FF_SERIAL_CLASSES");
    if (both) fork(ctx->side);
    launch_class(1, ns, gp.n_citems, both ? ctx->side : s);
    launch_class(0, 0, ns, s);
    if (both) join(ctx->side);
  }
  if (!generic_side) launch_generic(s);
  if (generic_side) join(ctx->side);
}

void launch_assembly(ff_form* f, const ff_mesh* m, ff_pattern* p, double* d_values, double* d_rhs, cudaStream_t s,
                     unsigned flags = 0);

// FF_SCATTER_AUTO_MODE: times both scatters (CUDA events on s, one warm-up
// then the mean of 3 runs each) and records the faster for (form, plan).
void calibrate_scatter(ff_form* f, const ff_mesh* m, ff_pattern* p, double* d_values, double* d_rhs, cudaStream_t s) {
  ensure_plan(p, m);
  const int w = p->slot_bytes;
  build_variant(f, w);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ffb::cuda_check(cudaEventCreate(&e0), "cudaEventCreate");
  ffb::cuda_check(cudaEventCreate(&e1), "cudaEventCreate");
  double ms[2] = {-1.0, -1.0};
  const unsigned fl[2] = {FF_SCATTER_GATHER, FF_SCATTER_ATOMIC};
  try {
    for (int v = 0; v < 2; ++v) {
      if (v == 0 && !gather_possible(f, p, w)) continue;
      launch_assembly(f, m, p, d_values, d_rhs, s, fl[v]);  // warm-up: plans, modules
      ffb::cuda_check(cudaEventRecord(e0, s), "event");
      for (int r = 0; r < 3; ++r) launch_assembly(f, m, p, d_values, d_rhs, s, fl[v]);
      ffb::cuda_check(cudaEventRecord(e1, s), "event");
      ffb::cuda_check(cudaEventSynchronize(e1), "calibration");
      float t = 0.f;
      ffb::cuda_check(cudaEventElapsedTime(&t, e0, e1), "event");
      ms[v] = t / 3.0;
    }
  } catch (...) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    throw;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  p->auto_ms[0] = ms[0];
  p->auto_ms[1] = ms[1];
  p->auto_mode = (ms[0] >= 0.0 && ms[0] <= ms[1]) ? FF_SCATTER_GATHER_MODE : FF_SCATTER_ATOMIC_MODE;
  p->auto_form = f->id;
  p->auto_generation = p->plan_generation;
  if (p->auto_mode == FF_SCATTER_GATHER_MODE)  // leave the chosen scatter's result in the buffers
    launch_assembly(f, m, p, d_values, d_rhs, s, FF_SCATTER_GATHER);
}

void launch_assembly(ff_form* f, const ff_mesh* m, ff_pattern* p, double* d_values, double* d_rhs, cudaStream_t s,
                     unsigned flags) {
  require(f->ctx && f->ctx == m->ctx && m->ctx == p->ctx, "form, mesh and pattern must share one context");
  require(f->dim == m->dim, "form and mesh dimensions differ");
  require(f->ncomp == m->bs && f->n_local == m->k * m->bs, "form and mesh have different DOFs per element");
  require(p->bs == m->bs, "mesh and sparsity pattern have different components per node");
  ensure_plan(p, m);
  const int w = p->slot_bytes;
  build_variant(f, w);
  ff_ctx* ctx = f->ctx;
  const int64_t n_rows = p->re - p->rb;
  if (ctx->scatter == FF_SCATTER_AUTO_MODE && flags == 0 &&
      !(p->auto_form == f->id && p->auto_generation == p->plan_generation && p->auto_mode)) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
      calibrate_scatter(f, m, p, d_values, d_rhs, s);
      return;  // the buffers hold the chosen scatter's assembly
    }
  }
  const int mode = select_scatter(f, p, flags, w);
  if (mode == FF_SCATTER_GATHER_MODE) {
    launch_gather(f, m, p, d_values, d_rhs, s, flags, w);
    return;
  }
  if (!(flags & FF_SKIP_ZERO))
    ffb::cuda_check(ffb::kernels::zero_fill(d_values, int64_t(p->bs) * p->bs * p->nnz, d_rhs, p->bs * n_rows,
                                            ctx->d_status, ctx->sm_count, s),
                    "K0");
  if (m->ne == 0 || (flags & FF_ZERO_ONLY)) return;
  const double* coords = m->coords;
  const int32_t* vconn = m->vconn;
  const int32_t* dconn = m->dconn;
  const void* slots = p->slots;
  long long ne = m->ne, rb = p->rb, re = p->re;
  const int64_t* row_ptr = p->row_ptr;
  unsigned long long* status = ctx->d_status;
  void* args[] = {&coords, &vconn, &dconn, &slots, &ne, &row_ptr, &d_values, &d_rhs, &rb, &re, &status};
  const unsigned grid = static_cast<unsigned>((m->ne + f->block - 1) / f->block);
  ffb::cuda_check(cudaLaunchKernel(reinterpret_cast<const void*>(f->kernel[w]), dim3(grid), dim3(f->block), args, 0, s),
                  "K2 launch");
}

void report_status(ff_ctx* ctx, ff_stats* stats) {
  ffb::cuda_check(cudaMemcpyAsync(ctx->h_status, ctx->d_status, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                  ctx->stream),
                  "status copy");
  ffb::cuda_check(cudaStreamSynchronize(ctx->stream), "assembly");
  const unsigned long long be = ctx->h_status[0], br = ctx->h_status[1];
  if (stats) {
    stats->bad_element = be == ~0ull ? -1 : static_cast<int64_t>(be);
    stats->bad_row = br == ~0ull ? -1 : static_cast<int64_t>(br);
  }
  if (be != ~0ull) throw Error(FF_E_DEGENERATE, "degenerate element " + std::to_string(be) + " (|det J| <= 1e-14)");
  if (br != ~0ull)
    throw Error(FF_E_PATTERN, "column not present in sparsity row " + std::to_string(br) + " (inconsistent sparsity pattern)");
}

// Everything a captured assembly depends on: replaying its graph is valid
// while none of these changed (buffers, plans, modules, scatter, stream).
std::vector<std::uint64_t> graph_key(const ff_form* f, const ff_mesh* m, const ff_pattern* p, const double* v,
                                     const double* r, cudaStream_t s) {
  auto u = [](const void* x) { return static_cast<std::uint64_t>(reinterpret_cast<std::uintptr_t>(x)); };
  return {f->id, u(m), m->generation, u(m->coords), u(m->vconn), u(m->dconn), u(p), p->plan_generation,
          p->gather_generation, u(p->slots), u(p->ginv), u(p->gather.crec), u(p->gather.rec), u(p->class_lib),
          u(v), u(r), u(s), static_cast<std::uint64_t>(f->ctx->scatter),
          static_cast<std::uint64_t>(f->ctx->class_min_rows)};
}

void drop_graph(ff_pattern* p) {
  if (p->graph_exec) cudaGraphExecDestroy(p->graph_exec);
  p->graph_exec = nullptr;
  p->graph_key.clear();
}

std::uint64_t next_form_id() {
  static std::atomic<std::uint64_t> n{0};
  return ++n;
}

// Connectivity generations are process-wide: plans keyed on (mesh, generation)
// can never match a new mesh that reuses a destroyed mesh's address.
std::uint64_t next_generation() {
  static std::atomic<std::uint64_t> n{0};
  return ++n;
}

// The MeshError message of element t (fem.cpp:17-34 wording and order:
// vertex index range, duplicate vertices, then orientation; the DOF checks of
// higher-order spaces sit between the two, with DOF wording).
std::string mesh_error(const ff_mesh* m, int64_t t, bool orient) {
  const int nn = m->dim + 1;
  std::vector<int32_t> v(nn), d(m->k);
  ffb::cuda_check(cudaMemcpy(v.data(), m->vconn + t * nn, nn * sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
  const std::string el = "element " + std::to_string(t) + ": ";
  for (int a = 0; a < nn; ++a)
    if (v[a] < 0 || v[a] >= m->nv) return el + "node index " + std::to_string(v[a]) + " out of range";
  for (int a = 0; a < nn; ++a)
    for (int b = a + 1; b < nn; ++b)
      if (v[a] == v[b]) return el + "duplicate node indices";
  if (m->dconn != m->vconn) {
    ffb::cuda_check(cudaMemcpy(d.data(), m->dconn + t * m->k, m->k * sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
    for (int a = 0; a < m->k; ++a)
      if (d[a] < 0 || d[a] >= m->n_dofs) return el + "DOF index " + std::to_string(d[a]) + " out of range";
    for (int a = 0; a < m->k; ++a)
      for (int b = a + 1; b < m->k; ++b)
        if (d[a] == d[b]) return el + "duplicate DOF indices";
  }
  (void)orient;
  return el + (m->dim == 2 ? "non-positive signed area" : "non-positive signed volume");
}

// Mesh::validate (fem.cpp:17-34) over the device-resident mesh; throws
// MeshError for the lowest failing element, like the reference's loop.
void validate_mesh(const ff_mesh* m, bool orient) {
  ff_ctx* ctx = m->ctx;
  unsigned long long* d_bad = ctx->d_status + 2;
  ffb::cuda_check(ffb::kernels::validate_mesh(m->coords, m->dim, m->nv, m->vconn, m->dconn != m->vconn ? m->dconn : nullptr,
                                              m->k, m->n_dofs, m->ne, orient, d_bad, ctx->sm_count, ctx->stream),
                  "mesh validation");
  unsigned long long bad = 0;
  ffb::cuda_check(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
  ffb::cuda_check(cudaStreamSynchronize(ctx->stream), "mesh validation");
  if (bad != ~0ull) throw fem::MeshError(mesh_error(m, static_cast<int64_t>(bad), orient));
}

void free_mesh(ff_mesh* m) {
  cudaFree(m->coords);
  if (m->dconn != m->vconn) cudaFree(m->dconn);
  cudaFree(m->vconn);
  cudaFree(m->stage);
  cudaFree(m->stage_d);
  delete m;
}

// Upload n ids into dst through the staging buffer; true when any id changed.
bool upload_conn(ff_mesh* m, int32_t* dst, const int32_t* src, int64_t n) {
  ff_ctx* ctx = m->ctx;
  // staging per array (vconn: m->stage, dconn: m->stage_d), sized for it
  int32_t*& stage = dst == m->vconn ? m->stage : m->stage_d;
  if (!stage) stage = device_alloc<int32_t>(std::max<int64_t>(n, 1), "connectivity staging");
  ffb::cuda_check(cudaMemcpyAsync(stage, src, n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream), "H2D");
  unsigned long long* d_diff = ctx->d_status + 2;
  ffb::cuda_check(cudaMemsetAsync(d_diff, 0, sizeof(unsigned long long), ctx->stream), "memset");
  ffb::cuda_check(ffb::kernels::copy_compare(stage, dst, n, d_diff, ctx->sm_count, ctx->stream), "compare");
  unsigned long long diff = 0;
  ffb::cuda_check(cudaMemcpyAsync(&diff, d_diff, sizeof diff, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
  ffb::cuda_check(cudaStreamSynchronize(ctx->stream), "connectivity upload");
  return diff != 0;
}

}  // namespace

extern "C" {

const char* ff_version(void) { return "femforge-b200 0.1 (sm_100a, NVRTC)"; }
const char* ff_last_error(void) { return g_error.c_str(); }

int ff_device_count(int* count) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    *count = n;
  });
}

int ff_init(int device, ff_ctx** out) {
  return guarded([&] {
    require(out != nullptr, "ff_init: out is NULL");
    auto c = std::make_unique<ff_ctx>();
    c->device = device;
    ffb::cuda_check(cudaSetDevice(device), "cudaSetDevice");
    ffb::cuda_check(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device), "attribute");
    ffb::cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ffb::cuda_check(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "cudaStreamCreate");
    ffb::cuda_check(cudaStreamCreateWithFlags(&c->upload, cudaStreamNonBlocking), "cudaStreamCreate");

    ffb::cuda_check(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming), "cudaEventCreate");
    ffb::cuda_check(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming), "cudaEventCreate");
    c->d_status = device_alloc<unsigned long long>(5, "status");  // [bad_elem, bad_row, scratch, 2 diffs]
    ffb::cuda_check(cudaMallocHost(&c->h_status, 4 * sizeof(unsigned long long)), "cudaMallocHost");
    ffb::cuda_check(cudaMemset(c->d_status, 0xff, 2 * sizeof(unsigned long long)), "memset");
    *out = c.release();
  });
}

int ff_ctx_destroy(ff_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    bind(ctx);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->d_status);
    cudaFreeHost(ctx->h_status);
    cudaStreamSynchronize(ctx->side);
    cudaStreamSynchronize(ctx->upload);
    cudaStreamDestroy(ctx->upload);
    cudaEventDestroy(ctx->fork);
    cudaEventDestroy(ctx->join);
    cudaStreamDestroy(ctx->side);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int ff_ctx_synchronize(ff_ctx* ctx) {
  return guarded([&] {
    require(ctx, "null context");
    bind(ctx);
    ffb::cuda_check(cudaStreamSynchronize(ctx->stream), "synchronize");
  });
}

void* ff_ctx_stream(ff_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int ff_ctx_set_scatter(ff_ctx* ctx, int mode) {
  return guarded([&] {
    require(ctx, "null context");
    require(mode == FF_SCATTER_ATOMIC_MODE || mode == FF_SCATTER_GATHER_MODE || mode == FF_SCATTER_AUTO_MODE,
            "unknown scatter mode");
    ctx->scatter = mode;
  });
}

int ff_ctx_set_gather_classes(ff_ctx* ctx, int64_t min_rows) {
  return guarded([&] {
    require(ctx && min_rows >= 0, "invalid argument");
    ctx->class_min_rows = min_rows;
  });
}

int ff_expr_eval(const char* expr, int dim, const double* pts, int64_t n, double* out) {
  return guarded([&] {
    require(expr && dim >= 1 && dim <= 3 && n >= 0 && (n == 0 || (pts && out)), "ff_expr_eval: invalid argument");
    const symbolic::Expr e = symbolic::parse(expr);
    static const char* const kNames[3] = {"x", "y", "z"};
    for (const std::string& s : symbolic::free_symbols(e)) {
      bool ok = false;
      for (int c = 0; c < dim; ++c) ok = ok || s == kNames[c];
      if (!ok) throw symbolic::SymbolicError("expression references symbol '" + s + "'");
    }
    std::map<std::string, double> at;
    for (int64_t i = 0; i < n; ++i) {
      for (int c = 0; c < dim; ++c) at[kNames[c]] = pts[i * dim + c];
      out[i] = symbolic::eval(e, at);
    }
  });
}

int ff_form_entry_text(const ff_form* f, int kind, int i, int j, char* buf, size_t cap, size_t* out_len) {
  return guarded([&] {
    require(f && !f->raw, "ff_form_entry_text: form without an instantiated weak form");
    const int n = f->inst.n_local;
    require(i >= 0 && i < n && (kind == 1 || (kind == 0 && j >= 0 && j < n)), "ff_form_entry_text: index out of range");
    const std::string s = symbolic::print(kind == 0 ? f->inst.bilinear[static_cast<std::size_t>(i) * n + j]
                                                    : f->inst.linear[i]);
    if (out_len) *out_len = s.size();
    if (buf && cap) {
      const std::size_t k = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), k);
      buf[k] = '\0';
    }
  });
}

int ff_class_source(const ff_form* f, int n, const int32_t* len, const int32_t* steps, const int32_t* local,
                    const uint8_t* slots, char* buf, size_t cap, size_t* out_len) {
  return guarded([&] {
    require(f && n >= 0 && (n == 0 || (len && steps && local && slots)), "null argument");
    require(f->plan.n_kinv > 0, "form has no reference-tensor plan (no row gather)");
    const int nsc = f->n_local / f->ncomp;  // slots per incidence (node rows of vector forms)
    std::vector<codegen::RowClass> rc(n);
    int64_t at = 0;
    for (int c = 0; c < n; ++c) {
      rc[c].len = len[c];
      rc[c].steps = steps[c];
      for (int q = 0; q < steps[c]; ++q) {
        rc[c].local.push_back(local[at + q]);
        for (int j = 0; j < nsc; ++j) rc[c].slots.push_back(slots[(at + q) * nsc + j]);
      }
      at += steps[c];
    }
    // FF_CLASS_PRE (analysis hook): the record prefix the plan would pick
    int pre = 1;
    if (const char* v = std::getenv("FF_CLASS_PRE")) pre = std::max(1, std::min(8, std::atoi(v)));
    for (const auto& c : rc) pre = std::min(pre, std::max(c.steps, 1));
    const std::string src = codegen::emit_class_source(f->plan, f->n_local, rc,
                                                       std::getenv("FF_SPLIT_CLASSES") == nullptr, f->ncomp, pre);
    if (out_len) *out_len = src.size();
    if (buf && cap) {
      const std::size_t k = std::min(cap - 1, src.size());
      std::memcpy(buf, src.data(), k);
      buf[k] = '\0';
    }
  });
}

int ff_form_create(ff_ctx* ctx, const ff_form_desc* d, ff_form** out) {
  return guarded([&] {
    require(d && out, "ff_form_create: null argument");
    require(d->dim == 2 || d->dim == 3, "form dimension must be 2 or 3");
    require(d->degree == 1 || d->degree == 2, "only Lagrange degree 1 and 2 are supported");
    require(d->bilinear && d->linear, "bilinear and linear integrands are required");
    auto f = std::make_unique<ff_form>();
    f->id = next_form_id();
    f->ctx = ctx;
    f->dim = d->dim;
    f->degree = d->degree;
    f->block = d->block_size > 0 ? d->block_size : 128;
    fem::WeakForm wf;
    wf.bilinear = symbolic::parse(d->bilinear);
    wf.linear = symbolic::parse(d->linear);
    wf.space.dim = d->dim;
    wf.space.degree = d->degree;
    const auto t0 = std::chrono::steady_clock::now();
    f->inst = fem::instantiate(wf);
    f->n_local = f->inst.n_local;
    f->params.block_size = f->block;
    f->params.quad_rule = d->quad_rule;
    f->params.strategy = static_cast<codegen::Strategy>(d->strategy);
    f->params.n_local = f->n_local;
    if (d->block_size <= 0) {
      // CTA size of the element kernels, by body: the pointwise quadrature body
      // needs ~254 registers, so its CTAs are one warp (config 4: 4.36 ms at 32
      // threads, 4.59 at 128, 5.73 at 256); reference-tensor bodies 128 (K2a:
      // NS 1.888 vs 1.901 ms, C2 0.493 vs 0.518 against 256)
      const int rule_id = d->quad_rule > 0 ? d->quad_rule : codegen::default_quad_rule(d->dim, d->degree);
      const codegen::ElementPlan plan =
          codegen::plan_element(f->inst, fem::quadrature_rule(d->dim, rule_id), f->params.strategy);
      f->block = plan.strategy == codegen::Strategy::Pointwise ? 32 : 128;
      f->params.block_size = f->block;
    }
    f->compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    build_variant(f.get(), 1);
    *out = f.release();
  });
}

int ff_form_create_blocked(ff_ctx* ctx, const ff_form_desc* d, int ncomp, const char* const* block_bilinear,
                           const char* const* block_linear, ff_form** out) {
  return guarded([&] {
    require(d && out && block_bilinear && block_linear, "ff_form_create_blocked: null argument");
    require(d->dim == 2 || d->dim == 3, "form dimension must be 2 or 3");
    require(d->degree == 1 || d->degree == 2, "only Lagrange degree 1 and 2 are supported");
    require(ncomp >= 1 && ncomp <= 3, "1 to 3 components per node");
    auto f = std::make_unique<ff_form>();
    f->id = next_form_id();
    f->ctx = ctx;
    f->dim = d->dim;
    f->degree = d->degree;
    f->block = d->block_size > 0 ? d->block_size : 128;
    std::vector<fem::WeakForm> blocks(ncomp * ncomp), lin(ncomp);
    for (int q = 0; q < ncomp * ncomp; ++q) {
      require(block_bilinear[q] != nullptr, "missing bilinear block");
      blocks[q].bilinear = symbolic::parse(block_bilinear[q]);
      blocks[q].linear = symbolic::integer(0);
      blocks[q].space.dim = d->dim;
      blocks[q].space.degree = d->degree;
    }
    for (int c = 0; c < ncomp; ++c) {
      require(block_linear[c] != nullptr, "missing linear component");
      lin[c].bilinear = symbolic::integer(0);
      lin[c].linear = symbolic::parse(block_linear[c]);
      lin[c].space.dim = d->dim;
      lin[c].space.degree = d->degree;
    }
    const auto t0 = std::chrono::steady_clock::now();
    f->inst = fem::instantiate_blocked(blocks, lin, ncomp);
    f->n_local = f->inst.n_local;
    f->ncomp = ncomp;
    f->params.block_size = f->block;
    f->params.quad_rule = d->quad_rule;
    f->params.strategy = static_cast<codegen::Strategy>(d->strategy);
    f->params.n_local = f->n_local;
    f->compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    build_variant(f.get(), 1);
    *out = f.release();
  });
}

int ff_mesh_set_components(ff_mesh* m, int ncomp) {
  return guarded([&] {
    require(m && ncomp >= 1 && ncomp <= 3, "invalid argument");
    m->bs = ncomp;
    m->generation = next_generation();  // process-wide: no plan keyed on an old value can match
  });
}

int ff_compile(ff_ctx* ctx, const char* src, int dim, int degree, int block_size, ff_form** out, char* log,
               size_t log_cap) {
  return guarded([&] {
    require(src && out, "ff_compile: null argument");
    auto f = std::make_unique<ff_form>();
    f->id = next_form_id();
    f->ctx = ctx;
    f->raw = true;
    f->dim = dim;
    f->degree = degree;
    f->n_local = fem::local_dofs(dim, degree);
    f->block = block_size > 0 ? block_size : 256;
    f->source[1] = src;
    try {
      f->module[1] = ffb::nvrtc_compile(f->source[1], "femforge_user.cu");
    } catch (const Error& e) {
      if (log && log_cap) {
        std::strncpy(log, e.what(), log_cap - 1);
        log[log_cap - 1] = '\0';
      }
      throw;
    }
    if (log && log_cap) {
      std::strncpy(log, f->module[1].log.c_str(), log_cap - 1);
      log[log_cap - 1] = '\0';
    }
    f->compile_ms = f->module[1].ms;
    load_module(f.get(), 1);
    *out = f.release();
  });
}

int ff_form_source(const ff_form* f, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    require(f, "null form");
    const std::string& s = f->source[1];
    if (len) *len = s.size();
    if (buf && cap) {
      const std::size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = '\0';
    }
  });
}

int ff_form_cubin(const ff_form* f, void* buf, size_t cap, size_t* len) {
  return guarded([&] {
    require(f, "null form");
    const std::string& s = f->module[1].cubin;
    if (len) *len = s.size();
    if (buf) std::memcpy(buf, s.data(), std::min(cap, s.size()));
  });
}

int ff_form_info_get(const ff_form* f, ff_form_info* o) {
  return guarded([&] {
    require(f && o, "null argument");
    o->dim = f->dim;
    o->degree = f->degree;
    o->n_local = f->n_local;
    o->n_quad = f->plan.n_quad;
    o->strategy = static_cast<int>(f->plan.strategy);
    o->n_invariants = f->plan.n_invariants;
    o->n_unique_entries = f->plan.n_unique_entries;
    o->flops_per_element = f->plan.flops;
    o->registers = f->module[1].registers;
    o->shared_bytes = f->module[1].shared_bytes;
    o->compile_ms = f->compile_ms;
    o->n_kinv = (!f->raw && codegen::gather_capable(f->plan, f->n_local, f->ncomp, f->block)) ? f->plan.n_kinv : 0;
    o->row_flops = f->plan.row_flops;
  });
}

int ff_form_destroy(ff_form* f) {
  return guarded([&] {
    if (!f) return;
    for (auto& lib : f->lib)
      if (lib) cudaLibraryUnload(lib);
    delete f;
  });
}

int ff_mesh_create(ff_ctx* ctx, int dim, const double* coords, int64_t nv, const int32_t* vconn, int64_t ne,
                   const int32_t* dconn, int32_t k, int64_t n_dofs, ff_mesh** out) {
  return guarded([&] {
    require(ctx && out && coords && vconn, "ff_mesh_create: null argument");
    require(dim == 2 || dim == 3, "mesh dimension must be 2 or 3");
    require(nv >= 0 && ne >= 0 && n_dofs >= 0, "negative size");
    require(n_dofs < (int64_t(1) << 31), "more than 2^31 DOFs per device are not supported");
    require(k == dim + 1 || dconn, "dconn is required when dofs_per_elem != dim+1");
    bind(ctx);
    auto m = std::make_unique<ff_mesh>();
    m->ctx = ctx;
    m->dim = dim;
    m->k = k;
    m->nv = nv;
    m->ne = ne;
    m->n_dofs = n_dofs;
    m->coords = device_alloc<double>(nv * dim, "coords");
    m->vconn = device_alloc<int32_t>(ne * (dim + 1), "vconn");
    m->dconn = dconn ? device_alloc<int32_t>(ne * k, "dconn") : m->vconn;
    ffb::cuda_check(cudaMemcpyAsync(m->coords, coords, nv * dim * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    ffb::cuda_check(cudaMemcpyAsync(m->vconn, vconn, ne * (dim + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    if (dconn)
      ffb::cuda_check(cudaMemcpyAsync(m->dconn, dconn, ne * k * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    ffb::cuda_check(cudaStreamSynchronize(ctx->stream), "mesh upload");
    m->generation = next_generation();
    // flatten_mesh validates first (device.cpp:49)
    try {
      validate_mesh(m.get(), true);
    } catch (...) {
      free_mesh(m.release());
      throw;
    }
    *out = m.release();
  });
}

int ff_mesh_update(ff_mesh* m, const double* coords, const int32_t* vconn, const int32_t* dconn) {
  return guarded([&] {
    require(m, "null mesh");
    ff_ctx* ctx = m->ctx;
    bind(ctx);
    if (coords)
      ffb::cuda_check(cudaMemcpyAsync(m->coords, coords, m->nv * m->dim * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    if (vconn)
      ffb::cuda_check(cudaMemcpyAsync(m->vconn, vconn, m->ne * (m->dim + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    if (dconn && m->dconn != m->vconn)
      ffb::cuda_check(cudaMemcpyAsync(m->dconn, dconn, m->ne * m->k * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    ffb::cuda_check(cudaStreamSynchronize(ctx->stream), "mesh update");
    if (vconn || dconn) {
      // new connectivity: slot and gather plans (and captured graphs) are
      // re-derived; it is a new mesh, so it is validated like one
      m->generation = next_generation();
      validate_mesh(m, true);
    }
    // coordinates alone are the flattened arrays changing under a validated
    // mesh (test_device.cpp:283-285): degenerate elements surface in assembly
  });
}

int ff_mesh_destroy(ff_mesh* m) {
  return guarded([&] {
    if (!m) return;
    bind(m->ctx);
    free_mesh(m);
  });
}

int ff_pattern_build(ff_ctx* ctx, const ff_mesh* m, int64_t rb, int64_t re, ff_pattern** out) {
  return guarded([&] {
    require(ctx && m && out, "ff_pattern_build: null argument");
    const int bs = m->bs;
    require(0 <= rb && rb <= re && re <= bs * m->n_dofs, "row block outside [0, n_dofs]");
    require(rb % bs == 0 && re % bs == 0, "row block of a vector space must cover whole nodes");
    rb /= bs;
    re /= bs;
    require(re - rb < (int64_t(1) << 31), "row block too large");
    bind(ctx);
    auto p = std::make_unique<ff_pattern>();
    p->ctx = ctx;
    p->rb = rb;
    p->re = re;
    p->bs = bs;
    p->k = m->k;
    validate_mesh(m, true);  // build_sparsity validates first (device.cpp:67)
    int mx = 0;
    ffb::cuda_check(ffb::kernels::build_pattern(m->dconn, m->ne, m->k, rb, re, ctx->sm_count, ctx->stream, &p->row_ptr,
                                                &p->col_idx, &p->nnz, &mx),
                    "K1 pattern build");
    p->max_row_len = mx;
    *out = p.release();
  });
}

int ff_pattern_info(const ff_pattern* p, int64_t* n_rows, int64_t* nnz, int32_t* max_row_len) {
  return guarded([&] {
    require(p, "null pattern");
    if (n_rows) *n_rows = p->bs * (p->re - p->rb);
    if (nnz) *nnz = int64_t(p->bs) * p->bs * p->nnz;
    if (max_row_len) *max_row_len = p->bs * p->max_row_len;
  });
}

// device CSR of the pattern as the user sees it (block-expanded for bs > 1)
void ensure_device_csr(ff_pattern* p) {
  if (p->bs == 1 || p->vrow_ptr) return;
  bind(p->ctx);
  const int64_t n = p->re - p->rb;
  p->vrow_ptr = device_alloc<int64_t>(p->bs * n + 1, "blocked row_ptr");
  p->vcol_idx = device_alloc<int32_t>(int64_t(p->bs) * p->bs * p->nnz, "blocked col_idx");
  ffb::cuda_check(ffb::kernels::expand_block_pattern(p->row_ptr, p->col_idx, n, p->bs, p->vrow_ptr, p->vcol_idx,
                                                     p->ctx->sm_count, p->ctx->stream),
                  "block pattern expansion");
  ffb::cuda_check(cudaStreamSynchronize(p->ctx->stream), "block pattern expansion");
}

int ff_pattern_export(const ff_pattern* p, int64_t* row_ptr, int32_t* col_idx) {
  return guarded([&] {
    require(p, "null pattern");
    bind(p->ctx);
    ff_pattern* q = const_cast<ff_pattern*>(p);  // the expansion is a cache
    ensure_device_csr(q);
    const int64_t* rp = p->bs == 1 ? p->row_ptr : p->vrow_ptr;
    const int32_t* ci = p->bs == 1 ? p->col_idx : p->vcol_idx;
    const int64_t n = p->bs * (p->re - p->rb), nnz = int64_t(p->bs) * p->bs * p->nnz;
    if (row_ptr) ffb::cuda_check(cudaMemcpy(row_ptr, rp, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
    if (col_idx) ffb::cuda_check(cudaMemcpy(col_idx, ci, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
  });
}

int ff_pattern_export_ell(const ff_pattern* p, int32_t max_nz, int32_t* row_len, int32_t* row_cols) {
  return guarded([&] {
    require(p && row_len && row_cols, "null argument");
    require(max_nz >= p->bs * p->max_row_len, "max_nz smaller than the longest row");
    const int64_t n = p->bs * (p->re - p->rb);
    std::vector<int64_t> rp(n + 1);
    std::vector<int32_t> ci(int64_t(p->bs) * p->bs * p->nnz);
    if (ff_pattern_export(p, rp.data(), ci.data()) != FF_OK) throw Error(FF_E_CUDA, g_error);
    for (int64_t i = 0; i < n; ++i) {
      row_len[i] = static_cast<int32_t>(rp[i + 1] - rp[i]);
      for (int32_t c = 0; c < max_nz; ++c)
        row_cols[i * max_nz + c] = c < row_len[i] ? ci[rp[i] + c] : -1;
    }
  });
}

int ff_pattern_device(const ff_pattern* p, const int64_t** row_ptr, const int32_t** col_idx) {
  return guarded([&] {
    require(p, "null pattern");
    ff_pattern* q = const_cast<ff_pattern*>(p);
    ensure_device_csr(q);
    if (row_ptr) *row_ptr = p->bs == 1 ? p->row_ptr : p->vrow_ptr;
    if (col_idx) *col_idx = p->bs == 1 ? p->col_idx : p->vcol_idx;
  });
}

int ff_pattern_destroy(ff_pattern* p) {
  return guarded([&] {
    if (!p) return;
    bind(p->ctx);
    cudaFree(p->row_ptr);
    cudaFree(p->col_idx);
    cudaFree(p->vrow_ptr);
    cudaFree(p->vcol_idx);
    cudaFree(p->slots);
    drop_graph(p);
    free_gather(p);
    cudaFree(p->ginv);
    cudaFree(p->bvec);
    cudaFree(p->e2e_values);
    cudaFree(p->e2e_rhs);
    delete p;
  });
}

int ff_pattern_prepare(ff_pattern* p, const ff_mesh* m) {
  return guarded([&] {
    require(p && m, "null argument");
    ensure_plan(p, m);
  });
}

int ff_pattern_gather_info(ff_pattern* p, const ff_mesh* m, ff_gather_info* out) {
  return guarded([&] {
    require(p && m && out, "null argument");
    require(m->k <= 12, "row gather supports at most 12 DOFs per element");
    ensure_gather_plan(p, m);
    out->n_items = p->gather.n_items;
    out->n_steps = p->gather.n_steps;
    out->n_incidences = p->gather.n_incidences;
    out->record_bytes = p->gather.rec_bytes;
    out->build_ms = p->gather_ms;
    out->n_classes = static_cast<int>(p->gather.classes.size());
    out->n_class_rows = p->gather.n_class_rows;
    out->n_class_items = p->gather.n_citems;
    // what launch_gather issues: K2a + the class kernel(s) + the non-empty
    // generic ranges
    const auto& g = p->gather;
    out->launches = (m->ne > 0 ? 1 : 0) + (g.n_citems_short > 0) + (g.n_citems > g.n_citems_short) +
                    (g.n_short > 0) + (g.n_items > g.n_short);
  });
}

int ff_scatter_selected(const ff_form* f, const ff_pattern* p, unsigned flags, int* mode) {
  return guarded([&] {
    require(f && p && mode, "null argument");
    *mode = select_scatter(f, p, flags, p->max_row_len <= 256 ? 1 : 2);
  });
}

int ff_assemble_device(ff_form* f, const ff_mesh* m, ff_pattern* p, double* d_values, double* d_rhs, void* stream) {
  return guarded([&] {
    require(f && m && p && d_values && d_rhs, "ff_assemble_device: null argument");
    bind(f->ctx);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : f->ctx->stream;
    // repeated assemblies replay one CUDA graph of the whole launch sequence
    // (K2a, class and generic row kernels with their side-stream fork/join, or
    // K0 + K2): one launch instead of 4-6, no host work per step. The first
    // call builds plans and modules; the second identical call is captured.
    // (scalar forms: the vector gather's sub-row kernels measured slower as a
    // graph, 70.1 vs 68.6 ms at config 5; created streams only: the legacy and
    // per-thread default streams are not captured)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (std::getenv("FF_NO_GRAPH") || f->raw || f->ncomp > 1 || s == nullptr || s == cudaStreamLegacy ||
        s == cudaStreamPerThread || cudaStreamIsCapturing(s, &cap) != cudaSuccess ||
        cap != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      launch_assembly(f, m, p, d_values, d_rhs, s);
      return;
    }
    const std::vector<std::uint64_t> key = graph_key(f, m, p, d_values, d_rhs, s);
    if (p->graph_exec && key == p->graph_key) {
      ffb::cuda_check(cudaGraphLaunch(p->graph_exec, s), "cudaGraphLaunch");
      return;
    }
    if (key != p->graph_warm_key) {
      launch_assembly(f, m, p, d_values, d_rhs, s);
      p->graph_warm_key = graph_key(f, m, p, d_values, d_rhs, s);
      return;
    }
    drop_graph(p);
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();  // not capturable here: plain launches from now on
      p->graph_warm_key.clear();
      launch_assembly(f, m, p, d_values, d_rhs, s);
      return;
    }
    cudaGraph_t g = nullptr;
    try {
      launch_assembly(f, m, p, d_values, d_rhs, s);
    } catch (...) {
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      throw;
    }
    ffb::cuda_check(cudaStreamEndCapture(s, &g), "cudaStreamEndCapture");
    const cudaError_t e = cudaGraphInstantiate(&p->graph_exec, g, 0);
    cudaGraphDestroy(g);
    ffb::cuda_check(e, "cudaGraphInstantiate");
    p->graph_key = key;
    ffb::cuda_check(cudaGraphLaunch(p->graph_exec, s), "cudaGraphLaunch");
  });
}

int ff_scatter_calibrate(ff_form* f, const ff_mesh* m, ff_pattern* p, double* d_values, double* d_rhs, void* stream,
                         ff_scatter_timing* out) {
  return guarded([&] {
    require(f && m && p && d_values && d_rhs, "ff_scatter_calibrate: null argument");
    require(f->ctx && f->ctx == m->ctx && m->ctx == p->ctx, "form, mesh and pattern must share one context");
    bind(f->ctx);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : f->ctx->stream;
    calibrate_scatter(f, m, p, d_values, d_rhs, s);
    if (out) {
      out->gather_ms = p->auto_ms[0];
      out->atomic_ms = p->auto_ms[1];
      out->chosen = p->auto_mode;
    }
  });
}

int ff_assemble_device_ex(ff_form* f, const ff_mesh* m, ff_pattern* p, double* d_values, double* d_rhs, void* stream,
                          unsigned flags) {
  return guarded([&] {
    require(f && m && p && d_values && d_rhs, "ff_assemble_device_ex: null argument");
    require(flags < 128, "unknown flags");
    bind(f->ctx);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : f->ctx->stream;
    launch_assembly(f, m, p, d_values, d_rhs, s, flags);
  });
}

int ff_check(ff_ctx* ctx, ff_stats* stats) {
  return guarded([&] {
    require(ctx, "null context");
    bind(ctx);
    ffb::cuda_check(cudaDeviceSynchronize(), "device");
    report_status(ctx, stats);
  });
}

int ff_assemble(ff_form* f, ff_mesh* m, ff_pattern* p, const double* coords, const int32_t* vconn, const int32_t* dconn,
                double* values_out, double* rhs_out, ff_stats* stats) {
  return guarded([&] {
    require(f && m && p && values_out && rhs_out, "ff_assemble: null argument");
    const auto t0 = std::chrono::steady_clock::now();
    ff_ctx* ctx = f->ctx;
    require(ctx, "form was compiled without a context");
    bind(ctx);
    // inputs: the flattened mesh (device.cpp:48-64 analogue), host -> device
    if (coords)
      ffb::cuda_check(cudaMemcpyAsync(m->coords, coords, m->nv * m->dim * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    const int64_t n_rows = p->bs * (p->re - p->rb);
    const int64_t nnz = int64_t(p->bs) * p->bs * p->nnz;
    if (!p->e2e_values) p->e2e_values = device_alloc<double>(nnz, "values");
    if (!p->e2e_rhs) p->e2e_rhs = device_alloc<double>(n_rows, "rhs");
    const bool has_d = dconn && m->dconn != m->vconn;
    auto assemble_and_copy = [&]() {
      launch_assembly(f, m, p, p->e2e_values, p->e2e_rhs, ctx->stream);
      ffb::cuda_check(cudaMemcpyAsync(values_out, p->e2e_values, nnz * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
      ffb::cuda_check(cudaMemcpyAsync(rhs_out, p->e2e_rhs, n_rows * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    };
    // The reference re-searches every column on every call (device.cpp:274-288);
    // here the connectivity goes through staging buffers and is compared
    // exactly with the resident copy: any change gives the mesh a new
    // generation, so the slot and gather plans are re-derived (and the missing
    // column check re-run), and the new connectivity is validated like a new
    // mesh (device.cpp:49). Once the (pattern, mesh) plans exist, the upload and
    // compare run on their own stream while the assembly runs with the resident
    // connectivity and its values go back to the host (H2D and D2H overlap on
    // the full-duplex link); a changed connectivity re-runs the assembly.
    const bool planned = p->plan_mesh == m && p->plan_generation == m->generation && p->slots;
    if ((vconn || has_d) && planned) {
      const int64_t nvc = m->ne * (m->dim + 1), ndc = m->ne * m->k;
      if (vconn && !m->stage) m->stage = device_alloc<int32_t>(std::max<int64_t>(nvc, 1), "connectivity staging");
      if (has_d && !m->stage_d) m->stage_d = device_alloc<int32_t>(std::max<int64_t>(ndc, 1), "connectivity staging");
      unsigned long long* d_diff = ctx->d_status + 3;
      cudaStream_t u = ctx->upload;
      ffb::cuda_check(cudaMemsetAsync(d_diff, 0, 2 * sizeof(unsigned long long), u), "memset");
      if (vconn) {
        ffb::cuda_check(cudaMemcpyAsync(m->stage, vconn, nvc * sizeof(int32_t), cudaMemcpyHostToDevice, u), "H2D");
        ffb::cuda_check(ffb::kernels::compare(m->stage, m->vconn, nvc, d_diff, ctx->sm_count, u), "compare");
      }
      if (has_d) {
        ffb::cuda_check(cudaMemcpyAsync(m->stage_d, dconn, ndc * sizeof(int32_t), cudaMemcpyHostToDevice, u), "H2D");
        ffb::cuda_check(ffb::kernels::compare(m->stage_d, m->dconn, ndc, d_diff + 1, ctx->sm_count, u), "compare");
      }
      ffb::cuda_check(cudaMemcpyAsync(ctx->h_status + 2, d_diff, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, u),
                      "D2H");
      assemble_and_copy();
      ffb::cuda_check(cudaStreamSynchronize(u), "connectivity upload");
      ffb::cuda_check(cudaStreamSynchronize(ctx->stream), "D2H");
      if (ctx->h_status[2] || ctx->h_status[3]) {  // changed: adopt it and assemble again
        if (vconn && ctx->h_status[2])
          ffb::cuda_check(cudaMemcpyAsync(m->vconn, m->stage, nvc * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream), "copy");
        if (has_d && ctx->h_status[3])
          ffb::cuda_check(cudaMemcpyAsync(m->dconn, m->stage_d, ndc * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream), "copy");
        m->generation = next_generation();
        validate_mesh(m, true);
        assemble_and_copy();
      }
    } else {
      bool changed = false;
      if (vconn) changed |= upload_conn(m, m->vconn, vconn, m->ne * (m->dim + 1));
      if (has_d) changed |= upload_conn(m, m->dconn, dconn, m->ne * m->k);
      if (changed) {
        m->generation = next_generation();
        validate_mesh(m, true);
      }
      assemble_and_copy();
    }
    report_status(ctx, stats);  // (also waits for the D2H copies)
    if (stats) stats->ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  });
}

// ---- downstream consumer ---------------------------------------------------

int ff_spmv(ff_pattern* p, const double* d_values, const double* d_x, double* d_y, void* stream) {
  return guarded([&] {
    require(p && d_values && d_x && d_y, "ff_spmv: null argument");
    bind(p->ctx);
    ensure_device_csr(p);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->ctx->stream;
    const int64_t n = p->bs * (p->re - p->rb);
    ffb::cuda_check(ffb::kernels::spmv(p->bs == 1 ? p->row_ptr : p->vrow_ptr, p->bs == 1 ? p->col_idx : p->vcol_idx,
                                       d_values, d_x, d_y, n, p->ctx->sm_count, s),
                    "spmv");
  });
}

int ff_cg_solve(ff_pattern* p, const double* d_values, const double* d_b, double* d_x, double tol, int max_iter,
                ff_cg_result* out) {
  return guarded([&] {
    require(p && d_values && d_b && d_x, "ff_cg_solve: null argument");
    require(p->rb == 0, "cg_solve needs the full system (row block starting at 0)");
    bind(p->ctx);
    ensure_device_csr(p);
    const int64_t n = p->bs * (p->re - p->rb);
    ffb::kernels::CgStats st;
    ffb::cuda_check(ffb::kernels::cg_solve(p->bs == 1 ? p->row_ptr : p->vrow_ptr,
                                           p->bs == 1 ? p->col_idx : p->vcol_idx, d_values, d_b, d_x, n, tol,
                                           max_iter, p->ctx->sm_count, p->ctx->stream, &st),
                    "cg_solve");
    if (st.breakdown == 1) throw Error(FF_E_ARG, "cg_solve: breakdown (non-finite step)");
    if (st.breakdown == 2) throw Error(FF_E_ARG, "cg_solve: breakdown (non-finite residual)");
    if (out) {
      out->iterations = st.iterations;
      out->residual = st.residual;
      out->converged = st.converged;
    }
  });
}

namespace {
void write_value(std::FILE* f, double v) { std::fprintf(f, "%.17g", v); }
struct OutFile {
  std::FILE* f;
  explicit OutFile(const char* path) : f(std::fopen(path, "w")) {
    if (!f) throw Error(FF_E_ARG, std::string("cannot open '") + path + "' for writing");
  }
  ~OutFile() {
    if (f) std::fclose(f);
  }
};
}  // namespace

int ff_export_matrix(ff_pattern* p, const double* values, const char* path, int fmt) {
  return guarded([&] {
    require(p && values && path, "ff_export_matrix: null argument");
    const int64_t n = p->bs * (p->re - p->rb), nnz = int64_t(p->bs) * p->bs * p->nnz;
    std::vector<int64_t> rp(n + 1);
    std::vector<int32_t> ci(std::max<int64_t>(nnz, 1));
    if (ff_pattern_export(p, rp.data(), ci.data()) != FF_OK) throw Error(FF_E_CUDA, g_error);
    if (ff_export_csr(n, rp.data(), ci.data(), values, path, fmt) != FF_OK) throw Error(FF_E_ARG, g_error);
  });
}

int ff_export_csr(int64_t n, const int64_t* rp, const int32_t* ci, const double* values, const char* path, int fmt) {
  return guarded([&] {
    require(rp && ci && values && path && n >= 0, "ff_export_csr: null argument");
    require(fmt == FF_EXPORT_MATRIX_MARKET || fmt == FF_EXPORT_CSV, "unknown export format");
    const int64_t nnz = rp[n];
    OutFile fh(path);
    // linalg.cpp:170-199: rows in order, sorted columns (the ELL order without padding)
    if (fmt == FF_EXPORT_MATRIX_MARKET) {
      std::fprintf(fh.f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n",
                   static_cast<long long>(n), static_cast<long long>(n), static_cast<long long>(nnz));
      for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
          std::fprintf(fh.f, "%lld %d ", static_cast<long long>(i + 1), ci[k] + 1);
          write_value(fh.f, values[k]);
          std::fputc('\n', fh.f);
        }
    } else {
      for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
          std::fprintf(fh.f, "%lld,%d,", static_cast<long long>(i), ci[k]);
          write_value(fh.f, values[k]);
          std::fputc('\n', fh.f);
        }
    }
  });
}

int ff_export_vector(const double* b, int64_t n, const char* path, int fmt) {
  return guarded([&] {
    require(b && path && n >= 0, "ff_export_vector: null argument");
    require(fmt == FF_EXPORT_MATRIX_MARKET || fmt == FF_EXPORT_CSV, "unknown export format");
    OutFile fh(path);
    if (fmt == FF_EXPORT_MATRIX_MARKET)
      std::fprintf(fh.f, "%%%%MatrixMarket matrix array real general\n%lld 1\n", static_cast<long long>(n));
    for (int64_t i = 0; i < n; ++i) {
      write_value(fh.f, b[i]);
      std::fputc('\n', fh.f);
    }
  });
}

// ---- host helpers ---------------------------------------------------------

int ff_unit_square_mesh(int n, double* coords, int32_t* conn) {
  return guarded([&] {
    const fem::Mesh m = meshgen::unit_square_mesh(n);
    const auto c = m.coords_flat();
    const auto e = m.conn_flat();
    std::memcpy(coords, c.data(), c.size() * sizeof(double));
    std::memcpy(conn, e.data(), e.size() * sizeof(int32_t));
  });
}

int ff_kuhn_mesh(int n, double* coords, int32_t* conn) {
  return guarded([&] {
    const fem::Mesh m = meshgen::kuhn_cube_mesh(n);
    const auto c = m.coords_flat();
    const auto e = m.conn_flat();
    std::memcpy(coords, c.data(), c.size() * sizeof(double));
    std::memcpy(conn, e.data(), e.size() * sizeof(int32_t));
  });
}

int ff_kuhn_p2_dofs(int n, const int32_t* vconn, int64_t ne, int32_t* dconn) {
  return guarded([&] {
    fem::Mesh m;
    m.dim = 3;
    m.elements.resize(ne);
    for (int64_t e = 0; e < ne; ++e)
      for (int a = 0; a < 4; ++a) m.elements[e].nodes[a] = vconn[4 * e + a];
    const fem::DofMap d = meshgen::kuhn_p2_dofs(n, m);
    std::memcpy(dconn, d.dofs.data(), d.dofs.size() * sizeof(int32_t));
  });
}

int ff_p2_dofs(int dim, const int32_t* vconn, int64_t ne, int64_t nv, int32_t* dconn, int64_t* n_dofs) {
  return guarded([&] {
    fem::Mesh m;
    m.dim = dim;
    m.nodes.resize(nv);
    m.elements.resize(ne);
    for (int64_t e = 0; e < ne; ++e)
      for (int a = 0; a <= dim; ++a) m.elements[e].nodes[a] = vconn[(dim + 1) * e + a];
    const fem::DofMap d = fem::lagrange_dofs(m, 2);
    std::memcpy(dconn, d.dofs.data(), d.dofs.size() * sizeof(int32_t));
    if (n_dofs) *n_dofs = d.n_dofs;
  });
}

int ff_partition_rows(int64_t n_dofs, int n_parts, int part, int64_t* rb, int64_t* re) {
  return guarded([&] {
    require(n_parts > 0 && part >= 0 && part < n_parts, "invalid partition");
    *rb = n_dofs * part / n_parts;
    *re = n_dofs * (part + 1) / n_parts;
  });
}

int ff_select_elements(const int32_t* dconn, int64_t ne, int32_t k, int64_t rb, int64_t re, int64_t* ids, int64_t* count) {
  return guarded([&] {
    require(dconn && count, "null argument");
    int64_t n = 0;
    for (int64_t e = 0; e < ne; ++e) {
      bool touch = false;
      for (int a = 0; a < k && !touch; ++a) touch = dconn[e * k + a] >= rb && dconn[e * k + a] < re;
      if (touch) {
        if (ids) ids[n] = e;
        ++n;
      }
    }
    *count = n;
  });
}

}  // extern "C"

/* femforge_b200.h -- the drop-in C ABI of the femforge-b200 assembly engine.
 *
 * The hot path of the reference (femforge, arXiv:1802.03433, mounted at
 * /root/reference/proj) sits behind these C++ entry points, which this ABI
 * replaces:
 *
 *   device::flatten_mesh     include/femforge/device/device.hpp:63   -> ff_mesh_create
 *   device::build_sparsity   include/femforge/device/device.hpp:74   -> ff_pattern_build
 *   codegen::compile_form /  include/femforge/codegen/kernel.hpp:65  -> ff_form_create
 *   codegen::emit_source     include/femforge/codegen/kernel.hpp:76  -> ff_form_source / ff_compile
 *   device::assemble_sparse  include/femforge/device/device.hpp:143-153 -> ff_assemble (host
 *                            buffers) / ff_assemble_device (device-resident, async)
 *   device::FormEvaluator    include/femforge/device/device.hpp:97-102 -> ff_form (the
 *                            compiled element kernel is the evaluator plug-in)
 *
 * Conventions: C linkage, plain pointers and sizes, no exceptions across the
 * ABI. Every function returns an ff_status (0 = FF_OK); on failure the
 * thread-local ff_last_error() carries the reference's message (e.g.
 * "degenerate element 7 (|det J| <= 1e-14)", "column 5 not present in
 * sparsity row 0 (inconsistent sparsity pattern)"). Caller-owned host arrays
 * go in, caller-allocated outputs come back; library-owned device memory
 * lives behind handles. Handles are immutable after creation except the
 * per-context stream; use one context per device and per host thread.
 *
 * Output layout: CSR with int64 row_ptr (n_rows+1), int32 col_idx (nnz,
 * sorted ascending within each row, diagonal always present -- device.cpp:70),
 * fp64 values (nnz) and fp64 rhs (n_rows). A row block [row_begin, row_end)
 * selects the rows a device owns (multi-GPU row partitioning).
 */
#ifndef FEMFORGE_B200_H
#define FEMFORGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ff_status {
  FF_OK = 0,
  FF_E_ARG = -1,        /* invalid argument / launch limit (DeviceError in device.cpp:90-97) */
  FF_E_DEGENERATE = -2, /* |det J| <= 1e-14; lowest element index in the message / stats */
  FF_E_PATTERN = -3,    /* column not present in sparsity row (device.cpp:285-288) */
  FF_E_NVRTC = -4,      /* runtime compilation failed (log in ff_last_error) */
  FF_E_CUDA = -5,       /* CUDA runtime error */
  FF_E_FORM = -6,       /* weak-form error (FormError / CodegenError) */
  FF_E_MESH = -7,       /* mesh validation error (MeshError) */
  FF_E_SYMBOLIC = -8,   /* parse / symbolic error (ParseError with offset) */
  FF_E_NOMEM = -9       /* device or host allocation failed */
} ff_status;

typedef struct ff_ctx ff_ctx;
typedef struct ff_form ff_form;
typedef struct ff_mesh ff_mesh;
typedef struct ff_pattern ff_pattern;

/* element body strategies (codegen::Strategy) */
enum { FF_STRATEGY_AUTO = 0, FF_STRATEGY_TENSOR = 1, FF_STRATEGY_POINTWISE = 2 };

typedef struct ff_form_desc {
  int dim;               /* 2 or 3 */
  int degree;            /* Lagrange degree 1 or 2 */
  int quad_rule;         /* 0 = default (2D: reference 3-point rule; 3D: 4-point degree 2) */
  int strategy;          /* FF_STRATEGY_* */
  int block_size;        /* threads per CTA of the element kernels; 0 = by body (pointwise 32, reference-tensor 128) */
  const char* bilinear;  /* integrand over u, u_x, u_y[, u_z], v, v_x, v_y[, v_z], x, y[, z] */
  const char* linear;    /* integrand over v, x, y[, z] */
} ff_form_desc;

typedef struct ff_form_info {
  int dim, degree, n_local, n_quad, strategy;
  int n_invariants;      /* reference-tensor strategy: merged geometric invariants */
  int n_unique_entries;  /* distinct local entries computed per element */
  int64_t flops_per_element;
  int registers;         /* per thread, from the loaded cubin (0 if not loaded) */
  int shared_bytes;      /* static shared memory per CTA */
  double compile_ms;     /* symbolic + emit + NVRTC */
  int n_kinv;            /* bilinear invariants stored per element by the row gather (0: no gather) */
  int64_t row_flops;     /* fp64 operations of the n_local gather rows of one element */
} ff_form_info;

typedef struct ff_stats {
  int64_t bad_element;   /* lowest degenerate element, or -1 */
  int64_t bad_row;       /* lowest row with a missing column, or -1 */
  double ms;             /* wall time of the call (host-synchronous entry points) */
} ff_stats;

/* ---- library / context ------------------------------------------------- */
const char* ff_version(void);
const char* ff_last_error(void);
int ff_device_count(int* count);
int ff_init(int device, ff_ctx** out);
int ff_ctx_destroy(ff_ctx* ctx);
int ff_ctx_synchronize(ff_ctx* ctx);
void* ff_ctx_stream(ff_ctx* ctx); /* cudaStream_t of the context */
/* Default scatter of the context; per-call flags override it.
 *   FF_SCATTER_GATHER_MODE (default): row gather -- element invariants, then one
 *     CSR row per lane accumulated in shared memory and written once
 *     (atomic-free, deterministic; needs a reference-tensor form, <= 12 DOFs
 *     per element and rows of <= 221 entries, else the atomic kernel runs);
 *   FF_SCATTER_ATOMIC_MODE: element-parallel fp64 RED after a zero-fill (the
 *     reference's parallel mode, device.cpp:193-200);
 *   FF_SCATTER_AUTO_MODE: measured choice -- the first device assembly of a
 *     (form, pattern, mesh) times both scatters on the caller's buffers and
 *     keeps the faster (ff_scatter_calibrate; the atomic scatter alone when
 *     the form/pattern cannot gather). */
enum { FF_SCATTER_ATOMIC_MODE = 1, FF_SCATTER_GATHER_MODE = 2, FF_SCATTER_AUTO_MODE = 3 };
int ff_ctx_set_scatter(ff_ctx* ctx, int mode);

/* ---- forms: weak form text -> symbolic -> CUDA source -> NVRTC (sm_100a) - */
/* ctx may be NULL: compile-only (no device needed; ff_assemble* then fail). */
int ff_form_create(ff_ctx* ctx, const ff_form_desc* desc, ff_form** out);
/* Vector-valued (ncomp-component) P1/P2 forms as blocks of scalar forms:
 * a(u,v) = sum_{c,d} a_cd(u_d, v_c) with block_bilinear[c*ncomp + d] the
 * scalar integrand over u*, v* (trial component d, test component c), and
 * l(v) = sum_c l_c(v_c) with block_linear[c]. Local DOF a*ncomp + c, global
 * DOF ncomp*node + c; the mesh must carry ncomp (ff_mesh_set_components). The
 * pattern is the ncomp x ncomp block expansion of the scalar pattern; the
 * scatter is the fp64-RED kernel (BASELINE config 5, elasticity). */
int ff_form_create_blocked(ff_ctx* ctx, const ff_form_desc* desc, int ncomp, const char* const* block_bilinear,
                           const char* const* block_linear, ff_form** out);
/* Raw template route: compile caller-provided CUDA source that defines
 * extern "C" __global__ ff_assemble_atomic with the template's signature. */
int ff_compile(ff_ctx* ctx, const char* cuda_src, int dim, int degree, int block_size, ff_form** out,
               char* log, size_t log_cap);
int ff_form_source(const ff_form* form, char* buf, size_t cap, size_t* len);
int ff_form_cubin(const ff_form* form, void* buf, size_t cap, size_t* len);
int ff_form_info_get(const ff_form* form, ff_form_info* out);
int ff_form_destroy(ff_form* form);

/* ---- meshes: host arrays copied to the device --------------------------- */
/* coords [n_vertices][dim] fp64; vconn [n_elems][dim+1] vertex ids;
 * dconn [n_elems][dofs_per_elem] DOF ids (NULL for P1: dconn = vconn). */
int ff_mesh_create(ff_ctx* ctx, int dim, const double* coords, int64_t n_vertices, const int32_t* vconn,
                   int64_t n_elems, const int32_t* dconn, int32_t dofs_per_elem, int64_t n_dofs,
                   ff_mesh** out);
/* Vector space on the mesh: ncomp components per node (DOF ncomp*node + c);
 * n_dofs of ff_mesh_create stays the node (scalar) DOF count. */
int ff_mesh_set_components(ff_mesh* mesh, int ncomp);
/* Re-upload coordinates/connectivity into an existing mesh (same sizes). */
int ff_mesh_update(ff_mesh* mesh, const double* coords, const int32_t* vconn, const int32_t* dconn);
int ff_mesh_destroy(ff_mesh* mesh);

/* ---- sparsity (K1: sort + unique over element DOF pairs) ----------------- */
int ff_pattern_build(ff_ctx* ctx, const ff_mesh* mesh, int64_t row_begin, int64_t row_end, ff_pattern** out);
int ff_pattern_info(const ff_pattern* p, int64_t* n_rows, int64_t* nnz, int32_t* max_row_len);
int ff_pattern_export(const ff_pattern* p, int64_t* row_ptr, int32_t* col_idx);
/* ELL view for API parity with SparsityPattern (device.hpp:67-72): row_len
 * [n_rows], row_cols [n_rows][max_nz] padded with -1. */
int ff_pattern_export_ell(const ff_pattern* p, int32_t max_nz, int32_t* row_len, int32_t* row_cols);
int ff_pattern_device(const ff_pattern* p, const int64_t** row_ptr, const int32_t** col_idx);
int ff_pattern_destroy(ff_pattern* p);
/* Element slot plan of (pattern, mesh): per element and local (a,b) the
 * position of column dof[b] inside row dof[a]. Built on first assembly;
 * exposed for tests. Returns FF_E_PATTERN on a missing column. */
int ff_pattern_prepare(ff_pattern* p, const ff_mesh* mesh);
/* Gather plan statistics (built by the first gather assembly or here):
 * warp items, lock-step steps (records / 32) and incidences (row, element). */
typedef struct ff_gather_info {
  int64_t n_items, n_steps, n_incidences;  /* generic items (rows outside the classes) */
  int record_bytes;
  double build_ms;
  int n_classes;                            /* row classes with a specialised kernel */
  int64_t n_class_rows, n_class_items;
  int launches;                             /* kernel launches per gather assembly (K2a, class, generic) */
} ff_gather_info;
/* Row classes of the gather plan: rows with identical incidence sequences
 * get an NVRTC kernel specialised to the class (slots as compile-time
 * register indices). Classes need >= min_rows rows (default 128); 0 turns
 * the specialisation off (every row takes the generic gather). */
int ff_ctx_set_gather_classes(ff_ctx* ctx, int64_t min_rows);
/* The class-specialised source for caller-given classes (tests / inspection):
 * n classes with len[c] entries and steps[c] incidences; local and slots are
 * the concatenated per-step local indices and [steps][n_local] slot bytes. */
int ff_class_source(const ff_form* form, int n, const int32_t* len, const int32_t* steps, const int32_t* local,
                    const uint8_t* slots, char* buf, size_t cap, size_t* out_len);
int ff_pattern_gather_info(ff_pattern* p, const ff_mesh* mesh, ff_gather_info* out);
/* Which scatter the next assembly of (form, pattern) runs: FF_SCATTER_*_MODE. */
int ff_scatter_selected(const ff_form* form, const ff_pattern* p, unsigned flags, int* mode);
/* Times the row gather and the atomic scatter of (form, mesh, pattern) on the
 * given device buffers (CUDA events on `stream`: one warm-up run, then the
 * mean of 3 runs each; gather_ms < 0 when the gather cannot run), records the
 * faster as the pattern's choice for FF_SCATTER_AUTO_MODE and returns it.
 * Blocking; leaves a valid assembly in the buffers. */
typedef struct ff_scatter_timing {
  double gather_ms, atomic_ms;
  int chosen;            /* FF_SCATTER_GATHER_MODE or FF_SCATTER_ATOMIC_MODE */
} ff_scatter_timing;
int ff_scatter_calibrate(ff_form* form, const ff_mesh* mesh, ff_pattern* p, double* d_values, double* d_rhs,
                         void* stream, ff_scatter_timing* out);

/* ---- numeric assembly (K0 zero-fill + K2 element kernel with scatter) ---- */
/* Device-resident, asynchronous on `stream` (NULL: the context stream).
 * d_values [nnz], d_rhs [n_rows] are caller-owned device buffers. Errors
 * detected on the device are reported by ff_check(). */
int ff_assemble_device(ff_form* form, const ff_mesh* mesh, ff_pattern* p, double* d_values, double* d_rhs,
                       void* stream);
/* Same with flags. Scatter flags override the context mode:
 * FF_SCATTER_ATOMIC (element-parallel fp64 RED, needs K0: FF_SKIP_ZERO = K2
 * only on already-zero buffers, FF_ZERO_ONLY = K0 only), FF_SCATTER_GATHER
 * (row gather; FF_GATHER_INVARIANTS_ONLY /
 * FF_GATHER_ROWS_ONLY launch only its first / second kernel, for timing). */
enum {
  FF_SKIP_ZERO = 1,
  FF_ZERO_ONLY = 2,
  FF_SCATTER_ATOMIC = 4,
  FF_SCATTER_GATHER = 16,
  FF_GATHER_INVARIANTS_ONLY = 32,
  FF_GATHER_ROWS_ONLY = 64
};
int ff_assemble_device_ex(ff_form* form, const ff_mesh* mesh, ff_pattern* p, double* d_values, double* d_rhs,
                          void* stream, unsigned flags);
/* Synchronises the context stream and reports device-side errors of the
 * last ff_assemble_device (degenerate element / missing column). */
int ff_check(ff_ctx* ctx, ff_stats* stats);
/* End-to-end with host buffers (the reference call shape): uploads the
 * mesh's coordinates and connectivity, assembles, downloads values and rhs,
 * synchronously. Host buffers may be pageable or pinned. */
int ff_assemble(ff_form* form, ff_mesh* mesh, ff_pattern* p, const double* coords, const int32_t* vconn,
                const int32_t* dconn, double* values_out, double* rhs_out, ff_stats* stats);

/* ---- downstream consumer of the assembled system --------- */
/* y = A x on the device, A the pattern's CSR with device values (replaces
 * linalg::matvec(EllMatrix), linalg.cpp:35-49). */
int ff_spmv(ff_pattern* p, const double* d_values, const double* d_x, double* d_y, void* stream);
typedef struct ff_cg_result {
  int iterations;
  double residual; /* final relative residual ||r|| / ||b|| */
  int converged;
} ff_cg_result;
/* Unpreconditioned CG on the device, the reference's algorithm and stopping
 * rule (linalg.cpp:61-96): x0 = 0, stop when ||r|| <= tol ||b||. Breakdown
 * (non-finite step / residual) fails with the reference's messages. */
int ff_cg_solve(ff_pattern* p, const double* d_values, const double* d_b, double* d_x, double tol, int max_iter,
                ff_cg_result* out);
/* Host export of an assembled system in the reference's formats
 * (linalg.cpp:148-210): MatrixMarket coordinate / CSV triplets, %.17g. */
enum { FF_EXPORT_MATRIX_MARKET = 0, FF_EXPORT_CSV = 1 };
int ff_export_matrix(ff_pattern* p, const double* values, const char* path, int fmt);
int ff_export_vector(const double* b, int64_t n, const char* path, int fmt);
/* Host-only export of caller CSR arrays (n rows) in the same formats. */
int ff_export_csr(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* values, const char* path,
                  int fmt);

/* ---- host helpers (CPU only; no device needed) --------------------------- */
/* Parses `expr` (symbolic::parse, expr.cpp) and evaluates it at n points
 * [n][dim] of (x, y[, z]) (symbolic::eval); a symbol other than the first
 * `dim` coordinates fails with FF_E_SYMBOLIC "expression references symbol
 * 's'" (the CLI's coefficient check, femforge.cpp:95-113, and l2_error's,
 * linalg.cpp:101-104). n = 0 only validates. */
int ff_expr_eval(const char* expr, int dim, const double* pts, int64_t n, double* out);
/* The instantiated integrand of entry (i, j) (kind 0: bilinear) or i (kind
 * 1: linear) as text (symbolic::print): the inspection view the CLI's
 * `codegen --out-ir` writes (femforge.cpp:203-231). Same length protocol
 * as ff_class_source. */
int ff_form_entry_text(const ff_form* form, int kind, int i, int j, char* buf, size_t cap, size_t* out_len);
/* meshgen.cpp:13-33 unit square; SURVEY.md Appendix C Kuhn cube + P2 lattice. */
int ff_unit_square_mesh(int n, double* coords, int32_t* conn);
int ff_kuhn_mesh(int n, double* coords, int32_t* conn);
int ff_kuhn_p2_dofs(int n, const int32_t* vconn, int64_t n_elems, int32_t* dconn);
/* Generic P2 numbering (vertices first, then edges by (min,max)); returns
 * n_dofs through *n_dofs. */
int ff_p2_dofs(int dim, const int32_t* vconn, int64_t n_elems, int64_t n_vertices, int32_t* dconn,
               int64_t* n_dofs);
/* Contiguous row block of part `part` of `n_parts` (balanced by DOF count). */
int ff_partition_rows(int64_t n_dofs, int n_parts, int part, int64_t* row_begin, int64_t* row_end);
/* Elements with at least one DOF in [row_begin,row_end) (owned + halo), in
 * ascending order; ids may be NULL to count only. */
int ff_select_elements(const int32_t* dconn, int64_t n_elems, int32_t dofs_per_elem, int64_t row_begin,
                       int64_t row_end, int64_t* ids, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* FEMFORGE_B200_H */

/* oracle/femoracle.c -- TEST INFRASTRUCTURE ONLY: the CPU checker (see
 * femoracle.h for the parity status). Plain C11 + OpenMP, no product code.
 *
 * Each function restates one piece of the reference algorithm; the
 * file:line anchors are into /root/reference/proj.
 */
#include "femoracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* meshes                                                                    */

void fo_unit_square_mesh(int n, double* coords, int32_t* conn) {
  /* meshgen.cpp:13-33 */
  const double h = 1.0 / n;
  int64_t t = 0;
  for (int j = 0; j <= n; ++j)
    for (int i = 0; i <= n; ++i) {
      coords[2 * t] = i * h;
      coords[2 * t + 1] = j * h;
      ++t;
    }
  t = 0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      int32_t v00 = j * (n + 1) + i, v10 = v00 + 1, v01 = v00 + (n + 1), v11 = v01 + 1;
      int32_t* e = conn + 6 * t;
      e[0] = v00; e[1] = v10; e[2] = v11;
      e[3] = v00; e[4] = v11; e[5] = v01;
      ++t;
    }
}

void fo_kuhn_mesh(int n, double* coords, int32_t* conn) {
  /* Appendix C; mirrors meshgen.cpp:13-33 (h = 1.0/n, i innermost) and the
   * CW->CCW swap of meshgen.cpp:100-103 (nodes[1] <-> nodes[2]). */
  const double h = 1.0 / n;
  const int64_t m = n + 1;
  int64_t t = 0;
  for (int k = 0; k <= n; ++k)
    for (int j = 0; j <= n; ++j)
      for (int i = 0; i <= n; ++i) {
        coords[3 * t] = i * h;
        coords[3 * t + 1] = j * h;
        coords[3 * t + 2] = k * h;
        ++t;
      }
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  static const int odd[6] = {0, 1, 1, 0, 0, 1};
  t = 0;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        for (int p = 0; p < 6; ++p) {
          int c[3] = {i, j, k};
          int32_t v[4];
          v[0] = (int32_t)(c[0] + m * (c[1] + m * c[2]));
          c[perms[p][0]] += 1;
          v[1] = (int32_t)(c[0] + m * (c[1] + m * c[2]));
          c[perms[p][1]] += 1;
          v[2] = (int32_t)(c[0] + m * (c[1] + m * c[2]));
          v[3] = (int32_t)((i + 1) + m * ((j + 1) + m * (k + 1)));
          if (odd[p]) { int32_t s = v[1]; v[1] = v[2]; v[2] = s; }
          memcpy(conn + 4 * t, v, sizeof v);
          ++t;
        }
}

void fo_p2_dofs_kuhn(int n, const int32_t* vconn, int64_t ne, int32_t* dconn) {
  /* Appendix C: vertex (i,j,k) -> lattice (2i,2j,2k); edge midpoint -> sum of
   * the endpoint lattice coordinates / 2 = (i_a+i_b, ...). */
  static const int edges[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  const int64_t m = n + 1, L = 2 * (int64_t)n + 1;
  for (int64_t e = 0; e < ne; ++e) {
    int64_t I[4], J[4], K[4];
    for (int a = 0; a < 4; ++a) {
      int64_t v = vconn[4 * e + a];
      I[a] = v % m; J[a] = (v / m) % m; K[a] = v / (m * m);
      dconn[10 * e + a] = (int32_t)(2 * I[a] + L * (2 * J[a] + L * 2 * K[a]));
    }
    for (int q = 0; q < 6; ++q) {
      int a = edges[q][0], b = edges[q][1];
      dconn[10 * e + 4 + q] = (int32_t)((I[a] + I[b]) + L * ((J[a] + J[b]) + L * (K[a] + K[b])));
    }
  }
}

/* ------------------------------------------------------------------------ */
/* sparsity: device.cpp:66-88 (std::set per row, diagonal inserted first)    */

struct fo_pattern {
  int64_t rb, re;
  int64_t* row_ptr;
  int32_t* col_idx;
};

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

static int64_t row_unique(const int64_t* inc_ptr, const int64_t* inc, const int32_t* dconn, int k,
                          int64_t r, int64_t rb, int32_t* buf) {
  int64_t len = 0;
  buf[len++] = (int32_t)r;
  for (int64_t p = inc_ptr[r - rb]; p < inc_ptr[r - rb + 1]; ++p) {
    const int32_t* d = dconn + inc[p] * k;
    for (int b = 0; b < k; ++b) buf[len++] = d[b];
  }
  qsort(buf, (size_t)len, sizeof(int32_t), cmp_i32);
  int64_t u = 0;
  for (int64_t t = 0; t < len; ++t)
    if (u == 0 || buf[t] != buf[u - 1]) buf[u++] = buf[t];
  return u;
}

fo_pattern* fo_build_pattern(const int32_t* dconn, int64_t ne, int k, int64_t n_dofs,
                             int64_t rb, int64_t re) {
  (void)n_dofs;
  const int64_t nr = re - rb;
  int64_t* inc_ptr = calloc((size_t)nr + 1, sizeof(int64_t));
  for (int64_t e = 0; e < ne; ++e)
    for (int a = 0; a < k; ++a) {
      int64_t r = dconn[e * k + a];
      if (r >= rb && r < re) inc_ptr[r - rb + 1]++;
    }
  for (int64_t r = 0; r < nr; ++r) inc_ptr[r + 1] += inc_ptr[r];
  int64_t* inc = malloc(sizeof(int64_t) * (size_t)(inc_ptr[nr] + 1));
  int64_t* fill = malloc(sizeof(int64_t) * (size_t)(nr + 1));
  memcpy(fill, inc_ptr, sizeof(int64_t) * (size_t)nr);
  for (int64_t e = 0; e < ne; ++e)
    for (int a = 0; a < k; ++a) {
      int64_t r = dconn[e * k + a];
      if (r >= rb && r < re) inc[fill[r - rb]++] = e;
    }
  free(fill);
  int64_t maxdeg = 0;
  for (int64_t r = 0; r < nr; ++r)
    if (inc_ptr[r + 1] - inc_ptr[r] > maxdeg) maxdeg = inc_ptr[r + 1] - inc_ptr[r];
  fo_pattern* p = calloc(1, sizeof(fo_pattern));
  p->rb = rb;
  p->re = re;
  p->row_ptr = calloc((size_t)nr + 1, sizeof(int64_t));
  const size_t cap = (size_t)(maxdeg * k + 1);
#pragma omp parallel
  {
    int32_t* buf = malloc(sizeof(int32_t) * cap);
#pragma omp for schedule(dynamic, 1024)
    for (int64_t r = rb; r < re; ++r) p->row_ptr[r - rb + 1] = row_unique(inc_ptr, inc, dconn, k, r, rb, buf);
    free(buf);
  }
  for (int64_t r = 0; r < nr; ++r) p->row_ptr[r + 1] += p->row_ptr[r];
  p->col_idx = malloc(sizeof(int32_t) * (size_t)(p->row_ptr[nr] + 1));
#pragma omp parallel
  {
    int32_t* buf = malloc(sizeof(int32_t) * cap);
#pragma omp for schedule(dynamic, 1024)
    for (int64_t r = rb; r < re; ++r) {
      int64_t u = row_unique(inc_ptr, inc, dconn, k, r, rb, buf);
      memcpy(p->col_idx + p->row_ptr[r - rb], buf, sizeof(int32_t) * (size_t)u);
    }
    free(buf);
  }
  free(inc_ptr);
  free(inc);
  return p;
}

int64_t fo_pattern_nnz(const fo_pattern* p) { return p->row_ptr[p->re - p->rb]; }

void fo_pattern_copy(const fo_pattern* p, int64_t* row_ptr, int32_t* col_idx) {
  const int64_t nr = p->re - p->rb;
  memcpy(row_ptr, p->row_ptr, sizeof(int64_t) * (size_t)(nr + 1));
  memcpy(col_idx, p->col_idx, sizeof(int32_t) * (size_t)p->row_ptr[nr]);
}

void fo_pattern_free(fo_pattern* p) {
  if (!p) return;
  free(p->row_ptr);
  free(p->col_idx);
  free(p);
}

/* ------------------------------------------------------------------------ */
/* quadrature: fem.cpp:43-48 (2D), Appendix C (3D)                           */

#define A4 0.1381966011250105151795413165634361882280
#define B4 0.5854101966249684544613760503096914353161

static int tet_rule(int id, double* p, double* w) {
  int n = 0;
#define ADD(a, b, c, ww) do { if (p) { p[3*n]=(a); p[3*n+1]=(b); p[3*n+2]=(c); w[n]=(ww);} ++n; } while (0)
#define PERM4(a, ww) do { double t_ = 1.0 - 3.0*(a); ADD(a,a,a,ww); ADD(t_,a,a,ww); ADD(a,t_,a,ww); ADD(a,a,t_,ww);} while (0)
#define PERM6(a, ww) do { double t_ = 0.5 - (a); ADD(a,a,t_,ww); ADD(a,t_,a,ww); ADD(t_,a,a,ww); \
                          ADD(a,t_,t_,ww); ADD(t_,a,t_,ww); ADD(t_,t_,a,ww);} while (0)
  switch (id) {
    case 1: ADD(0.25, 0.25, 0.25, 1.0 / 6.0); break;
    case 4:
      ADD(A4, A4, A4, 1.0 / 24.0); ADD(B4, A4, A4, 1.0 / 24.0);
      ADD(A4, B4, A4, 1.0 / 24.0); ADD(A4, A4, B4, 1.0 / 24.0);
      break;
    case 11:
      ADD(0.25, 0.25, 0.25, -74.0 / 5625.0);
      PERM4(1.0 / 14.0, 343.0 / 45000.0);
      PERM6(0.1005964238332007950038978525383593769, 56.0 / 2250.0);
      break;
    case 14:
      PERM4(0.09273525031089122640232391373703060, 0.01224884051939365825728503424772125);
      PERM4(0.31088591926330060979734573376345783, 0.01878132095300264179986427538888106);
      PERM6(0.04550370412564964949188052627933944, 0.00709100346284691107301157135337624);
      break;
    default: return 0;
  }
#undef ADD
#undef PERM4
#undef PERM6
  return n;
}

int fo_quad_size(int dim, int quad_id) {
  if (dim == 2) return quad_id == 3 ? 3 : quad_id == 1 ? 1 : 0;
  return tet_rule(quad_id, NULL, NULL);
}

void fo_quad_rule(int dim, int quad_id, double* pts, double* w) {
  if (dim == 2) {
    if (quad_id == 3) { /* fem.cpp:45-46 */
      const double p[6] = {1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0};
      memcpy(pts, p, sizeof p);
      w[0] = w[1] = w[2] = 1.0 / 6.0;
    } else {
      pts[0] = pts[1] = 1.0 / 3.0;
      w[0] = 0.5;
    }
    return;
  }
  tet_rule(quad_id, pts, w);
}

/* ------------------------------------------------------------------------ */
/* basis (fem.cpp:68-71 generalised): values and reference gradients          */

static int n_local(int dim, int degree) {
  if (dim == 2) return degree == 1 ? 3 : 6;
  return degree == 1 ? 4 : 10;
}

static void basis(int dim, int degree, const double* xi, double* phi, double* dphi /* [n][dim] */) {
  double l[4], dl[4][3];
  const int nv = dim + 1;
  memset(dl, 0, sizeof dl);
  l[0] = 1.0;
  for (int c = 0; c < dim; ++c) {
    l[0] -= xi[c];
    l[c + 1] = xi[c];
    dl[0][c] = -1.0;
    dl[c + 1][c] = 1.0;
  }
  if (degree == 1) {
    for (int a = 0; a < nv; ++a) {
      phi[a] = l[a];
      for (int c = 0; c < dim; ++c) dphi[a * dim + c] = dl[a][c];
    }
    return;
  }
  for (int a = 0; a < nv; ++a) {
    phi[a] = l[a] * (2.0 * l[a] - 1.0);
    for (int c = 0; c < dim; ++c) dphi[a * dim + c] = (4.0 * l[a] - 1.0) * dl[a][c];
  }
  static const int e3[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  static const int e2[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  const int ne = dim == 3 ? 6 : 3;
  for (int q = 0; q < ne; ++q) {
    int a = dim == 3 ? e3[q][0] : e2[q][0], b = dim == 3 ? e3[q][1] : e2[q][1];
    phi[nv + q] = 4.0 * l[a] * l[b];
    for (int c = 0; c < dim; ++c) dphi[(nv + q) * dim + c] = 4.0 * (dl[a][c] * l[b] + l[a] * dl[b][c]);
  }
}

/* coefficient fields of the form family (fem.cpp:99-107 + convection) */
static void coefficients(int form, int dim, const double* x, double sigma[3][3], double* lam,
                         double beta[3], double* f) {
  memset(sigma, 0, sizeof(double) * 9);
  memset(beta, 0, sizeof(double) * 3);
  *lam = 0.0;
  double r2 = 0.0;
  for (int c = 0; c < dim; ++c) r2 += x[c] * x[c];
  const double fdemo = -2.0 * r2 + 36.0;
  switch (form) {
    case FO_POISSON:
      for (int c = 0; c < dim; ++c) sigma[c][c] = 1.0;
      *f = fdemo;
      break;
    case FO_DEMO2D:
      sigma[0][0] = 1.0; sigma[0][1] = -x[0] - x[1];
      sigma[1][0] = x[0] + x[1]; sigma[1][1] = 1.0;
      *lam = 1.0;
      *f = fdemo;
      break;
    case FO_STIFFNESS:
      for (int c = 0; c < dim; ++c) sigma[c][c] = 1.0;
      *f = 0.0;
      break;
    case FO_MASS:
      *lam = 1.0;
      *f = 1.0;
      break;
    case FO_HELMHOLTZ:
      for (int c = 0; c < dim; ++c) sigma[c][c] = 1.0;
      *lam = 1.0;
      *f = fdemo;
      break;
    case FO_VARCOEF: {
      double s = dim == 3 ? 1.0 + x[0] * x[1] * x[2] : 1.0 + x[0] * x[1];
      for (int c = 0; c < dim; ++c) sigma[c][c] = s;
      *lam = 1.0 + x[0] * x[0];
      beta[0] = 1.0;
      beta[1] = x[0];
      if (dim == 3) beta[2] = -x[1];
      *f = fdemo;
      break;
    }
    default:
      *f = 0.0;
  }
}

/* Element kernel: fem.cpp:122-158 semantics (grad = J^{-T} grad_ref written as
 * cofactor/det, times det J) evaluated per quadrature point, summed in
 * ascending q as in device.cpp:176-192. Returns 0, or -1 if degenerate
 * (device.cpp:128, 180-186). */
static int element_local(int form, int dim, int degree, int nq, const double* qp, const double* qw,
                         const double* xv /* [dim+1][dim] */, double* ke, double* fe) {
  const int n = n_local(dim, degree);
  double J[3][3] = {{0}}, C[3][3] = {{0}}, det;
  for (int r = 0; r < dim; ++r)
    for (int c = 0; c < dim; ++c) J[r][c] = xv[(c + 1) * dim + r] - xv[r];
  if (dim == 2) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    C[0][0] = J[1][1]; C[0][1] = -J[1][0];
    C[1][0] = -J[0][1]; C[1][1] = J[0][0];
  } else {
    det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
          J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
          J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        int r1 = (r + 1) % 3, r2 = (r + 2) % 3, c1 = (c + 1) % 3, c2 = (c + 2) % 3;
        C[r][c] = J[r1][c1] * J[r2][c2] - J[r1][c2] * J[r2][c1];
      }
  }
  if (fabs(det) <= 1e-14) return -1;
  for (int t = 0; t < n * n; ++t) ke[t] = 0.0;
  for (int t = 0; t < n; ++t) fe[t] = 0.0;
  double phi[10], dref[30], g[10][3];
  for (int q = 0; q < nq; ++q) {
    const double* xi = qp + q * dim;
    basis(dim, degree, xi, phi, dref);
    for (int a = 0; a < n; ++a)
      for (int r = 0; r < dim; ++r) {
        double s = 0.0;
        for (int c = 0; c < dim; ++c) s += C[r][c] * dref[a * dim + c];
        g[a][r] = s / det;
      }
    double x[3] = {0, 0, 0};
    for (int r = 0; r < dim; ++r) {
      x[r] = xv[r];
      for (int c = 0; c < dim; ++c) x[r] += J[r][c] * xi[c];
    }
    double sigma[3][3], lam, beta[3], f;
    coefficients(form, dim, x, sigma, &lam, beta, &f);
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int r = 0; r < dim; ++r) {
          double sg = 0.0;
          for (int c = 0; c < dim; ++c) sg += sigma[r][c] * g[j][c];
          s += g[i][r] * sg;
        }
        double conv = 0.0;
        for (int c = 0; c < dim; ++c) conv += beta[c] * g[j][c];
        s += lam * phi[i] * phi[j] + conv * phi[i];
        ke[i * n + j] += qw[q] * (s * det);
      }
      fe[i] += qw[q] * (f * phi[i] * det);
    }
  }
  return 0;
}

int fo_element_matrix(int form, int dim, int degree, int quad_id, const double* xv, double* ke,
                      double* fe) {
  double qp[3 * 16], qw[16];
  int nq = fo_quad_size(dim, quad_id);
  if (nq <= 0) return -3;
  fo_quad_rule(dim, quad_id, qp, qw);
  return element_local(form, dim, degree, nq, qp, qw, xv, ke, fe);
}

static int64_t find_slot(const int64_t* row_ptr, const int32_t* col_idx, int64_t rl, int32_t j) {
  /* device.cpp:274-288 binary search */
  int64_t lo = row_ptr[rl], hi = row_ptr[rl + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (col_idx[mid] < j) lo = mid + 1; else hi = mid;
  }
  if (lo >= row_ptr[rl + 1] || col_idx[lo] != j) return -1;
  return lo;
}

int fo_assemble(int form, int dim, int degree, int quad_id, const double* coords,
                const int32_t* vconn, const int32_t* dconn, int64_t ne, const int64_t* row_ptr,
                const int32_t* col_idx, int64_t rb, int64_t re, double* values, double* rhs,
                int workers, int64_t* bad) {
  double qp[3 * 16], qw[16];
  const int nq = fo_quad_size(dim, quad_id);
  if (nq <= 0) return -3;
  fo_quad_rule(dim, quad_id, qp, qw);
  const int n = n_local(dim, degree), nv = dim + 1;
  memset(values, 0, sizeof(double) * (size_t)row_ptr[re - rb]);
  memset(rhs, 0, sizeof(double) * (size_t)(re - rb));
  int64_t first_bad = -1, first_miss = -1;
  int nthreads = workers > 1 ? workers : 1;
#pragma omp parallel num_threads(nthreads) if (workers > 1)
  {
    double xv[12], ke[100], fe[10];
#pragma omp for schedule(dynamic, 64)
    for (int64_t e = 0; e < ne; ++e) {
      for (int a = 0; a < nv; ++a)
        for (int c = 0; c < dim; ++c) xv[a * dim + c] = coords[(int64_t)vconn[e * nv + a] * dim + c];
      if (element_local(form, dim, degree, nq, qp, qw, xv, ke, fe) != 0) {
#pragma omp critical(fo_bad)
        if (first_bad < 0 || e < first_bad) first_bad = e;
        continue;
      }
      const int32_t* d = dconn + e * n;
      for (int i = 0; i < n; ++i) {
        int64_t gi = d[i];
        if (gi < rb || gi >= re) continue;
        for (int j = 0; j < n; ++j) {
          int64_t s = find_slot(row_ptr, col_idx, gi - rb, d[j]);
          if (s < 0) {
#pragma omp critical(fo_miss)
            if (first_miss < 0) first_miss = gi;
            continue;
          }
          if (workers > 1) {
#pragma omp atomic
            values[s] += ke[i * n + j];
          } else {
            values[s] += ke[i * n + j];
          }
        }
        if (workers > 1) {
#pragma omp atomic
          rhs[gi - rb] += fe[i];
        } else {
          rhs[gi - rb] += fe[i];
        }
      }
    }
  }
  if (first_bad >= 0) { if (bad) *bad = first_bad; return -1; }
  if (first_miss >= 0) { if (bad) *bad = first_miss; return -2; }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* vector P1/P2 linear elasticity (BASELINE.json config 5; no reference      */
/* implementation -- parity rests on the rigid-body-mode and block KATs in   */
/* the tests). Per element and quadrature point (ascending q, the device.cpp */
/* 176-192 order) K[(a,c),(b,d)] += w det (lam d_d phi_b d_c phi_a           */
/*   + mu d_c phi_b d_d phi_a + mu [c==d] grad phi_b . grad phi_a),          */
/* F[(a,c)] += w det f_c phi_a; local DOF a*dim + c, global dim*node + c,    */
/* binary-search scatter into the block-expanded CSR (device.cpp:274-288).   */
int fo_assemble_elasticity(int dim, int degree, int quad_id, const double* coords, const int32_t* vconn,
                           const int32_t* dconn, int64_t ne, const int64_t* row_ptr, const int32_t* col_idx,
                           int64_t rb, int64_t re, double lam, double mu, const double* force, double* values,
                           double* rhs, int64_t* bad) {
  double qp[3 * 16], qw[16];
  const int nq = fo_quad_size(dim, quad_id);
  if (nq <= 0) return -3;
  fo_quad_rule(dim, quad_id, qp, qw);
  const int k = n_local(dim, degree), nv = dim + 1, n = k * dim;
  memset(values, 0, sizeof(double) * (size_t)row_ptr[re - rb]);
  memset(rhs, 0, sizeof(double) * (size_t)(re - rb));
  double* ke = malloc(sizeof(double) * (size_t)(n * n));
  double fe[30];
  for (int64_t e = 0; e < ne; ++e) {
    double xv[12], J[3][3] = {{0}}, C[3][3] = {{0}}, det;
    for (int a = 0; a < nv; ++a)
      for (int c = 0; c < dim; ++c) xv[a * dim + c] = coords[(int64_t)vconn[e * nv + a] * dim + c];
    for (int r = 0; r < dim; ++r)
      for (int c = 0; c < dim; ++c) J[r][c] = xv[(c + 1) * dim + r] - xv[r];
    if (dim == 2) {
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      C[0][0] = J[1][1]; C[0][1] = -J[1][0];
      C[1][0] = -J[0][1]; C[1][1] = J[0][0];
    } else {
      det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
            J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          int r1 = (r + 1) % 3, r2 = (r + 2) % 3, c1 = (c + 1) % 3, c2 = (c + 2) % 3;
          C[r][c] = J[r1][c1] * J[r2][c2] - J[r1][c2] * J[r2][c1];
        }
    }
    if (fabs(det) <= 1e-14) {
      if (bad) *bad = e;
      free(ke);
      return -1;
    }
    for (int t = 0; t < n * n; ++t) ke[t] = 0.0;
    for (int t = 0; t < n; ++t) fe[t] = 0.0;
    double phi[10], dref[30], g[10][3];
    for (int q = 0; q < nq; ++q) {
      basis(dim, degree, qp + q * dim, phi, dref);
      for (int a = 0; a < k; ++a)
        for (int r = 0; r < dim; ++r) {
          double s = 0.0;
          for (int c = 0; c < dim; ++c) s += C[r][c] * dref[a * dim + c];
          g[a][r] = s / det;
        }
      for (int a = 0; a < k; ++a)
        for (int c = 0; c < dim; ++c) {
          for (int b = 0; b < k; ++b)
            for (int d = 0; d < dim; ++d) {
              double gg = 0.0;
              for (int r = 0; r < dim; ++r) gg += g[b][r] * g[a][r];
              double s = lam * g[b][d] * g[a][c] + mu * g[b][c] * g[a][d] + (c == d ? mu * gg : 0.0);
              ke[(a * dim + c) * n + b * dim + d] += qw[q] * (s * det);
            }
          fe[a * dim + c] += qw[q] * (force[c] * phi[a] * det);
        }
    }
    const int32_t* dd = dconn + e * k;
    for (int a = 0; a < k; ++a)
      for (int c = 0; c < dim; ++c) {
        const int64_t gi = (int64_t)dim * dd[a] + c;
        if (gi < rb || gi >= re) continue;
        for (int b = 0; b < k; ++b)
          for (int d = 0; d < dim; ++d) {
            const int64_t s = find_slot(row_ptr, col_idx, gi - rb, dim * dd[b] + d);
            if (s < 0) {
              if (bad) *bad = gi;
              free(ke);
              return -2;
            }
            values[s] += ke[(a * dim + c) * n + b * dim + d];
          }
        rhs[gi - rb] += fe[a * dim + c];
      }
  }
  free(ke);
  return 0;
}

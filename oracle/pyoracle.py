"""oracle/pyoracle.py -- TEST INFRASTRUCTURE ONLY (the checker).

ctypes bindings for the C restatement (oracle/liboracle.so) and for the
reference harness (oracle/_ref/libffref.so, built from /root/reference by
oracle/Makefile). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

FORMS = {"poisson": 0, "demo2d": 1, "stiffness": 2, "mass": 3, "helmholtz": 4, "varcoef": 5}

_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(os.path.join(HERE, "liboracle.so"))
        L.fo_unit_square_mesh.argtypes = [C.c_int, _f64p, _i32p]
        L.fo_kuhn_mesh.argtypes = [C.c_int, _f64p, _i32p]
        L.fo_p2_dofs_kuhn.argtypes = [C.c_int, _i32p, C.c_int64, _i32p]
        L.fo_build_pattern.restype = C.c_void_p
        L.fo_build_pattern.argtypes = [_i32p, C.c_int64, C.c_int, C.c_int64, C.c_int64, C.c_int64]
        L.fo_pattern_nnz.restype = C.c_int64
        L.fo_pattern_nnz.argtypes = [C.c_void_p]
        L.fo_pattern_copy.argtypes = [C.c_void_p, _i64p, _i32p]
        L.fo_pattern_free.argtypes = [C.c_void_p]
        L.fo_quad_size.argtypes = [C.c_int, C.c_int]
        L.fo_quad_rule.argtypes = [C.c_int, C.c_int, _f64p, _f64p]
        L.fo_assemble.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _f64p, _i32p, _i32p, C.c_int64,
                                  _i64p, _i32p, C.c_int64, C.c_int64, _f64p, _f64p, C.c_int,
                                  C.POINTER(C.c_int64)]
        L.fo_assemble_elasticity.argtypes = [C.c_int, C.c_int, C.c_int, _f64p, _i32p, _i32p, C.c_int64, _i64p,
                                             _i32p, C.c_int64, C.c_int64, C.c_double, C.c_double, _f64p, _f64p,
                                             _f64p, C.POINTER(C.c_int64)]
        L.fo_element_matrix.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _f64p, _f64p, _f64p]
        _lib = L
    return _lib


def unit_square_mesh(n):
    nv, ne = (n + 1) ** 2, 2 * n * n
    xy = np.empty((nv, 2)); conn = np.empty((ne, 3), np.int32)
    lib().fo_unit_square_mesh(n, xy, conn)
    return xy, conn


def kuhn_mesh(n):
    nv, ne = (n + 1) ** 3, 6 * n ** 3
    xyz = np.empty((nv, 3)); conn = np.empty((ne, 4), np.int32)
    lib().fo_kuhn_mesh(n, xyz, conn)
    return xyz, conn


def p2_dofs_kuhn(n, vconn):
    d = np.empty((vconn.shape[0], 10), np.int32)
    lib().fo_p2_dofs_kuhn(n, np.ascontiguousarray(vconn), vconn.shape[0], d)
    return d, (2 * n + 1) ** 3


def build_pattern(dconn, n_dofs, row_begin=0, row_end=None):
    row_end = n_dofs if row_end is None else row_end
    d = np.ascontiguousarray(dconn, dtype=np.int32)
    p = lib().fo_build_pattern(d, d.shape[0], d.shape[1], n_dofs, row_begin, row_end)
    nnz = lib().fo_pattern_nnz(p)
    rp = np.empty(row_end - row_begin + 1, np.int64); ci = np.empty(nnz, np.int32)
    lib().fo_pattern_copy(p, rp, ci)
    lib().fo_pattern_free(p)
    return rp, ci


def quad_rule(dim, quad_id):
    n = lib().fo_quad_size(dim, quad_id)
    pts = np.empty((n, dim)); w = np.empty(n)
    lib().fo_quad_rule(dim, quad_id, pts, w)
    return pts, w


class OracleError(RuntimeError):
    pass


def assemble(form, dim, degree, quad_id, coords, vconn, dconn, row_ptr, col_idx,
             row_begin=0, row_end=None, workers=1):
    row_end = row_begin + len(row_ptr) - 1 if row_end is None else row_end
    vals = np.empty(int(row_ptr[-1])); rhs = np.empty(row_end - row_begin)
    bad = C.c_int64(-1)
    rc = lib().fo_assemble(FORMS.get(form, form), dim, degree, quad_id,
                           np.ascontiguousarray(coords, np.float64),
                           np.ascontiguousarray(vconn, np.int32), np.ascontiguousarray(dconn, np.int32),
                           vconn.shape[0], row_ptr, col_idx, row_begin, row_end, vals, rhs, workers,
                           C.byref(bad))
    if rc == -1:
        raise OracleError(f"degenerate element {bad.value} (|det J| <= 1e-14)")
    if rc == -2:
        raise OracleError(f"column not present in sparsity row {bad.value}")
    if rc != 0:
        raise OracleError(f"oracle error {rc}")
    return vals, rhs


def block_pattern(row_ptr, col_idx, bs):
    """bs x bs block expansion of a scalar CSR (vector space DOF bs*node + c)."""
    n = len(row_ptr) - 1
    lens = np.diff(row_ptr)
    rp = np.zeros(bs * n + 1, np.int64)
    rp[1:] = np.cumsum(np.repeat(lens * bs, bs))
    ci = np.empty(int(rp[-1]), np.int32)
    for r in range(n):
        cols = col_idx[row_ptr[r]:row_ptr[r + 1]].astype(np.int64)
        blk = (bs * cols[:, None] + np.arange(bs)[None, :]).ravel()
        for c in range(bs):
            ci[rp[bs * r + c]:rp[bs * r + c + 1]] = blk
    return rp, ci


def assemble_elasticity(dim, degree, quad_id, coords, vconn, dconn, row_ptr, col_idx, lam=1.0, mu=1.0,
                        force=(0.0, 0.0, -1.0), row_begin=0, row_end=None):
    """Vector P2 elasticity restatement (femoracle.c) into a block-expanded CSR."""
    row_end = row_begin + len(row_ptr) - 1 if row_end is None else row_end
    vals = np.empty(int(row_ptr[-1])); rhs = np.empty(row_end - row_begin)
    bad = C.c_int64(-1)
    f = np.ascontiguousarray(list(force) + [0.0] * (3 - len(force)), np.float64)
    rc = lib().fo_assemble_elasticity(dim, degree, quad_id, np.ascontiguousarray(coords, np.float64),
                                      np.ascontiguousarray(vconn, np.int32), np.ascontiguousarray(dconn, np.int32),
                                      vconn.shape[0], np.ascontiguousarray(row_ptr, np.int64),
                                      np.ascontiguousarray(col_idx, np.int32), row_begin, row_end, lam, mu, f, vals,
                                      rhs, C.byref(bad))
    if rc != 0:
        raise OracleError(f"oracle error {rc} at {bad.value}")
    return vals, rhs


def element_matrix(form, dim, degree, quad_id, xv):
    n = {(2, 1): 3, (2, 2): 6, (3, 1): 4, (3, 2): 10}[(dim, degree)]
    ke = np.empty(n * n); fe = np.empty(n)
    rc = lib().fo_element_matrix(FORMS.get(form, form), dim, degree, quad_id,
                                 np.ascontiguousarray(xv, np.float64), ke, fe)
    if rc != 0:
        raise OracleError("degenerate element" if rc == -1 else f"oracle error {rc}")
    return ke.reshape(n, n), fe


# --------------------------------------------------------------------------
# the reference itself (oracle/_ref/libffref.so)

def ref_available():
    return os.path.exists(os.path.join(HERE, "_ref", "libffref.so"))


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(os.path.join(HERE, "_ref", "libffref.so"))
        L.ffref_last_error.restype = C.c_char_p
        L.ffref_create.restype = C.c_void_p
        L.ffref_create.argtypes = [C.c_int, C.c_int, _f64p, C.c_int64, _i32p, _i32p, C.c_int64,
                                   C.c_int64, C.c_char_p, C.c_char_p, C.c_int]
        L.ffref_destroy.argtypes = [C.c_void_p]
        L.ffref_nnz.restype = C.c_int64
        L.ffref_nnz.argtypes = [C.c_void_p]
        L.ffref_pattern.argtypes = [C.c_void_p, _i64p, _i32p]
        L.ffref_assemble.argtypes = [C.c_void_p, C.c_int, C.c_int64, _f64p, _f64p]
        L.ffref_create3_on_pattern.restype = C.c_void_p
        L.ffref_create3_on_pattern.argtypes = [C.c_int, _f64p, C.c_int64, _i32p, _i32p, C.c_int64, C.c_int64,
                                               C.c_char_p, C.c_char_p, C.c_int, _i64p, _i32p]
        L.ffref_assemble_sample.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, _f64p, _f64p]
        L.ffref_emit_demo_source.argtypes = [C.c_char_p, C.c_int64]
        L.ffref_max_threads.restype = C.c_int
        L.ffref_build_info.restype = C.c_char_p
        L.ffref_export.argtypes = [C.c_void_p, _f64p, _f64p, C.c_char_p, C.c_char_p, C.c_int]
        L.ffref_cg.argtypes = [C.c_void_p, _f64p, _f64p, C.c_double, C.c_int, _f64p, C.POINTER(C.c_int),
                               C.POINTER(C.c_double)]
        _ref = L
    return _ref


# Weak-form text of the oracle's form family over the reference's reserved
# symbols (fem.cpp:36-41 / fem.hpp:50-55, extended with z, u_z, v_z).
def form_text(form, dim):
    g = ["x", "y", "z"][:dim]
    f = "(-2*(" + "+".join(c + "^2" for c in g) + ")+36)"
    grad = " + ".join(f"u_{c}*v_{c}" for c in g)
    if form == "poisson":
        return grad, f + "*v"
    if form == "stiffness":
        return grad, "0"
    if form == "mass":
        return "u*v", "v"
    if form == "helmholtz":
        return grad + " + u*v", f + "*v"
    if form == "demo2d":
        # helmholtz_form(sigma={1,-x-y,x+y,1}, 1, f) (test_device.cpp:38-42)
        return "v_x*(u_x + (-x-y)*u_y) + v_y*((x+y)*u_x + u_y) + u*v", f + "*v"
    if form == "varcoef":
        s = "(1+x*y*z)" if dim == 3 else "(1+x*y)"
        beta = "(u_x + x*u_y - y*u_z)" if dim == 3 else "(u_x + x*u_y)"
        return f"{s}*({grad}) + (1+x^2)*u*v + {beta}*v", f + "*v"
    raise ValueError(form)


class RefHarness:
    """The reference's own pipeline (2D P1) / CAS + IR VM (3D), see
    oracle/ref_harness.cpp."""

    def __init__(self, dim, degree, coords, vconn, dconn, n_dofs, form, quad_id=4, pattern=None):
        """pattern=(row_ptr, col_idx): 3D only -- search this prebuilt CSR
        (kept alive here) instead of building the std::set pattern."""
        bil, lin = form_text(form, dim) if isinstance(form, str) else form
        self.L = ref()
        self.coords = np.ascontiguousarray(coords, np.float64)
        self.vconn = np.ascontiguousarray(vconn, np.int32)
        self.dconn = np.ascontiguousarray(dconn, np.int32)
        self.n_dofs = n_dofs
        self.n_elems = vconn.shape[0]
        if pattern is not None:
            self._rp = np.ascontiguousarray(pattern[0], np.int64)
            self._ci = np.ascontiguousarray(pattern[1], np.int32)
            self.h = self.L.ffref_create3_on_pattern(degree, self.coords, coords.shape[0], self.vconn, self.dconn,
                                                     vconn.shape[0], n_dofs, bil.encode(), lin.encode(), quad_id,
                                                     self._rp, self._ci)
        else:
            self.h = self.L.ffref_create(dim, degree, self.coords, coords.shape[0], self.vconn, self.dconn,
                                         vconn.shape[0], n_dofs, bil.encode(), lin.encode(), quad_id)
        if not self.h:
            raise OracleError(self.L.ffref_last_error().decode())
        self.nnz = self.L.ffref_nnz(self.h)

    def pattern(self):
        rp = np.empty(self.n_dofs + 1, np.int64); ci = np.empty(self.nnz, np.int32)
        self.L.ffref_pattern(self.h, rp, ci)
        return rp, ci

    def assemble(self, workers=1, elem_limit=0):
        vals = np.empty(self.nnz); rhs = np.empty(self.n_dofs)
        if self.L.ffref_assemble(self.h, workers, elem_limit, vals, rhs) != 0:
            raise OracleError(self.L.ffref_last_error().decode())
        return vals, rhs


    def assemble_sample(self, values, rhs, workers, first, stride, count):
        """Accumulate elements first, first+stride, ... (count) into values/rhs
        (no zero fill): a bounded timing sample of the full-mesh 3D loop."""
        if self.L.ffref_assemble_sample(self.h, workers, first, stride, count, values, rhs) != 0:
            raise OracleError(self.L.ffref_last_error().decode())

    def export(self, values, rhs, mpath, vpath, fmt=0):
        """The reference's export_matrix / export_vector of this 2D system."""
        if ref().ffref_export(self.h, np.ascontiguousarray(values, np.float64), np.ascontiguousarray(rhs, np.float64),
                              str(mpath).encode(), str(vpath).encode(), fmt) != 0:
            raise OracleError(ref().ffref_last_error().decode())

    def cg(self, values, rhs, tol=1e-10, max_iter=10000):
        """The reference's cg_solve on this 2D system: (x, iterations, residual, converged)."""
        x = np.empty(len(rhs))
        it, res = C.c_int(0), C.c_double(0.0)
        rc = ref().ffref_cg(self.h, np.ascontiguousarray(values, np.float64), np.ascontiguousarray(rhs, np.float64),
                            tol, max_iter, x, C.byref(it), C.byref(res))
        if rc < 0:
            raise OracleError(ref().ffref_last_error().decode())
        return x, it.value, res.value, rc == 0
    def __del__(self):
        if getattr(self, "h", None):
            self.L.ffref_destroy(self.h)
            self.h = None

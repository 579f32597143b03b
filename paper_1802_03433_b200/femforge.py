"""Python bindings of the femforge-b200 C ABI (include/femforge_b200.h).

A thin ctypes layer: every call goes to ``libfemforge_b200.so`` (the in-tree
CUDA/NVRTC engine). There is no CPU fallback -- if the library or a GPU is
missing the calls raise.

Names follow the reference's device/fem API (/root/reference/proj/include/
femforge/device/device.hpp): ``build_sparsity``, ``assemble_sparse``,
``flatten_mesh`` map onto Pattern, assemble and Mesh.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfemforge_b200.so")

FF_OK, FF_E_ARG, FF_E_DEGENERATE, FF_E_PATTERN, FF_E_NVRTC, FF_E_CUDA, FF_E_FORM, FF_E_MESH, FF_E_SYMBOLIC, FF_E_NOMEM = \
    0, -1, -2, -3, -4, -5, -6, -7, -8, -9
STRATEGY = {"auto": 0, "tensor": 1, "pointwise": 2}
SCATTER_MODE = {"atomic": 1, "gather": 2, "auto": 3}
SCATTER_NAME = {v: k for k, v in SCATTER_MODE.items()}


class FFError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class DeviceError(FFError):
    """device::DeviceError (device.hpp:15-17): degenerate element, pattern mismatch, launch limits."""


class FormError(FFError):
    pass


class MeshError(FFError):
    pass


class SymbolicError(FFError):
    pass


class CompileError(FFError):
    pass


_ERRTYPE = {FF_E_DEGENERATE: DeviceError, FF_E_PATTERN: DeviceError, FF_E_ARG: DeviceError, FF_E_CUDA: DeviceError,
            FF_E_NOMEM: DeviceError, FF_E_FORM: FormError, FF_E_MESH: MeshError, FF_E_SYMBOLIC: SymbolicError,
            FF_E_NVRTC: CompileError}


class _FormDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("degree", C.c_int), ("quad_rule", C.c_int), ("strategy", C.c_int),
                ("block_size", C.c_int), ("bilinear", C.c_char_p), ("linear", C.c_char_p)]


class FormInfo(C.Structure):
    _fields_ = [("dim", C.c_int), ("degree", C.c_int), ("n_local", C.c_int), ("n_quad", C.c_int),
                ("strategy", C.c_int), ("n_invariants", C.c_int), ("n_unique_entries", C.c_int),
                ("flops_per_element", C.c_int64), ("registers", C.c_int), ("shared_bytes", C.c_int),
                ("compile_ms", C.c_double), ("n_kinv", C.c_int), ("row_flops", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class GatherInfo(C.Structure):
    _fields_ = [("n_items", C.c_int64), ("n_steps", C.c_int64), ("n_incidences", C.c_int64),
                ("record_bytes", C.c_int), ("build_ms", C.c_double), ("n_classes", C.c_int),
                ("n_class_rows", C.c_int64), ("n_class_items", C.c_int64),
                ("launches", C.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class CgResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("residual", C.c_double), ("converged", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("bad_element", C.c_int64), ("bad_row", C.c_int64), ("ms", C.c_double)]


class ScatterTiming(C.Structure):
    _fields_ = [("gather_ms", C.c_double), ("atomic_ms", C.c_double), ("chosen", C.c_int)]


_P = C.c_void_p
_i64 = C.c_int64
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

# (name, restype, argtypes) of every exported entry point of femforge_b200.h
SIGNATURES = [
    ("ff_version", C.c_char_p, []),
    ("ff_last_error", C.c_char_p, []),
    ("ff_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("ff_init", C.c_int, [C.c_int, C.POINTER(_P)]),
    ("ff_ctx_destroy", C.c_int, [_P]),
    ("ff_ctx_synchronize", C.c_int, [_P]),
    ("ff_ctx_stream", _P, [_P]),
    ("ff_ctx_set_scatter", C.c_int, [_P, C.c_int]),
    ("ff_ctx_set_gather_classes", C.c_int, [_P, _i64]),
    ("ff_class_source", C.c_int, [_P, C.c_int, _P, _P, _P, _P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("ff_expr_eval", C.c_int, [C.c_char_p, C.c_int, _P, _i64, _P]),
    ("ff_form_entry_text", C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("ff_form_create", C.c_int, [_P, C.POINTER(_FormDesc), C.POINTER(_P)]),
    ("ff_compile", C.c_int, [_P, C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_P), C.c_char_p, C.c_size_t]),
    ("ff_form_create_blocked", C.c_int, [_P, C.POINTER(_FormDesc), C.c_int, C.POINTER(C.c_char_p),
                                         C.POINTER(C.c_char_p), C.POINTER(_P)]),
    ("ff_mesh_set_components", C.c_int, [_P, C.c_int]),
    ("ff_form_source", C.c_int, [_P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("ff_form_cubin", C.c_int, [_P, _P, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("ff_form_info_get", C.c_int, [_P, C.POINTER(FormInfo)]),
    ("ff_form_destroy", C.c_int, [_P]),
    ("ff_mesh_create", C.c_int, [_P, C.c_int, _P, _i64, _P, _i64, _P, C.c_int32, _i64, C.POINTER(_P)]),
    ("ff_mesh_update", C.c_int, [_P, _P, _P, _P]),
    ("ff_mesh_destroy", C.c_int, [_P]),
    ("ff_pattern_build", C.c_int, [_P, _P, _i64, _i64, C.POINTER(_P)]),
    ("ff_pattern_info", C.c_int, [_P, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(C.c_int32)]),
    ("ff_pattern_export", C.c_int, [_P, _P, _P]),
    ("ff_pattern_export_ell", C.c_int, [_P, C.c_int32, _P, _P]),
    ("ff_pattern_device", C.c_int, [_P, C.POINTER(_P), C.POINTER(_P)]),
    ("ff_pattern_destroy", C.c_int, [_P]),
    ("ff_pattern_prepare", C.c_int, [_P, _P]),
    ("ff_pattern_gather_info", C.c_int, [_P, _P, C.POINTER(GatherInfo)]),
    ("ff_scatter_selected", C.c_int, [_P, _P, C.c_uint, C.POINTER(C.c_int)]),
    ("ff_scatter_calibrate", C.c_int, [_P, _P, _P, _P, _P, _P, C.POINTER(ScatterTiming)]),
    ("ff_assemble_device", C.c_int, [_P, _P, _P, _P, _P, _P]),
    ("ff_assemble_device_ex", C.c_int, [_P, _P, _P, _P, _P, _P, C.c_uint]),
    ("ff_check", C.c_int, [_P, C.POINTER(Stats)]),
    ("ff_assemble", C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, C.POINTER(Stats)]),
    ("ff_spmv", C.c_int, [_P, _P, _P, _P, _P]),
    ("ff_cg_solve", C.c_int, [_P, _P, _P, _P, C.c_double, C.c_int, C.POINTER(CgResult)]),
    ("ff_export_matrix", C.c_int, [_P, _f64p, C.c_char_p, C.c_int]),
    ("ff_export_vector", C.c_int, [_f64p, _i64, C.c_char_p, C.c_int]),
    ("ff_export_csr", C.c_int, [_i64, _i64p, _i32p, _f64p, C.c_char_p, C.c_int]),
    ("ff_unit_square_mesh", C.c_int, [C.c_int, _f64p, _i32p]),
    ("ff_kuhn_mesh", C.c_int, [C.c_int, _f64p, _i32p]),
    ("ff_kuhn_p2_dofs", C.c_int, [C.c_int, _i32p, _i64, _i32p]),
    ("ff_p2_dofs", C.c_int, [C.c_int, _i32p, _i64, _i64, _i32p, C.POINTER(_i64)]),
    ("ff_partition_rows", C.c_int, [_i64, C.c_int, C.c_int, C.POINTER(_i64), C.POINTER(_i64)]),
    ("ff_select_elements", C.c_int, [_i32p, _i64, C.c_int32, _i64, _i64, _P, C.POINTER(_i64)]),
]

_lib = None


def lib():
    """Loads the engine. Raises (never falls back) when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"femforge-b200 engine not built: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ok(rc):
    if rc != FF_OK:
        msg = lib().ff_last_error().decode(errors="replace")
        raise _ERRTYPE.get(rc, FFError)(rc, msg)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def device_count():
    n = C.c_int(0)
    _ok(lib().ff_device_count(C.byref(n)))
    return n.value


class Context:
    def __init__(self, device=0):
        h = _P()
        _ok(lib().ff_init(device, C.byref(h)))
        self.h = h
        self.device = device

    @property
    def stream(self):
        return lib().ff_ctx_stream(self.h)

    def synchronize(self):
        _ok(lib().ff_ctx_synchronize(self.h))

    def set_scatter(self, mode):
        """'gather' (row gather, atomic-free, default), 'atomic' (fp64 RED
        after a zero-fill) or 'auto' (the first device assembly of a (form,
        pattern, mesh) times both and keeps the faster)."""
        _ok(lib().ff_ctx_set_scatter(self.h, SCATTER_MODE[mode]))
        self.scatter = mode

    def set_gather_classes(self, min_rows):
        """Row classes with >= min_rows rows get a specialised gather kernel; 0: off."""
        _ok(lib().ff_ctx_set_gather_classes(self.h, int(min_rows)))

    def check(self):
        st = Stats()
        _ok(lib().ff_check(self.h, C.byref(st)))
        return st

    def close(self):
        if getattr(self, "h", None):
            lib().ff_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


class Form:
    """Weak form -> symbolic instantiation -> CUDA source -> NVRTC (sm_100a).

    ctx=None compiles without a device (source/cubin/info only)."""

    def __init__(self, ctx, dim, degree, bilinear, linear, quad_rule=0, strategy="auto", block_size=0):
        d = _FormDesc(dim, degree, quad_rule, STRATEGY.get(strategy, strategy), block_size,
                      bilinear.encode(), linear.encode())
        h = _P()
        _ok(lib().ff_form_create(ctx.h if ctx else None, C.byref(d), C.byref(h)))
        self.h, self.ctx, self.dim, self.degree = h, ctx, dim, degree

    @classmethod
    def blocked(cls, ctx, dim, degree, ncomp, block_bilinear, block_linear, quad_rule=0, strategy="auto",
                block_size=128):
        """Vector-valued form: block_bilinear[c*ncomp+d] (test c, trial d) and
        block_linear[c] scalar integrands (ff_form_create_blocked)."""
        self = cls.__new__(cls)
        d = _FormDesc(dim, degree, quad_rule, STRATEGY.get(strategy, strategy), block_size, b"0", b"0")
        bb = (C.c_char_p * len(block_bilinear))(*[t.encode() for t in block_bilinear])
        bl = (C.c_char_p * len(block_linear))(*[t.encode() for t in block_linear])
        h = _P()
        _ok(lib().ff_form_create_blocked(ctx.h if ctx else None, C.byref(d), ncomp, bb, bl, C.byref(h)))
        self.h, self.ctx, self.dim, self.degree, self.ncomp = h, ctx, dim, degree, ncomp
        return self

    @classmethod
    def from_source(cls, ctx, source, dim, degree, block_size=256):
        self = cls.__new__(cls)
        h = _P()
        log = C.create_string_buffer(1 << 16)
        _ok(lib().ff_compile(ctx.h if ctx else None, source.encode(), dim, degree, block_size, C.byref(h), log, len(log)))
        self.h, self.ctx, self.dim, self.degree = h, ctx, dim, degree
        self.log = log.value.decode()
        return self

    @property
    def source(self):
        n = C.c_size_t(0)
        _ok(lib().ff_form_source(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _ok(lib().ff_form_source(self.h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    @property
    def cubin(self):
        n = C.c_size_t(0)
        _ok(lib().ff_form_cubin(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _ok(lib().ff_form_cubin(self.h, C.cast(buf, C.c_void_p), n.value, C.byref(n)))
        return buf.raw

    @property
    def info(self):
        i = FormInfo()
        _ok(lib().ff_form_info_get(self.h, C.byref(i)))
        return i.as_dict()

    def class_source(self, classes):
        """Specialised gather source for classes [(len, [local i], [[slot bytes]])]."""
        n = len(classes)
        ln = np.array([c[0] for c in classes], np.int32)
        st = np.array([len(c[1]) for c in classes], np.int32)
        lo = np.ascontiguousarray(np.concatenate([np.asarray(c[1], np.int32) for c in classes]) if n else np.zeros(1, np.int32))
        sl = np.ascontiguousarray(np.concatenate([np.asarray(c[2], np.uint8).ravel() for c in classes]) if n else np.zeros(1, np.uint8))
        m = C.c_size_t(0)
        fn = lib().ff_class_source
        _ok(fn(self.h, n, _ptr(ln), _ptr(st), _ptr(lo), _ptr(sl), None, 0, C.byref(m)))
        buf = C.create_string_buffer(m.value + 1)
        _ok(fn(self.h, n, _ptr(ln), _ptr(st), _ptr(lo), _ptr(sl), buf, m.value + 1, C.byref(m)))
        return buf.value.decode()

    def entry_text(self, kind, i, j=0):
        """Instantiated integrand of bilinear entry (i, j) (kind "bilinear") or
        linear entry i (kind "linear") as text (ff_form_entry_text)."""
        k = 0 if kind == "bilinear" else 1
        m = C.c_size_t(0)
        _ok(lib().ff_form_entry_text(self.h, k, i, j, None, 0, C.byref(m)))
        buf = C.create_string_buffer(m.value + 1)
        _ok(lib().ff_form_entry_text(self.h, k, i, j, buf, m.value + 1, C.byref(m)))
        return buf.value.decode()

    def close(self):
        if getattr(self, "h", None):
            lib().ff_form_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


class Mesh:
    """Device copy of coordinates [nv][dim], vertex connectivity [ne][dim+1]
    and DOF connectivity [ne][k] (None for P1)."""

    def __init__(self, ctx, dim, coords, vconn, dconn=None, n_dofs=None, ncomp=1):
        self.coords = np.ascontiguousarray(coords, np.float64)
        self.vconn = np.ascontiguousarray(vconn, np.int32)
        self.dconn = None if dconn is None else np.ascontiguousarray(dconn, np.int32)
        self.k = dim + 1 if dconn is None else self.dconn.shape[1]
        self.n_dofs = self.coords.shape[0] if n_dofs is None else int(n_dofs)
        self.n_elems = self.vconn.shape[0]
        self.dim = dim
        h = _P()
        _ok(lib().ff_mesh_create(ctx.h, dim, _ptr(self.coords), self.coords.shape[0], _ptr(self.vconn), self.n_elems,
                                 _ptr(self.dconn), self.k, self.n_dofs, C.byref(h)))
        self.h, self.ctx = h, ctx
        self.ncomp = ncomp
        if ncomp > 1:
            _ok(lib().ff_mesh_set_components(h, ncomp))

    def update(self, coords=None, vconn=None, dconn=None):
        coords, vconn, dconn = _mesh_arrays(self, coords, vconn, dconn)
        _ok(lib().ff_mesh_update(self.h, _ptr(coords), _ptr(vconn), _ptr(dconn)))

    def close(self):
        if getattr(self, "h", None):
            lib().ff_mesh_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


class Pattern:
    """K1: CSR sparsity of rows [row_begin, row_end) (build_sparsity, device.cpp:66-88)."""

    def __init__(self, ctx, mesh, row_begin=0, row_end=None):
        row_end = mesh.n_dofs * getattr(mesh, "ncomp", 1) if row_end is None else row_end
        h = _P()
        _ok(lib().ff_pattern_build(ctx.h, mesh.h, row_begin, row_end, C.byref(h)))
        self.h, self.ctx, self.row_begin, self.row_end = h, ctx, row_begin, row_end
        n, nnz, mx = _i64(), _i64(), C.c_int32()
        _ok(lib().ff_pattern_info(h, C.byref(n), C.byref(nnz), C.byref(mx)))
        self.n_rows, self.nnz, self.max_row_len = n.value, nnz.value, mx.value

    def export(self):
        rp = np.empty(self.n_rows + 1, np.int64)
        ci = np.empty(max(self.nnz, 1), np.int32)
        _ok(lib().ff_pattern_export(self.h, _ptr(rp), _ptr(ci)))
        return rp, ci[: self.nnz]

    def export_ell(self, max_nz=None):
        max_nz = self.max_row_len if max_nz is None else max_nz
        rl = np.empty(self.n_rows, np.int32)
        rc = np.empty(self.n_rows * max_nz, np.int32)
        _ok(lib().ff_pattern_export_ell(self.h, max_nz, _ptr(rl), _ptr(rc)))
        return rl, rc.reshape(self.n_rows, max_nz)

    def device_pointers(self):
        rp, ci = _P(), _P()
        _ok(lib().ff_pattern_device(self.h, C.byref(rp), C.byref(ci)))
        return rp.value, ci.value

    def prepare(self, mesh):
        _ok(lib().ff_pattern_prepare(self.h, mesh.h))

    def gather_info(self, mesh):
        """Builds (if needed) and describes the row-gather plan of (pattern, mesh)."""
        gi = GatherInfo()
        _ok(lib().ff_pattern_gather_info(self.h, mesh.h, C.byref(gi)))
        return gi.as_dict()

    def scatter_for(self, form, flags=0):
        """Name of the scatter the next assembly with `form` runs."""
        m = C.c_int(0)
        _ok(lib().ff_scatter_selected(form.h, self.h, flags, C.byref(m)))
        return SCATTER_NAME[m.value]

    def calibrate_scatter(self, form, mesh, values_ptr, rhs_ptr, stream=None):
        """Times the row gather and the atomic scatter on device buffers and
        records the faster for 'auto': {gather_ms, atomic_ms, chosen}."""
        t = ScatterTiming()
        _ok(lib().ff_scatter_calibrate(form.h, mesh.h, self.h, C.c_void_p(values_ptr), C.c_void_p(rhs_ptr),
                                       _stream(stream), C.byref(t)))
        return {"gather_ms": t.gather_ms if t.gather_ms >= 0 else None, "atomic_ms": t.atomic_ms,
                "chosen": SCATTER_NAME[t.chosen]}

    def close(self):
        if getattr(self, "h", None):
            lib().ff_pattern_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def _stream(s):
    """None -> the context stream; 0 (torch's default stream) -> cudaStreamLegacy."""
    return None if s is None else C.c_void_p(1 if s == 0 else s)


def assemble_device(form, mesh, pattern, values_ptr, rhs_ptr, stream=None):
    """K0 + K2 on device buffers, asynchronous on `stream` (a cudaStream_t int)."""
    _ok(lib().ff_assemble_device(form.h, mesh.h, pattern.h, C.c_void_p(values_ptr), C.c_void_p(rhs_ptr),
                                 _stream(stream)))


FF_SKIP_ZERO, FF_ZERO_ONLY, FF_SCATTER_ATOMIC, FF_SCATTER_GATHER = 1, 2, 4, 16
FF_GATHER_INVARIANTS_ONLY, FF_GATHER_ROWS_ONLY = 32, 64


def assemble_device_ex(form, mesh, pattern, values_ptr, rhs_ptr, stream=None, flags=0):
    _ok(lib().ff_assemble_device_ex(form.h, mesh.h, pattern.h, C.c_void_p(values_ptr), C.c_void_p(rhs_ptr),
                                    _stream(stream), flags))


def _mesh_arrays(mesh, coords, vconn, dconn):
    """Caller mesh arrays as the C ABI reads them: C-contiguous float64 /
    int32 of exactly the mesh's sizes (the library copies nv*dim, ne*(dim+1)
    and ne*k values from the raw pointers)."""
    def conv(a, dtype, n, what):
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype)
        if a.size != n:
            raise ValueError(f"{what}: {a.size} values, the mesh needs {n}")
        return a
    coords = conv(coords, np.float64, mesh.coords.shape[0] * mesh.dim, "coords")
    vconn = conv(vconn, np.int32, mesh.n_elems * (mesh.dim + 1), "vconn")
    if dconn is not None and mesh.dconn is None:
        raise ValueError("dconn given for a mesh whose DOFs are its vertices")
    dconn = conv(dconn, np.int32, mesh.n_elems * mesh.k, "dconn")
    return coords, vconn, dconn


def _out_array(a, n, what):
    if a is None:
        return np.empty(n)
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.size == n
            and a.flags.writeable):
        raise ValueError(f"{what}: needs a writable C-contiguous float64 array of {n} values")
    return a


def assemble(form, mesh, pattern, coords=None, vconn=None, dconn=None, values=None, rhs=None):
    """End-to-end with host buffers (assemble_sparse's call shape): uploads the
    given mesh arrays, assembles, returns host (values, rhs)."""
    coords, vconn, dconn = _mesh_arrays(mesh, coords, vconn, dconn)
    values = _out_array(values, pattern.nnz, "values")
    rhs = _out_array(rhs, pattern.n_rows, "rhs")
    st = Stats()
    _ok(lib().ff_assemble(form.h, mesh.h, pattern.h, _ptr(coords), _ptr(vconn), _ptr(dconn), _ptr(values), _ptr(rhs),
                          C.byref(st)))
    return values, rhs


# ---- downstream consumer ---------------------------------

EXPORT_FORMAT = {"matrix_market": 0, "csv": 1}


def spmv(pattern, values_ptr, x_ptr, y_ptr, stream=None):
    """y = A x on the device (linalg::matvec, linalg.cpp:35-49)."""
    _ok(lib().ff_spmv(pattern.h, C.c_void_p(values_ptr), C.c_void_p(x_ptr), C.c_void_p(y_ptr), _stream(stream)))


def cg_solve(pattern, values_ptr, b_ptr, x_ptr, tol=1e-10, max_iter=10000):
    """The reference's unpreconditioned CG (linalg.cpp:61-96) on the device.
    Returns {iterations, residual, converged}; x is written in place."""
    r = CgResult()
    _ok(lib().ff_cg_solve(pattern.h, C.c_void_p(values_ptr), C.c_void_p(b_ptr), C.c_void_p(x_ptr), tol, max_iter,
                          C.byref(r)))
    return {"iterations": r.iterations, "residual": r.residual, "converged": bool(r.converged)}


def export_matrix(pattern, values, path, fmt="matrix_market"):
    _ok(lib().ff_export_matrix(pattern.h, np.ascontiguousarray(values, np.float64), str(path).encode(),
                               EXPORT_FORMAT[fmt]))


def export_vector(b, path, fmt="matrix_market"):
    b = np.ascontiguousarray(b, np.float64)
    _ok(lib().ff_export_vector(b, b.size, str(path).encode(), EXPORT_FORMAT[fmt]))


def export_csr(row_ptr, col_idx, values, path, fmt="matrix_market"):
    _ok(lib().ff_export_csr(len(row_ptr) - 1, np.ascontiguousarray(row_ptr, np.int64),
                            np.ascontiguousarray(col_idx, np.int32), np.ascontiguousarray(values, np.float64),
                            str(path).encode(), EXPORT_FORMAT[fmt]))


# ---- host helpers -----------------------------------------------------------

def unit_square_mesh(n):
    xy = np.empty(((n + 1) ** 2, 2)); conn = np.empty((2 * n * n, 3), np.int32)
    _ok(lib().ff_unit_square_mesh(n, xy, conn))
    return xy, conn


def kuhn_mesh(n):
    xyz = np.empty(((n + 1) ** 3, 3)); conn = np.empty((6 * n ** 3, 4), np.int32)
    _ok(lib().ff_kuhn_mesh(n, xyz, conn))
    return xyz, conn


def kuhn_p2_dofs(n, vconn):
    d = np.empty((vconn.shape[0], 10), np.int32)
    _ok(lib().ff_kuhn_p2_dofs(n, np.ascontiguousarray(vconn, np.int32), vconn.shape[0], d))
    return d, (2 * n + 1) ** 3


def p2_dofs(dim, vconn, n_vertices):
    k = 6 if dim == 2 else 10
    d = np.empty((vconn.shape[0], k), np.int32)
    nd = _i64()
    _ok(lib().ff_p2_dofs(dim, np.ascontiguousarray(vconn, np.int32), vconn.shape[0], n_vertices, d, C.byref(nd)))
    return d, nd.value


def partition_rows(n_dofs, n_parts, part):
    rb, re = _i64(), _i64()
    _ok(lib().ff_partition_rows(n_dofs, n_parts, part, C.byref(rb), C.byref(re)))
    return rb.value, re.value


def select_elements(dconn, row_begin, row_end):
    d = np.ascontiguousarray(dconn, np.int32)
    cnt = _i64()
    _ok(lib().ff_select_elements(d, d.shape[0], d.shape[1], row_begin, row_end, None, C.byref(cnt)))
    ids = np.empty(cnt.value, np.int64)
    _ok(lib().ff_select_elements(d, d.shape[0], d.shape[1], row_begin, row_end, _ptr(ids), C.byref(cnt)))
    return ids


# ---- weak-form text (the reference's helmholtz_form, fem.cpp:99-107) ---------

def expr_eval(expr, dim, pts=None):
    """Evaluates a coefficient / exact-solution expression over (x, y[, z]) at
    points [n][dim] (ff_expr_eval); pts None only validates it (raises
    SymbolicError on a parse error or a foreign symbol)."""
    if pts is None:
        _ok(lib().ff_expr_eval(expr.encode(), dim, None, 0, None))
        return None
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, dim)
    out = np.empty(pts.shape[0])
    _ok(lib().ff_expr_eval(expr.encode(), dim, _ptr(pts), pts.shape[0], _ptr(out)))
    return out


def helmholtz_text(dim, sigma=None, lam="0", f="0", beta=None):
    """bilinear = grad v . sigma grad u + lam u v [+ (beta . grad u) v]; linear = f v."""
    c = ["x", "y", "z"][:dim]
    if sigma is None:
        sigma = [["1" if r == s else "0" for s in range(dim)] for r in range(dim)]
    terms = []
    for r in range(dim):
        inner = " + ".join(f"({sigma[r][s]})*u_{c[s]}" for s in range(dim))
        terms.append(f"v_{c[r]}*({inner})")
    bil = " + ".join(terms) + f" + ({lam})*v*u"
    if beta is not None:
        bil += " + (" + " + ".join(f"({beta[s]})*u_{c[s]}" for s in range(dim)) + ")*v"
    return bil, f"({f})*v"


POISSON_F = {2: "-2*(x^2+y^2)+36", 3: "-2*(x^2+y^2+z^2)+36"}   # femforge.cpp:28


def named_form(name, dim):
    """The oracle's form family (oracle/femoracle.h) as weak-form text."""
    f = POISSON_F[dim]
    if name == "poisson":
        return helmholtz_text(dim, f=f)
    if name == "stiffness":
        return helmholtz_text(dim)
    if name == "mass":
        return helmholtz_text(dim, sigma=[["0"] * dim for _ in range(dim)], lam="1", f="1")
    if name == "helmholtz":
        return helmholtz_text(dim, lam="1", f=f)
    if name == "demo2d":
        return helmholtz_text(2, sigma=[["1", "-x-y"], ["x+y", "1"]], lam="1", f=f)
    if name == "varcoef":
        s = "1+x*y*z" if dim == 3 else "1+x*y"
        sig = [[s if r == q else "0" for q in range(dim)] for r in range(dim)]
        beta = ["1", "x", "-y"][:dim]
        return helmholtz_text(dim, sigma=sig, lam="1+x^2", f=f, beta=beta)
    raise ValueError(name)


def elasticity_text(dim, lam="1", mu="1", f=("0", "0", "-1")):
    """Isotropic linear elasticity as block integrands (BASELINE config 5):
    block (c, d) = lam u_d v_c + mu u_c v_d + mu [c == d] grad u . grad v over
    the scalar basis (u_x = d/dx of the trial basis function), l_c = f_c v."""
    ax = ["x", "y", "z"][:dim]
    blocks = []
    for c in range(dim):
        for d in range(dim):
            t = f"({lam})*u_{ax[d]}*v_{ax[c]} + ({mu})*u_{ax[c]}*v_{ax[d]}"
            if c == d:
                t += f" + ({mu})*(" + " + ".join(f"u_{a}*v_{a}" for a in ax) + ")"
            blocks.append(t)
    return blocks, [f"({f[c]})*v" for c in range(dim)]


"""Generates the committed golden fixtures from the REFERENCE itself.

Runs here (where /root/reference exists): oracle/_ref/libffref.so is the
unmodified reference library (built by `make -C oracle ref`) plus the harness
in oracle/ref_harness.cpp. Fixtures (tests/golden/*.npz):

  ref2d_<form>_n<n>.npz  2D P1 via the reference pipeline end to end
                         (helmholtz_form -> instantiate -> compile_form ->
                         build_sparsity -> assemble_sparse det mode), ELL->CSR
  ref3d_p<d>_<form>_n<n>_q<q>.npz  3D via the reference CAS + IR VM
                         (restated 3D instantiate / device loop)
  kat_tet.npz            SURVEY.md Appendix B exact element matrices (sympy)
  demo_kernel.cu.golden.sha256  hash of the reference's emit_source output

Usage: python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrs):
    np.savez_compressed(os.path.join(OUT, name), **arrs)
    print("wrote", name, {k: v.shape for k, v in arrs.items()})


def ref2d(form, n):
    xy, conn = po.unit_square_mesh(n)
    h = po.RefHarness(2, 1, xy, conn, conn, xy.shape[0], form)
    rp, ci = h.pattern()
    v, b = h.assemble()
    save(f"ref2d_{form}_n{n}.npz", row_ptr=rp, col_idx=ci, values=v, rhs=b)


def ref3d(degree, form, n, q):
    xyz, vc = po.kuhn_mesh(n)
    if degree == 1:
        dc, nd = vc, xyz.shape[0]
    else:
        dc, nd = po.p2_dofs_kuhn(n, vc)
    h = po.RefHarness(3, degree, xyz, vc, dc, nd, form, q)
    rp, ci = h.pattern()
    v, b = h.assemble()
    save(f"ref3d_p{degree}_{form}_n{n}_q{q}.npz", row_ptr=rp, col_idx=ci, values=v, rhs=b)


def kats():
    import sympy as sp
    xi, eta, zeta = sp.symbols("xi eta zeta")
    lam = [1 - xi - eta - zeta, xi, eta, zeta]
    p1 = lam
    p2 = [l * (2 * l - 1) for l in lam] + [4 * lam[a] * lam[b] for a, b in
                                           [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]]

    def integ(f):
        return sp.integrate(sp.integrate(sp.integrate(f, (zeta, 0, 1 - xi - eta)), (eta, 0, 1 - xi)), (xi, 0, 1))

    out = {}
    for name, basis in (("p1", p1), ("p2", p2)):
        g = [[sp.diff(f, v) for v in (xi, eta, zeta)] for f in basis]
        K = [[integ(sum(g[i][c] * g[j][c] for c in range(3))) for j in range(len(basis))] for i in range(len(basis))]
        M = [[integ(basis[i] * basis[j]) for j in range(len(basis))] for i in range(len(basis))]
        F = [integ(f) for f in basis]
        out[f"{name}_K"] = np.array([[float(v) for v in r] for r in K])
        out[f"{name}_M"] = np.array([[float(v) for v in r] for r in M])
        out[f"{name}_F"] = np.array([float(v) for v in F])
    save("kat_tet.npz", **out)


def demo_source_hash():
    buf = po.C.create_string_buffer(1 << 20)
    n = po.ref().ffref_emit_demo_source(buf, len(buf))
    src = buf.value[:n]
    with open(os.path.join(OUT, "demo_kernel.cu.golden.sha256"), "w") as f:
        f.write(hashlib.sha256(src).hexdigest() + "\n")
    print("reference emit_source sha256", hashlib.sha256(src).hexdigest())


if __name__ == "__main__":
    if not po.ref_available():
        sys.exit("oracle/_ref/libffref.so missing: run `make -C oracle ref` (needs /root/reference)")
    for form in ("demo2d", "poisson", "stiffness", "mass"):
        for n in (1, 4, 8):
            ref2d(form, n)
    ref2d("demo2d", 16)
    for deg in (1, 2):
        for form in ("poisson", "helmholtz"):
            ref3d(deg, form, 2, 4)
        ref3d(deg, "varcoef", 2, 14)
        ref3d(deg, "mass", 1, 14)
    ref3d(2, "poisson", 3, 4)
    kats()
    demo_source_hash()

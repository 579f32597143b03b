"""The oracle (oracle/femoracle.c) pinned against the reference's own outputs
and against exact known answers. CPU only."""
import glob
import os

import numpy as np
import pytest

import pyoracle as po
from conftest import GOLDEN, normwise


def _golden(pattern):
    return sorted(glob.glob(os.path.join(GOLDEN, pattern)))


@pytest.mark.parametrize("path", _golden("ref2d_*.npz"), ids=os.path.basename)
def test_oracle_matches_reference_2d(path):
    g = np.load(path)
    _, form, n = os.path.basename(path)[:-4].split("_")
    n = int(n[1:])
    xy, conn = po.unit_square_mesh(n)
    rp, ci = po.build_pattern(conn, xy.shape[0])
    assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(ci, g["col_idx"])
    v, b = po.assemble(form, 2, 1, 3, xy, conn, conn, rp, ci)
    assert normwise(v, g["values"]) <= 1e-14
    assert normwise(b, g["rhs"]) <= 1e-14


@pytest.mark.parametrize("path", _golden("ref3d_*.npz"), ids=os.path.basename)
def test_oracle_matches_reference_cas_3d(path):
    g = np.load(path)
    _, p, form, n, q = os.path.basename(path)[:-4].split("_")
    deg, n, q = int(p[1:]), int(n[1:]), int(q[1:])
    xyz, vc = po.kuhn_mesh(n)
    dc, nd = (vc, xyz.shape[0]) if deg == 1 else po.p2_dofs_kuhn(n, vc)
    rp, ci = po.build_pattern(dc, nd)
    assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(ci, g["col_idx"])
    v, b = po.assemble(form, 3, deg, q, xyz, vc, dc, rp, ci)
    assert normwise(v, g["values"]) <= 1e-13
    assert normwise(b, g["rhs"]) <= 1e-13


REF_TET = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float)


@pytest.mark.parametrize("deg", [1, 2])
def test_oracle_known_answers_appendix_b(deg):
    kat = np.load(os.path.join(GOLDEN, "kat_tet.npz"))
    p = f"p{deg}"
    K, _ = po.element_matrix("stiffness", 3, deg, 4, REF_TET)  # 4-point rule is exact for K
    assert np.max(np.abs(K - kat[p + "_K"])) <= 1e-14
    M, F = po.element_matrix("mass", 3, deg, 14, REF_TET)      # degree-5 rule exact for M
    assert np.max(np.abs(M - kat[p + "_M"])) <= 1e-15
    assert np.max(np.abs(F - kat[p + "_F"])) <= 1e-15
    assert np.max(np.abs(K.sum(axis=1))) <= 1e-14             # zero row sums


def test_oracle_unit_triangle_fixtures():
    # test_fem.cpp:157-179 / acceptance criterion 1
    tri = np.array([[0, 0], [1, 0], [0, 1]], dtype=float)
    K, F = po.element_matrix("stiffness", 2, 1, 3, tri)
    assert np.max(np.abs(K - np.array([[1, -.5, -.5], [-.5, .5, 0], [-.5, 0, .5]]))) <= 1e-14
    M, F = po.element_matrix("mass", 2, 1, 3, tri)
    assert np.max(np.abs(M - (np.ones((3, 3)) + np.eye(3)) / 24)) <= 1e-14
    assert np.max(np.abs(F - 1 / 6)) <= 1e-14


@pytest.mark.parametrize("dim,qid,deg", [(2, 3, 2), (3, 1, 1), (3, 4, 2), (3, 11, 4), (3, 14, 5)])
def test_quadrature_exactness(dim, qid, deg):
    from math import factorial
    pts, w = po.quad_rule(dim, qid)
    for a in range(deg + 1):
        for b in range(deg + 1 - a):
            for c in range(deg + 1 - a - b if dim == 3 else 1):
                exact = factorial(a) * factorial(b) * factorial(c) / factorial(a + b + c + dim)
                got = np.sum(w * pts[:, 0] ** a * pts[:, 1] ** b * (pts[:, 2] ** c if dim == 3 else 1))
                assert abs(got - exact) <= 1e-15


@pytest.mark.parametrize("n", [3, 5, 7])
def test_nnz_formulas_appendix_a(n):
    xy, conn = po.unit_square_mesh(n)
    assert po.build_pattern(conn, xy.shape[0])[0][-1] == 7 * n * n + 6 * n + 1
    xyz, vc = po.kuhn_mesh(n)
    assert po.build_pattern(vc, xyz.shape[0])[0][-1] == 15 * n ** 3 + 21 * n ** 2 + 9 * n + 1
    dc, nd = po.p2_dofs_kuhn(n, vc)
    assert po.build_pattern(dc, nd)[0][-1] == 230 * n ** 3 + 138 * n ** 2 + 24 * n + 1


def test_oracle_degenerate_and_mismatch():
    xy, conn = po.unit_square_mesh(2)
    rp, ci = po.build_pattern(conn, xy.shape[0])
    bad = xy.copy()
    bad[conn[5]] = 0.25  # collapse element 5 (and neighbours share nodes -> lowest reported)
    with pytest.raises(po.OracleError, match="degenerate element"):
        po.assemble("stiffness", 2, 1, 3, bad, conn, conn, rp, ci)
    other = conn.copy()
    other[0] = [0, 1, 5]  # pair (0,5) absent from the pattern (test_device.cpp:268-278)
    with pytest.raises(po.OracleError, match="not present"):
        po.assemble("stiffness", 2, 1, 3, xy, other, other, rp, ci)


@pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")
def test_oracle_vs_live_reference_2d_n32():
    xy, conn = po.unit_square_mesh(32)
    h = po.RefHarness(2, 1, xy, conn, conn, xy.shape[0], "demo2d")
    rp, ci = h.pattern()
    v, b = h.assemble()
    rp2, ci2 = po.build_pattern(conn, xy.shape[0])
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2)
    v2, b2 = po.assemble("demo2d", 2, 1, 3, xy, conn, conn, rp2, ci2)
    assert normwise(v2, v) <= 1e-14 and normwise(b2, b) <= 1e-14
    # the reference's parallel mode agrees with its deterministic mode (test_device.cpp:298-311)
    vp, bp = h.assemble(workers=4)
    assert normwise(vp, v) <= 1e-12


@pytest.mark.parametrize("n", [1, 2, 3])
def test_elasticity_oracle_rigid_body_modes(n):
    """Vector P2 elasticity (config 5) has no reference implementation; the
    restatement is pinned by physics: translations and rotations are in the
    kernel of K, K is symmetric, and sum(rhs_c) = integral of f_c."""
    import scipy.sparse as sp
    c, v = po.kuhn_mesh(n)
    d, nd = po.p2_dofs_kuhn(n, v)
    rp, ci = po.build_pattern(d, nd)
    vrp, vci = po.block_pattern(rp, ci, 3)
    vals, rhs = po.assemble_elasticity(3, 2, 4, c, v, d, vrp, vci, lam=2.0, mu=0.5, force=(0.0, 1.0, -1.0))
    K = sp.csr_matrix((vals, vci, vrp), shape=(3 * nd, 3 * nd))
    L = 2 * n + 1
    idx = np.arange(nd)
    X = np.stack([idx % L, (idx // L) % L, idx // (L * L)], 1) / (L - 1)
    scale = np.abs(vals).max()
    modes = []
    for t in range(3):
        u = np.zeros(3 * nd)
        u[t::3] = 1.0
        modes.append(u)
    for a, b in [(0, 1), (1, 2), (0, 2)]:
        u = np.zeros(3 * nd)
        u[a::3] = -X[:, b]
        u[b::3] = X[:, a]
        modes.append(u)
    for u in modes:
        assert np.abs(K @ u).max() <= 1e-12 * scale
    assert abs(K - K.T).max() <= 1e-14 * scale
    assert abs(rhs[1::3].sum() - 1.0) <= 1e-12 and abs(rhs[2::3].sum() + 1.0) <= 1e-12 and abs(rhs[0::3].sum()) <= 1e-14


@pytest.mark.skipif(not po.ref_available(), reason="needs oracle/_ref")
@pytest.mark.parametrize("fmt", ["matrix_market", "csv"])
def test_export_matches_reference_bytes(fmt, tmp_path):
    """ff_export_csr / ff_export_vector write exactly what the reference's
    linalg::export_matrix(EllMatrix) / export_vector write (linalg.cpp:148-210)."""
    from paper_1802_03433_b200 import femforge as ff
    xy, conn = po.unit_square_mesh(4)
    h = po.RefHarness(2, 1, xy, conn, conn, xy.shape[0], "demo2d")
    rp, ci = h.pattern()
    v, b = h.assemble()
    code = {"matrix_market": 0, "csv": 1}[fmt]
    h.export(v, b, tmp_path / "ref.mtx", tmp_path / "ref_b.mtx", code)
    ff.export_csr(rp, ci, v, tmp_path / "ours.mtx", fmt)
    ff.export_vector(b, tmp_path / "ours_b.mtx", fmt)
    assert (tmp_path / "ours.mtx").read_bytes() == (tmp_path / "ref.mtx").read_bytes()
    assert (tmp_path / "ours_b.mtx").read_bytes() == (tmp_path / "ref_b.mtx").read_bytes()
    if fmt == "matrix_market":
        assert (tmp_path / "ours.mtx").read_text().splitlines()[1] == f"25 25 {len(ci)}"


@pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")
def test_reference_build_reproduces_its_golden_kernel_source():
    """Pins the oracle/_ref build to the reference: its emit_source output for
    the demo form hashes to the committed fixture, which is the hash of the
    reference's own golden (proj/tests/data/demo_kernel.cu.golden,
    test_codegen.cpp:199-206) when the reference tree is present."""
    import hashlib
    buf = po.C.create_string_buffer(1 << 20)
    n = po.ref().ffref_emit_demo_source(buf, len(buf))
    got = hashlib.sha256(buf.value[:n]).hexdigest()
    with open(os.path.join(GOLDEN, "demo_kernel.cu.golden.sha256")) as f:
        assert got == f.read().strip()
    golden = "/root/reference/proj/tests/data/demo_kernel.cu.golden"
    if os.path.exists(golden):
        with open(golden, "rb") as f:
            assert got == hashlib.sha256(f.read()).hexdigest()

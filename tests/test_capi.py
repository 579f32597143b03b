"""The C ABI and the host side of the engine, without a GPU: library loads,
exports every symbol of include/femforge_b200.h, NVRTC compiles the emitted
kernels for sm_100a, host helpers agree with the oracle, error behaviour."""
import os
import re
import subprocess

import numpy as np
import pytest

import pyoracle as po
from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "femforge_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|void\*)\s+(ff_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol(ff):
    out = subprocess.run(["nm", "-D", "--defined-only", ff.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (ff_\w+)", out))
    declared = header_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    bound = {name for name, _, _ in ff.SIGNATURES}
    assert set(declared) == bound


def test_no_driver_library_link(ff):
    # the engine must load on a GPU-less host (driver resolved at run time)
    out = subprocess.run(["ldd", ff.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcuda.so" not in out


@pytest.mark.parametrize("dim,deg,form,quad,strategy,reg_cap", [
    (2, 1, "demo2d", 3, "auto", 96), (2, 2, "helmholtz", 1, "auto", 128), (3, 1, "poisson", 4, "auto", 96),
    (3, 2, "poisson", 4, "auto", 168), (3, 2, "poisson", 4, "pointwise", 255), (3, 2, "varcoef", 14, "auto", 255),
])
def test_nvrtc_compiles_for_sm100a(ff, dim, deg, form, quad, strategy, reg_cap):
    bil, lin = ff.named_form(form, dim)
    f = ff.Form(None, dim, deg, bil, lin, quad_rule=quad, strategy=strategy)
    info = f.info
    assert info["n_local"] == {(2, 1): 3, (2, 2): 6, (3, 1): 4, (3, 2): 10}[(dim, deg)]
    assert 0 < info["registers"] <= reg_cap
    cubin = f.cubin
    assert cubin[:4] == b"\x7fELF"
    src = f.source
    assert "{{" not in src and "ff_assemble_atomic" in src
    # byte-deterministic emission (criterion 7)
    assert ff.Form(None, dim, deg, bil, lin, quad_rule=quad, strategy=strategy).source == src


def test_reference_tensor_collapses_poisson_p2(ff):
    bil, lin = ff.named_form("stiffness", 3)
    info = ff.Form(None, 3, 2, bil, lin).info
    # K = sum_t C_t (det J^{-1} J^{-T})_t: six geometric invariants, 55 symmetric entries
    assert info["strategy"] == 1 and info["n_invariants"] <= 7
    assert info["n_unique_entries"] <= 56


def test_form_errors(ff):
    with pytest.raises(ff.SymbolicError, match="offset 5"):
        ff.Form(None, 2, 1, "sin(x", "v")
    with pytest.raises(ff.FormError, match="outside the reserved set"):
        ff.Form(None, 2, 1, "u*v + rogue", "v")
    with pytest.raises(ff.FormError, match="outside the reserved set"):
        ff.Form(None, 2, 1, "u*v", "u")  # trial symbol not allowed in the linear form
    with pytest.raises(ff.FormError):
        ff.Form(None, 2, 1, "u_z*v_z", "v")  # 3D symbol in a 2D form
    with pytest.raises(ff.FFError):
        ff.Form(None, 3, 2, "u*v", "v", quad_rule=7)
    with pytest.raises(ff.FFError):
        ff.Form(None, 3, 3, "u*v", "v")


def test_nonpolynomial_integrand_falls_back_to_pointwise(ff):
    f = ff.Form(None, 2, 1, "u_x*v_x + u_y*v_y + u*v", "(19.739208802178716 + 1)*cos(3.141592653589793*x)*cos(3.141592653589793*y)*v")
    assert f.info["strategy"] == 2
    with pytest.raises(ff.FormError, match="not polynomial"):
        ff.Form(None, 2, 1, "u*v", "sin(x)*v", strategy="tensor")


@pytest.mark.parametrize("n", [1, 3, 8])
def test_mesh_generators_match_oracle(ff, n):
    assert all(np.array_equal(a, b) for a, b in zip(ff.unit_square_mesh(n), po.unit_square_mesh(n)))
    (c, v), (oc, ov) = ff.kuhn_mesh(n), po.kuhn_mesh(n)
    assert np.array_equal(c, oc) and np.array_equal(v, ov)
    assert np.array_equal(ff.kuhn_p2_dofs(n, v)[0], po.p2_dofs_kuhn(n, ov)[0])


def test_kuhn_tets_positively_oriented(ff):
    c, v = ff.kuhn_mesh(3)
    x = c[v]
    det = np.linalg.det(np.stack([x[:, 1] - x[:, 0], x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]], axis=-1))
    assert np.all(det > 0) and np.allclose(det, 1 / 27)


def test_generic_p2_dofs(ff):
    c, v = ff.kuhn_mesh(3)
    d, nd = ff.p2_dofs(3, v, c.shape[0])
    lat, nl = ff.kuhn_p2_dofs(3, v)
    assert nd == nl == 7 ** 3
    # same DOF sets up to renumbering: identical pattern size
    assert po.build_pattern(d, nd)[0][-1] == po.build_pattern(lat, nl)[0][-1]
    assert np.array_equal(d[:, :4], v)  # vertices first


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_partition_and_halo_selection(ff, parts):
    c, v = ff.kuhn_mesh(4)
    d, nd = ff.kuhn_p2_dofs(4, v)
    bounds = [ff.partition_rows(nd, parts, p) for p in range(parts)]
    assert bounds[0][0] == 0 and bounds[-1][1] == nd
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(parts - 1))
    covered = np.zeros(v.shape[0], int)
    for rb, re in bounds:
        ids = ff.select_elements(d, rb, re)
        expect = np.nonzero(((d >= rb) & (d < re)).any(axis=1))[0]
        assert np.array_equal(ids, expect)
        covered[ids] += 1
    assert covered.min() >= 1  # every element assembled by at least one block


def test_cpp_host_suites():
    exe = os.path.join(ROOT, "build", "tests", "test_host")
    if not os.path.exists(exe):
        pytest.skip("C++ test binary not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


def test_integration_binding_is_the_documented_one():
    """tests/cpp/ref_side/device_b200.cpp (compiled against the reference into
    oracle/_ref/test_integration, run by the GPU suite) is INTEGRATION.md §2's
    snippet verbatim, and it builds wherever the reference sources exist."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    a = doc.index("```cpp\n// src/device/device_b200.cpp") + len("```cpp\n")
    snippet = doc[a:doc.index("```", a)]
    src = open(os.path.join(ROOT, "tests", "cpp", "ref_side", "device_b200.cpp")).read()
    assert src.endswith(snippet)
    if os.path.isdir("/root/reference/proj/src"):
        assert os.path.exists(os.path.join(ROOT, "oracle", "_ref", "test_integration"))


def _row_classes(dconn, n_dofs, row_ptr, col_idx, min_rows):
    """Row classes as the gather plan defines them: rows whose incidences,
    sorted by (local index, slot bytes, element), and lengths coincide."""
    import collections
    k = dconn.shape[1]
    inc = collections.defaultdict(list)
    for e in range(dconn.shape[0]):
        for i in range(k):
            r = dconn[e, i]
            cols = col_idx[row_ptr[r]:row_ptr[r + 1]]
            inc[r].append((i, tuple(int(np.searchsorted(cols, dconn[e, j])) for j in range(k)), e))
    sig = collections.Counter()
    for r in range(n_dofs):
        seq = tuple((i, sl) for i, sl, e in sorted(inc[r]))
        sig[(int(row_ptr[r + 1] - row_ptr[r]), seq)] += 1
    return [(ln, [i for i, _ in seq], [list(sl) for _, sl in seq])
            for (ln, seq), c in sig.most_common() if c >= min_rows]


def test_class_specialised_source_compiles(ff):
    """The per-class gather kernels (rows in registers, compile-time slots) of
    a 3D P2 Kuhn mesh compile for sm_100a through NVRTC."""
    import pyoracle as po
    c, v = po.kuhn_mesh(4)
    d, nd = po.p2_dofs_kuhn(4, v)
    rp, ci = po.build_pattern(d, nd)
    classes = _row_classes(d, nd, rp, ci, 8)
    assert len(classes) >= 8 and max(c[0] for c in classes) == 65
    bil, lin = ff.named_form("poisson", 3)
    f = ff.Form(None, 3, 2, bil, lin, quad_rule=4)
    src = f.class_source(classes)
    assert "ff_gather_classes_s" in src and "ff_gather_classes_l" in src
    assert f.class_source(classes) == src  # byte-deterministic
    g = ff.Form.from_source(None, src, 3, 2)
    assert g.cubin[:4] == b"\x7fELF"


def test_blocked_elasticity_form_compiles(ff):
    """Vector P2 elasticity (3x3 blocks of scalar forms, 30 DOFs per element)
    through instantiate_blocked -> tensor plan -> NVRTC for sm_100a, with the
    component-pair row gather (K2a + generic sub-row kernel) in the module."""
    b, l = ff.elasticity_text(3)
    f = ff.Form.blocked(None, 3, 2, 3, b, l, quad_rule=4)
    info = f.info
    assert info["n_local"] == 30 and info["n_kinv"] == 36
    assert f.cubin[:4] == b"\x7fELF" and "#define FF_BS 3" in f.source
    assert "ff_gather_invariants" in f.source and "ff_gather_apply<29>(r, g, d, arow)" in f.source


def _vrow_terms(src, nsc):
    import re
    terms = []
    for a in range(nsc):
        body = src[src.index(f"void ff_vrow<{a}>("):]
        body = body[:body.index("}")]
        terms += [0 if e == "0.0" else e.count("g[") for e in re.findall(r"v\[\d+\] = (.*?);", body)]
    return terms


@pytest.mark.parametrize("lam,mu,nbq,nkinv", [("1", "1", 6, 36), ("2", "0.5", 10, 90)])
def test_vector_record_is_block_uniform(ff, lam, mu, nbq, nkinv):
    """Vector forms: every (test, trial) component block's entries are one
    linear map (ff_vrow) of that block's own record quantities
    (element_plan.cpp: uniform_block_basis). Elasticity: 6 quantities per
    block for lambda = mu ((c,d) and (d,c) share them: 36 in the record), 9
    (padded to 10) otherwise; every entry of the P2 node-pair map reads <= 6
    resp. 9 quantities -- the diagonal blocks' 18-invariant entries are gone."""
    import re
    b, l = ff.elasticity_text(3, lam=lam, mu=mu)
    f = ff.Form.blocked(None, 3, 2, 3, b, l, quad_rule=4)
    src = f.source
    assert f.info["n_kinv"] == nkinv
    assert re.search(r"#define FF_NBQ (\d+)", src).group(1) == str(nbq)
    q = [int(x) for x in re.search(r"ff_block_q\[9\] = \{(.*?)\}", src).group(1).split(",")]
    assert all(o % 2 == 0 and o + nbq <= nkinv for o in q)
    if lam == mu:
        assert q[1] == q[3] and q[2] == q[6] and q[5] == q[7]  # (c,d) and (d,c) share
    t = _vrow_terms(src, 10)
    assert len(t) == 100 and max(t) <= (6 if lam == mu else 9)

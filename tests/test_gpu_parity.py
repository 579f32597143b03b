"""GPU parity: the CUDA path (through the C ABI) against the reference's own
golden outputs, the oracle, and size-independent properties at the
BASELINE.json sizes. Tolerances: sparsity bit-exact; values/rhs <= 1e-12
normwise (acceptance.cpp:58-67; BASELINE.json north star)."""
import glob
import os

import numpy as np
import pytest

import pyoracle as po
from conftest import GOLDEN, normwise

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _golden(pattern):
    return sorted(glob.glob(os.path.join(GOLDEN, pattern)))


SCATTERS = ["gather", "atomic"]


def gpu_system(ff, ctx, dim, deg, form, coords, vconn, dconn, n_dofs, quad=0, strategy="auto",
               row_begin=0, row_end=None, block=256, scatter="gather"):
    ctx.set_scatter(scatter)
    bil, lin = ff.named_form(form, dim) if isinstance(form, str) else form
    f = ff.Form(ctx, dim, deg, bil, lin, quad_rule=quad, strategy=strategy, block_size=block)
    m = ff.Mesh(ctx, dim, coords, vconn, None if deg == 1 else dconn, n_dofs)
    p = ff.Pattern(ctx, m, row_begin, row_end)
    rp, ci = p.export()
    v, b = ff.assemble(f, m, p)
    return rp, ci, v, b, f, m, p


@pytest.mark.parametrize("path", _golden("ref2d_*.npz"), ids=os.path.basename)
@pytest.mark.parametrize("scatter", SCATTERS)
def test_gpu_matches_reference_2d(ff, ctx, path, scatter):
    g = np.load(path)
    _, form, n = os.path.basename(path)[:-4].split("_")
    xy, conn = ff.unit_square_mesh(int(n[1:]))
    rp, ci, v, b, *_ = gpu_system(ff, ctx, 2, 1, form, xy, conn, conn, xy.shape[0], scatter=scatter)
    assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(ci, g["col_idx"])
    assert normwise(v, g["values"]) <= TOL
    assert normwise(b, g["rhs"]) <= TOL


@pytest.mark.parametrize("path", _golden("ref3d_*.npz"), ids=os.path.basename)
@pytest.mark.parametrize("strategy", ["tensor", "pointwise"])
@pytest.mark.parametrize("scatter", SCATTERS)
def test_gpu_matches_reference_cas_3d(ff, ctx, path, strategy, scatter):
    g = np.load(path)
    _, p, form, n, q = os.path.basename(path)[:-4].split("_")
    deg, n, q = int(p[1:]), int(n[1:]), int(q[1:])
    xyz, vc = ff.kuhn_mesh(n)
    dc, nd = (vc, xyz.shape[0]) if deg == 1 else ff.kuhn_p2_dofs(n, vc)
    rp, ci, v, b, *_ = gpu_system(ff, ctx, 3, deg, form, xyz, vc, dc, nd, quad=q, strategy=strategy, scatter=scatter)
    assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(ci, g["col_idx"])
    assert normwise(v, g["values"]) <= TOL
    assert normwise(b, g["rhs"]) <= TOL


CASES = [  # (dim, degree, form, n, quad)
    (2, 1, "demo2d", 96, 3),
    (2, 1, "poisson", 64, 3),
    (2, 2, "helmholtz", 24, 1),
    (3, 1, "poisson", 14, 4),
    (3, 1, "varcoef", 8, 14),
    (3, 2, "poisson", 10, 4),
    (3, 2, "helmholtz", 8, 11),
    (3, 2, "varcoef", 6, 14),
]


def _mesh(ff, dim, deg, n):
    if dim == 2:
        c, v = ff.unit_square_mesh(n)
        d, nd = (v, c.shape[0]) if deg == 1 else ff.p2_dofs(2, v, c.shape[0])
    else:
        c, v = ff.kuhn_mesh(n)
        d, nd = (v, c.shape[0]) if deg == 1 else ff.kuhn_p2_dofs(n, v)
    return c, v, d, nd


@pytest.mark.parametrize("dim,deg,form,n,quad", CASES)
@pytest.mark.parametrize("scatter", SCATTERS)
def test_gpu_matches_oracle(ff, ctx, dim, deg, form, n, quad, scatter):
    c, v, d, nd = _mesh(ff, dim, deg, n)
    rp, ci, val, rhs, *_ = gpu_system(ff, ctx, dim, deg, form, c, v, d, nd, quad=quad, scatter=scatter)
    orp, oci = po.build_pattern(d, nd)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    ov, ob = po.assemble(form, dim, deg, quad, c, v, d, orp, oci, workers=8)
    assert normwise(val, ov) <= TOL
    assert normwise(rhs, ob) <= TOL


def test_ell_view_matches_reference_layout(ff, ctx):
    g = np.load(os.path.join(GOLDEN, "ref2d_demo2d_n8.npz"))
    xy, conn = ff.unit_square_mesh(8)
    *_, p = gpu_system(ff, ctx, 2, 1, "demo2d", xy, conn, conn, xy.shape[0])
    assert p.max_row_len == 7  # MAX_NZ 7 (test_device.cpp:85-90)
    rl, rc = p.export_ell()
    assert np.array_equal(rl, np.diff(g["row_ptr"]))
    for i in range(p.n_rows):
        assert np.array_equal(rc[i, :rl[i]], g["col_idx"][g["row_ptr"][i]:g["row_ptr"][i + 1]])
        assert np.all(rc[i, rl[i]:] == -1)


@pytest.mark.parametrize("scatter", SCATTERS)
def test_device_path_equals_e2e_path(ff, ctx, scatter):
    import torch
    c, v, d, nd = _mesh(ff, 3, 2, 6)
    rp, ci, val, rhs, f, m, p = gpu_system(ff, ctx, 3, 2, "poisson", c, v, d, nd, scatter=scatter)
    dv = torch.empty(p.nnz, dtype=torch.float64, device="cuda")
    db = torch.empty(p.n_rows, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        ff.assemble_device(f, m, p, dv.data_ptr(), db.data_ptr(), s)
    torch.cuda.synchronize()
    ctx.check()
    # same kernel, atomics reorder fp64 adds only
    assert normwise(dv.cpu().numpy(), val) <= 1e-14
    assert normwise(db.cpu().numpy(), rhs) <= 1e-14


@pytest.mark.parametrize("scatter", SCATTERS)
def test_graph_replay_follows_the_mesh(ff, ctx, scatter):
    """Repeated ff_assemble_device calls on a created stream replay one CUDA
    graph (first call plain, second captured): the replay reads the current
    coordinates, and a connectivity update (new plans) re-captures; every
    result equals the host-buffer path on the same mesh."""
    import torch
    c, v, d, nd = _mesh(ff, 3, 2, 6)
    rp, ci, val, rhs, f, m, p = gpu_system(ff, ctx, 3, 2, "helmholtz", c, v, d, nd, quad=4, scatter=scatter)
    stream = torch.cuda.Stream()
    dv = torch.empty(p.nnz, dtype=torch.float64, device="cuda")
    db = torch.empty(p.n_rows, dtype=torch.float64, device="cuda")

    def run(k):
        out = []
        for _ in range(k):
            dv.fill_(float("nan"))
            torch.cuda.synchronize()
            ff.assemble_device(f, m, p, dv.data_ptr(), db.data_ptr(), stream.cuda_stream)
            torch.cuda.synchronize()
            ctx.check()
            out.append((dv.cpu().numpy().copy(), db.cpu().numpy().copy()))
        return out

    for a, b in run(4):
        assert normwise(a, val) <= 1e-14 and normwise(b, rhs) <= 1e-14
    rng = np.random.default_rng(7)
    c2 = c.copy()
    inner = np.all((c > 1e-12) & (c < 1 - 1e-12), axis=1)
    c2[inner] += rng.uniform(-0.02, 0.02, size=(inner.sum(), 3)) / 6
    val2, rhs2 = ff.assemble(f, m, p, coords=c2)   # uploads the new coordinates
    torch.cuda.synchronize()
    for a, b in run(2):
        assert normwise(a, val2) <= 1e-14 and normwise(b, rhs2) <= 1e-14
    perm = rng.permutation(v.shape[0])
    v3, d3 = np.ascontiguousarray(v[perm]), np.ascontiguousarray(d[perm])
    val3, rhs3 = ff.assemble(f, m, p, coords=c2, vconn=v3, dconn=d3)
    torch.cuda.synchronize()
    for a, b in run(3):
        assert normwise(a, val3) <= 1e-14 and normwise(b, rhs3) <= 1e-14
    assert normwise(val3, val2) <= 1e-13


@pytest.mark.parametrize("scatter", SCATTERS)
def test_degenerate_element_reported_by_lowest_index(ff, ctx, scatter):
    ctx.set_scatter(scatter)
    xy, conn = ff.unit_square_mesh(4)
    b, l = ff.named_form("stiffness", 2)
    f = ff.Form(ctx, 2, 1, b, l)
    m = ff.Mesh(ctx, 2, xy, conn)
    p = ff.Pattern(ctx, m)
    bad = xy.copy()
    bad[conn[9]] = [0.3, 0.35]  # collapse element 9 (and every element sharing an edge with it)
    x = bad[conn]
    det = (x[:, 1, 0] - x[:, 0, 0]) * (x[:, 2, 1] - x[:, 0, 1]) - (x[:, 2, 0] - x[:, 0, 0]) * (x[:, 1, 1] - x[:, 0, 1])
    lowest = int(np.nonzero(np.abs(det) <= 1e-14)[0].min())
    with pytest.raises(ff.DeviceError, match=f"degenerate element {lowest} "):
        ff.assemble(f, m, p, coords=bad)
    ff.assemble(f, m, p, coords=xy)  # recovers


@pytest.mark.parametrize("scatter", SCATTERS)
def test_pattern_from_other_mesh_is_a_hard_error(ff, ctx, scatter):
    ctx.set_scatter(scatter)
    # test_device.cpp:262-279: same node count, disjoint connectivity
    xy, conn = ff.unit_square_mesh(2)
    b, l = ff.named_form("demo2d", 2)
    f = ff.Form(ctx, 2, 1, b, l)
    m = ff.Mesh(ctx, 2, xy, conn)
    p = ff.Pattern(ctx, m)
    other = conn.copy()
    other[0] = [0, 1, 5]
    with pytest.raises(ff.DeviceError, match="not present in sparsity row"):
        ff.assemble(f, m, p, vconn=other)


@pytest.mark.parametrize("scatter", SCATTERS)
def test_isolated_dofs_and_tiny_meshes(ff, ctx, scatter):
    """Edge cases of the pattern rules (device.cpp:66-88: the diagonal is
    always present): a node no element touches keeps a diagonal-only row whose
    value and load are exactly 0 (the atomic-free scatters write every value,
    nothing is zero-filled for them); one-cell meshes in 2D and 3D match the
    oracle."""
    ctx.set_scatter(scatter)
    xy, conn = ff.unit_square_mesh(3)
    xy = np.vstack([xy, [[2.0, 2.0]]])          # node 16: no element
    rp, ci, v, b, *_ = gpu_system(ff, ctx, 2, 1, "demo2d", xy, conn, conn, xy.shape[0], scatter=scatter)
    assert rp[-1] - rp[-2] == 1 and ci[-1] == 16 and v[-1] == 0.0 and b[-1] == 0.0
    orp, oci = po.build_pattern(conn, xy.shape[0])
    ov, ob = po.assemble("demo2d", 2, 1, 3, xy, conn, conn, orp, oci)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    assert normwise(v, ov) <= TOL and normwise(b, ob) <= TOL
    for dim, deg in [(2, 1), (3, 1), (3, 2)]:
        c, vc, d, nd = _mesh(ff, dim, deg, 1)
        form = "demo2d" if dim == 2 else "helmholtz"
        rp, ci, v, b, *_ = gpu_system(ff, ctx, dim, deg, form, c, vc, d, nd, quad=3 if dim == 2 else 4,
                                      scatter=scatter)
        orp, oci = po.build_pattern(d, nd)
        ov, ob = po.assemble(form, dim, deg, 3 if dim == 2 else 4, c, vc, d, orp, oci)
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
        assert normwise(v, ov) <= TOL and normwise(b, ob) <= TOL


@pytest.mark.parametrize("parts", [2, 3, 4])
@pytest.mark.parametrize("scatter", SCATTERS)
def test_row_blocks_concatenate_to_full_system(ff, ctx, parts, scatter):
    c, v, d, nd = _mesh(ff, 3, 2, 6)
    rp, ci, val, rhs, *_ = gpu_system(ff, ctx, 3, 2, "poisson", c, v, d, nd, scatter=scatter)
    rp_parts, cis, vals, rhss, off = [], [], [], [], 0
    for part in range(parts):
        rb, re = ff.partition_rows(nd, parts, part)
        ids = ff.select_elements(d, rb, re)  # owned + halo elements, duplicated across blocks
        sub = gpu_system(ff, ctx, 3, 2, "poisson", c, v[ids], d[ids], nd, row_begin=rb, row_end=re, scatter=scatter)
        rp_parts.append(sub[0][:-1] + off)
        off += sub[0][-1]
        cis.append(sub[1]); vals.append(sub[2]); rhss.append(sub[3])
    rp_cat = np.concatenate(rp_parts + [np.array([off])])
    assert np.array_equal(rp_cat, rp)
    assert np.array_equal(np.concatenate(cis), ci)
    assert normwise(np.concatenate(vals), val) <= TOL
    assert normwise(np.concatenate(rhss), rhs) <= TOL


ATOMIC_FREE = [  # (scatter, dim, degree, n, form, quad)
    ("gather", 3, 1, 20, "helmholtz", 4),
    ("gather", 3, 2, 12, "poisson", 4),
    ("gather", 2, 1, 128, "demo2d", 3),
    ("gather", 2, 2, 40, "helmholtz", 3),
]


@pytest.mark.parametrize("scatter,dim,deg,n,form,quad", ATOMIC_FREE)
def test_atomic_free_scatter_is_bitwise_reproducible_and_matches_atomic(ff, ctx, scatter, dim, deg, n, form, quad):
    """Atomic-free scatters: fixed summation order -> identical bits on every
    run (the reference's deterministic-mode property, criterion 7/8)."""
    c, v, d, nd = _mesh(ff, dim, deg, n)
    rp, ci, v1, b1, f, m, p = gpu_system(ff, ctx, dim, deg, form, c, v, d, nd, quad=quad, scatter=scatter)
    assert p.scatter_for(f) == scatter
    v2, b2 = ff.assemble(f, m, p)
    assert v1.tobytes() == v2.tobytes() and b1.tobytes() == b2.tobytes()
    ctx.set_scatter("atomic")
    va, ba = ff.assemble(f, m, p)
    ctx.set_scatter(scatter)
    assert normwise(va, v1) <= 1e-14 and normwise(ba, b1) <= 1e-14


@pytest.mark.parametrize("dim,deg,n", [(3, 2, 8), (3, 1, 12), (2, 1, 32), (2, 2, 16)])
def test_gather_plan_covers_every_incidence(ff, ctx, dim, deg, n):
    c, v, d, nd = _mesh(ff, dim, deg, n)
    ctx.set_scatter("gather")
    b, l = ff.named_form("poisson", dim)
    f = ff.Form(ctx, dim, deg, b, l)
    m = ff.Mesh(ctx, dim, c, v, None if deg == 1 else d, nd)
    p = ff.Pattern(ctx, m)
    gi = p.gather_info(m)
    k = d.shape[1]
    assert gi["n_incidences"] == d.shape[0] * k           # every (element, local row) once
    # every row is either in a specialised row class or in a generic item
    assert gi["n_items"] == -(-(nd - gi["n_class_rows"]) // 32)
    assert gi["n_class_items"] * 32 >= gi["n_class_rows"]
    assert gi["record_bytes"] == (8 if k <= 4 else 16)
    assert f.info["n_kinv"] > 0


def test_gather_falls_back_to_atomic_for_pointwise_forms(ff, ctx):
    c, v, d, nd = _mesh(ff, 3, 2, 4)
    ctx.set_scatter("gather")
    b, l = ff.named_form("varcoef", 3)
    f = ff.Form(ctx, 3, 2, b, l, quad_rule=14)
    assert f.info["strategy"] == 2 and f.info["n_kinv"] == 0
    m = ff.Mesh(ctx, 3, c, v, d, nd)
    p = ff.Pattern(ctx, m)
    assert p.scatter_for(f) == "atomic"


def test_gather_phases_compose(ff, ctx):
    """K2a (invariants) then K2b (rows) launched separately == one call."""
    import torch
    c, v, d, nd = _mesh(ff, 3, 2, 6)
    rp, ci, val, rhs, f, m, p = gpu_system(ff, ctx, 3, 2, "poisson", c, v, d, nd, scatter="gather")
    dv = torch.full((p.nnz,), float("nan"), dtype=torch.float64, device="cuda")
    db = torch.full((p.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ff.assemble_device_ex(f, m, p, dv.data_ptr(), db.data_ptr(), s, ff.FF_GATHER_INVARIANTS_ONLY)
    ff.assemble_device_ex(f, m, p, dv.data_ptr(), db.data_ptr(), s, ff.FF_GATHER_ROWS_ONLY)
    torch.cuda.synchronize()
    ctx.check()
    assert dv.cpu().numpy().tobytes() == val.tobytes() and db.cpu().numpy().tobytes() == rhs.tobytes()


def test_north_star_size_properties(ff, ctx):
    """Kuhn 128^3 P2 Poisson (12.58M tets): nnz cubic, zero row sums of the
    stiffness, symmetry, and sum(rhs) = integral of f (partition of unity;
    the 4-point rule is exact for the quadratic f) -- checked on the GPU."""
    import torch
    n = 128
    c, v, d, nd = _mesh(ff, 3, 2, n)
    b, l = ff.named_form("poisson", 3)
    ctx.set_scatter("gather")
    f = ff.Form(ctx, 3, 2, b, l)
    m = ff.Mesh(ctx, 3, c, v, d, nd)
    p = ff.Pattern(ctx, m)
    assert p.nnz == 230 * n ** 3 + 138 * n ** 2 + 24 * n + 1
    vals = torch.empty(p.nnz, dtype=torch.float64, device="cuda")
    rhs = torch.empty(p.n_rows, dtype=torch.float64, device="cuda")
    ff.assemble_device(f, m, p, vals.data_ptr(), rhs.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ctx.check()
    rp_ptr, ci_ptr = p.device_pointers()
    rp, ci = p.export()
    rp_t = torch.from_numpy(rp).cuda()
    ci_t = torch.from_numpy(ci).cuda().long()
    rows = torch.repeat_interleave(torch.arange(p.n_rows, device="cuda"), rp_t[1:] - rp_t[:-1])
    amax = vals.abs().max()
    rowsum = torch.zeros(p.n_rows, dtype=torch.float64, device="cuda").index_add_(0, rows, vals)
    rowmax = torch.zeros(p.n_rows, dtype=torch.float64, device="cuda").index_reduce_(0, rows, vals.abs(), "amax")
    assert float((rowsum.abs() / rowmax).max()) <= 1e-12
    # symmetry: value of (i,j) equals value of (j,i); keys sorted => compare via sort
    key = rows * nd + ci_t
    tkey = ci_t * nd + rows
    order = torch.argsort(tkey)
    assert torch.equal(tkey[order], key)  # pattern symmetric
    assert float((vals[order] - vals).abs().max() / amax) <= 1e-12
    assert abs(float(rhs.sum()) - 34.0) <= 1e-9
    # the atomic-free gather against the element-parallel fp64-RED kernel
    va = torch.empty_like(vals)
    ra = torch.empty_like(rhs)
    ff.assemble_device_ex(f, m, p, va.data_ptr(), ra.data_ptr(), torch.cuda.current_stream().cuda_stream,
                          ff.FF_SCATTER_ATOMIC)
    torch.cuda.synchronize()
    ctx.check()
    assert float((va - vals).abs().max() / amax) <= 1e-12
    assert float((ra - rhs).abs().max() / rhs.abs().max()) <= 1e-12


@pytest.mark.parametrize("dim,deg,n,form", [(3, 2, 10, "poisson"), (3, 1, 12, "helmholtz"), (2, 1, 64, "demo2d"),
                                            (2, 2, 24, "helmholtz")])
def test_class_specialised_gather_equals_generic(ff, ctx, dim, deg, n, form):
    """Row classes (slots as compile-time register indices) sum every CSR slot
    in the same incidence order as the generic gather."""
    c, v, d, nd = _mesh(ff, dim, deg, n)
    ctx.set_scatter("gather")
    quad = 4 if dim == 3 else 3
    b, l = ff.named_form(form, dim)
    f = ff.Form(ctx, dim, deg, b, l, quad_rule=quad)
    m = ff.Mesh(ctx, dim, c, v, None if deg == 1 else d, nd)
    p = ff.Pattern(ctx, m)
    try:
        ctx.set_gather_classes(16)
        gi = p.gather_info(m)
        assert gi["n_classes"] > 0 and gi["n_class_rows"] > nd // 2
        assert gi["n_class_rows"] + gi["n_items"] * 32 >= nd
        v1, b1 = ff.assemble(f, m, p)
        ctx.set_gather_classes(0)
        assert p.gather_info(m)["n_classes"] == 0
        v0, b0 = ff.assemble(f, m, p)
        v2, b2 = ff.assemble(f, m, p)
    finally:
        ctx.set_gather_classes(128)
    # same summation order; the two NVRTC modules may contract fp64 FMAs
    # differently, so the paths agree to rounding (each is bitwise reproducible)
    assert normwise(v1, v0) <= 1e-15 and normwise(b1, b0) <= 1e-15
    assert v2.tobytes() == v0.tobytes() and b2.tobytes() == b0.tobytes()
    orp, oci = po.build_pattern(d, nd)
    ov, ob = po.assemble(form, dim, deg, quad, c, v, d, orp, oci, workers=8)
    assert normwise(v1, ov) <= TOL and normwise(b1, ob) <= TOL




def _elasticity_system(ff, ctx, n, row_begin=0, row_end=None, ids=None, lam="1", mu="1", force=("0", "0", "-1"),
                       scatter="gather"):
    ctx.set_scatter(scatter)
    c, v = ff.kuhn_mesh(n)
    d, nd = ff.kuhn_p2_dofs(n, v)
    if ids is not None:
        v, d = np.ascontiguousarray(v[ids]), np.ascontiguousarray(d[ids])
    b, l = ff.elasticity_text(3, lam, mu, force)
    f = ff.Form.blocked(ctx, 3, 2, 3, b, l, quad_rule=4)
    m = ff.Mesh(ctx, 3, c, v, d, nd, ncomp=3)
    p = ff.Pattern(ctx, m, row_begin, row_end)
    rp, ci = p.export()
    val, rhs = ff.assemble(f, m, p)
    return c, v, d, nd, rp, ci, val, rhs, f, m, p


@pytest.mark.parametrize("n", [2, 5])
@pytest.mark.parametrize("scatter", ["gather", "atomic"])
def test_elasticity_matches_oracle(ff, ctx, n, scatter):
    """Config 5 (vector P2 elasticity): block-expanded pattern bit-exact, values
    and RHS <= 1e-12 normwise against the C restatement, through the row
    gather (block-uniform records, the three trial components of a row in
    neighbouring lanes) and the atomic scatter."""
    c, v, d, nd, rp, ci, val, rhs, f, m, p = _elasticity_system(ff, ctx, n, lam="2", mu="0.5", force=("0", "1", "-1"),
                                                                scatter=scatter)
    assert p.scatter_for(f) == scatter and p.n_rows == 3 * nd
    orp, oci = po.build_pattern(d, nd)
    vrp, vci = po.block_pattern(orp, oci, 3)
    assert np.array_equal(rp, vrp) and np.array_equal(ci, vci)
    ov, ob = po.assemble_elasticity(3, 2, 4, c, v, d, vrp, vci, lam=2.0, mu=0.5, force=(0.0, 1.0, -1.0))
    assert normwise(val, ov) <= TOL and normwise(rhs, ob) <= TOL


@pytest.mark.parametrize("lam,mu", [("1", "1"), ("2", "0.5")])
def test_elasticity_class_gather_matches_atomic(ff, ctx, lam, mu):
    """Vector forms through the class-specialised gather (node-row classes,
    lanes = (row, trial component), rows staged in CSR order and written by
    TMA; short- and long-row kernels): equal to the atomic scatter to
    rounding, bitwise reproducible run to run."""
    n = 8
    ctx.set_gather_classes(200)
    try:
        *_, val_a, rhs_a, f, m, p = _elasticity_system(ff, ctx, n, lam=lam, mu=mu, scatter="atomic")
        ctx.set_scatter("gather")
        val_g, rhs_g = ff.assemble(f, m, p)
        val_g2, rhs_g2 = ff.assemble(f, m, p)
        gi = p.gather_info(m)
    finally:
        ctx.set_gather_classes(128)
    assert gi["n_class_rows"] > 0 and gi["n_classes"] >= 8
    assert normwise(val_g, val_a) <= 1e-15 and normwise(rhs_g, rhs_a) <= 1e-15
    assert np.array_equal(val_g, val_g2) and np.array_equal(rhs_g, rhs_g2)


def test_elasticity_rigid_body_modes_and_row_blocks(ff, ctx):
    """Size-independent properties at n=16 (24.6k tets, 107k DOFs): rigid-body
    modes in the kernel, symmetry, sum of the load; 3 node-aligned row blocks
    concatenate to the 1-GPU system (SURVEY §8e for config 5)."""
    import scipy.sparse as sp
    n = 16
    ctx.set_gather_classes(0)  # generic sub-row gather here (classes: the test above)
    try:
        _elasticity_rbm(ff, ctx, sp, n)
    finally:
        ctx.set_gather_classes(128)


def _elasticity_rbm(ff, ctx, sp, n):
    c, v, d, nd, rp, ci, val, rhs, *_ = _elasticity_system(ff, ctx, n)
    K = sp.csr_matrix((val, ci, rp), shape=(3 * nd, 3 * nd))
    L = 2 * n + 1
    idx = np.arange(nd)
    X = np.stack([idx % L, (idx // L) % L, idx // (L * L)], 1) / (L - 1)
    scale = np.abs(val).max()
    for a, b in [(0, 1), (1, 2), (0, 2)]:
        u = np.zeros(3 * nd)
        u[a::3] = -X[:, b]
        u[b::3] = X[:, a]
        assert np.abs(K @ u).max() <= 1e-11 * scale
    for t in range(3):
        u = np.zeros(3 * nd)
        u[t::3] = 1.0
        assert np.abs(K @ u).max() <= 1e-11 * scale
    assert abs(K - K.T).max() <= 1e-12 * scale
    assert abs(rhs[2::3].sum() + 1.0) <= 1e-10
    parts, off, pieces = 3, 0, []
    for part in range(parts):
        sb, se = ff.partition_rows(nd, parts, part)
        ids = ff.select_elements(d, sb, se)
        sub = _elasticity_system(ff, ctx, n, 3 * sb, 3 * se, ids)
        pieces.append((sub[4][:-1] + off, sub[5], sub[6], sub[7]))
        off += sub[4][-1]
    rp_cat = np.concatenate([x[0] for x in pieces] + [np.array([off])])
    assert np.array_equal(rp_cat, rp) and np.array_equal(np.concatenate([x[1] for x in pieces]), ci)
    assert normwise(np.concatenate([x[2] for x in pieces]), val) <= TOL
    assert normwise(np.concatenate([x[3] for x in pieces]), rhs) <= TOL


def test_elasticity_zero_load_vector(ff, ctx):
    """A load vector that is identically zero in every component (f = 0): the
    element record stores no load-vector entry at all, the row kernels never
    load one, and the RHS comes out exactly zero; the matrix equals the atomic
    scatter's."""
    n = 8
    ctx.set_gather_classes(64)
    try:
        *_, val_a, rhs_a, f, m, p = _elasticity_system(ff, ctx, n, force=("0", "0", "0"), scatter="atomic")
        ctx.set_scatter("gather")
        val_g, rhs_g = ff.assemble(f, m, p)
        assert p.gather_info(m)["n_class_rows"] > 0
    finally:
        ctx.set_gather_classes(128)
    assert not rhs_g.any() and not rhs_a.any()
    assert normwise(val_g, val_a) <= 1e-15


def test_elasticity_class_gather_row_blocks(ff, ctx):
    """The vector class gather (lane-triple items of 10 node rows, CSR-order
    staging, TMA row write-out, short/long-row kernels) over 3 node-aligned row
    blocks with their halo elements: the concatenated blocks equal the 1-GPU
    system (SURVEY §8e for config 5), every block compared with the oracle."""
    n = 8
    ctx.set_gather_classes(32)
    try:
        c, v, d, nd, rp, ci, val, rhs, *_ = _elasticity_system(ff, ctx, n, lam="2", mu="0.5")
        parts, off, pieces = 3, 0, []
        for part in range(parts):
            sb, se = ff.partition_rows(nd, parts, part)
            ids = ff.select_elements(d, sb, se)
            sub = _elasticity_system(ff, ctx, n, 3 * sb, 3 * se, ids, lam="2", mu="0.5")
            assert sub[-1].gather_info(sub[-2])["n_class_rows"] > 0
            pieces.append((sub[4][:-1] + off, sub[5], sub[6], sub[7]))
            off += sub[4][-1]
    finally:
        ctx.set_gather_classes(128)
    rp_cat = np.concatenate([x[0] for x in pieces] + [np.array([off])])
    assert np.array_equal(rp_cat, rp) and np.array_equal(np.concatenate([x[1] for x in pieces]), ci)
    assert normwise(np.concatenate([x[2] for x in pieces]), val) <= TOL
    assert normwise(np.concatenate([x[3] for x in pieces]), rhs) <= TOL
    orp, oci = po.build_pattern(d, nd)
    vrp, vci = po.block_pattern(orp, oci, 3)
    ov, ob = po.assemble_elasticity(3, 2, 4, c, v, d, vrp, vci, lam=2.0, mu=0.5, force=(0.0, 0.0, -1.0))
    assert normwise(val, ov) <= TOL and normwise(rhs, ob) <= TOL


@pytest.mark.parametrize("deg", [1, 2])
@pytest.mark.parametrize("scatter", ["gather", "atomic"])
def test_elasticity_2d_matches_oracle(ff, ctx, deg, scatter):
    """2D vector elasticity (2 components: lane pairs in the class gather, the
    CSR-order staging at pitch = 2 mod 16) on a 48^2 unit square, P1 and P2,
    lambda != mu: block pattern bit-exact and values / RHS <= 1e-12 against
    the C restatement, through the class + generic row gather and the atomic
    scatter."""
    n = 48
    ctx.set_scatter(scatter)
    ctx.set_gather_classes(64)
    try:
        xy, v = ff.unit_square_mesh(n)
        if deg == 2:
            d, nd = ff.p2_dofs(2, v, xy.shape[0])
        else:
            d, nd = v, xy.shape[0]
        b, l = ff.elasticity_text(2, lam="2", mu="0.5", f=("1", "-1"))
        f = ff.Form.blocked(ctx, 2, deg, 2, b, l)
        m = ff.Mesh(ctx, 2, xy, v, d if deg == 2 else None, nd if deg == 2 else None, ncomp=2)
        p = ff.Pattern(ctx, m)
        rp, ci = p.export()
        val, rhs = ff.assemble(f, m, p)
        if scatter == "gather":
            assert p.gather_info(m)["n_class_rows"] > 0
    finally:
        ctx.set_gather_classes(128)
    orp, oci = po.build_pattern(d, nd)
    vrp, vci = po.block_pattern(orp, oci, 2)
    assert np.array_equal(rp, vrp) and np.array_equal(ci, vci)
    # the default 2D rule is the reference's 3-point rule (fem.cpp:43-48), quad id 3
    ov, ob = po.assemble_elasticity(2, deg, 3, xy, v, d, vrp, vci, lam=2.0, mu=0.5, force=(1.0, -1.0))
    assert normwise(val, ov) <= TOL and normwise(rhs, ob) <= TOL


def test_bench_two_ranks_on_one_gpu(ff):
    """The multi-rank bench path (row blocks, halo elements, global nnz, max
    over ranks) with 2 ranks sharing the one GPU over gloo: one JSON line, the
    whole-job nnz equal to the 1-rank pattern's."""
    import json
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FF_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29533", os.path.join(root, "bench.py"), "--gpus", "2", "--config", "c3",
           "--size", "16", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    n = 16
    # strong scaling (default): row blocks of the one 16^3 mesh
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["nnz"] == 230 * n ** 3 + 138 * n ** 2 + 24 * n + 1
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    # weak scaling: the 16^3 cell stacked twice, one slab per rank
    out = subprocess.run(cmd + ["--scaling", "weak"], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    from paper_1802_03433_b200 import rowblocks
    import pyoracle as po
    nnz = 0
    for r in range(2):
        c, v, dc, nd, rb, re, ne = rowblocks.weak_slab(ff, 3, 2, n, 2, r)
        nnz += int(po.build_pattern(dc, nd, rb, re)[0][-1])
    assert d["scaling"] == "weak" and d["config"]["elements"] == 2 * 6 * n ** 3 and d["config"]["nnz"] == nnz
    assert d["value"] > 0 and d["e2e"]["value"] > 0


@pytest.mark.parametrize("deg", [1, 2])
def test_jittered_permuted_mesh(ff, ctx, deg):
    """SURVEY §8d stress variant (seed 42, as test_device.cpp:219): interior
    vertices jittered by <= 0.1 h (orientation kept), elements randomly
    permuted (no element-order locality). Sparsity bit-exact, values <= 1e-12
    against the oracle, through the default row gather."""
    n = 10
    c, v = ff.kuhn_mesh(n)
    rng = np.random.default_rng(42)
    h = 1.0 / n
    interior = np.all((c > 1e-12) & (c < 1 - 1e-12), axis=1)
    c = c.copy()
    c[interior] += rng.uniform(-0.1 * h, 0.1 * h, size=(interior.sum(), 3))
    perm = rng.permutation(v.shape[0])
    v = np.ascontiguousarray(v[perm])
    d, nd = (v, c.shape[0]) if deg == 1 else ff.kuhn_p2_dofs(n, v)
    rp, ci, val, rhs, f, m, p = gpu_system(ff, ctx, 3, deg, "helmholtz", c, v, d, nd, quad=4, scatter="gather")
    assert p.scatter_for(f) == "gather"
    orp, oci = po.build_pattern(d, nd)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    ov, ob = po.assemble("helmholtz", 3, deg, 4, c, v, d, orp, oci, workers=8)
    assert normwise(val, ov) <= TOL and normwise(rhs, ob) <= TOL


@pytest.mark.parametrize("form,quad,gather_ok", [("poisson", 4, True), ("varcoef", 14, False)])
def test_auto_scatter_is_the_measured_faster_one(ff, ctx, form, quad, gather_ok):
    """North star (3): FF_SCATTER_AUTO_MODE times the row gather and the fp64
    RED scatter on the caller's buffers and keeps the faster; the assembly it
    leaves (and every later one) matches the oracle."""
    import torch
    n = 10
    c, v, d, nd = _mesh(ff, 3, 2, n)
    b, l = ff.named_form(form, 3)
    f = ff.Form(ctx, 3, 2, b, l, quad_rule=quad)
    m = ff.Mesh(ctx, 3, c, v, d, nd)
    p = ff.Pattern(ctx, m)
    ctx.set_scatter("auto")
    try:
        vals = torch.empty(p.nnz, dtype=torch.float64, device="cuda")
        rhs = torch.empty(p.n_rows, dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        t = p.calibrate_scatter(f, m, vals.data_ptr(), rhs.data_ptr(), s)
        assert t["atomic_ms"] > 0
        if gather_ok:
            assert t["gather_ms"] > 0
            assert t["chosen"] == ("gather" if t["gather_ms"] <= t["atomic_ms"] else "atomic")
        else:
            assert t["gather_ms"] is None and t["chosen"] == "atomic"
        assert p.scatter_for(f) == t["chosen"]
        orp, oci = po.build_pattern(d, nd)
        ov, ob = po.assemble(form, 3, 2, quad, c, v, d, orp, oci, workers=8)
        torch.cuda.synchronize()
        assert normwise(vals.cpu().numpy(), ov) <= TOL and normwise(rhs.cpu().numpy(), ob) <= TOL
        v2, b2 = ff.assemble(f, m, p)  # later calls run the choice
        assert normwise(v2, ov) <= TOL and normwise(b2, ob) <= TOL
    finally:
        ctx.set_scatter("gather")

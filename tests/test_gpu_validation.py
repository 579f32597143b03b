"""Mesh validation and connectivity re-upload through the C ABI.

The reference validates every mesh before flattening it and before building
its sparsity (fem.cpp:17-34, called from device.cpp:49 and :67): node index
out of range, duplicate node indices, non-positive signed area -- the lowest
failing element, in that check order, with its index in the message. The
engine runs the same checks on the device at ff_mesh_create, ff_mesh_update
(new connectivity), ff_pattern_build and when ff_assemble uploads connectivity
that differs from the resident one."""
import numpy as np
import pytest

import pyoracle as po
from conftest import normwise

pytestmark = pytest.mark.gpu


def _p1_2d(ff, n=4):
    xy, conn = ff.unit_square_mesh(n)
    return xy, conn.copy()


def test_out_of_range_node_is_reported_by_lowest_element(ff, ctx):
    xy, conn = _p1_2d(ff)
    conn[7, 1] = xy.shape[0]
    conn[3, 2] = -1
    with pytest.raises(ff.MeshError, match=r"^element 3: node index -1 out of range$"):
        ff.Mesh(ctx, 2, xy, conn)


def test_duplicate_nodes(ff, ctx):
    xy, conn = _p1_2d(ff)
    conn[5] = [conn[5, 0], conn[5, 0], conn[5, 2]]
    with pytest.raises(ff.MeshError, match=r"^element 5: duplicate node indices$"):
        ff.Mesh(ctx, 2, xy, conn)


def test_range_is_checked_before_duplicates_and_orientation(ff, ctx):
    xy, conn = _p1_2d(ff)
    conn[2] = conn[2, ::-1]                       # clockwise
    conn[2, 0] = 10 ** 6                          # and out of range: range wins
    with pytest.raises(ff.MeshError, match=r"^element 2: node index 1000000 out of range$"):
        ff.Mesh(ctx, 2, xy, conn)


def test_clockwise_triangle(ff, ctx):
    xy, conn = _p1_2d(ff)
    conn[11] = conn[11, [0, 2, 1]]
    with pytest.raises(ff.MeshError, match=r"^element 11: non-positive signed area$"):
        ff.Mesh(ctx, 2, xy, conn)


def test_negative_tet_and_bad_p2_dofs(ff, ctx):
    xyz, vc = ff.kuhn_mesh(3)
    dc, nd = ff.kuhn_p2_dofs(3, vc)
    bad = vc.copy()
    bad[17] = bad[17, [1, 0, 2, 3]]
    with pytest.raises(ff.MeshError, match=r"^element 17: non-positive signed volume$"):
        ff.Mesh(ctx, 3, xyz, bad, dc, nd)
    d2 = dc.copy()
    d2[4, 9] = nd
    with pytest.raises(ff.MeshError, match=rf"^element 4: DOF index {nd} out of range$"):
        ff.Mesh(ctx, 3, xyz, vc, d2, nd)
    d3 = dc.copy()
    d3[6, 8] = d3[6, 4]
    with pytest.raises(ff.MeshError, match=r"^element 6: duplicate DOF indices$"):
        ff.Mesh(ctx, 3, xyz, vc, d3, nd)
    ff.Mesh(ctx, 3, xyz, vc, dc, nd).close()      # the untouched mesh passes


def test_update_validates_new_connectivity_but_not_coordinates(ff, ctx):
    xy, conn = _p1_2d(ff)
    m = ff.Mesh(ctx, 2, xy, conn)
    bad = conn.copy()
    bad[9, 0] = -5
    with pytest.raises(ff.MeshError, match=r"^element 9: node index -5 out of range$"):
        m.update(vconn=bad)
    m.update(vconn=conn)
    # coordinates alone: the flattened arrays change under a validated mesh
    # (test_device.cpp:283-285); degenerate elements surface in assembly
    flat = xy.copy()
    flat[conn[0]] = [0.5, 0.5]
    m.update(coords=flat)


def test_pattern_build_validates(ff, ctx):
    xy, conn = _p1_2d(ff)
    m = ff.Mesh(ctx, 2, xy, conn)
    flat = xy.copy()
    flat[:, 1] = -flat[:, 1]                      # mirrored: every triangle clockwise
    m.update(coords=flat)
    with pytest.raises(ff.MeshError, match=r"^element 0: non-positive signed area$"):
        ff.Pattern(ctx, m)


@pytest.mark.parametrize("scatter", ["gather", "atomic"])
def test_update_then_reassemble_rederives_plans(ff, ctx, scatter):
    """assemble(Y), update(X), assemble, assemble(Y) again must
    give Y's system, not X's plans run over Y's connectivity."""
    ctx.set_scatter(scatter)
    n = 4
    xyz, vc = ff.kuhn_mesh(n)
    dc, nd = ff.kuhn_p2_dofs(n, vc)
    b, l = ff.named_form("poisson", 3)
    f = ff.Form(ctx, 3, 2, b, l)
    m = ff.Mesh(ctx, 3, xyz, vc, dc, nd)
    p = ff.Pattern(ctx, m)
    rp, ci = p.export()
    ov, ob = po.assemble("poisson", 3, 2, 4, xyz, vc, dc, rp, ci)
    # X: the same elements listed in another order (same sparsity)
    perm = np.random.default_rng(3).permutation(vc.shape[0])
    vx, dx = np.ascontiguousarray(vc[perm]), np.ascontiguousarray(dc[perm])
    v1, b1 = ff.assemble(f, m, p, vconn=vc, dconn=dc)
    m.update(vconn=vx, dconn=dx)
    v2, b2 = ff.assemble(f, m, p)
    v3, b3 = ff.assemble(f, m, p, vconn=vc, dconn=dc)
    for v, bb in ((v1, b1), (v2, b2), (v3, b3)):
        assert normwise(v, ov) <= 1e-12 and normwise(bb, ob) <= 1e-12


def test_e2e_upload_of_invalid_connectivity_is_rejected(ff, ctx):
    ctx.set_scatter("gather")
    xy, conn = _p1_2d(ff)
    b, l = ff.named_form("poisson", 2)
    f = ff.Form(ctx, 2, 1, b, l)
    m = ff.Mesh(ctx, 2, xy, conn)
    p = ff.Pattern(ctx, m)
    good_v, good_b = ff.assemble(f, m, p)
    bad = conn.copy()
    bad[12, 2] = bad[12, 1]
    with pytest.raises(ff.MeshError, match=r"^element 12: duplicate node indices$"):
        ff.assemble(f, m, p, vconn=bad)
    v, bb = ff.assemble(f, m, p, vconn=conn)
    assert np.array_equal(v, good_v) and np.array_equal(bb, good_b)


def test_python_boundary_checks_dtype_and_size(ff, ctx):
    xy, conn = _p1_2d(ff)
    b, l = ff.named_form("poisson", 2)
    f = ff.Form(ctx, 2, 1, b, l)
    m = ff.Mesh(ctx, 2, xy, conn)
    p = ff.Pattern(ctx, m)
    v0, b0 = ff.assemble(f, m, p)
    v1, b1 = ff.assemble(f, m, p, vconn=conn.astype(np.int64))   # coerced, not misread
    assert np.array_equal(v0, v1) and np.array_equal(b0, b1)
    with pytest.raises(ValueError):
        ff.assemble(f, m, p, vconn=conn[:-1])
    with pytest.raises(ValueError):
        ff.assemble(f, m, p, values=np.empty(p.nnz, np.float32))
    with pytest.raises(ValueError):
        ff.assemble(f, m, p, rhs=np.empty(p.n_rows - 1))


def test_pattern_of_scalar_mesh_rejected_for_vector_form(ff, ctx):
    xyz, vc = ff.kuhn_mesh(2)
    dc, nd = ff.kuhn_p2_dofs(2, vc)
    bl, ll = ff.elasticity_text(3)
    f = ff.Form.blocked(ctx, 3, 2, 3, bl, ll, quad_rule=4)
    m = ff.Mesh(ctx, 3, xyz, vc, dc, nd)
    p = ff.Pattern(ctx, m)                          # built before the components are set
    m2 = ff.Mesh(ctx, 3, xyz, vc, dc, nd, ncomp=3)
    with pytest.raises(ff.DeviceError, match="components per node"):
        ff.assemble(f, m2, p)


def test_reference_side_binding_matches_reference_assemble_sparse():
    """INTEGRATION.md §2 compiled for real (oracle/_ref/test_integration: the
    unmodified reference objects + the documented binding + libfemforge_b200.so):
    assemble_sparse_b200 == the reference's assemble_sparse on 2D n=64 (demo
    Helmholtz and Poisson): identical ELL columns, values/RHS <= 1e-12."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "oracle", "_ref", "test_integration")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/test_integration not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert r.stdout.count("-> ok") == 2 and "integration ok" in r.stdout

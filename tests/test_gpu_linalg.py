"""Downstream consumer of the assembled system on the GPU:
SpMV against scipy, CG against the reference's own cg_solve (oracle/_ref),
and the reference's criterion 5 (acceptance.cpp:201-223): L2 convergence
order >= 1.9 on the manufactured cosine problem, assembled and solved on the
device."""
import math

import numpy as np
import pytest

import pyoracle as po
from conftest import normwise

pytestmark = pytest.mark.gpu


def _system(ff, ctx, bil, lin, n):
    xy, conn = ff.unit_square_mesh(n)
    f = ff.Form(ctx, 2, 1, bil, lin, quad_rule=3)
    m = ff.Mesh(ctx, 2, xy, conn)
    p = ff.Pattern(ctx, m)
    v, b = ff.assemble(f, m, p)
    return xy, conn, f, m, p, v, b


@pytest.mark.parametrize("dim,deg,n", [(2, 1, 32), (3, 2, 6)])
def test_spmv_matches_scipy(ff, ctx, dim, deg, n):
    import scipy.sparse as sp
    import torch
    if dim == 2:
        c, v = ff.unit_square_mesh(n)
        d, nd = v, c.shape[0]
    else:
        c, v = ff.kuhn_mesh(n)
        d, nd = ff.kuhn_p2_dofs(n, v)
    bil, lin = ff.named_form("helmholtz", dim)
    f = ff.Form(ctx, dim, deg, bil, lin)
    m = ff.Mesh(ctx, dim, c, v, None if deg == 1 else d, nd)
    p = ff.Pattern(ctx, m)
    vals, _ = ff.assemble(f, m, p)
    rp, ci = p.export()
    x = np.random.default_rng(7).standard_normal(p.n_rows)
    dv, dx = torch.from_numpy(vals).cuda(), torch.from_numpy(x).cuda()
    dy = torch.empty_like(dx)
    ff.spmv(p, dv.data_ptr(), dx.data_ptr(), dy.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    want = sp.csr_matrix((vals, ci, rp), shape=(p.n_rows, p.n_rows)) @ x
    assert normwise(dy.cpu().numpy(), want) <= 1e-14


@pytest.mark.skipif(not po.ref_available(), reason="needs oracle/_ref")
def test_cg_matches_reference_cg(ff, ctx):
    """GPU CG == the reference's cg_solve (linalg.cpp:61-96) on the same SPD
    system (2D Helmholtz, n=32): same stopping rule, same solution."""
    import torch
    bil, lin = ff.named_form("helmholtz", 2)
    xy, conn, f, m, p, v, b = _system(ff, ctx, bil, lin, 32)
    dv, db = torch.from_numpy(v).cuda(), torch.from_numpy(b).cuda()
    dx = torch.empty_like(db)
    res = ff.cg_solve(p, dv.data_ptr(), db.data_ptr(), dx.data_ptr(), tol=1e-10)
    assert res["converged"] and res["residual"] <= 1e-10
    h = po.RefHarness(2, 1, xy, conn, conn, xy.shape[0], "helmholtz")
    xr, itr, resr, conv = h.cg(v, b, 1e-10, 10000)
    assert conv and abs(res["iterations"] - itr) <= 2
    assert normwise(dx.cpu().numpy(), xr) <= 1e-8


def test_criterion5_convergence_order(ff, ctx):
    """acceptance.cpp:201-223 on the GPU: -lap u + u = (2 pi^2 + 1) cos(pi x)
    cos(pi y) (natural BCs), P1 on 16/32/64, CG to 1e-10; L2 errors with the
    reference's 3-point rule (linalg.cpp:101-127) must drop with order >= 1.9."""
    import torch
    pi = math.pi
    bil = "u_x*v_x + u_y*v_y + 1*u*v"
    lin = f"({2 * pi * pi + 1!r})*cos({pi!r}*x)*cos({pi!r}*y)*v"
    qp = np.array([[1 / 6, 1 / 6], [2 / 3, 1 / 6], [1 / 6, 2 / 3]])
    errs = []
    for n in (16, 32, 64):
        xy, conn, f, m, p, v, b = _system(ff, ctx, bil, lin, n)
        dv, db = torch.from_numpy(v).cuda(), torch.from_numpy(b).cuda()
        dx = torch.empty_like(db)
        res = ff.cg_solve(p, dv.data_ptr(), db.data_ptr(), dx.data_ptr(), tol=1e-10, max_iter=10000)
        assert res["converged"]
        x = dx.cpu().numpy()
        p0, p1, p2 = xy[conn[:, 0]], xy[conn[:, 1]], xy[conn[:, 2]]
        det = (p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1]) - (p2[:, 0] - p0[:, 0]) * (p1[:, 1] - p0[:, 1])
        tot = 0.0
        for xi, eta in qp:
            px = p0 + (p1 - p0) * xi + (p2 - p0) * eta
            uh = (1 - xi - eta) * x[conn[:, 0]] + xi * x[conn[:, 1]] + eta * x[conn[:, 2]]
            d = uh - np.cos(pi * px[:, 0]) * np.cos(pi * px[:, 1])
            tot += np.sum(d * d * det) / 6.0
        errs.append(math.sqrt(tot))
    o1, o2 = math.log2(errs[0] / errs[1]), math.log2(errs[1] / errs[2])
    assert o1 >= 1.9 and o2 >= 1.9, (errs, o1, o2)

"""Full-size parity gates: every BASELINE.json configuration at its stated
size, the GPU system (through the C ABI) against the CPU oracle -- or, for the
2D config, against the reference library itself (oracle/_ref). Sparsity
bit-exact; values / RHS <= 1e-12 normwise (acceptance.cpp:58-67, the
north-star gate "3D P2 Poisson with >= 10M tets").

  NS  3D P2 Poisson, Kuhn 128^3 (12.58M tets, 485M nnz)  vs fo_build_pattern / fo_assemble
  C1  2D P1 512^2, Poisson + the demo Helmholtz form     vs the reference's assemble_sparse (par mode)
  C2  3D P1 Poisson, Kuhn 128^3                          vs the oracle
  C3  3D P2 Poisson, Kuhn 96^3                           vs the oracle
  C4  3D P2 var-coef, Kuhn 96^3, 14-point rule           vs the oracle
  C5  vector P2 elasticity, Kuhn 160^3 (8.5e9 nnz)       rows whose CSR offsets pass 2^31 and 2^32
                                                         vs fo_assemble_elasticity on those rows;
                                                         rigid-body modes of the whole system via ff_spmv
  rows NS in 8 row blocks (halo elements duplicated) concatenated == the 1-GPU CSR
"""
import os

import numpy as np
import pytest

import pyoracle as po
from conftest import normwise

pytestmark = pytest.mark.gpu
TOL = 1e-12
WORKERS = os.cpu_count() or 1


def _kuhn(ff, n, deg):
    c, v = ff.kuhn_mesh(n)
    d, nd = (v, c.shape[0]) if deg == 1 else ff.kuhn_p2_dofs(n, v)
    return c, v, d, nd


def _system(ff, ctx, dim, deg, form, c, v, d, nd, quad):
    ctx.set_scatter("gather")
    b, l = ff.named_form(form, dim)
    f = ff.Form(ctx, dim, deg, b, l, quad_rule=quad)
    m = ff.Mesh(ctx, dim, c, v, None if deg == 1 else d, nd)
    p = ff.Pattern(ctx, m)
    return f, m, p


def _check_vs_oracle(ff, ctx, dim, deg, form, n, quad, expect_scatter):
    c, v, d, nd = _kuhn(ff, n, deg)
    f, m, p = _system(ff, ctx, dim, deg, form, c, v, d, nd, quad)
    assert p.scatter_for(f) == expect_scatter
    rp, ci = p.export()
    orp, oci = po.build_pattern(d, nd)
    assert np.array_equal(rp, orp), "row_ptr differs from the oracle"
    assert np.array_equal(ci, oci), "col_idx differs from the oracle"
    del ci
    val, rhs = ff.assemble(f, m, p)
    ov, ob = po.assemble(form, dim, deg, quad, c, v, d, orp, oci, workers=WORKERS)
    ev, eb = normwise(val, ov), normwise(rhs, ob)
    assert ev <= TOL and eb <= TOL, (ev, eb)
    return f, m, p


def test_ns_p2_poisson_128_full_system_vs_oracle(ff, ctx):
    """The north-star gate: 12,582,912 tets, 16,974,593 DOFs, 484,609,025 nnz;
    the default row gather (class kernels + generic rows) at full size."""
    f, m, p = _check_vs_oracle(ff, ctx, 3, 2, "poisson", 128, 4, "gather")
    gi = p.gather_info(m)
    assert p.nnz == 484_609_025 and gi["n_classes"] >= 8 and gi["n_class_rows"] > p.n_rows // 2


def test_c2_p1_poisson_128_vs_oracle(ff, ctx):
    _check_vs_oracle(ff, ctx, 3, 1, "poisson", 128, 4, "gather")


def test_c3_p2_poisson_96_vs_oracle(ff, ctx):
    _check_vs_oracle(ff, ctx, 3, 2, "poisson", 96, 4, "gather")


def test_c4_varcoef_96_q14_vs_oracle(ff, ctx):
    c, v, d, nd = _kuhn(ff, 96, 2)
    f, m, p = _system(ff, ctx, 3, 2, "varcoef", c, v, d, nd, 14)
    rp, ci = p.export()
    orp, oci = po.build_pattern(d, nd)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    del ci
    val, rhs = ff.assemble(f, m, p)
    ov, ob = po.assemble("varcoef", 3, 2, 14, c, v, d, orp, oci, workers=WORKERS)
    assert normwise(val, ov) <= TOL and normwise(rhs, ob) <= TOL


@pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref (the reference library) not built")
@pytest.mark.parametrize("form", ["poisson", "demo2d"])
def test_c1_512_vs_reference_library(ff, ctx, form):
    """Config 1 against the UNMODIFIED reference (build_sparsity +
    assemble_sparse(CompiledEvaluator) in parallel mode on every host thread,
    device.cpp:66-88, 265-305): ELL -> CSR pattern bit-exact, values and RHS
    <= 1e-12 normwise (par-mode atomic order differs run to run)."""
    xy, conn = ff.unit_square_mesh(512)
    h = po.RefHarness(2, 1, xy, conn, conn, xy.shape[0], form)
    hrp, hci = h.pattern()
    hv, hb = h.assemble(workers=WORKERS)
    f, m, p = _system(ff, ctx, 2, 1, form, xy, conn, conn, xy.shape[0], 3)
    rp, ci = p.export()
    assert p.n_rows == 263_169 and p.nnz == 1_838_081
    assert np.array_equal(rp, hrp) and np.array_equal(ci, hci)
    val, rhs = ff.assemble(f, m, p)
    assert normwise(val, hv) <= TOL and normwise(rhs, hb) <= TOL


def test_ns_row_blocks_concatenate_to_full_system(ff, ctx):
    """SURVEY §8e at the north-star size: 8 contiguous DOF row blocks, each
    assembled from its owned + halo elements (what one rank of `bench.py
    --gpus 8` does), concatenate to the 1-GPU CSR; values equal to 1e-12."""
    from paper_1802_03433_b200 import rowblocks
    n = 128
    c, v, d, nd = _kuhn(ff, n, 2)
    f, m, p = _system(ff, ctx, 3, 2, "poisson", c, v, d, nd, 4)
    rp, ci = p.export()
    val, rhs = ff.assemble(f, m, p)
    scale_v, scale_b = np.abs(val).max(), np.abs(rhs).max()
    world = 8
    for r in range(world):
        rb, re = rowblocks.row_block(nd, world, r)
        ids = rowblocks.local_elements(d, rb, re)
        vl, dl = np.ascontiguousarray(v[ids]), np.ascontiguousarray(d[ids])
        ml = ff.Mesh(ctx, 3, c, vl, dl, nd)
        pl = ff.Pattern(ctx, ml, rb, re)
        lrp, lci = pl.export()
        assert np.array_equal(lrp + rp[rb], rp[rb:re + 1]), f"row_ptr of block {r}"
        assert np.array_equal(lci, ci[rp[rb]:rp[re]]), f"col_idx of block {r}"
        lv, lb = ff.assemble(f, ml, pl)
        assert np.abs(lv - val[rp[rb]:rp[re]]).max() <= TOL * scale_v
        assert np.abs(lb - rhs[rb:re]).max() <= TOL * scale_b
        pl.close()
        ml.close()


class _DevArray:
    """A device allocation owned by the library, seen by torch (no copy)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def test_c5_elasticity_160_offsets_past_2_31_vs_oracle(ff, ctx):
    """Config 5 on one B200 (99.2M DOFs, 8.51e9 nnz: int64 row_ptr). Rows
    whose CSR offsets straddle 2^31 and 2^32, and the last rows, are compared
    with the C restatement restricted to those rows (fo_assemble_elasticity
    takes row_begin/row_end); the whole system is checked for the six
    rigid-body modes (K u = 0) through ff_spmv, and sum(rhs_z) = -|Omega|."""
    import torch
    n = 160
    c, v, d, nd = _kuhn(ff, n, 2)
    ctx.set_scatter("gather")
    bb, bl = ff.elasticity_text(3)
    f = ff.Form.blocked(ctx, 3, 2, 3, bb, bl, quad_rule=4)
    m = ff.Mesh(ctx, 3, c, v, d, nd, ncomp=3)
    p = ff.Pattern(ctx, m)
    N = 3 * nd
    assert p.n_rows == N and p.nnz == 8_510_549_769
    vals = torch.empty(p.nnz, dtype=torch.float64, device="cuda")
    rhs = torch.empty(N, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ff.assemble_device(f, m, p, vals.data_ptr(), rhs.data_ptr(), s)
    torch.cuda.synchronize()
    ctx.check()
    rpp, cip = p.device_pointers()
    rp = torch.as_tensor(_DevArray(rpp, N + 1, "<i8"), device="cuda")
    ci = torch.as_tensor(_DevArray(cip, p.nnz, "<i4"), device="cuda")
    assert int(rp[-1]) == p.nnz
    chunk = 1 << 28   # no 68 GB temporaries
    scale = max(float(vals[i:i + chunk].abs().max()) for i in range(0, p.nnz, chunk))

    # rows past 2^31 / 2^32 and the last rows, against the oracle
    rph = rp.cpu().numpy()
    blocks = []
    for off in (2 ** 31, 2 ** 32, p.nnz - 1):
        row = int(np.searchsorted(rph, off, side="right")) - 1
        node = row // 3
        blocks.append((max(node - 150, 0), min(node + 150, nd)))
    for nb, ne in blocks:
        orp, oci = po.build_pattern(d, nd, nb, ne)
        vrp, vci = po.block_pattern(orp, oci, 3)
        ids = ff.select_elements(d, nb, ne)
        ov, ob = po.assemble_elasticity(3, 2, 4, c, v[ids], d[ids], vrp, vci, row_begin=3 * nb, row_end=3 * ne)
        r0, r1 = 3 * nb, 3 * ne
        lo, hi = int(rph[r0]), int(rph[r1])
        assert hi - lo == vrp[-1] and np.array_equal(rph[r0:r1 + 1] - lo, vrp)
        assert np.array_equal(ci[lo:hi].cpu().numpy(), vci)
        assert normwise(vals[lo:hi].cpu().numpy(), ov) <= TOL
        assert normwise(rhs[r0:r1].cpu().numpy(), ob) <= TOL
    assert any(int(rph[3 * nb]) < 2 ** 31 < int(rph[3 * ne]) for nb, ne in blocks)
    assert any(int(rph[3 * nb]) < 2 ** 32 < int(rph[3 * ne]) for nb, ne in blocks)

    # the whole system: rigid-body modes and the load
    L = 2 * n + 1
    idx = torch.arange(nd, device="cuda", dtype=torch.float64)
    X = torch.stack([idx % L, torch.div(idx, L, rounding_mode="floor") % L,
                     torch.div(idx, L * L, rounding_mode="floor")], 1) / (L - 1)
    y = torch.empty(N, dtype=torch.float64, device="cuda")
    modes = []
    for t in range(3):
        u = torch.zeros(N, dtype=torch.float64, device="cuda")
        u[t::3] = 1.0
        modes.append(u)
    for a, b in [(0, 1), (1, 2), (0, 2)]:
        u = torch.zeros(N, dtype=torch.float64, device="cuda")
        u[a::3] = -X[:, b]
        u[b::3] = X[:, a]
        modes.append(u)
    for u in modes:
        ff.spmv(p, vals.data_ptr(), u.data_ptr(), y.data_ptr(), s)
        torch.cuda.synchronize()
        assert float(y.abs().max()) <= 1e-11 * scale
    assert abs(float(rhs[2::3].sum()) + 1.0) <= 1e-9
    assert abs(float(rhs[0::3].sum())) <= 1e-9

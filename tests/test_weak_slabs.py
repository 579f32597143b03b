"""Weak-scaling slabs (bench.py --gpus N --scaling weak): rank r of W meshes the r-th
cell of a box stacked W cells high, exactly as the library meshes one cell.
Host logic only (CPU): the 1-rank slab is the library mesh itself, and the
ranks' owned rows together are the pattern of the whole box, checked against
an independent construction (the same box cut out of a larger Kuhn cube /
unit square)."""
import numpy as np
import pytest

import pyoracle as po


@pytest.fixture(scope="module")
def ff():
    import paper_1802_03433_b200.femforge as ff
    ff.lib()
    return ff


@pytest.mark.parametrize("dim,deg", [(2, 1), (3, 1), (3, 2)])
def test_one_rank_slab_is_the_library_mesh(ff, dim, deg):
    from paper_1802_03433_b200 import rowblocks
    n = 4
    c, v, d, nd, rb, re, ne = rowblocks.weak_slab(ff, dim, deg, n, 1, 0)
    if dim == 3:
        C, V = ff.kuhn_mesh(n)
        D, ND = (V, C.shape[0]) if deg == 1 else ff.kuhn_p2_dofs(n, V)
    else:
        C, V = ff.unit_square_mesh(n)
        D, ND = V, C.shape[0]
    assert np.array_equal(v, V) and np.allclose(c, C) and nd == ND and (rb, re) == (0, ND) and ne == V.shape[0]
    assert np.array_equal(v if d is None else d, D)


@pytest.mark.parametrize("dim,deg", [(2, 1), (3, 1), (3, 2)])
def test_stacked_slabs_are_the_box(ff, dim, deg):
    from paper_1802_03433_b200 import rowblocks
    n, W = 3, 3
    M = n * W
    if dim == 3:
        C, V = ff.kuhn_mesh(M)
        D = V if deg == 1 else ff.kuhn_p2_dofs(M, V)[0]
    else:
        C, V = ff.unit_square_mesh(M)
        D = V
    inside = np.all(C[V].mean(1)[:, :dim - 1] < n / M, axis=1)   # the n x .. x M box
    u, inv = np.unique(D[inside], return_inverse=True)
    rp, _ = po.build_pattern(inv.reshape(-1, D.shape[1]).astype(np.int32), len(u))
    nnz, rows, elems = 0, 0, 0
    for r in range(W):
        c, v, d, nd, rb, re, ne = rowblocks.weak_slab(ff, dim, deg, n, W, r)
        assert v.max() < c.shape[0] and ne == inside.sum()
        # every owned row is covered by the slab's elements
        dd = v if d is None else d
        assert np.isin(np.arange(rb, re), dd).all()
        prp, _ = po.build_pattern(dd, nd, rb, re)
        nnz += int(prp[-1])
        rows += re - rb
    assert rows == len(u) and nnz == int(rp[-1])

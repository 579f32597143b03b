"""World-size-2 row-block path on CPU (gloo): the host logic of the multi-GPU
flow (partition, owned + halo element selection, global row/nnz offsets,
block gather) with each rank's block computed by the CPU oracle. The
concatenation must equal the single-rank system: sparsity bit-exact, values
and RHS <= 1e-12 normwise."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import pyoracle as po
from conftest import normwise


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_dir):
    import torch.distributed as dist

    from paper_1802_03433_b200 import rowblocks

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dim, deg, form, n, quad = case
        if dim == 2:
            c, v = po.unit_square_mesh(n)
            d, nd = v, c.shape[0]
        else:
            c, v = po.kuhn_mesh(n)
            d, nd = (v, c.shape[0]) if deg == 1 else po.p2_dofs_kuhn(n, v)
        rb, re = rowblocks.row_block(nd, world, rank)
        ids = rowblocks.local_elements(d, rb, re)
        vl, dl = np.ascontiguousarray(v[ids]), np.ascontiguousarray(d[ids])
        rp, ci = po.build_pattern(dl, nd, rb, re)
        vals, rhs = po.assemble(form, dim, deg, quad, c, vl, dl, rp, ci, row_begin=rb, row_end=re)
        r0, z0, n_tot, nnz_tot = rowblocks.global_offsets(int(rp[-1]), re - rb)
        assert r0 == rb and n_tot == nd
        full = rowblocks.gather_csr(rp, ci, vals, rhs)
        if rank == 0:
            np.savez(os.path.join(out_dir, "cat.npz"), row_ptr=full[0], col_idx=full[1], values=full[2],
                     rhs=full[3], nnz_tot=nnz_tot)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [(3, 2, "poisson", 4, 4), (3, 1, "helmholtz", 5, 4), (2, 1, "demo2d", 16, 3)])
def test_two_rank_row_blocks_equal_single_rank(case, tmp_path):
    import paper_1802_03433_b200.femforge as ff
    ff.lib()  # host helpers of the C ABI (no GPU needed)
    mp.start_processes(_worker, args=(2, _free_port(), case, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(tmp_path / "cat.npz")
    dim, deg, form, n, quad = case
    if dim == 2:
        c, v = po.unit_square_mesh(n)
        d, nd = v, c.shape[0]
    else:
        c, v = po.kuhn_mesh(n)
        d, nd = (v, c.shape[0]) if deg == 1 else po.p2_dofs_kuhn(n, v)
    rp, ci = po.build_pattern(d, nd)
    vals, rhs = po.assemble(form, dim, deg, quad, c, v, d, rp, ci)
    assert int(got["nnz_tot"]) == int(rp[-1])
    assert np.array_equal(got["row_ptr"], rp) and np.array_equal(got["col_idx"], ci)
    assert normwise(got["values"], vals) <= 1e-12
    assert normwise(got["rhs"], rhs) <= 1e-12

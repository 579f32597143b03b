"""Multi-GPU row blocks: one process per GPU, contiguous DOF
row blocks, halo elements duplicated, no collective on the data path.

Host logic only -- the partition and halo selection are the C ABI helpers
(``ff_partition_rows``, ``ff_select_elements``); ``torch.distributed`` is
used for the global CSR row offsets (an exclusive prefix over the per-rank
nnz, the "host prefix sum over 8 integers" of §8e) and for gathering blocks
on one rank for validation. The reference has no distributed path
(SPEC.md:504); these helpers are what a caller of ``assemble_sparse`` would
run per rank.
"""
from __future__ import annotations

import numpy as np

from . import femforge as ff


def row_block(n_dofs, world, rank):
    """[row_begin, row_end) owned by `rank` (balanced by DOF count)."""
    return ff.partition_rows(n_dofs, world, rank)


def local_elements(dconn, row_begin, row_end):
    """Ids of the elements with at least one DOF in the block (owned + halo)."""
    return ff.select_elements(dconn, row_begin, row_end)


def _all_gather_i64(values, group=None):
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(values, dtype=torch.int64, device=dev)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return np.stack([o.cpu().numpy() for o in out])


def global_offsets(local_nnz, local_rows, group=None):
    """(row offset, nnz offset, total rows, total nnz) of this rank's block in
    the global CSR: exclusive prefix sums over the ranks' (rows, nnz)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    allv = _all_gather_i64([local_rows, local_nnz], group)
    rows, nnz = allv[:, 0], allv[:, 1]
    return int(rows[:rank].sum()), int(nnz[:rank].sum()), int(rows.sum()), int(nnz.sum())


def gather_csr(row_ptr, col_idx, values, rhs, group=None, dst=0):
    """Concatenates the ranks' CSR blocks on rank `dst` (validation / export
    only; not on the hot path). Returns (row_ptr, col_idx, values, rhs) on
    `dst`, None elsewhere."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n_rows = len(row_ptr) - 1
    nnz = int(row_ptr[-1])
    r0, z0, n_tot, nnz_tot = global_offsets(nnz, n_rows, group)
    sizes = _all_gather_i64([n_rows, nnz], group)

    def cat(local, count_col, dtype):
        # gather needs equal sizes: pad every block to the largest, trim on dst
        cap = int(sizes[:, count_col].max())
        buf = np.zeros(cap, dtype)
        buf[: len(local)] = local
        t = torch.from_numpy(buf)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        if rank == dst:
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.gather(t, parts, dst=dst, group=group)
            return np.concatenate([parts[r].cpu().numpy()[: int(sizes[r, count_col])] for r in range(world)])
        dist.gather(t, None, dst=dst, group=group)
        return None

    rp = cat(np.asarray(row_ptr[:-1]) + z0, 0, np.int64)
    ci = cat(col_idx, 1, np.int32)
    va = cat(values, 1, np.float64)
    rh = cat(rhs, 0, np.float64)
    if rank != dst:
        return None
    return np.concatenate([rp, np.array([nnz_tot], np.int64)]), ci, va, rh

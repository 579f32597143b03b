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


# ---- weak scaling: a stack of `world` unit cells (squares / cubes) -----------
#
# Rank r of W owns the r-th n x n (x n) cell of a box [0,1]^(d-1) x [0,W] meshed
# exactly as the library's unit-square / Kuhn-cube meshes (the same per-cell
# subdivision, vertex and P2 DOF numbering, stacked along the last axis), so
# its work is that of the single-GPU workload whatever W is. Each rank builds
# only its slab: its cells plus one halo layer below (the elements touching
# its lowest row layer); rows are the DOF lattice layers it owns.

def _cell_pattern(ff, dim, degree):
    if dim == 2:
        c1, v1 = ff.unit_square_mesh(1)
        d1 = v1 if degree == 1 else ff.p2_dofs(2, v1, c1.shape[0])[0]
    else:
        c1, v1 = ff.kuhn_mesh(1)
        d1 = v1 if degree == 1 else ff.kuhn_p2_dofs(1, v1)[0]
    lat = np.rint(c1).astype(np.int64)  # vertex lattice coordinates of the unit cell
    if degree == 1:
        dl = lat[d1]
    else:  # node lattice coordinates on the refined (x2) lattice, 3 points per axis
        dl = np.stack([(d1 // 3 ** a) % 3 for a in range(dim)], -1)
    return lat[v1], dl


def weak_slab(ff, dim, degree, n, world, rank):
    """(coords, vconn, dconn, n_dofs, row_begin, row_end, n_elems_global) of
    rank `rank`'s slab of the stacked box, numbered locally (vertices and
    DOFs from the slab's lowest layer; the global ids are these plus a
    per-rank constant, so the CSR block is the global one shifted). dconn is
    None for P1, whose DOFs are the vertices."""
    if degree == 2 and dim == 2:
        raise ValueError("weak slabs: P2 in 3D only (BASELINE configs)")
    vpat, dpat = _cell_pattern(ff, dim, degree)
    z0 = max(0, n * rank - 1)                 # one halo cell layer below
    z1 = n * (rank + 1)
    nz = z1 - z0
    axes = [np.arange(n)] * (dim - 1) + [np.arange(nz)]
    grid = np.meshgrid(*axes, indexing="ij")
    cell = np.stack([g.ravel(order="F") for g in grid], -1)   # first axis fastest
    N1 = n + 1
    vx = cell[:, None, None, :] + vpat[None]
    vid = vx[..., 0] + N1 * vx[..., 1] if dim == 2 else vx[..., 0] + N1 * (vx[..., 1] + N1 * vx[..., 2])
    vconn = vid.reshape(-1, dim + 1).astype(np.int32)
    lay = [np.arange(N1)] * (dim - 1) + [np.arange(nz + 1)]
    lg = np.meshgrid(*lay[::-1], indexing="ij")[::-1]          # last axis slowest
    coords = np.stack([g.ravel() for g in lg], -1).astype(np.float64)
    coords[:, -1] += z0
    coords /= n
    if degree == 1:
        L, f, dconn = N1, 1, None
    else:
        L, f = 2 * n + 1, 2
        px = f * cell[:, None, None, :] + dpat[None]
        dconn = (px[..., 0] + L * (px[..., 1] + L * px[..., 2])).reshape(-1, dpat.shape[1]).astype(np.int32)
    plane = L ** (dim - 1)                                     # DOFs per lattice layer
    n_dofs = plane * (f * nz + 1)
    rb = plane * f * (n * rank - z0)
    re = n_dofs if rank == world - 1 else plane * f * (n * (rank + 1) - z0)
    return coords, vconn, dconn, n_dofs, rb, re, n ** (dim - 1) * n * world * vpat.shape[0]

"""One-process-per-GPU partitioning of the PENCIL nests, over torch.distributed
(NCCL on B200s, gloo for the CPU tests).  The data path per step:

  * CSR SpMV / gemv — row blocks balanced by non-zeros (pencil_shard_rows_by_nnz).  Each rank owns
    rows [r0, r1) of A and the same slice of x; a step all-gathers x (one NCCL all_gather into a
    rank-padded buffer) and runs the local SpMV.  Column indices are remapped once, at setup,
    into the padded layout (col -> owner*max_rows + col - bounds[owner]) so no unpad copy runs
    per step.
  * 5x5 stencils — equal row bands; each rank exchanges 2 halo rows with each neighbour
    (send/recv) and runs the stencil on its band extended by the halos.

The local compute is a callable so the same plumbing is exercised on CPU (gloo + the oracle)
and on GPUs (NCCL + the CUDA kernels).
"""
import ctypes

import numpy as np

from . import _lib


def shard_rows_by_nnz(rowptr, nshards):
    lib = _lib.load()
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int32)
    bounds = np.zeros(nshards + 1, dtype=np.int32)
    st = lib.pencil_shard_rows_by_nnz(rowptr.ctypes.data, rowptr.size - 1, nshards, bounds.ctypes.data)
    if st:
        raise ValueError("pencil_shard_rows_by_nnz failed")
    return bounds


def shard_bands(h, nshards):
    lib = _lib.load()
    bounds = np.zeros(nshards + 1, dtype=np.int32)
    if lib.pencil_shard_bands(h, nshards, bounds.ctypes.data):
        raise ValueError("pencil_shard_bands failed")
    return bounds


def shard_gemm_grid(m, n, nshards):
    lib = _lib.load()
    r, c = ctypes.c_int(), ctypes.c_int()
    if lib.pencil_shard_gemm_grid(m, n, nshards, ctypes.byref(r), ctypes.byref(c)):
        raise ValueError("pencil_shard_gemm_grid failed")
    return r.value, c.value


class RowShardedCsr:
    """Local piece of a row-sharded square CSR matrix plus the x all-gather plumbing."""

    def __init__(self, rowptr, col, val, rank, world, bounds=None):
        self.rank, self.world = rank, world
        self.bounds = shard_rows_by_nnz(rowptr, world) if bounds is None else np.asarray(bounds, np.int32)
        r0, r1 = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.r0, self.r1 = r0, r1
        self.max_rows = int(np.max(self.bounds[1:] - self.bounds[:-1]))
        p0, p1 = int(rowptr[r0]), int(rowptr[r1])
        self.rowptr = (rowptr[r0:r1 + 1] - p0).astype(np.int32)
        c = col[p0:p1].astype(np.int64)
        owner = np.searchsorted(self.bounds, c, side="right") - 1
        self.col = (owner * self.max_rows + (c - self.bounds[owner])).astype(np.int32)
        self.val = val[p0:p1]
        self.nrows, self.nnz = r1 - r0, p1 - p0
        self.ncols_padded = self.max_rows * world

    def pad_local_x(self, x_local, like=None):
        """x_local (this rank's rows) into a max_rows buffer for the all-gather."""
        import torch
        buf = torch.zeros(self.max_rows, dtype=torch.float32, device=x_local.device)
        buf[: x_local.numel()] = x_local
        return buf

    def allgather_x(self, x_local_padded, out=None):
        import torch
        import torch.distributed as dist
        if out is None:
            out = torch.empty(self.ncols_padded, dtype=torch.float32, device=x_local_padded.device)
        if dist.get_backend() == "nccl":
            dist.all_gather_into_tensor(out, x_local_padded)
        else:  # gloo (CPU tests): list form
            dist.all_gather(list(out.view(self.world, self.max_rows).unbind(0)), x_local_padded)
        return out


class BandShardedImage:
    """Row band of an h x w image with the 2-row halos a 5x5 stencil needs."""

    HALO = 2

    def __init__(self, h, w, rank, world):
        self.h, self.w, self.rank, self.world = h, w, rank, world
        b = shard_bands(h, world)
        self.b0, self.b1 = int(b[rank]), int(b[rank + 1])
        self.top = self.HALO if rank > 0 else 0          # halo rows present above the band
        self.bot = self.HALO if rank < world - 1 else 0  # and below
        self.rows = self.b1 - self.b0 + self.top + self.bot

    def exchange_halos(self, ext):
        """ext: (rows, w) tensor = [top halo | own band | bottom halo]; fills the halos from the
        neighbours' edge rows (send own first/last 2 rows, receive theirs)."""
        import torch.distributed as dist
        H, reqs = self.HALO, []
        own0, own1 = self.top, self.top + (self.b1 - self.b0)
        if self.rank > 0:
            reqs.append(dist.isend(ext[own0:own0 + H].contiguous(), self.rank - 1))
            top = ext[0:H].clone()
            reqs.append(dist.irecv(top, self.rank - 1))
        if self.rank < self.world - 1:
            reqs.append(dist.isend(ext[own1 - H:own1].contiguous(), self.rank + 1))
            bot = ext[own1:own1 + H].clone()
            reqs.append(dist.irecv(bot, self.rank + 1))
        for r in reqs:
            r.wait()
        if self.rank > 0:
            ext[0:H] = top
        if self.rank < self.world - 1:
            ext[own1:own1 + H] = bot
        return ext

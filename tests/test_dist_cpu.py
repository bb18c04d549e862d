"""Multi-process (world_size 2, gloo on CPU) coverage of the N>1 data path of bench.py: row
shards balanced by nnz with an x all-gather for SpMV, and row bands with a 2-row halo exchange
for the 5x5 stencils.  The local compute is the oracle (the CUDA kernels replace it on GPUs);
the assembled result must equal the single-process result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spmv_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import RowShardedCsr
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rowptr, col, val, x, _ = synth.csr_powerlaw(5000, maxlen=700, seed=3)
        sh = RowShardedCsr(rowptr, col, val, rank, world)
        xl = sh.pad_local_x(torch.from_numpy(x[sh.r0:sh.r1].copy()))
        xg = sh.allgather_x(xl)
        y = oracle.spmv_f32(sh.nrows, sh.ncols_padded, sh.nnz, sh.rowptr, sh.col, sh.val, xg.numpy())
        ypad = torch.zeros(sh.max_rows)
        ypad[: sh.nrows] = torch.from_numpy(y)
        parts = [torch.zeros(sh.max_rows) for _ in range(world)]
        dist.all_gather(parts, ypad)
        if rank == 0:
            full = np.concatenate([parts[r][: sh.bounds[r + 1] - sh.bounds[r]].numpy() for r in range(world)])
            ref = oracle.spmv_f32(rowptr.size - 1, x.size, col.size, rowptr, col, val, x)
            q.put((bool(np.array_equal(full.view(np.uint32), ref.view(np.uint32))),
                   [int(rowptr[sh.bounds[r + 1]] - rowptr[sh.bounds[r]]) for r in range(world)]))
    finally:
        dist.destroy_process_group()


def _conv_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import BandShardedImage
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h, w = 61, 37
        img = synth.u8_i32(h * w, seed=5).reshape(h, w)
        band = BandShardedImage(h, w, rank, world)
        ext = torch.zeros(band.rows, w, dtype=torch.int32)
        ext[band.top:band.top + band.b1 - band.b0] = torch.from_numpy(img[band.b0:band.b1])
        band.exchange_halos(ext)
        out = oracle.conv5x5_u8(band.rows, w, 256, ext.numpy().reshape(-1).copy(), synth.BINOMIAL).reshape(band.rows, w)
        mine = out[band.top:band.top + band.b1 - band.b0]
        ref = oracle.conv5x5_u8(h, w, 256, img.reshape(-1).copy(), synth.BINOMIAL).reshape(h, w)[band.b0:band.b1]
        ok = torch.tensor([int(np.array_equal(mine, ref))])
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if rank == 0:
            q.put(bool(ok.item()))
    finally:
        dist.destroy_process_group()


def _run(worker, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(worker, args=(world, free_port(), q), nprocs=world, join=True, start_method="spawn")
    return q.get()


def test_row_sharded_spmv_allgather_gloo():
    ok, nnz_per_rank = _run(_spmv_worker)
    assert ok
    assert max(nnz_per_rank) <= 1.1 * min(nnz_per_rank) + 700  # balanced by non-zeros


def test_band_sharded_stencil_halo_exchange_gloo():
    assert _run(_conv_worker)

"""Multi-process (world_size 2, gloo on CPU) coverage of the N>1 data path of bench.py: row
shards balanced by nnz with an x all-gather for SpMV, and row bands with a 2-row halo exchange
for the 5x5 stencils, plus the dense rows of SURVEY §8e: gemv row blocks (x replicated by an
all-gather of its shards), gemv_t column blocks (no collective), dot ranges + one all-reduce,
axpy ranges, and gemm on the R x C tile grid.  The local compute is the oracle (the CUDA kernels
replace it on GPUs); the assembled result must equal the single-process result bit for bit
(dot: the fp64 partials re-associate, checked to 1e-12 relative)."""
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


def _fused_worker(rank, world, port, q, multicast=False):
    """The fused SpMV -> all-gather step (FusedSpmvAllgather) with its device stores emulated:
    every rank keeps a persistent two-half gathered-vector buffer at a fake base address; in
    step k it gathers x from half k & 1 and 'stores' its row results at the addresses
    pingpong_targets gives for half (k + 1) & 1 (peer bases, or a fake multicast base); every
    rank applies the writes that land in its own buffer, and no write may touch the half any rank
    reads in that step.  Three chained iterations A(A(A x)) must equal the single-process result
    bit for bit."""
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import RowShardedCsr, pingpong_targets, step_halves
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rowptr, col, val, x, _ = synth.csr_powerlaw(3000, maxlen=500, seed=11)
        sh = RowShardedCsr(rowptr, col, val, rank, world)
        n = sh.ncols_padded
        bases = [(r + 1) << 36 for r in range(world)]
        MC = 7 << 40
        offset = 256
        tg = pingpong_targets(bases, offset, MC if multicast else 0, rank, sh.max_rows, n)
        for peers, mc in tg:
            assert (mc != 0) == multicast and (len(peers) == (0 if multicast else world))
        xg = sh.allgather_x(sh.pad_local_x(torch.from_numpy(x[sh.r0:sh.r1].copy())))
        mem = np.full(2 * n, np.nan, np.float32)  # this rank's two halves, back to back
        mem[:n] = xg.numpy()
        mine = MC if multicast else bases[rank]
        for k in range(3):
            src, dst = step_halves(k)
            y = oracle.spmv_f32(sh.nrows, n, sh.nnz, sh.rowptr, sh.col, sh.val, mem[src * n:(src + 1) * n].copy())
            peers, mc = tg[dst]
            allw = [None] * world
            dist.all_gather_object(allw, [(t, y) for t in (peers if not mc else [mc])])
            for wr in allw:
                for t, yy in wr:
                    if not multicast and not (bases[rank] <= t < bases[rank] + (1 << 36)):
                        continue  # a store into another rank's buffer
                    start = (t - mine - offset) // 4
                    assert (t - mine - offset) % 4 == 0
                    # the race the ping-pong removes: a store into the half being read this step
                    assert dst * n <= start and start + yy.size <= (dst + 1) * n, "store into the read half"
                    mem[start:start + yy.size] = yy
            # everything the remapped columns read next step was written this step
            assert not np.isnan(mem[dst * n + np.unique(sh.col)]).any()
            mem[src * n:(src + 1) * n] = np.nan  # the old x is dead: a stale read would show as NaN
        y3 = mem[step_halves(3)[0] * n:][:n]
        ref = x
        for _ in range(3):
            ref = oracle.spmv_f32(rowptr.size - 1, x.size, col.size, rowptr, col, val, ref)
        got = y3[sh.rank * sh.max_rows:][: sh.nrows]
        ok = torch.tensor([int(np.array_equal(got.view(np.uint32), ref[sh.r0:sh.r1].view(np.uint32)))])
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if rank == 0:
            q.put(bool(ok.item()))
    finally:
        dist.destroy_process_group()


def _fused_worker_mc(rank, world, port, q):
    _fused_worker(rank, world, port, q, multicast=True)


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


def _dense_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200 import dist as pd
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        # gemv: row blocks, x all-gathered from its shards, y gathered
        m, n = 203, 77
        A, x, y = synth.f32(m * n, 1), synth.f32(n, 2), synth.f32(m, 3)
        g = pd.RowShardedGemv(m, n, rank, world)
        lo, hi = pd.shard_range(n, world, rank, align=1)
        xr = pd.allgather_vector(torch.from_numpy(x[lo:hi].copy()), n, world, rank, align=1).numpy()
        yl = g.step(lambda mm, nn, a, b, AA, xx, yy: oracle.gemv(mm, nn, a, b, AA, xx, yy).astype(np.float32),
                    1.5, 0.5, A[g.r0 * n:g.r1 * n], xr, y[g.r0:g.r1])
        full = g.gather_y(torch.from_numpy(yl)).numpy()
        ref = oracle.gemv(m, n, 1.5, 0.5, A, x, y).astype(np.float32)
        res["gemv"] = bool(np.array_equal(full.view(np.uint32), ref.view(np.uint32)))
        # gemv_t: column blocks of the strided view, no collective
        m, n, lda, incx, incy = 41, 90, 96, 2, 3
        A, x, y = synth.f32(m * lda, 4), synth.f32(m * incx, 5), synth.f32(n * incy, 6)
        gt = pd.ColShardedGemvT(m, n, rank, world, lda=lda, incx=incx, incy=incy)  # views from the affine forms
        Av, yv = gt.views(A, y)
        mine = oracle.gemv_t(m, gt.j1 - gt.j0, lda, incx, incy, 1.0, 0.25, Av.copy(), x, yv.copy())
        ref = oracle.gemv_t(m, n, lda, incx, incy, 1.0, 0.25, A, x, y)
        js = np.arange(gt.j1 - gt.j0) * incy
        res["gemv_t"] = bool(np.array_equal(mine[js], ref[gt.j0 * incy + js]))
        # dot / axpy: contiguous ranges; dot adds one all-reduce
        n = 10007
        x, y = synth.f32(n, 7), synth.f32(n, 8)
        lo, hi = pd.shard_range(n, world, rank)
        d = pd.dot_sharded(lambda a, b: oracle.dot(a.numel(), a.numpy(), b.numpy()),
                           torch.from_numpy(x[lo:hi].copy()), torch.from_numpy(y[lo:hi].copy()))
        dref = oracle.dot(n, x, y)
        res["dot"] = abs(d - dref) <= 1e-12 * float(np.sum(np.abs(x.astype(np.float64) * y)))
        ya = oracle.axpy_f32(hi - lo, np.float32(0.75), x[lo:hi].copy(), y[lo:hi].copy())
        res["axpy"] = bool(np.array_equal(ya, oracle.axpy_f32(n, np.float32(0.75), x, y)[lo:hi]))
        # gemm: R x C tile grid, C assembled on every rank
        m, n, k = 37, 45, 19
        A, B, C = synth.f32(m * k, 9), synth.f32(k * n, 10), synth.f32(m * n, 11)
        tg = pd.GemmTileGrid(m, n, k, rank, world)
        Ap, Bp = tg.panels(A, B)
        Ct = C.reshape(m, n)[tg.m0:tg.m1, tg.n0:tg.n1].copy().reshape(-1)
        tile = tg.step(lambda mm, nn, kk, a, b, AA, BB, CC: oracle.gemm(mm, nn, kk, a, b, AA, BB, CC),
                       1.0, 0.5, Ap.copy(), Bp, Ct)
        full = tg.gather_c(torch.from_numpy(tile)).numpy()
        res["gemm"] = bool(np.array_equal(full.reshape(-1), oracle.gemm(m, n, k, 1.0, 0.5, A, B, C)))
        res["grid"] = (tg.R, tg.C)
        flags = torch.tensor([int(all(v for kk, v in res.items() if kk != "grid"))])
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        if rank == 0:
            q.put((bool(flags.item()), res))
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


@pytest.mark.parametrize("world", [2, 4])
def test_dense_shards_gemv_gemvt_dot_axpy_gemm_gloo(world):
    ok, res = _run(_dense_worker, world)
    assert ok, res
    assert res["grid"][0] * res["grid"][1] == world


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("multicast", [False, True])
def test_fused_spmv_allgather_targets_gloo(world, multicast):
    """Three iterations (x -> Ax -> A^2x -> A^3x) through the fused step's store targets."""
    assert _run(_fused_worker_mc if multicast else _fused_worker, world)


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_fused_band_halo_addresses_resolve_to_neighbour_rows(world):
    """The fused halo exchange (FusedBandStencil): the row addresses band_halo_rows gives each
    rank for fake per-rank band buffers, resolved back to (rank, row), rebuild the halo-extended
    band; the oracle stencils on it equal the whole image's rows bit for bit (u8 clamp-to-edge at
    the image edges through the repeated own rows; f32 interior rows via band_interior)."""
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import band_halo_rows, band_interior, shard_bands
    h, w = 53, 24
    img = synth.u8_i32(h * w, seed=9).reshape(h, w)
    imgf = synth.f32(h * w, seed=9).reshape(h, w)
    b = shard_bands(h, world)
    rows = [int(b[q + 1] - b[q]) for q in range(world)]
    esize, bases = 4, [(q + 1) << 32 for q in range(world)]

    def resolve(addr):
        q = next(q for q in range(world) if bases[q] <= addr < bases[q] + rows[q] * w * esize)
        off = addr - bases[q]
        assert off % (w * esize) == 0
        return q, off // (w * esize)

    ref_u8 = oracle.conv5x5_u8(h, w, 256, img.reshape(-1).copy(), synth.BINOMIAL).reshape(h, w)
    ref_f = oracle.conv5x5_f32_f32(h, w, imgf.reshape(-1).copy(), (synth.BINOMIAL / 256.0).astype(np.float32),
                                   np.zeros(h * w, np.float32)).reshape(h, w)
    for rank in range(world):
        top, bot = band_halo_rows(bases, rows, rank, w, esize)
        b0, b1 = int(b[rank]), int(b[rank + 1])
        pick = lambda a, qr: a[int(b[qr[0]]) + qr[1]]  # noqa: E731
        for src, ref, f32 in ((img, ref_u8, False), (imgf, ref_f, True)):
            ext = np.concatenate([np.stack([pick(src, resolve(t)) for t in top]), src[b0:b1],
                                  np.stack([pick(src, resolve(t)) for t in bot])])
            n = ext.shape[0]
            if not f32:
                out = oracle.conv5x5_u8(n, w, 256, ext.reshape(-1).copy(), synth.BINOMIAL).reshape(n, w)[2:-2]
                assert np.array_equal(out, ref[b0:b1])
            else:
                out = oracle.conv5x5_f32_f32(n, w, ext.reshape(-1).copy(), (synth.BINOMIAL / 256.0).astype(np.float32),
                                             np.zeros(n * w, np.float32)).reshape(n, w)[2:-2]
                lo, hi = band_interior(h, b0, b1)
                assert np.array_equal(out[lo:hi].view(np.uint32), ref[b0 + lo:b0 + hi].view(np.uint32))


def _emulate_fused_concurrent(world, pingpong, multicast=False, steps=3, seed=21):
    """All ranks of the fused SpMV -> all-gather step in one process, worst-case interleaved: the
    ranks advance one row at a time, round robin, and every store is visible to every reader at
    once (the way NVLink stores of one rank land while another rank's warps are still gathering).
    Rows fold in source order (the emitted C's fp32 rounding).  pingpong=False models the single
    buffer of round 1 (gather from and store into the same half)."""
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import RowShardedCsr, pingpong_targets, step_halves
    rowptr, col, val, x, _ = synth.csr_powerlaw(600, maxlen=60, seed=seed)
    shards = [RowShardedCsr(rowptr, col, val, r, world) for r in range(world)]
    n = shards[0].ncols_padded
    bases, MC, offset = [(r + 1) << 36 for r in range(world)], 7 << 40, 64
    span = 8 * n + offset
    mem = [np.zeros(2 * n, np.float32) for _ in range(world)]
    for r, sh in enumerate(shards):
        for q, shq in enumerate(shards):
            mem[r][q * shq.max_rows:q * shq.max_rows + shq.nrows] = x[shq.r0:shq.r1]
    tgs = [pingpong_targets(bases, offset, MC if multicast else 0, r, sh.max_rows, n) for r, sh in enumerate(shards)]

    def store(addr, v):
        if multicast:
            i = (addr - MC - offset) // 4
            for m in mem:
                m[i] = v
            return
        r = next(r for r in range(world) if bases[r] <= addr < bases[r] + span)
        mem[r][(addr - bases[r] - offset) // 4] = v

    for k in range(steps):
        src, dst = step_halves(k) if pingpong else (0, 0)
        cursors = [0] * world
        while any(c < sh.nrows for c, sh in zip(cursors, shards)):
            for r, sh in enumerate(shards):
                i = cursors[r]
                if i >= sh.nrows:
                    continue
                xs = mem[r][src * n:(src + 1) * n]
                s = np.float32(0)
                for kk in range(sh.rowptr[i], sh.rowptr[i + 1]):
                    s = np.float32(s + np.float32(sh.val[kk] * xs[sh.col[kk]]))
                peers, mc = tgs[r][dst]
                for t in (peers if not mc else [mc]):
                    store(t + 4 * i, s)
                cursors[r] += 1
    last = step_halves(steps)[0] if pingpong else 0
    got = np.concatenate([mem[0][last * n + q * sh.max_rows:][: sh.nrows] for q, sh in enumerate(shards)])
    return got, (rowptr, col, val, x)


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("multicast", [False, True])
def test_fused_spmv_pingpong_survives_concurrent_overwrite(world, multicast):
    """Chained in-place steps under the worst-case interleaving of stores and gathers: with the
    ping-pong halves the result is A(A(A x)) bit for bit; the single-buffer variant (round 1's
    FusedSpmvAllgather) is not — the model has teeth."""
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    got, (rowptr, col, val, x) = _emulate_fused_concurrent(world, True, multicast)
    ref = x
    for _ in range(3):
        ref = oracle.spmv_f32(rowptr.size - 1, x.size, col.size, rowptr, col, val, ref)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    bad, _ = _emulate_fused_concurrent(world, False, multicast)
    assert not np.array_equal(bad.view(np.uint32), ref.view(np.uint32))

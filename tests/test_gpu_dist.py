"""The N>1 data path of bench.py on the real stack, at world size 1 (this run has one GPU): NCCL
process group, RowShardedCsr (rank-padded x all-gather + column remap) feeding the CUDA SpMV
through a CsrPlan, the band-sharded stencil with its halo buffers, and the dense shards — each
against the single-process CUDA result.  The multi-rank exchange itself is covered by the gloo
tests (test_dist_cpu.py, world 2 and 4)."""
import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl(cuda):
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


def test_row_sharded_spmv_over_nccl(nccl):
    import torch
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import RowShardedCsr
    rowptr, col, val, x, _ = synth.csr_powerlaw(200000, maxlen=2048, seed=5)
    nrows, nnz = rowptr.size - 1, col.size
    sh = RowShardedCsr(rowptr, col, val, 0, 1)
    rp, cd, vd = (torch.from_numpy(a).cuda() for a in (sh.rowptr, sh.col, sh.val))
    xl = sh.pad_local_x(torch.from_numpy(x[sh.r0:sh.r1]).cuda())
    xg = sh.allgather_x(xl)
    y = torch.empty(sh.nrows, device="cuda")
    plan = pb.device.CsrPlan(sh.nrows, sh.ncols_padded, sh.nnz, rp, mode=0)
    plan.spmv(rp, cd, vd, xg, y)
    pb.device.sync_status()
    ref = torch.empty(nrows, device="cuda")
    rp0 = torch.from_numpy(rowptr).cuda()
    pb.device.CsrPlan(nrows, nrows, nnz, rp0, mode=0).spmv(rp0, torch.from_numpy(col).cuda(),
                                                          torch.from_numpy(val).cuda(), torch.from_numpy(x).cuda(), ref)
    assert torch.equal(y.view(torch.int32), ref.view(torch.int32))


def test_dense_shards_over_nccl(nccl):
    import torch
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200 import dist as pd
    n = 4096 + 13
    x = torch.from_numpy(synth.f32(n, 3)).cuda()
    lo, hi = pd.shard_range(n, 1, 0)
    full = pd.allgather_vector(x[lo:hi].contiguous(), n, 1, 0)
    assert torch.equal(full, x)
    r = torch.zeros(1, device="cuda")
    d = pd.dot_sharded(lambda a, b: (pb.device.dot(a.numel(), a, b, r), float(r.item()))[1], x, x)
    pb.device.dot(n, x, x, r)
    assert d == float(r.item())
    m, k, nn = 96, 64, 160
    A, B, C = synth.f32(m * k, 1), synth.f32(k * nn, 2), synth.f32(m * nn, 3)
    tg = pd.GemmTileGrid(m, nn, k, 0, 1)
    Ap, Bp = tg.panels(torch.from_numpy(A), torch.from_numpy(B))
    Ct = torch.from_numpy(C.copy()).cuda()
    tg.step(lambda mm, n2, kk, a, b, AA, BB, CC: pb.device.gemm(mm, n2, kk, a, b, AA, BB, CC), 1.0, 0.5,
            Ap.cuda(), Bp.cuda(), Ct)
    out = tg.gather_c(Ct)
    ref = torch.from_numpy(C.copy()).cuda()
    pb.device.gemm(m, nn, k, 1.0, 0.5, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), ref)
    assert torch.equal(out.reshape(-1), ref)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("aligned", [True, False])
def test_spmv_dist_peer_stores(cuda, mode, aligned):
    """pencil_spmv_dev_dist with three peer targets (plain device buffers standing in for the
    NVLink mappings, at different slot offsets): y and every target equal the plain SpMV bit for
    bit.  Unaligned col/val take the regular executor + the row-distribution launch."""
    import torch
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import synth
    rowptr, col, val, x, _ = synth.csr_powerlaw(70000, maxlen=3000, seed=9)
    nrows, nnz = rowptr.size - 1, col.size
    sh = 0 if aligned else 1
    rp = torch.from_numpy(rowptr).cuda()
    cd = torch.zeros(nnz + sh, dtype=torch.int32, device="cuda")[sh:]
    vd = torch.zeros(nnz + sh, device="cuda")[sh:]
    cd.copy_(torch.from_numpy(col))
    vd.copy_(torch.from_numpy(val))
    xd = torch.from_numpy(x).cuda()
    plan = pb.device.CsrPlan(nrows, nrows, nnz, rp, mode=mode)
    ref = torch.empty(nrows, device="cuda")
    plan.spmv(rp, cd, vd, xd, ref)
    bufs = [torch.full((nrows + 1000 * q,), float("nan"), device="cuda") for q in range(3)]
    peers = [b.data_ptr() + 4 * 1000 * q for q, b in enumerate(bufs)]
    y = torch.empty(nrows, device="cuda")
    plan.spmv_dist(rp, cd, vd, xd, y, peers)
    pb.device.sync_status()
    assert torch.equal(y.view(torch.int32), ref.view(torch.int32))
    for q, b in enumerate(bufs):
        assert torch.equal(b[1000 * q:].view(torch.int32), ref.view(torch.int32))
        assert torch.isnan(b[:1000 * q]).all()  # nothing outside the slot


def test_fused_spmv_allgather_world1(nccl):
    """FusedSpmvAllgather on a real NCCL group + torch symmetric memory (world 1): the gathered
    buffer holds the rank's rows after the barrier; multicast is used when the group has it."""
    import torch
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import RowShardedCsr, FusedSpmvAllgather
    rowptr, col, val, x, _ = synth.csr_powerlaw(100000, maxlen=2048, seed=6)
    sh = RowShardedCsr(rowptr, col, val, 0, 1)
    rp, cd, vd = (torch.from_numpy(a).cuda() for a in (sh.rowptr, sh.col, sh.val))
    xg = sh.allgather_x(sh.pad_local_x(torch.from_numpy(x).cuda()))
    plan = pb.device.CsrPlan(sh.nrows, sh.ncols_padded, sh.nnz, rp, mode=1)
    fz = FusedSpmvAllgather(sh, torch.device("cuda", torch.cuda.current_device()))
    y = torch.empty(sh.nrows, device="cuda")
    out = fz.step(plan, rp, cd, vd, xg, y)
    ref = torch.empty(sh.nrows, device="cuda")
    plan.spmv(rp, cd, vd, xg, ref)
    torch.cuda.synchronize()
    pb.device.sync_status()
    assert torch.equal(y.view(torch.int32), ref.view(torch.int32))
    assert torch.equal(out[: sh.nrows].view(torch.int32), ref.view(torch.int32))
    print("multicast" if fz.mc else "peer stores", len(fz.peers))


@pytest.mark.parametrize("mode", [0, 1])
def test_fused_spmv_allgather_chained_in_place(nccl, mode):
    """Iterated in place, as INTEGRATION.md shows it: x = fz.step(..., None, y) four times, each
    step gathering from the buffer the previous step stored into.  Source order (mode 0) must
    equal oracle.spmv_f32 applied four times bit for bit; reassociated (mode 1) within 1e-5
    normwise per step against the oracle applied to the GPU's own previous iterate."""
    import torch
    import oracle
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import RowShardedCsr, FusedSpmvAllgather
    from conftest import normwise_err
    rowptr, col, val, x, _ = synth.csr_powerlaw(60000, maxlen=1500, seed=12)
    n, nnz = rowptr.size - 1, col.size
    sh = RowShardedCsr(rowptr, col, val, 0, 1)
    rp, cd, vd = (torch.from_numpy(a).cuda() for a in (sh.rowptr, sh.col, sh.val))
    plan = pb.device.CsrPlan(sh.nrows, sh.ncols_padded, sh.nnz, rp, mode=mode)
    fz = FusedSpmvAllgather(sh, torch.device("cuda", torch.cuda.current_device()))
    fz.load(sh.pad_local_x(torch.from_numpy(x).cuda()))
    y = torch.empty(sh.nrows, device="cuda")
    ref = x.copy()
    for it in range(4):
        prev = fz.current()[: n].cpu().numpy()
        xn = fz.step(plan, rp, cd, vd, None, y)
        torch.cuda.synchronize()
        pb.device.sync_status()
        got = xn[: n].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), y.cpu().numpy().view(np.uint32))
        if mode == 0:
            ref = oracle.spmv_f32(n, n, nnz, rowptr, col, val, ref)
            assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), f"step {it}"
        else:
            r64 = oracle.spmv(n, n, nnz, rowptr, col, val, prev)
            terms = np.abs(val.astype(np.float64) * prev.astype(np.float64)[col])
            scale = np.add.reduceat(np.append(terms, 0.0), rowptr[:-1]) * (np.diff(rowptr) > 0)
            assert normwise_err(got, r64, scale) <= 1e-5, f"step {it}"
    # an explicit x that aliases the half the step stores into is refused
    with pytest.raises(ValueError):
        fz.step(plan, rp, cd, vd, fz.halves[(fz.k + 1) & 1], y)


@pytest.mark.parametrize("h,w,world", [(200, 256, 3), (67, 132, 4), (41, 512, 2)])
@pytest.mark.parametrize("case", ["binomial", "sharpen", "scale3", "nonbyte", "bigtaps", "f32", "f32tiny", "f32generic"])
def test_band_kernels_read_halos_in_place(cuda, h, w, world, case):
    """The band-sharded sweep (pencil_conv5x5_*_band_dev) on `world` separately allocated bands,
    each reading its halo rows straight out of its neighbours' buffers (the addresses
    band_halo_rows gives; peer mappings on a multi-GPU box): the bands' rows equal the
    whole-image call bit for bit — separable and 25-tap kernels, non-power-of-two scale, the exact
    repair pass (a non-byte pixel; taps too large for the fp32 path) and the fp32 interior."""
    import torch
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import band_halo_rows, band_interior, shard_bands
    b = shard_bands(h, world)
    rows = [int(b[q + 1] - b[q]) for q in range(world)]
    f32 = case.startswith("f32")
    if f32:
        himg = synth.f32(h * w, seed=3)
        if case == "f32tiny":  # products of the fused power-of-two taps round: the guarded repair pass
            himg[h // 2 * w + 9] = np.float32(3e-39)
            himg[(rows[0] - 1) * w + 11] = np.float32(-2e-38)  # in a halo row of rank 1
        img = torch.from_numpy(himg).cuda()
        k = synth.f32(25, 9) if case == "f32generic" else (synth.BINOMIAL / 256.0).astype(np.float32)
        whole = torch.zeros(h * w, device="cuda")
        pb.device.conv5x5_f32(h, w, img, k, whole)
        ref_c = oracle.conv5x5_f32_f32(h, w, himg, k, np.zeros(h * w, np.float32))  # the emitted C as written
        assert np.array_equal(whole.cpu().numpy().view(np.uint32), ref_c.view(np.uint32))
    else:
        img = torch.from_numpy(synth.u8_i32(h * w, seed=3)).cuda()
        k, scale = {"binomial": (synth.BINOMIAL, 256), "sharpen": (synth.SHARPEN, 1), "scale3": (synth.SHARPEN, 3),
                    "nonbyte": (synth.BINOMIAL, 256), "bigtaps": (synth.BINOMIAL * 1000, 256000)}[case]
        if case == "nonbyte":
            img[h // 2 * w + 7] = 300
            img[(rows[0] - 1) * w + 5] = -4  # in a halo row of rank 1
        whole = torch.empty(h * w, dtype=torch.int32, device="cuda")
        pb.device.conv5x5_u8(h, w, scale, img, k, whole)
    bands = [img[int(b[q]) * w:int(b[q + 1]) * w].clone() for q in range(world)]  # separate allocations
    ptrs = [t.data_ptr() for t in bands]
    for q in range(world):
        top, bot = band_halo_rows(ptrs, rows, q, w, 4)
        b0, b1 = int(b[q]), int(b[q + 1])
        if f32:
            out = torch.zeros(rows[q] * w, device="cuda")
            lo, hi = band_interior(h, b0, b1)
            pb.device.conv5x5_f32_band(rows[q], w, lo, hi, bands[q], top, bot, k, out)
            got, ref = out.view(rows[q], w)[lo:hi], whole.view(h, w)[b0 + lo:b0 + hi]
            assert torch.equal(got.view(torch.int32), ref.contiguous().view(torch.int32))
        else:
            out = torch.empty(rows[q] * w, dtype=torch.int32, device="cuda")
            pb.device.conv5x5_u8_band(rows[q], w, scale, bands[q], top, bot, k, out)
            assert torch.equal(out, whole[b0 * w:b1 * w])


def test_band_kernel_rejects_unaligned_rows(cuda):
    import torch
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import synth
    img = torch.from_numpy(synth.u8_i32(16 * 64)).cuda()
    out = torch.empty_like(img)
    p = img.data_ptr()
    with pytest.raises(pb.PencilError):
        pb.device.conv5x5_u8_band(16, 64, 256, img, (p + 4, p), (p, p), synth.BINOMIAL, out)


def test_fused_band_stencil_symmetric_memory(nccl):
    """FusedBandStencil at world 1 on the real stack (symmetric memory rendezvous, barriers,
    the band launch): the whole image, so both edges clamp through the band's own rows."""
    import torch
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import FusedBandStencil
    h, w = 96, 256
    img = torch.from_numpy(synth.u8_i32(h * w, seed=4)).cuda()
    fb = FusedBandStencil(h, w, 0, 1, torch.int32, torch.device("cuda", torch.cuda.current_device()))
    fb.band().copy_(img)
    out = torch.empty(h * w, dtype=torch.int32, device="cuda")
    fb.step_u8(256, synth.BINOMIAL, out)
    ref = torch.empty_like(out)
    pb.device.conv5x5_u8(h, w, 256, img, synth.BINOMIAL, ref)
    assert torch.equal(out, ref)
    fbf = FusedBandStencil(h, w, 0, 1, torch.float32, torch.device("cuda", torch.cuda.current_device()))
    imgf = torch.from_numpy(synth.f32(h * w, seed=4)).cuda()
    fbf.band().copy_(imgf)
    k = (synth.BINOMIAL / 256.0).astype(np.float32)
    outf, reff = torch.zeros(h * w, device="cuda"), torch.zeros(h * w, device="cuda")
    fbf.step_f32(k, outf)
    pb.device.conv5x5_f32(h, w, imgf, k, reff)
    assert torch.equal(outf.view(torch.int32), reff.view(torch.int32))

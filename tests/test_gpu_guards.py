"""Out-of-bounds writes and run-to-run races, checked without compute-sanitizer (closed on this
GPU pool: runs under it have left GPUs needing a reset).  Every output array sits between two
16 KB guard zones filled with a sentinel; after the launch the guards must be untouched, and the
elements a kernel must NOT store to (gemv_t's y between incy strides, conv5x5_f32's border, rows
of y outside a spmv_dist slot) must keep their sentinel too.  Kernels that split a reduction
across threads / CTAs (dot, gemv_t split-K, SpMV row folds, gemm) run three times on the same
inputs and must agree bit for bit: their combine order is fixed, so a race shows up as a
difference.  The values themselves are checked against the oracle."""
import numpy as np
import pytest

import oracle
from paper_1302_5586_b200 import synth

pytestmark = pytest.mark.gpu
G = 4096  # guard elements on each side


def guarded(torch, n, dtype, fill):
    base = torch.full((n + 2 * G,), fill, dtype=dtype, device="cuda")
    return base, base[G:G + n]


def guards_intact(base, n, fill):
    import torch
    g = torch.cat([base[:G], base[G + n:]])
    if g.dtype.is_floating_point and fill != fill:  # NaN sentinel
        return bool(torch.isnan(g).all())
    return bool((g == fill).all())


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("aligned", [True, False])
def test_spmv_guards_and_determinism(cuda, mode, aligned):
    import paper_1302_5586_b200 as pb
    torch = cuda
    rowptr, col, val, x, _ = synth.csr_powerlaw(20000, maxlen=1500, seed=31)
    n, nnz = rowptr.size - 1, col.size
    s = 0 if aligned else 1
    cd = torch.zeros(nnz + s, dtype=torch.int32, device="cuda")[s:]
    vd = torch.zeros(nnz + s, device="cuda")[s:]
    cd.copy_(torch.from_numpy(col))
    vd.copy_(torch.from_numpy(val))
    rp, xd = dev(torch, rowptr), dev(torch, x)
    plan = pb.device.CsrPlan(n, n, nnz, rp, mode=mode)
    outs = []
    for _ in range(3):
        base, y = guarded(torch, n, torch.float32, float("nan"))
        plan.spmv(rp, cd, vd, xd, y)
        torch.cuda.synchronize()
        assert guards_intact(base, n, float("nan"))
        outs.append(y.clone())
    pb.device.sync_status()
    assert all(torch.equal(o.view(torch.int32), outs[0].view(torch.int32)) for o in outs)
    if mode == 0:
        assert np.array_equal(outs[0].cpu().numpy().view(np.uint32),
                              oracle.spmv_f32(n, n, nnz, rowptr, col, val, x).view(np.uint32))
    # fused stores: a peer slot in the middle of a guarded buffer
    base, _ = guarded(torch, n + 100, torch.float32, float("nan"))
    y = torch.empty(n, device="cuda")
    plan.spmv_dist(rp, cd, vd, xd, y, [base.data_ptr() + 4 * (G + 100)])
    torch.cuda.synchronize()
    assert torch.isnan(base[:G + 100]).all() and torch.isnan(base[G + 100 + n:]).all()
    assert torch.equal(base[G + 100:G + 100 + n].view(torch.int32), y.view(torch.int32))


def test_dense_blas_guards_and_determinism(cuda):
    import paper_1302_5586_b200 as pb
    torch = cuda
    m, k = 1000, 777
    A, xv, yv = synth.f32(m * k, 1), synth.f32(k, 2), synth.f32(m, 3)
    base, y = guarded(torch, m, torch.float32, float("nan"))
    y.copy_(torch.from_numpy(yv))
    pb.device.gemv(m, k, 1.5, 0.5, dev(torch, A), dev(torch, xv), y)
    torch.cuda.synchronize()
    assert guards_intact(base, m, float("nan"))
    assert np.max(np.abs(y.cpu().numpy() - oracle.gemv(m, k, 1.5, 0.5, A, xv, yv))) < 1e-3
    # gemv_t: y[j*incy] only; the incy-1 elements in between keep the sentinel
    mm, nn, lda, incx, incy = 3000, 1500, 1504, 2, 3
    A2, xt, yt = synth.f32(mm * lda, 4), synth.f32(mm * incx, 5), synth.f32(nn * incy, 6)
    outs = []
    for _ in range(3):
        base, y = guarded(torch, nn * incy, torch.float32, float("nan"))
        y[::incy] = torch.from_numpy(yt[::incy]).cuda()
        pb.device.gemv_t(mm, nn, lda, incx, incy, 1.0, 0.25, dev(torch, A2), dev(torch, xt), y)
        torch.cuda.synchronize()
        assert guards_intact(base, nn * incy, float("nan"))
        yy = y.view(nn, incy)
        assert torch.isnan(yy[:, 1:]).all()
        outs.append(yy[:, 0].clone())
    assert all(torch.equal(o.view(torch.int32), outs[0].view(torch.int32)) for o in outs)
    ref = oracle.gemv_t(mm, nn, lda, incx, incy, 1.0, 0.25, A2, xt, yt)[::incy]
    assert np.max(np.abs(outs[0].cpu().numpy() - ref)) < 1e-3
    # dot: one float written, fixed-order combine
    n = (1 << 22) + 5
    a, b = synth.f32(n, 7), synth.f32(n, 8)
    vals = []
    for _ in range(3):
        base, r = guarded(torch, 1, torch.float32, float("nan"))
        pb.device.dot(n, dev(torch, a), dev(torch, b), r)
        torch.cuda.synchronize()
        assert guards_intact(base, 1, float("nan"))
        vals.append(float(r.item()))
    assert vals[0] == vals[1] == vals[2]
    assert abs(vals[0] - oracle.dot(n, a, b)) <= 1e-5 * float(np.sum(np.abs(a.astype(np.float64) * b)))
    base, y = guarded(torch, n, torch.float32, float("nan"))
    y.copy_(torch.from_numpy(b))
    pb.device.axpy(n, 0.75, dev(torch, a), y)
    torch.cuda.synchronize()
    assert guards_intact(base, n, float("nan"))
    assert np.array_equal(y.cpu().numpy().view(np.uint32), oracle.axpy_f32(n, np.float32(0.75), a, b).view(np.uint32))


@pytest.mark.parametrize("h,w", [(70, 256), (33, 132), (9, 60)])
def test_stencil_guards(cuda, h, w):
    import paper_1302_5586_b200 as pb
    torch = cuda
    img = synth.u8_i32(h * w, 9)
    for taps, scale in ((synth.BINOMIAL, 256), (synth.SHARPEN, 1), (np.arange(25, dtype=np.int32) % 7, 5)):
        ref = oracle.conv5x5_u8(h, w, scale, img, taps)
        base, out = guarded(torch, h * w, torch.int32, -7)
        pb.device.conv5x5_u8(h, w, scale, dev(torch, img), taps, out)
        torch.cuda.synchronize()
        assert guards_intact(base, h * w, -7)
        assert np.array_equal(out.cpu().numpy(), ref)
        base8, o8 = guarded(torch, h * w, torch.uint8, 0xA5)
        pb.device.conv5x5_u8_bytes(h, w, scale, dev(torch, img.astype(np.uint8)), taps, o8)
        torch.cuda.synchronize()
        assert guards_intact(base8, h * w, 0xA5)
        assert np.array_equal(o8.cpu().numpy().astype(np.int64), ref)
    imgf = synth.f32(h * w, 10)
    for taps in ((synth.BINOMIAL / 256.0).astype(np.float32), synth.f32(25, 11)):
        base, out = guarded(torch, h * w, torch.float32, float("nan"))
        pb.device.conv5x5_f32(h, w, dev(torch, imgf), taps, out)
        torch.cuda.synchronize()
        assert guards_intact(base, h * w, float("nan"))
        o = out.cpu().numpy().reshape(h, w)
        # the 2-pixel border is never stored to (interior-only nest)
        border = np.ones((h, w), bool)
        border[2:h - 2, 2:w - 2] = False
        assert np.isnan(o[border]).all()
        ref = oracle.conv5x5_f32_f32(h, w, imgf, taps, np.full(h * w, np.nan, np.float32)).reshape(h, w)
        assert np.array_equal(o[~border].view(np.uint32), ref[~border].view(np.uint32))


@pytest.mark.parametrize("shape", [(257, 260, 100), (128, 256, 32), (300, 517, 1000)])
def test_gemm_guards_and_determinism(cuda, shape):
    import paper_1302_5586_b200 as pb
    torch = cuda
    m, n, k = shape
    A, B, C = synth.f32(m * k, 13), synth.f32(k * n, 14), synth.f32(m * n, 15)
    outs = []
    for _ in range(3):
        base, c = guarded(torch, m * n, torch.float32, float("nan"))
        c.copy_(torch.from_numpy(C))
        pb.device.gemm(m, n, k, 1.0, 0.5, dev(torch, A), dev(torch, B), c)
        torch.cuda.synchronize()
        assert guards_intact(base, m * n, float("nan"))
        outs.append(c.clone())
    assert all(torch.equal(o.view(torch.int32), outs[0].view(torch.int32)) for o in outs)
    ref = A.reshape(m, k).astype(np.float64) @ B.reshape(k, n) + 0.5 * C.reshape(m, n)
    scale = np.abs(A.reshape(m, k)).astype(np.float64) @ np.abs(B.reshape(k, n)) + 0.5 * np.abs(C.reshape(m, n))
    assert float(np.max(np.abs(outs[0].cpu().numpy().reshape(m, n) - ref) / scale)) < 1e-5

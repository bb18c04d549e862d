"""Full-size parity on the BASELINE.json configs (run with -m gpu).  Inputs are the SURVEY §8d
synthetic streams; the checker is the C restatement of the interpreter (oracle port, fp64/int64)
and, for source-order kernels, the fp32 semantics of the reference-emitted C — both pinned to
the reference on the golden vectors (tests/test_oracle.py)."""
import numpy as np
import pytest

import oracle
from conftest import normwise_err
from paper_1302_5586_b200 import synth

pytestmark = pytest.mark.gpu
TOL = 1e-5


def dev(torch, a):
    return torch.from_numpy(a).cuda()


def test_gemv_8192(cuda):
    import paper_1302_5586_b200 as pb
    torch = cuda
    m = n = 8192
    A, x, y = synth.f32(m * n, 42), synth.f32(n, 42, m * n), synth.f32(m, 42, m * n + n)
    for alpha, beta in [(1.0, 0.0), (1.5, 0.5)]:
        yd = dev(torch, y.copy())
        pb.device.gemv(m, n, alpha, beta, dev(torch, A), dev(torch, x), yd)
        ref = oracle.gemv(m, n, alpha, beta, A, x, y)
        scale = abs(alpha) * (np.abs(A.reshape(m, n)).astype(np.float64) @ np.abs(x)) + abs(beta) * np.abs(y)
        assert normwise_err(yd.cpu().numpy(), ref, scale) <= TOL


def test_gemv_t_vobla_view_16384(cuda):
    import paper_1302_5586_b200 as pb
    torch = cuda
    m = n = lda = 16384
    incx, incy = 2, 3
    A = synth.f32(m * lda, 42)
    x = synth.f32(m * incx, 42, m * lda)
    y = synth.f32(n * incy, 42, m * lda + m * incx)
    yd = dev(torch, y.copy())
    pb.device.gemv_t(m, n, lda, incx, incy, 1.0, 0.5, dev(torch, A), dev(torch, x), yd)
    ref = oracle.gemv_t(m, n, lda, incx, incy, 1.0, 0.5, A, x, y)
    got = yd.cpu().numpy()
    js = np.arange(n) * incy
    At = np.abs(A.reshape(m, lda)).astype(np.float32)
    scale = np.zeros(n * incy)
    scale[js] = (np.abs(x[np.arange(m) * incx]) @ At).astype(np.float64) + 0.5 * np.abs(y[js])
    assert normwise_err(got, ref, scale) <= TOL
    untouched = np.setdiff1d(np.arange(n * incy), js)
    assert np.array_equal(got[untouched], y[untouched])


def test_dot_axpy_chain_2e28(cuda):
    import paper_1302_5586_b200 as pb
    torch = cuda
    n = 1 << 28
    x, y = synth.f32(n, 42), synth.f32(n, 42, n)
    xd, yd = dev(torch, x), dev(torch, y.copy())
    r = torch.zeros(1, device="cuda")
    pb.device.dot(n, xd, yd, r)
    d = float(r.item())
    ref = oracle.dot(n, x, y)
    scale = float(np.sum(np.abs(x.astype(np.float64) * y)))
    assert abs(d - ref) <= TOL * scale
    pb.device.axpy_ptr(n, r, xd, yd)  # axpy(dot(x, y), x, y) without a host hop
    exact = oracle.axpy_f32(n, np.float32(d), x, y)
    assert np.array_equal(yd.cpu().numpy().view(np.uint32), exact.view(np.uint32))


@pytest.fixture(scope="module")
def big_csr():
    return synth.csr_powerlaw(1 << 24)


@pytest.mark.parametrize("mode", [0, 1], ids=["source_order", "reassociated"])
def test_spmv_powerlaw_16M_rows(cuda, big_csr, mode):
    import paper_1302_5586_b200 as pb
    torch = cuda
    rowptr, col, val, x, _ = big_csr
    nrows, nnz = rowptr.size - 1, col.size
    assert abs(nnz - 16 * nrows) <= 0.01 * 16 * nrows
    rp, cd, vd, xd = dev(torch, rowptr), dev(torch, col), dev(torch, val), dev(torch, x)
    y = torch.empty(nrows, device="cuda")
    plan = pb.device.CsrPlan(nrows, nrows, nnz, rp, mode=mode)
    plan.spmv(rp, cd, vd, xd, y)
    pb.device.sync_status()
    got = y.cpu().numpy()
    if mode == 0:  # bit-exact vs the emitted C's fp32 source-order semantics
        exact = oracle.spmv_f32(nrows, nrows, nnz, rowptr, col, val, x)
        assert np.array_equal(got.view(np.uint32), exact.view(np.uint32))
    ref = oracle.spmv(nrows, nrows, nnz, rowptr, col, val, x)
    terms = np.abs(val.astype(np.float64)) * np.abs(x[col])
    cs = np.concatenate([[0.0], np.cumsum(terms)])
    assert normwise_err(got, ref, cs[rowptr[1:]] - cs[rowptr[:-1]]) <= TOL


@pytest.mark.parametrize("mode", [0, 1], ids=["source_order", "reassociated"])
def test_spmv_dropin_host_arrays_pipelined(cuda, big_csr, mode):
    """Host arrays at full size take the pipelined drop-in (chunked upload, one launch per block of
    tiles, per-block y download): results are bit-identical to the device-resident path."""
    import paper_1302_5586_b200 as pb
    torch = cuda
    rowptr, col, val, x, _ = big_csr
    nrows, nnz = rowptr.size - 1, col.size
    rp = dev(torch, rowptr)
    yd = torch.empty(nrows, device="cuda")
    plan = pb.device.CsrPlan(nrows, nrows, nnz, rp, mode=mode)
    plan.spmv(rp, dev(torch, col), dev(torch, val), dev(torch, x), yd)
    pb.device.sync_status()
    y = np.full(nrows, np.nan, np.float32)
    (pb.dropin.spmv_vec if mode else pb.dropin.spmv_inline)(nrows, nrows, nnz, rowptr, col, val, x, y)
    assert np.array_equal(y.view(np.uint32), yd.cpu().numpy().view(np.uint32))


def test_spmv_dropin_pipelined_non_monotone_and_fault(cuda):
    import paper_1302_5586_b200 as pb
    nrows = 1 << 18
    lens = np.full(nrows, 17, np.int64)
    rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    nnz = int(rowptr[-1])
    assert nnz >= 1 << 22
    col = (synth.u8_i32(nnz, seed=5).astype(np.int64) * 4099 % nrows).astype(np.int32)
    val, x = synth.f32(nnz, seed=6), synth.f32(nrows, seed=7)
    bad = rowptr.copy()
    bad[nrows // 2] = bad[nrows // 2 + 1] + 5  # row nrows/2 - 1 reads past, row nrows/2 is empty
    y = np.zeros(nrows, np.float32)
    pb.dropin.spmv_inline(nrows, nrows, nnz, bad, col, val, x, y)
    exact = oracle.spmv_f32(nrows, nrows, nnz, bad, col, val, x)
    assert np.array_equal(y.view(np.uint32), exact.view(np.uint32))
    col_bad = col.copy()
    col_bad[nnz - 3] = nrows + 11
    with pytest.raises(pb.PencilError) as e:
        pb.dropin.spmv_vec(nrows, nrows, nnz, rowptr, col_bad, val, x, y)
    assert e.value.code == "E-INTERP"


def test_conv5x5_u8_16384(cuda):
    """The whole 16384^2 image against the oracle (the interpreter's int64 semantics, OpenMP C),
    bit for bit: int32-storage kernels (separable binomial, diamond sharpen) and the packed-byte
    kernels (SWAR binomial, DIA sharpen) — every pixel, borders included."""
    import paper_1302_5586_b200 as pb
    torch = cuda
    h = w = 16384
    img = synth.u8_i32(h * w, 42)
    imgd = dev(torch, img)
    img8 = dev(torch, img.astype(np.uint8))
    for k, scale in [(synth.BINOMIAL, 256), (synth.SHARPEN, 1)]:
        ref = oracle.conv5x5_u8(h, w, scale, img, k)
        out = torch.empty(h * w, dtype=torch.int32, device="cuda")
        pb.device.conv5x5_u8(h, w, scale, imgd, k, out)
        got = out.cpu().numpy()
        bad = np.flatnonzero(got != ref)
        assert bad.size == 0, (int(k[12]), bad[:8])
        del got, out
        out8 = torch.empty(h * w, dtype=torch.uint8, device="cuda")
        pb.device.conv5x5_u8_bytes(h, w, scale, img8, k, out8)
        got8 = out8.cpu().numpy()
        bad = np.flatnonzero(got8 != ref)
        assert bad.size == 0, ("bytes", int(k[12]), bad[:8])
        del got8, out8, ref


def _gemm_scale(A, B, C, alpha, beta, m, n, k):
    return abs(alpha) * (np.abs(A.reshape(m, k)).astype(np.float64) @ np.abs(B.reshape(k, n))) + \
        abs(beta) * np.abs(C.reshape(m, n))


@pytest.mark.parametrize("shape", [(2048, 2048, 2048, 1.0, 0.0), (1000, 777, 333, 1.25, 0.5), (128, 256, 32, 1.0, 0.0),
                                   (129, 257, 33, -0.5, 2.0)])
def test_gemm_3xtf32_vs_fp64(cuda, shape):
    import paper_1302_5586_b200 as pb
    torch = cuda
    m, n, k, alpha, beta = shape
    A, B, C = synth.f32(m * k, 42), synth.f32(k * n, 43), synth.f32(m * n, 44)
    Cd = dev(torch, C.copy())
    pb.device.gemm(m, n, k, alpha, beta, dev(torch, A), dev(torch, B), Cd)
    ref = alpha * (A.reshape(m, k).astype(np.float64) @ B.reshape(k, n).astype(np.float64)) + beta * C.reshape(m, n)
    err = normwise_err(Cd.cpu().numpy().reshape(m, n), ref, _gemm_scale(A, B, C, alpha, beta, m, n, k))
    assert err <= TOL, err


def test_gemm_16384_sampled(cuda):
    import paper_1302_5586_b200 as pb
    torch = cuda
    m = n = k = 16384
    A, B = synth.f32(m * k, 42), synth.f32(k * n, 43)
    Cd = torch.zeros(m * n, device="cuda")
    pb.device.gemm(m, n, k, 1.0, 0.0, dev(torch, A), dev(torch, B), Cd)
    got = Cd.view(m, n)
    rng = np.random.default_rng(0)
    rows, cols = rng.integers(0, m, 64), rng.integers(0, n, 64)
    A2, B2 = A.reshape(m, k), B.reshape(k, n)
    sub = got[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy()
    ref = A2[rows].astype(np.float64) @ B2[:, cols].astype(np.float64)
    scale = np.abs(A2[rows]).astype(np.float64) @ np.abs(B2[:, cols]).astype(np.float64)
    assert normwise_err(sub, ref, scale) <= TOL  # 4096 sampled entries of C


def test_conv5x5_f32_16384(cuda):
    import paper_1302_5586_b200 as pb
    torch = cuda
    h = w = 16384
    img = synth.f32(h * w, 42)
    k = (synth.BINOMIAL.astype(np.float32) / 256.0).astype(np.float32)
    out0 = synth.f32(h * w, 42, h * w)
    out = dev(torch, out0.copy())
    pb.device.conv5x5_f32(h, w, dev(torch, img), k, out)
    exact = oracle.conv5x5_f32_f32(h, w, img, k, out0)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), exact.view(np.uint32))

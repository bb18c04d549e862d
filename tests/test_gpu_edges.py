"""Edge cases of the CUDA path (run with -m gpu): schedules the golden shapes do not reach —
non-monotone CSR rowptr (the generic per-row schedule), ragged widths that take the scalar
stencil kernels, misaligned device pointers, views that leave their declared extent, faults."""
import numpy as np
import pytest

import oracle
from conftest import normwise_err
from paper_1302_5586_b200 import synth

pytestmark = pytest.mark.gpu


def test_spmv_non_monotone_rowptr_takes_generic_schedule(cuda):
    import paper_1302_5586_b200 as pb
    # row 1 has end < start: an empty row in PENCIL semantics (the k loop does not run)
    rowptr = np.array([0, 3, 1, 4, 6], np.int32)
    col = np.array([0, 2, 1, 3, 0, 1], np.int32)
    val = synth.f32(6, seed=3)
    x = synth.f32(4, seed=4)
    for fn in (pb.dropin.spmv_inline, pb.dropin.spmv_vec):
        y = np.zeros(4, np.float32)
        fn(4, 4, 6, rowptr, col, val, x, y)
        ref = oracle.spmv_f32(4, 4, 6, rowptr, col, val, x)
        assert np.array_equal(y.view(np.uint32), ref.view(np.uint32))


def test_spmv_out_of_range_column_faults_then_recovers(cuda):
    import paper_1302_5586_b200 as pb
    rowptr = np.array([0, 2, 3], np.int32)
    col = np.array([0, 9, 1], np.int32)
    with pytest.raises(pb.PencilError) as e:
        pb.dropin.spmv_vec(2, 4, 3, rowptr, col, synth.f32(3), synth.f32(4), np.zeros(2, np.float32))
    assert e.value.code == "E-INTERP"
    # the fault word was collected and cleared: the next good call succeeds
    y = np.zeros(2, np.float32)
    pb.dropin.spmv_vec(2, 4, 3, rowptr, np.array([0, 3, 1], np.int32), synth.f32(3), synth.f32(4), y)


def test_spmv_all_rows_empty_and_single_long_row(cuda):
    import paper_1302_5586_b200 as pb
    torch = cuda
    for lens in ([0] * 1000, [0] * 10 + [5000] + [0] * 10, [4096] * 3 + [1] * 5000):
        rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        nnz, nrows = int(rowptr[-1]), len(lens)
        col = (synth.u8_i32(max(nnz, 1), seed=7)[:nnz] * 3) % 977
        val, x = synth.f32(max(nnz, 1), seed=8)[:nnz], synth.f32(977, seed=9)
        for mode in (0, 1):
            rp = torch.from_numpy(rowptr).cuda()
            plan = pb.device.CsrPlan(nrows, 977, nnz, rp, mode=mode)
            y = torch.full((nrows,), 7.0, device="cuda")
            plan.spmv(rp, torch.from_numpy(col.astype(np.int32)).cuda(), torch.from_numpy(val).cuda(),
                      torch.from_numpy(x).cuda(), y)
            pb.device.sync_status()
            got = y.cpu().numpy()
            ref64 = oracle.spmv(nrows, 977, nnz, rowptr, col.astype(np.int32), val, x)
            if mode == 0:
                exact = oracle.spmv_f32(nrows, 977, nnz, rowptr, col.astype(np.int32), val, x)
                assert np.array_equal(got.view(np.uint32), exact.view(np.uint32))
            terms = np.abs(val.astype(np.float64)) * np.abs(x[col])
            cs = np.concatenate([[0.0], np.cumsum(terms)])
            assert normwise_err(got, ref64, cs[rowptr[1:]] - cs[rowptr[:-1]]) <= 1e-5


@pytest.mark.parametrize("h,w", [(13, 37), (64, 130), (5, 5), (130, 6)])
def test_stencils_ragged_widths(cuda, h, w):
    import paper_1302_5586_b200 as pb
    img = synth.u8_i32(h * w, seed=h * w)
    for k, scale in ((synth.BINOMIAL, 256), (synth.SHARPEN, 1), (synth.BINOMIAL, 7)):
        out = np.zeros(h * w, np.int32)
        pb.dropin.conv5x5_u8(h, w, scale, img, k, out)
        assert np.array_equal(out.astype(np.int64), oracle.conv5x5_u8(h, w, scale, img, k))
    imgf, kf, o0 = synth.f32(h * w, seed=5), synth.f32(25, seed=6), synth.f32(h * w, seed=7)
    outf = o0.copy()
    pb.dropin.conv5x5_f32(h, w, imgf, kf, outf)
    exact = oracle.conv5x5_f32_f32(h, w, imgf, kf, o0)
    assert np.array_equal(outf.view(np.uint32), exact.view(np.uint32))


def test_conv_u8_int32_storage_not_an_8bit_image(cuda):
    """int32 storage may hold any int: the warp-rows with values outside [0, 255] take the exact
    int32 path inside the fast kernel."""
    import paper_1302_5586_b200 as pb
    h, w = 70, 256
    img = synth.u8_i32(h * w, seed=11)
    img[5 * w + 17] = 100000
    img[40 * w + 200] = -77
    out = np.zeros(h * w, np.int32)
    pb.dropin.conv5x5_u8(h, w, 256, img, synth.BINOMIAL, out)
    assert np.array_equal(out.astype(np.int64), oracle.conv5x5_u8(h, w, 256, img, synth.BINOMIAL))
    big = synth.BINOMIAL * 1000  # taps beyond the fp32-exact range -> exact int path
    pb.dropin.conv5x5_u8(h, w, 7, img, big, out)
    assert np.array_equal(out.astype(np.int64), oracle.conv5x5_u8(h, w, 7, img, big))


def test_conv_u8_bytes_matches_int32_storage_ragged(cuda):
    import paper_1302_5586_b200 as pb
    torch = cuda
    # ring kernel (w % 4 == 0, |k| <= 657) incl. strips narrower than a warp; w % 4 != 0 and
    # taps beyond 657 take the dp4a / scalar kernels
    for h, w in ((33, 512), (20, 1000), (9, 16), (70, 132), (11, 1002), (5, 4)):
        img = synth.u8_i32(h * w, seed=w)
        for k, scale in ((synth.BINOMIAL, 256), (synth.SHARPEN, 1), (synth.BINOMIAL * 3, 5),
                         (synth.SHARPEN * 82, 3), (synth.BINOMIAL * 18, 1000), (synth.BINOMIAL * 20, 1000)):
            out8 = torch.empty(h * w, dtype=torch.uint8, device="cuda")
            pb.device.conv5x5_u8_bytes(h, w, scale, torch.from_numpy(img.astype(np.uint8)).cuda(), k, out8)
            ref = oracle.conv5x5_u8(h, w, scale, img, k)
            assert np.array_equal(out8.cpu().numpy().astype(np.int64), ref), (h, w, scale)


def test_misaligned_device_pointers(cuda):
    """views starting one element into a buffer are not 16-byte aligned: scalar paths"""
    import paper_1302_5586_b200 as pb
    torch = cuda
    m, n = 37, 101
    A, x, y = synth.f32(m * n + 1), synth.f32(n + 1, 3), synth.f32(m + 1, 4)
    Ad, xd, yd = (torch.from_numpy(a).cuda() for a in (A, x, y))
    pb.device.gemv(m, n, 1.0, 0.5, Ad[1:], xd[1:], yd[1:])
    ref = oracle.gemv(m, n, 1.0, 0.5, A[1:], x[1:], y[1:])
    scale = np.abs(A[1:].reshape(m, n)).astype(np.float64) @ np.abs(x[1:]) + 0.5 * np.abs(y[1:])
    assert normwise_err(yd[1:].cpu().numpy(), ref, scale) <= 1e-5
    nv = 1001
    a, b = synth.f32(nv + 1, 5), synth.f32(nv + 1, 6)
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    r = torch.zeros(1, device="cuda")
    pb.device.dot(nv, ad[1:], bd[1:], r)
    assert abs(r.item() - oracle.dot(nv, a[1:], b[1:])) <= 1e-5 * float(np.sum(np.abs(a[1:].astype(np.float64) * b[1:])))


def test_gemv_t_view_leaving_its_extent_faults(cuda):
    import paper_1302_5586_b200 as pb
    with pytest.raises(pb.PencilError) as e:
        pb.dropin.gemv_t(4, 9, 8, 1, 1, 1.0, 0.0, synth.f32(32), synth.f32(4), np.zeros(9, np.float32))
    assert e.value.code == "E-INTERP"


def test_interpreter_mirror_errors(cuda):
    import paper_1302_5586_b200 as pb
    it = pb.CudaInterpreter(0)
    it.set_array("A", synth.f32(6))
    with pytest.raises(pb.PencilError, match="no function named"):
        it.call("nope", [])
    with pytest.raises(pb.PencilError, match="wrong argument count"):
        it.call("dot", [pb.Arg.scalar(3)])
    with pytest.raises(pb.PencilError, match="needs an array"):
        it.call("dot", [pb.Arg.scalar(3), pb.Arg.scalar(1), pb.Arg.array("A")])
    with pytest.raises(pb.PencilError, match="no array storage"):
        it.call("dot", [pb.Arg.scalar(3), pb.Arg.array("A"), pb.Arg.array("B")])
    # an array shorter than its C99 static extent: the interpreter would fault on the first
    # load past its end
    with pytest.raises(pb.PencilError) as e:
        it.call("dot", [pb.Arg.scalar(7), pb.Arg.array("A"), pb.Arg.array("A")])
    assert e.value.code == "E-INTERP"
    assert it.call("dot", [pb.Arg.scalar(6), pb.Arg.array("A"), pb.Arg.array("A")]) > 0


SEPARABLE = [  # integer rank-1 taps k = u (x) v: the SEP kernels (horizontal pass on row entry)
    (np.outer([1, 4, 6, 4, 1], [1, 4, 6, 4, 1]), 256),
    (np.outer([1, -2, 1, 0, 0], [-1, 0, 2, 0, -1]), 1),
    (np.outer([0, 3, 0, -3, 0], [2, 4, 6, 4, 2]), 10),      # v not primitive: factored as 2 * (1,2,3,2,1)
    (np.outer([5, 5, 5, 5, 5], [5, 5, 5, 5, 5]), 625),      # near the fp32-exact bound
    (np.outer([0, 0, 1, 0, 0], [0, 0, 1, 0, 0]), 1),        # identity
    (np.outer([-1, -1, -1, -1, -1], [1, 1, 1, 1, 1]), 3),   # all-negative sums clamp to 0
]


@pytest.mark.parametrize("h,w", [(67, 256), (9, 132), (130, 516), (5, 4)])
def test_conv_u8_separable_taps_bit_exact(cuda, h, w):
    """Rank-1 integer taps take the separable kernels (int32 storage and packed bytes): bit-exact
    against the 25-tap oracle, edges clamped, pow2 and non-pow2 scales."""
    import paper_1302_5586_b200 as pb
    torch = cuda
    img = synth.u8_i32(h * w, seed=h + w)
    for k, scale in SEPARABLE:
        k = np.ascontiguousarray(k.reshape(-1), np.int32)
        ref = oracle.conv5x5_u8(h, w, scale, img, k)
        out = np.zeros(h * w, np.int32)
        pb.dropin.conv5x5_u8(h, w, scale, img, k, out)
        assert np.array_equal(out.astype(np.int64), ref), (k, scale)
        out8 = torch.empty(h * w, dtype=torch.uint8, device="cuda")
        pb.device.conv5x5_u8_bytes(h, w, scale, torch.from_numpy(img.astype(np.uint8)).cuda(), k, out8)
        assert np.array_equal(out8.cpu().numpy().astype(np.int64), ref), (k, scale)
    # a non-byte value in int32 storage still diverts to the exact repair pass
    bad = img.copy()
    bad[h // 2 * w + 1] = 4000
    k = np.ascontiguousarray(SEPARABLE[1][0].reshape(-1), np.int32)
    out = np.zeros(h * w, np.int32)
    pb.dropin.conv5x5_u8(h, w, 1, bad, k, out)
    assert np.array_equal(out.astype(np.int64), oracle.conv5x5_u8(h, w, 1, bad, k))


def _diamond_taps(rng, lim):
    k = rng.integers(-lim, lim + 1, size=(5, 5)).astype(np.int32)
    for di in range(5):
        for dj in range(5):
            if abs(di - 2) + abs(dj - 2) > 2:
                k[di, dj] = 0
    return k.reshape(-1)


@pytest.mark.parametrize("h,w", [(67, 256), (9, 132), (130, 516), (5, 4)])
def test_conv_u8_diamond_taps_bit_exact(cuda, h, w):
    """Taps supported on the radius-2 diamond (the 12 corner taps zero: the sharpen of the bench
    suite, Laplacian shapes) take the DIA kernels, which skip the zero taps: bit-exact against
    the 25-tap oracle on int32 storage and packed bytes, pow2 / non-pow2 / unit scales, signed
    taps, and the exact repair pass for a non-byte pixel."""
    import paper_1302_5586_b200 as pb
    torch = cuda
    rng = np.random.default_rng(h * 1000 + w)
    img = synth.u8_i32(h * w, seed=h + 2 * w)
    cases = [(np.ascontiguousarray(synth.SHARPEN), 1), (np.ascontiguousarray(synth.SHARPEN), 3)]
    cases += [(_diamond_taps(rng, lim), scale) for lim, scale in ((3, 16), (40, 77), (657, 4096), (1, 1))]
    for k, scale in cases:
        ref = oracle.conv5x5_u8(h, w, scale, img, k)
        out = np.zeros(h * w, np.int32)
        pb.dropin.conv5x5_u8(h, w, scale, img, k, out)
        assert np.array_equal(out.astype(np.int64), ref), (k, scale)
        out8 = torch.empty(h * w, dtype=torch.uint8, device="cuda")
        pb.device.conv5x5_u8_bytes(h, w, scale, torch.from_numpy(img.astype(np.uint8)).cuda(), k, out8)
        assert np.array_equal(out8.cpu().numpy().astype(np.int64), ref), (k, scale)
    bad = img.copy()
    bad[h // 2 * w + 3] = -7
    out = np.zeros(h * w, np.int32)
    pb.dropin.conv5x5_u8(h, w, 1, bad, synth.SHARPEN, out)
    assert np.array_equal(out.astype(np.int64), oracle.conv5x5_u8(h, w, 1, bad, synth.SHARPEN))


def test_spmv_source_order_long_rows(cuda):
    """Source order (spmv_inline / ACCESS spmv) with long rows: lengths around 64, rows spanning
    many 1024-non-zero tiles, long rows at tile edges, empty rows between long ones, and an
    out-of-range column inside a long row (fault): bit-identical to the emitted C's fp32 chain,
    through the device plan and the host-array drop-in."""
    import paper_1302_5586_b200 as pb
    torch = cuda
    rng = np.random.default_rng(17)
    lens = [63, 64, 65, 66, 0, 1, 3000, 0, 65, 1023, 1024, 1025, 2, 9000] + list(rng.integers(0, 200, 3000))
    lens += [64, 65] * 200 + list(rng.integers(0, 5, 5000))
    rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    nrows, nnz, ncols = len(lens), int(rowptr[-1]), 50021
    col = rng.integers(0, ncols, nnz).astype(np.int32)
    val, x = synth.f32(nnz, seed=21), synth.f32(ncols, seed=22)
    exact = oracle.spmv_f32(nrows, ncols, nnz, rowptr, col, val, x)
    rp = torch.from_numpy(rowptr).cuda()
    plan = pb.device.CsrPlan(nrows, ncols, nnz, rp, mode=0)
    y = torch.full((nrows,), 7.0, device="cuda")
    plan.spmv(rp, torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(), torch.from_numpy(x).cuda(), y)
    pb.device.sync_status()
    assert np.array_equal(y.cpu().numpy().view(np.uint32), exact.view(np.uint32))
    yh = np.full(nrows, np.nan, np.float32)
    pb.dropin.spmv_inline(nrows, ncols, nnz, rowptr, col, val, x, yh)
    assert np.array_equal(yh.view(np.uint32), exact.view(np.uint32))
    # an out-of-range column inside the 9000-long row: E-INTERP, and the row's other products
    bad = col.copy()
    bad[int(rowptr[13]) + 4500] = ncols + 5
    with pytest.raises(pb.PencilError) as e:
        pb.dropin.spmv_inline(nrows, ncols, nnz, rowptr, bad, val, x, np.zeros(nrows, np.float32))
    assert e.value.code == "E-INTERP"


def _conv_f32_exact(pb, h, w, img, k, seed=7):
    o0 = synth.f32(h * w, seed=seed)
    out = o0.copy()
    pb.dropin.conv5x5_f32(h, w, img, k, out)
    exact = oracle.conv5x5_f32_f32(h, w, img, k, o0)
    return np.array_equal(out.view(np.uint32), exact.view(np.uint32))


@pytest.mark.parametrize("h,w", [(70, 256), (64, 520), (9, 132)])
def test_conv_f32_pow2_taps_fused_bit_exact(cuda, h, w):
    """Power-of-two taps take the PF kernels (one FMA per tap: the product is exact, so one rounding
    equals the emitted C's two): binomial/256 fuses the 16 off-centre taps, an all-power-of-two
    kernel (with zeros and signs) all 25.  Taps > 1 or non-powers stay on the as-written path."""
    import paper_1302_5586_b200 as pb
    img = synth.f32(h * w, seed=h + w)
    binom = (synth.BINOMIAL.astype(np.float32) / 256.0).astype(np.float32)
    rng = np.random.default_rng(3)
    allp2 = (rng.choice([-1.0, 1.0], 25) * 2.0 ** rng.integers(-20, 1, 25)).astype(np.float32)
    allp2[[0, 7, 24]] = 0.0
    allp2[3] = -0.0
    big = binom.copy()
    big[0] = 2.0  # exponent > 0: not fusable
    for k in (binom, allp2, big, synth.f32(25, seed=6)):
        assert _conv_f32_exact(pb, h, w, img, k)


def test_conv_f32_pow2_guard_diverts_tiny_pixels(cuda):
    """Pixels whose scaled product would round below 2^-126 (here 2^-120 * 2^-8) flag the launch;
    the exact pass recomputes the image as written and re-arms the flag for the next call."""
    import paper_1302_5586_b200 as pb
    h, w = 70, 256
    binom = (synth.BINOMIAL.astype(np.float32) / 256.0).astype(np.float32)
    img = synth.f32(h * w, seed=21)
    tiny = img.copy().reshape(h, w)
    tiny[26:38, 90:150] = (tiny[26:38, 90:150] * np.float32(2.0 ** -118)).astype(np.float32)
    tiny = tiny.reshape(-1)
    # a fused FMA per power-of-two tap differs from the as-written sum on 49 pixels of this block
    # (numpy emulation, checked when the test was written), so the guard is what keeps it exact
    assert _conv_f32_exact(pb, h, w, tiny, binom)
    assert _conv_f32_exact(pb, h, w, img, binom)  # flag re-armed: the fast path again, still exact
    assert _conv_f32_exact(pb, h, w, tiny, binom)


@pytest.mark.parametrize("h,w", [(70, 256), (33, 520), (64, 264), (9, 8), (5, 512), (130, 1024), (40, 1040), (12, 16), (21, 1552)])
def test_conv_u8_bytes_swar_bit_exact(cuda, h, w):
    """Non-negative rank-1 taps with 16-bit sums take the SWAR kernel (two pixels per register,
    16 pixels per lane when w % 16 == 0, else 8; scale 256: byte-select requantisation, other powers of two: shift + mask;
    mirror-symmetric factors: the shared-pair-sum form, others the general one);
    strips at both image edges, strips narrower than a warp, and the non-SWAR cases (signed taps,
    sums >= 2^16, a clamp needed) beside them."""
    import paper_1302_5586_b200 as pb
    torch = cuda
    img = synth.u8_i32(h * w, seed=h * 7 + w)
    img[: min(h * w, 3 * w)] = 255  # saturated rows: the largest sums
    box = np.outer([1, 2, 2, 2, 1], [1, 2, 2, 2, 1]).astype(synth.BINOMIAL.dtype).reshape(-1)
    neg = -synth.BINOMIAL
    skew = np.outer([1, 3, 5, 2, 0], [2, 1, 4, 6, 3]).astype(synth.BINOMIAL.dtype).reshape(-1)  # not symmetric
    half = np.outer([1, 4, 6, 4, 1], [0, 1, 5, 3, 1]).astype(synth.BINOMIAL.dtype).reshape(-1)  # one factor symmetric
    for k, scale in ((synth.BINOMIAL, 256), (box, 64), (box, 32), (neg, 256), (synth.BINOMIAL, 128),
                     (synth.BINOMIAL * 2, 512), (synth.SHARPEN, 1), (skew, 256), (skew, 64), (half, 128)):
        out8 = torch.empty(h * w, dtype=torch.uint8, device="cuda")
        pb.device.conv5x5_u8_bytes(h, w, scale, torch.from_numpy(img.astype(np.uint8)).cuda(), k, out8)
        ref = oracle.conv5x5_u8(h, w, scale, img, k)
        assert np.array_equal(out8.cpu().numpy().astype(np.int64), ref), (h, w, scale)


LAPLACE25 = np.array([[-1, -1, -1, -1, -1], [-1, -1, -1, -1, -1], [-1, -1, 48, -1, -1],
                      [-1, -1, -1, -1, -1], [-1, -1, -1, -1, -1]], np.int32).reshape(-1)
LAPLACE13 = np.array([[0, 0, -1, 0, 0], [0, -1, -2, -1, 0], [-1, -2, 16, -2, -1],
                      [0, -1, -2, -1, 0], [0, 0, -1, 0, 0]], np.int32).reshape(-1)
SYM25 = np.array([[-1, -2, -3, -2, -1], [-2, -4, -6, -4, -2], [-3, -6, 120, -6, -3],  # mirror-symmetric,
                  [-2, -4, -6, -4, -2], [-1, -2, -3, -2, -1]], np.int32).reshape(-1)  # all 5 tap values
ASYM13 = np.array([[0, 0, -1, 0, 0], [0, -2, -1, -3, 0], [-1, -3, 20, -2, 0],      # diamond, no mirror
                   [0, -1, -2, 0, 0], [0, 0, -4, 0, 0]], np.int32).reshape(-1)
ASYM25 = np.array([[-1, 0, -2, 0, -3], [0, -1, -1, -5, 0], [-2, -1, 30, -1, -1],   # full support, no mirror
                   [-1, 0, 0, -2, 0], [0, -1, -1, 0, -4]], np.int32).reshape(-1)


@pytest.mark.parametrize("h,w", [(70, 256), (33, 520), (64, 264), (9, 8), (5, 512), (130, 1024), (40, 1040),
                                 (12, 16), (21, 1552), (3, 64), (1, 32), (2, 24)])
def test_conv_u8_bytes_signed_swar_bit_exact(cuda, h, w):
    """Centre-positive, off-centre non-positive taps (sharpen, Laplacians) with a power-of-two
    scale take the signed SWAR kernel (biased 16-bit sums, per-lane clamp): diamond and full 5x5
    supports, mirror-symmetric (the shared-partial form) and not, scales 1 .. 256, saturated rows, images shorter than the
    window, strips at both edges and narrower than a warp — bit-exact against the oracle; taps
    outside that shape (a positive off-centre tap, a negative centre, sums >= 2^16) take the other
    kernels, also exact."""
    import paper_1302_5586_b200 as pb
    torch = cuda
    img = synth.u8_i32(h * w, seed=h * 11 + w)
    img[: min(h * w, 2 * w)] = 255
    img[-min(h * w, w):] = 0
    mixed = synth.SHARPEN.copy()
    mixed[0] = 1  # a positive corner tap: not the signed SWAR shape
    for k, scale in ((synth.SHARPEN, 1), (synth.SHARPEN, 2), (LAPLACE13, 1), (LAPLACE13, 4), (LAPLACE25, 1),
                     (LAPLACE25, 16), (synth.SHARPEN * 7, 256), (LAPLACE25 * 10, 8), (mixed, 1),
                     (-synth.SHARPEN, 1), (synth.SHARPEN, 3), (SYM25, 1), (SYM25, 64), (ASYM13, 1),
                     (ASYM13, 8), (ASYM25, 2), (ASYM25, 1)):
        out8 = torch.empty(h * w, dtype=torch.uint8, device="cuda")
        pb.device.conv5x5_u8_bytes(h, w, scale, torch.from_numpy(img.astype(np.uint8)).cuda(), k, out8)
        ref = oracle.conv5x5_u8(h, w, scale, img, k)
        got = out8.cpu().numpy().astype(np.int64)
        assert np.array_equal(got, ref), (h, w, scale, int(k[12]), np.flatnonzero(got != ref)[:5])


@pytest.mark.parametrize("every", [2, 3, 50])
def test_spmv_empty_rows_take_the_segmented_executor(cuda, every):
    """A power-law matrix with an empty row inserted after every `every`-th row (runs of empty
    rows at tile edges included): the segmented executor names rows by their ordinal among the
    non-empty ones (plan ordinals) and the empty rows' y is zeroed — source order bit-exact against
    the emitted C semantics, reassociated within the normwise bound, through the device API and the
    drop-in door on host arrays."""
    import paper_1302_5586_b200 as pb
    torch = cuda
    rowptr, col, val, x, _ = synth.csr_powerlaw(1 << 18, seed=every)
    n = rowptr.size - 1
    lens = np.diff(rowptr)
    nl = np.zeros(n + n // every + 7, np.int64)
    nl[np.arange(n) + np.arange(n) // every] = lens  # plus 7 trailing empty rows
    rp2 = np.concatenate([[0], np.cumsum(nl)]).astype(np.int32)
    n2, nnz = rp2.size - 1, col.size
    ref = oracle.spmv_f32(n2, x.size, nnz, rp2, col, val, x)
    rp, cd, vd, xd = (torch.from_numpy(a).cuda() for a in (rp2, col, val, x))
    for mode in (0, 1):
        y = torch.full((n2,), float("nan"), device="cuda")
        plan = pb.device.CsrPlan(n2, x.size, nnz, rp, mode=mode)
        plan.spmv(rp, cd, vd, xd, y)
        pb.device.sync_status()
        got = y.cpu().numpy()
        if mode == 0:
            assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
        else:
            r64 = oracle.spmv(n2, x.size, nnz, rp2, col, val, x)
            terms = np.abs(val.astype(np.float64) * x.astype(np.float64)[col])
            scale = np.add.reduceat(np.append(terms, 0.0), rp2[:-1]) * (np.diff(rp2) > 0)
            assert normwise_err(got, r64, scale) <= 1e-5
        plan.close()
    yh = np.full(n2, np.nan, np.float32)
    pb.dropin.spmv_inline(n2, x.size, nnz, rp2, col, val, x, yh)
    assert np.array_equal(yh.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("mode", [0, 1])
def test_spmv_tapered_tiles_across_the_tail_start(cuda, mode):
    """The plan cuts full-size tiles (TILE non-zeros), then 1024-non-zero ones for the last quarter
    wave of the launch's warps (k_spmv.cu csr_tile_schedule): a 16 M non-zero matrix has both, with
    long rows (and empty rows) straddling the switch; source order bit-identical to the emitted C's
    fp32 chain, reassociated within the normwise bound, tile count as the schedule states."""
    TILE, WAVES = 8192, 0.25
    import paper_1302_5586_b200 as pb
    torch = cuda
    rng = np.random.default_rng(23)
    target = 16_000_000
    lens = list(rng.integers(0, 40, target // 19))
    rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    # long rows and an empty row wherever the tail may start (either mode's launch width)
    warps = 148 * (5 if mode else 4) * 8
    tail = int(WAVES * warps * TILE)
    start = (int(rowptr[-1]) - tail) // TILE * TILE
    r = int(np.searchsorted(rowptr, start))
    lens[r - 1:r - 1] = [9000, 0, 4097, 1025, 1]
    rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    nrows, nnz, ncols = len(lens), int(rowptr[-1]), 1 << 20
    col = rng.integers(0, ncols, nnz).astype(np.int32)
    val, x = synth.f32(nnz, seed=31), synth.f32(ncols, seed=32)
    rp = torch.from_numpy(rowptr).cuda()
    plan = pb.device.CsrPlan(nrows, ncols, nnz, rp, mode=mode)
    nt, tn = plan.info()
    s0 = max(0, nnz - tail) // TILE * TILE
    assert tn == TILE and nt == s0 // TILE + (nnz - s0 + 1023) // 1024
    y = torch.full((nrows,), 7.0, device="cuda")
    plan.spmv(rp, torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(), torch.from_numpy(x).cuda(), y)
    pb.device.sync_status()
    got = y.cpu().numpy()
    if mode == 0:
        exact = oracle.spmv_f32(nrows, ncols, nnz, rowptr, col, val, x)
        assert np.array_equal(got.view(np.uint32), exact.view(np.uint32))
    else:
        ref = oracle.spmv(nrows, ncols, nnz, rowptr, col, val, x)
        scale = oracle.spmv(nrows, ncols, nnz, rowptr, col, np.abs(val), np.abs(x))
        assert normwise_err(got, ref, scale) < 1e-5

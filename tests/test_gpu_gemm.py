"""gemm (3xTF32 on tcgen05) edge cases against fp64 (run with -m gpu): operands read in place by
TMA (K-major A, MN-major B), the padded-pitch copies for rows that are not 16-byte multiples or
misaligned bases, K = 0 and K below one K block, ragged tiles, more tiles than CTA pairs (the
persistent loop and both TMEM accumulators), and operands whose low mantissa bits are all set (the
hi / lo split: a wrong split shows up as ~2^-11 relative error, far above the bound).
Normwise bound: max |C - ref| / (|alpha| |A||B| + |beta| |C0|) <= 1e-5."""
import numpy as np
import pytest

from conftest import normwise_err
from paper_1302_5586_b200 import synth

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _check(pb, torch, m, n, k, alpha, beta, A, B, C, offset=0):
    """device gemm on views starting `offset` floats into their buffers"""
    def dev(a):
        buf = torch.zeros(a.size + offset + 1, dtype=torch.float32, device="cuda")
        buf[offset:offset + a.size] = torch.from_numpy(a).cuda()
        return buf, buf[offset:offset + a.size]
    _, Ad = dev(A)
    _, Bd = dev(B)
    cbuf, Cd = dev(C)
    pb.device.gemm(m, n, k, alpha, beta, Ad, Bd, Cd)
    torch.cuda.synchronize()
    A2, B2, C2 = (A.reshape(m, k).astype(np.float64), B.reshape(k, n).astype(np.float64),
                  C.reshape(m, n).astype(np.float64))
    ref = alpha * (A2 @ B2) + beta * C2
    scale = abs(alpha) * (np.abs(A2) @ np.abs(B2)) + abs(beta) * np.abs(C2)
    got = Cd.cpu().numpy().reshape(m, n)
    # guard floats around C untouched
    assert float(cbuf[-1].item()) == 0.0 and (offset == 0 or float(cbuf[0].item()) == 0.0)
    return normwise_err(got, ref, scale)


@pytest.mark.parametrize("shape", [
    (256, 256, 16), (1, 1, 1), (1, 300, 7), (300, 1, 9), (5, 6, 3),       # tiny / one K block
    (255, 257, 18), (513, 130, 61), (100, 260, 1000),                        # ragged tiles, K % 4 != 0
    (2560, 2560, 64),                                                        # 100 tiles > 74 CTA pairs
    (4096, 4096, 96),                                                        # 256 tiles: 3-4 per pair
])
def test_gemm_shapes(cuda, shape):
    import paper_1302_5586_b200 as pb
    m, n, k = shape
    A, B, C = synth.f32(m * k, 7), synth.f32(k * n, 8), synth.f32(m * n, 9)
    assert _check(pb, cuda, m, n, k, 1.0, 0.5, A, B, C) <= TOL


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_gemm_misaligned_operands(cuda, offset):
    """bases not 16-byte aligned: A and B go through the padded-pitch copy, C through scalar stores"""
    import paper_1302_5586_b200 as pb
    m, n, k = 300, 260, 72
    A, B, C = synth.f32(m * k, 1), synth.f32(k * n, 2), synth.f32(m * n, 3)
    assert _check(pb, cuda, m, n, k, -1.5, 0.25, A, B, C, offset) <= TOL


def test_gemm_k_zero(cuda):
    """empty sum: C = alpha * 0 + beta * C"""
    import paper_1302_5586_b200 as pb
    torch = cuda
    m, n = 37, 45
    C = synth.f32(m * n, 5)
    Cd = torch.from_numpy(C.copy()).cuda()
    pb.device.gemm(m, n, 0, 2.0, 0.5, torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda"), Cd)
    assert np.array_equal(Cd.cpu().numpy(), (np.float32(0.5) * C).astype(np.float32))


def test_gemm_full_mantissa_wide_exponents(cuda):
    """operands with every low mantissa bit set and exponents over 2^-30..2^30: the split must
    carry the 13 bits the tensor core drops from the hi operand"""
    import paper_1302_5586_b200 as pb
    rng = np.random.default_rng(5)
    m, n, k = 384, 320, 512

    def full_mantissa(size):
        bits = (rng.integers(0, 1 << 23, size, dtype=np.int64) | 0x1fff).astype(np.uint32)
        exp = rng.integers(127 - 30, 127 + 30, size).astype(np.uint32)
        sign = rng.integers(0, 2, size).astype(np.uint32) << 31
        return (sign | (exp << 23) | bits).view(np.float32)
    A, B, C = full_mantissa(m * k), full_mantissa(k * n), full_mantissa(m * n)
    err = _check(pb, cuda, m, n, k, 1.0, 1.0, A, B, C)
    assert err <= TOL, err


@pytest.mark.parametrize("pitches", [(0, 0, 0), (4, 8, 12), (3, 5, 1)])
def test_gemm_strided_views(cuda, pitches):
    """A, B, C as views into wider arrays (row pitches lda > k, ldb > n, ldc > n); odd pitches
    take the padded copies; the elements between the views' rows are left alone"""
    import paper_1302_5586_b200 as pb
    torch = cuda
    m, n, k = 300, 260, 72
    lda, ldb, ldc = k + pitches[0], n + pitches[1], n + pitches[2]
    rng = np.random.default_rng(11)
    Aw = rng.random((m, lda), dtype=np.float32) - 0.5
    Bw = rng.random((k, ldb), dtype=np.float32) - 0.5
    Cw = rng.random((m, ldc), dtype=np.float32) - 0.5
    Ad, Bd, Cd = (torch.from_numpy(a.reshape(-1).copy()).cuda() for a in (Aw, Bw, Cw))
    pb.device.gemm_strided(m, n, k, 1.25, 0.5, Ad, lda, Bd, ldb, Cd, ldc)
    got = Cd.cpu().numpy().reshape(m, ldc)
    A2, B2 = Aw[:, :k].astype(np.float64), Bw[:, :n].astype(np.float64)
    ref = 1.25 * (A2 @ B2) + 0.5 * Cw[:, :n]
    scale = 1.25 * (np.abs(A2) @ np.abs(B2)) + 0.5 * np.abs(Cw[:, :n])
    assert normwise_err(got[:, :n], ref, scale) <= TOL
    assert np.array_equal(got[:, n:], Cw[:, n:])  # the gaps between C's rows are untouched


def test_gemm_tile_grid_on_views(cuda):
    """GemmTileGrid.step_views: every rank's tile from views of the replicated A, B straight into
    its place in C (no panel copies); the assembled C equals one whole-matrix gemm bit for bit
    (same tiles, same K order per output)"""
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200.dist import GemmTileGrid
    torch = cuda
    m, n, k, world = 1000, 1200, 256, 8
    A, B = synth.f32(m * k, 5), synth.f32(k * n, 6)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C = torch.zeros(m * n, device="cuda")
    for rank in range(world):
        GemmTileGrid(m, n, k, rank, world).step_views(pb.device.gemm_strided, 1.0, 0.0, Ad, Bd, C)
    whole = torch.zeros(m * n, device="cuda")
    pb.device.gemm(m, n, k, 1.0, 0.0, Ad, Bd, whole)
    A2, B2 = A.reshape(m, k).astype(np.float64), B.reshape(k, n).astype(np.float64)
    assert normwise_err(C.cpu().numpy().reshape(m, n), A2 @ B2, np.abs(A2) @ np.abs(B2)) <= TOL
    assert torch.equal(C, whole)


def test_gemm_beta_zero_reads_c_as_written(cuda):
    """the fixture computes alpha * s + beta * C[i*n+j] as written: with beta = 0 a NaN or an
    infinity in C still gives NaN (0 * NaN, 0 * Inf), finite entries give alpha * s"""
    import paper_1302_5586_b200 as pb
    torch = cuda
    m, n, k = 300, 260, 40
    A, B, C = synth.f32(m * k, 1), synth.f32(k * n, 2), synth.f32(m * n, 3)
    C[[0, 7, 300 * 5 + 3]] = [np.nan, np.inf, -np.inf]
    Cd = torch.from_numpy(C.copy()).cuda()
    pb.device.gemm(m, n, k, 1.0, 0.0, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), Cd)
    got = Cd.cpu().numpy()
    bad = np.zeros(m * n, bool)
    bad[[0, 7, 300 * 5 + 3]] = True
    assert np.isnan(got[bad]).all() and np.isfinite(got[~bad]).all()
    ref = (A.reshape(m, k).astype(np.float64) @ B.reshape(k, n)).reshape(-1)
    scale = (np.abs(A.reshape(m, k)).astype(np.float64) @ np.abs(B.reshape(k, n))).reshape(-1)
    assert np.max(np.abs(got[~bad] - ref[~bad]) / scale[~bad]) <= TOL


@pytest.mark.parametrize("shape", [(2100, 2000, 300), (1500, 2803, 97)])
def test_gemm_dropin_host_arrays_pipelined(cuda, shape):
    """the drop-in gemm on host arrays (pipelined by row blocks: B, then each block's A / C rows,
    its gemm on strided views, its C rows back) equals the device call bit for bit — pageable
    (numpy) and pinned arrays, pitches that are and are not 16-byte multiples"""
    import paper_1302_5586_b200 as pb
    torch = cuda
    m, n, k = shape
    A, B, C = synth.f32(m * k, 21), synth.f32(k * n, 22), synth.f32(m * n, 23)
    Cd = torch.from_numpy(C.copy()).cuda()
    pb.device.gemm(m, n, k, 0.75, -0.5, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), Cd)
    ref = Cd.cpu().numpy()
    c_pg = C.copy()
    pb.dropin.gemm(m, n, k, 0.75, -0.5, A, B, c_pg)
    assert np.array_equal(c_pg.view(np.uint32), ref.view(np.uint32))
    c_pin = torch.from_numpy(C.copy()).pin_memory()
    pb.dropin.gemm(m, n, k, 0.75, -0.5, torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory(), c_pin)
    assert np.array_equal(c_pin.numpy().view(np.uint32), ref.view(np.uint32))

"""Randomised parity stress on the GPU (not part of the test suite): random CSR matrices (empty rows,
long rows, ragged sizes) through both SpMV modes and the drop-in, random stencil shapes / taps
through every kernel family (int32 storage, packed bytes, fp32), random gemm shapes — each against
the oracle (bit-exact where the contract is, normwise 1e-5 otherwise) until the time budget runs out.
--large: host-array sizes that take the pipelined drop-ins (SpMV >= 4 M non-zeros, stencils and
axpy >= 64 MB), fewer cases.
usage: python tools/stress.py [seconds] [--large]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
import paper_1302_5586_b200 as pb  # noqa: E402
from conftest import normwise_err  # noqa: E402
from paper_1302_5586_b200 import synth  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 240.0
LARGE = "--large" in sys.argv
t_end = time.time() + budget
rng = np.random.default_rng(int(time.time()) & 0xffff)
counts = {"spmv": 0, "conv_u8": 0, "conv_bytes": 0, "conv_f32": 0, "gemm": 0}
fails = []


def spmv_case():
    nrows = int(rng.integers(300_000, 2_000_000)) if LARGE else int(rng.integers(1, 300_000))
    ncols = int(rng.integers(1, 2_000_000 if LARGE else 200_000))
    lens = rng.integers(0, 40, nrows)
    if rng.random() < 0.5:
        lens[rng.integers(0, nrows, 3)] = rng.integers(0, 20_000, 3)  # long rows
    if rng.random() < 0.5:
        lens[rng.random(nrows) < rng.random()] = 0  # runs of empty rows
    rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    nnz = int(rowptr[-1])
    col = rng.integers(0, ncols, nnz).astype(np.int32)
    val, x = synth.f32(nnz, int(rng.integers(1, 1 << 30))), synth.f32(ncols, int(rng.integers(1, 1 << 30)))
    exact = oracle.spmv_f32(nrows, ncols, nnz, rowptr, col, val, x)
    ref = oracle.spmv(nrows, ncols, nnz, rowptr, col, val, x)
    scale = oracle.spmv(nrows, ncols, nnz, rowptr, col, np.abs(val), np.abs(x))
    y = np.full(nrows, np.nan, np.float32)
    pb.dropin.spmv_inline(nrows, ncols, nnz, rowptr, col, val, x, y)
    if not np.array_equal(y.view(np.uint32), exact.view(np.uint32)):
        fails.append(("spmv_inline", nrows, ncols, nnz))
    y = np.full(nrows, np.nan, np.float32)
    pb.dropin.spmv_vec(nrows, ncols, nnz, rowptr, col, val, x, y)
    if not normwise_err(y, ref, scale) <= 1e-5:
        fails.append(("spmv_vec", nrows, ncols, nnz))
    counts["spmv"] += 1


def taps_case():
    kind = rng.integers(0, 4)
    if kind == 0:  # separable non-negative
        u, v = rng.integers(0, 6, 5), rng.integers(0, 6, 5)
        return np.outer(u, v).astype(np.int32).reshape(-1)
    if kind == 1:  # centre-positive, off-centre non-positive (symmetric or not)
        k = -rng.integers(0, 4, 25)
        if rng.random() < 0.5:
            k = k.reshape(5, 5)
            k = np.minimum(k, k[::-1]); k = np.minimum(k, k[:, ::-1]); k = k.reshape(-1)
        k[12] = rng.integers(0, 60)
        return k.astype(np.int32)
    if kind == 2:  # diamond
        k = rng.integers(-5, 6, 25).reshape(5, 5)
        for i in range(5):
            for j in range(5):
                if abs(i - 2) + abs(j - 2) > 2:
                    k[i, j] = 0
        return k.astype(np.int32).reshape(-1)
    return rng.integers(-700, 700, 25).astype(np.int32)  # generic, some beyond the fp32-exact range


def conv_case():
    if LARGE:  # >= 64 MB of int32 / fp32 (and of bytes for the larger ones): the pipelined drop-ins
        h, w = int(rng.integers(4100, 9000)), int(rng.integers(4100, 9000)) // 4 * 4
        if rng.random() < 0.5:
            w = w // 16 * 16
    else:
        h, w = int(rng.integers(1, 700)), int(rng.integers(1, 1500))
        if rng.random() < 0.5:
            w = (w // 16 + 1) * 16
    img = synth.u8_i32(h * w, int(rng.integers(1, 1 << 30)))
    k = taps_case()
    scale = int(rng.choice([1, 2, 4, 16, 256, 3, 7, 1000]))
    ref = oracle.conv5x5_u8(h, w, scale, img, k)
    out = np.full(h * w, -1, np.int32)
    pb.dropin.conv5x5_u8(h, w, scale, img, k, out)
    if not np.array_equal(out.astype(np.int64), ref):
        fails.append(("conv5x5_u8", h, w, scale, k.tolist()))
    counts["conv_u8"] += 1
    out8 = np.zeros(h * w, np.uint8)
    pb.dropin.conv5x5_u8_bytes(h, w, scale, img.astype(np.uint8), k, out8)
    if not np.array_equal(out8.astype(np.int64), ref):
        fails.append(("conv5x5_u8_bytes", h, w, scale, k.tolist()))
    counts["conv_bytes"] += 1
    if h >= 5 and w >= 5:
        f = synth.f32(h * w, int(rng.integers(1, 1 << 30)))
        kf = synth.f32(25, int(rng.integers(1, 1 << 30))) if rng.random() < 0.5 else \
            (rng.choice([0, 1, 2, 4, -1, -8], 25) / 64.0).astype(np.float32)
        o0 = synth.f32(h * w, 5)
        o = o0.copy()
        pb.dropin.conv5x5_f32(h, w, f, kf, o)
        if not np.array_equal(o.view(np.uint32), oracle.conv5x5_f32_f32(h, w, f, kf, o0).view(np.uint32)):
            fails.append(("conv5x5_f32", h, w))
        counts["conv_f32"] += 1


def axpy_case():
    n = int(rng.integers(1 << 24, 1 << 26))
    x, y = synth.f32(n, int(rng.integers(1, 1 << 30))), synth.f32(n, int(rng.integers(1, 1 << 30)))
    a = np.float32(rng.normal())
    ref = oracle.axpy_f32(n, a, x, y)
    yy = y.copy()
    pb.dropin.axpy(n, float(a), x, yy)
    if not np.array_equal(yy.view(np.uint32), ref.view(np.uint32)):
        fails.append(("axpy", n))
    counts["axpy"] = counts.get("axpy", 0) + 1


def blas_case():
    m, n = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
    lda = n + int(rng.integers(0, 9))
    incx, incy = int(rng.integers(1, 5)), int(rng.integers(1, 5))
    A = synth.f32(m * lda, int(rng.integers(1, 1 << 30)))
    alpha, beta = float(rng.choice([1.0, -0.5, 2.0])), float(rng.choice([0.0, 1.0, 0.5]))
    x, y = synth.f32(n, 3), synth.f32(m, 4)
    ref = oracle.gemv(m, n, alpha, beta, A[: m * n], x, y)
    scale = oracle.gemv(m, n, abs(alpha), abs(beta), np.abs(A[: m * n]), np.abs(x), np.abs(y))
    yy = y.copy()
    pb.dropin.gemv(m, n, alpha, beta, A[: m * n].copy(), x, yy)
    if not normwise_err(yy, ref, scale) <= 1e-5:
        fails.append(("gemv", m, n))
    xt, yt = synth.f32(m * incx, 5), synth.f32(n * incy, 6)
    ref = oracle.gemv_t(m, n, lda, incx, incy, alpha, beta, A, xt, yt)
    scale = oracle.gemv_t(m, n, lda, incx, incy, abs(alpha), abs(beta), np.abs(A), np.abs(xt), np.abs(yt))
    yy = yt.copy()
    pb.dropin.gemv_t(m, n, lda, incx, incy, alpha, beta, A, xt, yy)
    if not normwise_err(yy, ref, scale) <= 1e-5:
        fails.append(("gemv_t", m, n, lda, incx, incy))
    nd = int(rng.integers(1, 5_000_000))
    xd, yd = synth.f32(nd, 7), synth.f32(nd, 8)
    got, ref, sc = pb.dropin.dot(nd, xd, yd), oracle.dot(nd, xd, yd), oracle.dot(nd, np.abs(xd), np.abs(yd))
    if not abs(got - ref) <= 1e-5 * sc:
        fails.append(("dot", nd))
    counts["blas"] = counts.get("blas", 0) + 1


def gemm_case():
    m, n, k = (int(v) for v in rng.integers(1, 700, 3))
    A, B, C = synth.f32(m * k, 1), synth.f32(k * n, 2), synth.f32(m * n, 3)
    alpha, beta = float(rng.choice([1.0, 0.5, -2.0])), float(rng.choice([0.0, 1.0, 0.25]))
    ref = oracle.gemm(m, n, k, alpha, beta, A, B, C)
    scale = oracle.gemm(m, n, k, abs(alpha), abs(beta), np.abs(A), np.abs(B), np.abs(C))
    Cg = C.copy()
    pb.dropin.gemm(m, n, k, alpha, beta, A, B, Cg)
    if not normwise_err(Cg, ref, scale) <= 1e-5:
        fails.append(("gemm", m, n, k, alpha, beta))
    counts["gemm"] += 1


while time.time() < t_end and not fails:
    spmv_case()
    conv_case()
    if LARGE:
        axpy_case()
    else:
        gemm_case()
        blas_case()
print("cases", counts, "fails", fails[:5], flush=True)
sys.exit(1 if fails else 0)

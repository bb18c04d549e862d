"""Synthetic inputs of SURVEY.md §8d (deterministic LCG, seed 42 per config) — numpy front end of
lib/libpencil_synth.so.  Shared by tests, the golden-vector script and both bench arms."""
import ctypes

import numpy as np

from . import _lib

SEED = 42


def f32(n, seed=SEED, first=0):
    out = np.empty(n, dtype=np.float32)
    _lib.load_synth().pencil_synth_f32(out.ctypes.data, n, seed, first)
    return out


def u8_i32(n, seed=SEED, first=0):
    out = np.empty(n, dtype=np.int32)
    _lib.load_synth().pencil_synth_u8_i32(out.ctypes.data, n, seed, first)
    return out


def u8(n, seed=SEED, first=0):
    out = np.empty(n, dtype=np.uint8)
    _lib.load_synth().pencil_synth_u8(out.ctypes.data, n, seed, first)
    return out


def csr_powerlaw(nrows, ncols=None, avg_per_row=16.0, alpha=1.5, maxlen=4096, seed=SEED):
    """Power-law CSR: returns (rowptr int32[nrows+1], col int32[nnz], val f32[nnz], x f32[ncols], xm)."""
    ncols = nrows if ncols is None else ncols
    s = _lib.load_synth()
    rowptr = np.empty(nrows + 1, dtype=np.int32)
    xm = ctypes.c_double()
    nnz = s.pencil_synth_csr_rowptr(nrows, avg_per_row, alpha, maxlen, seed, rowptr.ctypes.data,
                                    ctypes.byref(xm))
    if nnz < 0:
        raise ValueError("nnz overflows int32")
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float32)
    s.pencil_synth_csr_fill(nrows, ncols, seed, rowptr.ctypes.data, col.ctypes.data, val.ctypes.data)
    x = f32(ncols, seed, nrows + 2 * nnz)
    return rowptr, col, val, x, xm.value


# 5x5 kernels of the stencil config: binomial (1,4,6,4,1)x(1,4,6,4,1) / 256 and a signed sharpen
BINOMIAL = np.outer([1, 4, 6, 4, 1], [1, 4, 6, 4, 1]).astype(np.int32).reshape(-1)
SHARPEN = np.array([0, 0, -1, 0, 0,
                    0, -1, -2, -1, 0,
                    -1, -2, 17, -2, -1,
                    0, -1, -2, -1, 0,
                    0, 0, -1, 0, 0], dtype=np.int32)

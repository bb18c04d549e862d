"""Python calls of the drop-in C ABI (include/pencil_b200.h §1) on host numpy arrays or CUDA
torch tensors.  Each function has exactly the emitted-C parameter list; arrays are passed as
pointers, outputs are written in place, and a failed call raises PencilError."""
import numpy as np

from . import _lib
from .interp import check_status


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return a.ctypes.data
    return a.data_ptr()  # torch tensor (host or device)


def _call(name, *args):
    lib = _lib.load()
    fn = getattr(lib, name)
    conv = [_ptr(a) if (isinstance(a, np.ndarray) or hasattr(a, "data_ptr")) else a for a in args]
    r = fn(*conv)
    check_status()
    return r


def gemv(m, n, alpha, beta, A, x, y):
    _call("gemv", m, n, alpha, beta, A, x, y)


def gemv_t(m, n, lda, incx, incy, alpha, beta, A, x, y):
    _call("gemv_t", m, n, lda, incx, incy, alpha, beta, A, x, y)


def dot(n, x, y):
    return _call("dot", n, x, y)


def axpy(n, a, x, y):
    _call("axpy", n, a, x, y)


def spmv_vec(nrows, ncols, nnz, rowptr, col, val, x, y):
    _call("spmv_vec", nrows, ncols, nnz, rowptr, col, val, x, y)


def spmv_inline(nrows, ncols, nnz, rowptr, col, val, x, y):
    _call("spmv_inline", nrows, ncols, nnz, rowptr, col, val, x, y)


def spmv(nrows, ncols, nnz, rowptr, col, val, x, y):
    _call("spmv", nrows, ncols, nnz, rowptr, col, val, x, y)


def spmv_row(nrows, ncols, nnz, i, rowptr, col, val, x, y):
    _call("spmv_row", nrows, ncols, nnz, i, rowptr, col, val, x, y)


def conv5x5_u8(h, w, scale, img, k, out):
    _call("conv5x5_u8", h, w, scale, img, k, out)


def conv5x5_f32(h, w, img, k, out):
    _call("conv5x5_f32", h, w, img, k, out)


def gemm(m, n, k, alpha, beta, A, B, C):
    _call("gemm", m, n, k, alpha, beta, A, B, C)


def conv5x5_u8_bytes(h, w, scale, img, k, out):
    """The packed 8-bit stencil (an extension of the PENCIL ABI: uint8 arrays) on host numpy
    arrays / torch tensors — pencil_conv5x5_u8_bytes."""
    if hasattr(k, "data_ptr"):  # a torch tensor (host or device)
        ok = k.numel() == 25 and str(k.dtype) == "torch.int32" and k.is_contiguous()
        kk = k
    else:
        kk = np.ascontiguousarray(np.asarray(k, dtype=np.int32).reshape(-1))
        ok = kk.size == 25
    if not ok:
        raise ValueError("a 5x5 stencil needs 25 contiguous int32 taps")
    _call("pencil_conv5x5_u8_bytes", h, w, scale, img, kk, out)

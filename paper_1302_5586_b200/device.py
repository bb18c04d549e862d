"""Stream-ordered device API (include/pencil_b200.h §3) on CUDA torch tensors.

Launches go to torch's current CUDA stream unless ``stream`` is given, so they order with
torch work; nothing here synchronizes except ``sync_status``.  PyTorch is only the allocator
and stream provider here — every launch is one of the library's own kernels."""
import ctypes

import numpy as np

from . import _lib
from .interp import PencilError, _CODES


def _stream(stream):
    if stream is not None:
        return stream
    import torch
    return torch.cuda.current_stream().cuda_stream


def _chk(st):
    if st:
        lib = _lib.load()
        raise PencilError(_CODES.get(st, "E-?"), (lib.pencil_cuda_last_error() or b"").decode())


def gemv(m, n, alpha, beta, A, x, y, stream=None):
    _chk(_lib.load().pencil_gemv_dev(_stream(stream), m, n, alpha, beta, A.data_ptr(), x.data_ptr(),
                                     y.data_ptr()))


def gemv_t(m, n, lda, incx, incy, alpha, beta, A, x, y, stream=None):
    _chk(_lib.load().pencil_gemv_t_dev(_stream(stream), m, n, lda, incx, incy, alpha, beta, A.data_ptr(),
                                       x.data_ptr(), y.data_ptr()))


def dot(n, x, y, result, stream=None):
    _chk(_lib.load().pencil_dot_dev(_stream(stream), n, x.data_ptr(), y.data_ptr(), result.data_ptr()))


def axpy(n, a, x, y, stream=None):
    _chk(_lib.load().pencil_axpy_dev(_stream(stream), n, a, x.data_ptr(), y.data_ptr()))


def axpy_ptr(n, a_dev, x, y, stream=None):
    _chk(_lib.load().pencil_axpy_dev_ptr(_stream(stream), n, a_dev.data_ptr(), x.data_ptr(), y.data_ptr()))


def _taps(k, dtype):
    k = np.ascontiguousarray(np.asarray(k, dtype=dtype).reshape(-1))
    if k.size != 25:
        raise ValueError("a 5x5 stencil needs 25 taps")
    return k


def conv5x5_u8(h, w, scale, img, k, out, stream=None):
    kk = _taps(k, np.int32)
    _chk(_lib.load().pencil_conv5x5_u8_dev(_stream(stream), h, w, scale, img.data_ptr(), kk.ctypes.data,
                                           out.data_ptr()))


def conv5x5_u8_bytes(h, w, scale, img, k, out, stream=None):
    kk = _taps(k, np.int32)
    _chk(_lib.load().pencil_conv5x5_u8_bytes_dev(_stream(stream), h, w, scale, img.data_ptr(),
                                                 kk.ctypes.data, out.data_ptr()))


def _ptr2(ptrs):
    return (ctypes.c_void_p * 2)(*[int(p) for p in ptrs])


def conv5x5_u8_band(h, w, scale, img, top, bot, k, out, stream=None):
    """One rank's row band (h rows at img / out) with its halo rows read in place: top = device
    addresses of rows -2, -1, bot = of rows h, h + 1 (peer mappings of the neighbours' edge rows,
    or the band's own edge row at the image's top / bottom) — pencil_conv5x5_u8_band_dev."""
    kk = _taps(k, np.int32)
    _chk(_lib.load().pencil_conv5x5_u8_band_dev(_stream(stream), h, w, scale, img.data_ptr(), _ptr2(top),
                                                _ptr2(bot), kk.ctypes.data, out.data_ptr()))


def conv5x5_f32_band(h, w, out_lo, out_hi, img, top, bot, k, out, stream=None):
    """As conv5x5_u8_band for the fp32 stencil; writes band rows [out_lo, out_hi)."""
    kk = _taps(k, np.float32)
    _chk(_lib.load().pencil_conv5x5_f32_band_dev(_stream(stream), h, w, out_lo, out_hi, img.data_ptr(),
                                                 _ptr2(top), _ptr2(bot), kk.ctypes.data, out.data_ptr()))


def conv5x5_f32(h, w, img, k, out, stream=None):
    kk = _taps(k, np.float32)
    _chk(_lib.load().pencil_conv5x5_f32_dev(_stream(stream), h, w, img.data_ptr(), kk.ctypes.data,
                                            out.data_ptr()))


def gemm(m, n, k, alpha, beta, A, B, C, stream=None):
    _chk(_lib.load().pencil_gemm_dev(_stream(stream), m, n, k, alpha, beta, A.data_ptr(), B.data_ptr(),
                                     C.data_ptr()))


def gemm_strided(m, n, k, alpha, beta, A, lda, B, ldb, C, ldc, stream=None):
    """gemm on strided views (pencil_gemm_strided_dev): A, B, C are tensors whose first element is
    the view's (0, 0); rows are lda / ldb / ldc elements apart."""
    _chk(_lib.load().pencil_gemm_strided_dev(_stream(stream), m, n, k, alpha, beta, A.data_ptr(), lda,
                                             B.data_ptr(), ldb, C.data_ptr(), ldc))


class CsrPlan:
    """Inspector for one CSR sparsity structure (mode 0: row sums in source order — spmv_inline,
    spmv; mode 1: reassociation licensed — spmv_vec)."""

    def __init__(self, nrows, ncols, nnz, rowptr, mode=0, stream=None):
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        _chk(self._lib.pencil_csr_plan_create(_stream(stream), nrows, ncols, nnz, rowptr.data_ptr(), mode,
                                              ctypes.byref(h)))
        self.handle = h
        self.nrows, self.ncols, self.nnz, self.mode = nrows, ncols, nnz, mode

    def info(self):
        nt, tn = ctypes.c_int(), ctypes.c_int()
        _chk(self._lib.pencil_csr_plan_info(self.handle, ctypes.byref(nt), ctypes.byref(tn)))
        return nt.value, tn.value

    def spmv(self, rowptr, col, val, x, y, stream=None):
        _chk(self._lib.pencil_spmv_dev(_stream(stream), self.handle, rowptr.data_ptr(), col.data_ptr(),
                                       val.data_ptr(), x.data_ptr(), y.data_ptr()))

    def spmv_dist(self, rowptr, col, val, x, y, peers=(), mc=0, stream=None):
        """Fused SpMV -> all-gather (pencil_spmv_dev_dist): y as spmv(), and every row result
        also stored at peers[q] + 4*i (device addresses, ints) or once at the multicast
        address mc + 4*i."""
        arr = (ctypes.c_void_p * max(1, len(peers)))(*[int(p) for p in peers])
        _chk(self._lib.pencil_spmv_dev_dist(_stream(stream), self.handle, rowptr.data_ptr(), col.data_ptr(),
                                            val.data_ptr(), x.data_ptr(), y.data_ptr(), arr, len(peers),
                                            int(mc) or None))

    def close(self):
        if self.handle:
            self._lib.pencil_csr_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sync_status(stream=None):
    _chk(_lib.load().pencil_sync_status(_stream(stream)))


def l2_flush(stream=None):
    _chk(_lib.load().pencil_l2_flush(_stream(stream)))

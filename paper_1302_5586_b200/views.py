"""Array and view descriptors (include/pencil_b200.h §10).

* ``affine_accesses(source, fn, **scalars)`` — every array access of a PENCIL function with its
  enclosing loops and the symbolic affine form of its index (coefficients may be scalar parameters
  such as ``lda``; the reference's affine_form, depanalysis.cpp:163-193, keeps constants only),
  evaluated under the given bindings.
* ``View`` — base / offset / extents / strides of a nest's view of an array (ctypes mirror of
  ``pencil_view``); ``gemv_t_views`` derives the gemv_t fixture's views from its affine forms,
  ``View.slice`` cuts a sub-view (a column block of a sharded gemv_t).
* ``ArrayDesc`` — element type, extent, shard spec, per-shard device pointers, host mirror.
"""
import ctypes

import numpy as np

from . import _lib
from .interp import check_status

DTYPES = {np.dtype(np.int32): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2, np.dtype(np.uint8): 3}


class View:
    def __init__(self, c=None):
        self.c = c if c is not None else _lib.pencil_view()

    @property
    def offset(self):
        return self.c.offset

    @property
    def rank(self):
        return self.c.rank

    @property
    def extent(self):
        return tuple(self.c.extent[:self.c.rank])

    @property
    def stride(self):
        return tuple(self.c.stride[:self.c.rank])

    def on(self, base):
        """The same view over device memory at `base` (a torch tensor or an address)."""
        v = View(_lib.pencil_view.from_buffer_copy(self.c))
        v.c.base = base.data_ptr() if hasattr(base, "data_ptr") else int(base)
        return v

    def slice(self, dim, lo, hi):
        out = _lib.pencil_view()
        _lib.load().pencil_view_slice(ctypes.byref(self.c), dim, lo, hi, ctypes.byref(out))
        check_status()
        return View(out)

    def __repr__(self):
        return f"View(offset={self.offset}, extent={self.extent}, stride={self.stride})"


def affine_accesses(source, fn, **scalars):
    """[{array, write, affine, loops: [(name, lo, hi)], stride: [..], offset, form}] for fn."""
    lib = _lib.load()
    names = list(scalars)
    arr_n = (ctypes.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
    arr_v = (ctypes.c_longlong * max(1, len(names)))(*[int(scalars[n]) for n in names])
    cap = 64
    out = (_lib.pencil_access_form * cap)()
    k = lib.pencil_affine_accesses(source.encode(), fn.encode(), len(names), arr_n, arr_v, out, cap)
    if k < 0:
        check_status()
    res = []
    for r in out[:min(k, cap)]:
        nl = r.nloops
        res.append({"array": r.array.decode(), "write": bool(r.is_write), "affine": bool(r.affine),
                    "loops": [(r.loop[d].value.decode(), r.lo[d], r.hi[d]) for d in range(nl)],
                    "stride": [r.stride[d] for d in range(nl)], "offset": r.offset, "form": r.form.decode()})
    return res


def fixture_source(name):
    s = _lib.load().pencil_fixture_source(name.encode())
    if s is None:
        raise KeyError(name)
    return s.decode()


def dist_plan(source, fn):
    """Distribution plan of fn's parallel loop nest (pencil_dist_plan, csrc/distplan.cpp): per
    loop dimension, each array's class (block / view / via / all) and the derived sets `owned`,
    `halo`, `replicated` (all-gathered when produced sharded) and the loop's reduction variables
    (all-reduced).  `source` is a unit's text or a fixture name ("spmv", "gemm", ...)."""
    import json
    lib = _lib.load()
    if "(" not in source:
        source = fixture_source(source)
    n = lib.pencil_dist_plan(source.encode(), fn.encode(), None, 0)
    if n < 0:
        check_status()
        raise KeyError(fn)
    buf = ctypes.create_string_buffer(n + 1)
    lib.pencil_dist_plan(source.encode(), fn.encode(), buf, n + 1)
    return json.loads(buf.value.decode())


def gemv_t_views(m, n, lda, incx, incy):
    """(A, x, y) views of the gemv_t fixture for these scalars, from its affine forms."""
    arr = (_lib.pencil_view * 3)()
    _lib.load().pencil_gemv_t_views(m, n, lda, incx, incy, arr)
    check_status()
    return tuple(View(_lib.pencil_view.from_buffer_copy(arr[i])) for i in range(3))


def gemv_t_view(alpha, beta, A, x, y, stream=None):
    """gemv_t over views (pencil_gemv_t_view_dev): y(j) = alpha sum_i A(i, j) x(i) + beta y(j)."""
    from .device import _stream, _chk
    _chk(_lib.load().pencil_gemv_t_view_dev(_stream(stream), alpha, beta, ctypes.byref(A.c), ctypes.byref(x.c),
                                            ctypes.byref(y.c)))


class ArrayDesc:
    """pencil_array: dtype, n, shard bounds (ordered ranges partitioning [0, n)), per-shard device
    pointers known to this process, host mirror."""

    def __init__(self, dtype, n, bounds=None):
        self._lib = _lib.load()
        self.dtype = np.dtype(dtype)
        b = None if bounds is None else (ctypes.c_longlong * len(bounds))(*[int(v) for v in bounds])
        self.h = self._lib.pencil_array_create(DTYPES[self.dtype], int(n), 1 if bounds is None else len(bounds) - 1, b)
        if not self.h:
            check_status()
        self._keep = None

    def close(self):
        if self.h:
            self._lib.pencil_array_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def nshards(self):
        ns = ctypes.c_int()
        self._lib.pencil_array_info(self.h, None, None, ctypes.byref(ns), None)
        return ns.value

    def shard(self, s):
        lo, hi, dev, ptr = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_int(), ctypes.c_void_p()
        self._lib.pencil_array_shard(self.h, s, ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(dev), ctypes.byref(ptr))
        check_status()
        return lo.value, hi.value, dev.value, ptr.value

    def attach(self, s, device, ptr):
        self._lib.pencil_array_attach(self.h, s, device, ptr.data_ptr() if hasattr(ptr, "data_ptr") else int(ptr))
        check_status()

    def set_mirror(self, host):
        """Host mirror: a numpy array (kept alive here) of n elements."""
        self._keep = host
        self._lib.pencil_array_set_mirror(self.h, host.ctypes.data)
        check_status()

    def owner(self, index):
        return self._lib.pencil_array_owner(self.h, int(index))

    def sync(self, s, to_device, stream=None):
        from .device import _stream
        self._lib.pencil_array_sync(self.h, s, 1 if to_device else 0, _stream(stream))
        check_status()

    def view(self, s):
        v = _lib.pencil_view()
        self._lib.pencil_array_view(self.h, s, ctypes.byref(v))
        check_status()
        return View(v)

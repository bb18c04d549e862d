"""CudaInterpreter: the reference Interpreter's surface over the CUDA backend.

``pencil::Interpreter`` (reference proj/core/include/pencil/interp.hpp:27-72) keeps arrays in a
name-addressed store (``set_array`` / ``arrays()``), passes arrays to functions by store name and
scalars by value (``Arg::array`` / ``Arg::scalar``), and raises ``PencilError("E-INTERP", ...)``
on runtime faults (interp.cpp:95-122, 186-195, 273-279).  This class offers the same calls; the
arrays live in device memory and ``call`` launches the kernel the mapper selected from the
fixture's loop verdicts (runtime: csrc/dispatch.cpp pencil_runtime_call).
"""
import ctypes

import numpy as np

from . import _lib

_DTYPES = {np.dtype(np.int32): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2, np.dtype(np.uint8): 3}
_NP = {0: np.int32, 1: np.float32, 2: np.float64, 3: np.uint8}
_CODES = {1: "E-INTERP", 2: "E-ARG", 3: "E-CUDA", 4: "E-NOMEM", 5: "E-UNSUPPORTED", 6: "E-OP2-SHAPE",
          7: "E-OP2-RANGE", 8: "E-OP2-KERNEL", 9: "E-OP2-CONFLICT", 10: "E-OPTIML-SHAPE", 11: "E-OPTIML-RANGE"}


class PencilError(RuntimeError):
    """Mirror of pencil::PencilError (diag.hpp:44-55): ``code`` is the stable machine code."""

    def __init__(self, code, message):
        super().__init__(message if message.startswith(code) else f"{code}: {message}")
        self.code = code


def check_status():
    """Raise PencilError if the last C-ABI call on this thread failed."""
    lib = _lib.load()
    st = lib.pencil_cuda_last_status()
    if st:
        msg = (lib.pencil_cuda_last_error() or b"").decode()
        raise PencilError(_CODES.get(st, "E-?"), msg)


class Arg:
    """Interpreter::Arg (interp.hpp:29-36)."""

    def __init__(self, value=None, array_name=None):
        self.value = value
        self.array_name = array_name

    @property
    def is_array(self):
        return self.array_name is not None

    @staticmethod
    def scalar(v):
        return Arg(value=v)

    @staticmethod
    def array(name):
        return Arg(array_name=name)


class CudaInterpreter:
    def __init__(self, device=0):
        self._lib = _lib.load()
        self._rt = self._lib.pencil_runtime_create(device)
        if not self._rt:
            raise PencilError("E-CUDA", f"cannot open CUDA device {device}")
        self._names = {}

    def close(self):
        if self._rt:
            self._lib.pencil_runtime_destroy(self._rt)
            self._rt = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_array(self, name, data):
        """Interpreter::set_array: copy host data into a named device array."""
        a = np.asarray(data)
        if a.dtype.kind in "iub" and a.dtype != np.uint8:
            a = a.astype(np.int32)
        elif a.dtype.kind == "f" and a.dtype != np.float64:
            a = a.astype(np.float32)
        a = np.ascontiguousarray(a.reshape(-1))
        dt = _DTYPES[a.dtype]
        st = self._lib.pencil_runtime_set_array(self._rt, name.encode(), dt, a.ctypes.data, a.size)
        if st:
            raise PencilError(_CODES.get(st, "E-?"), f"set_array('{name}') failed")
        self._names[name] = (dt, a.size)

    def bind_device_array(self, name, tensor):
        """Bind a CUDA torch tensor under a name without copying."""
        dt = {"torch.int32": 0, "torch.float32": 1, "torch.float64": 2, "torch.uint8": 3}[str(tensor.dtype)]
        st = self._lib.pencil_runtime_bind_array(self._rt, name.encode(), dt, tensor.data_ptr(), tensor.numel())
        if st:
            raise PencilError(_CODES.get(st, "E-?"), f"bind_array('{name}') failed")
        self._names[name] = (dt, tensor.numel())

    def get_array(self, name):
        dt, n = self._names[name]
        out = np.empty(n, dtype=_NP[dt])
        st = self._lib.pencil_runtime_get_array(self._rt, name.encode(), out.ctypes.data, n)
        if st:
            raise PencilError(_CODES.get(st, "E-?"), f"no array storage for '{name}'")
        return out

    def arrays(self):
        """Interpreter::arrays(): every named array, downloaded."""
        return {k: self.get_array(k) for k in self._names}

    def call(self, fn, args):
        """Interpreter::call(fn, args) -> return value (float for `dot`, else None)."""
        n = len(args)
        cargs = (_lib.pencil_arg * max(n, 1))()
        keep = []
        for i, a in enumerate(args):
            if a.is_array:
                b = a.array_name.encode()
                keep.append(b)
                cargs[i].kind, cargs[i].array = 2, b
            elif isinstance(a.value, (int, np.integer)):
                cargs[i].kind, cargs[i].i = 0, int(a.value)
            else:
                cargs[i].kind, cargs[i].f = 1, float(a.value)
        ret = _lib.pencil_value()
        st = self._lib.pencil_runtime_call(self._rt, fn.encode(), n, ctypes.cast(cargs, ctypes.c_void_p),
                                           ctypes.byref(ret))
        if st:
            msg = (self._lib.pencil_cuda_last_error() or b"").decode()
            raise PencilError(_CODES.get(st, "E-?"), msg)
        if ret.kind == 1:
            return ret.f
        if ret.kind == 0:
            return ret.i
        return None

    def last_kernel(self):
        """The kernel variant the mapper chose for the last call (what was launched)."""
        return (self._lib.pencil_runtime_last_kernel(self._rt) or b"").decode()

    def fp_reordered(self):
        """The `fp-reduction-reorders-results` flag of the last call (pencilc.cpp:157-161)."""
        return bool(self._lib.pencil_runtime_fp_reordered(self._rt))

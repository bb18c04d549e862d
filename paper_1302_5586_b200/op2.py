"""OP2 mesh models on the GPU (include/pencil_b200.h §8; reference core/include/pencil/op2.hpp).

``Op2Model(doc)`` takes the reference's mesh-model document (docs/op2-input.md: sets, maps, dats,
kernels, par_loops; a dict or JSON text) and mirrors the reference's entry points:

  * construction = ``load_op2_model`` (op2.hpp:79) plus the kernel checks of ``lower_op2_model``
    (E-OP2-SHAPE / E-OP2-RANGE / E-OP2-KERNEL / E-OP2-CONFLICT raise ``PencilError``);
  * ``run()`` = ``interpret_op2_reference`` (op2.hpp:114): every par_loop in declaration order,
    on the device; ``dats()`` returns the final contents (int64), like its result map;
  * ``lowered`` = the PENCIL text of ``lower_op2_model`` (one driver per par_loop).
"""
import ctypes
import json

import numpy as np

from . import _lib
from .interp import check_status

STRATEGIES = {0: "parallel", 1: "levels", 2: "serial"}


class Op2Model:
    def __init__(self, doc):
        lib = _lib.load()
        text = doc if isinstance(doc, str) else json.dumps(doc)
        self._lib = lib
        self._h = lib.pencil_op2_load(text.encode())
        if not self._h:
            check_status()
            raise RuntimeError("pencil_op2_load failed without a status")
        self._doc = doc if isinstance(doc, dict) else None  # parsed lazily (large meshes)
        self._text = None if isinstance(doc, dict) else text

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pencil_op2_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- execution ---------------------------------------------------------------------------
    def prepare(self):
        self._lib.pencil_op2_prepare(self._h)
        check_status()

    def run(self):
        """All par_loops in order (synchronous); device faults raise PencilError('E-INTERP')."""
        self._lib.pencil_op2_run(self._h)
        check_status()
        return self

    def run_loop_async(self, i):
        self._lib.pencil_op2_run_loop_async(self._h, i)
        check_status()

    def sync(self):
        self._lib.pencil_op2_sync(self._h)
        check_status()

    @property
    def stream(self):
        return self._lib.pencil_op2_stream(self._h)

    # -- data --------------------------------------------------------------------------------
    def dat(self, name, out=None):
        """The dat's values (int64); `out`: an int64 array of the dat's size to fill instead of a new one."""
        n = self._lib.pencil_op2_dat_size(self._h, name.encode())
        if n < 0:
            raise KeyError(name)
        if out is None:
            out = np.empty(n, np.int64)
        elif out.dtype != np.int64 or out.size != n or not out.flags["C_CONTIGUOUS"]:
            raise ValueError("out must be a contiguous int64 array of the dat's size")
        self._lib.pencil_op2_get_dat(self._h, name.encode(), out.ctypes.data, n)
        check_status()
        return out

    def set_dat(self, name, values):
        v = np.ascontiguousarray(values, dtype=np.int64)
        self._lib.pencil_op2_set_dat(self._h, name.encode(), v.ctypes.data, v.size)
        check_status()

    def dats(self):
        if self._doc is None:
            self._doc = json.loads(self._text)
        return {d["name"]: self.dat(d["name"]) for d in self._doc.get("dats", [])}

    # -- introspection -----------------------------------------------------------------------
    def loop_info(self, i):
        s, lv = ctypes.c_int(), ctypes.c_int()
        self._lib.pencil_op2_loop_info(self._h, i, ctypes.byref(s), ctypes.byref(lv))
        check_status()
        return STRATEGIES[s.value], lv.value

    @property
    def num_loops(self):
        return self._lib.pencil_op2_num_loops(self._h)

    @property
    def cuda_source(self):
        return self._lib.pencil_op2_cuda_source(self._h).decode()

    @property
    def lowered(self):
        return self._lib.pencil_op2_lowered(self._h).decode()


class JitUnit:
    """Any PENCIL unit on the GPU (include/pencil_b200.h §9; csrc/jit.cpp), with the surface of
    pencil::Interpreter (interp.hpp:38-51): ``set_array(name, values)``, ``call(fn, args)``
    (args: ints / floats / ``Arg.array(name)``), ``get_array(name)``.  Values follow the
    interpreter: int64 or fp64 per element; ``get_array`` returns fp64 values, the exact int64
    of integer elements and the per-element is-double flags."""

    def __init__(self, source):
        lib = _lib.load()
        self._lib = lib
        self._h = lib.pencil_jit_load(source.encode())
        if not self._h:
            check_status()
            raise RuntimeError("pencil_jit_load failed without a status")

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pencil_jit_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def set_array(self, name, values):
        a = np.ascontiguousarray(values)
        dt = {np.dtype(np.int32): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2, np.dtype(np.uint8): 3}
        if a.dtype not in dt:
            a = a.astype(np.float64 if a.dtype.kind == "f" else np.int32)
        self._lib.pencil_jit_set_array(self._h, name.encode(), dt[a.dtype], a.ctypes.data, a.size)
        check_status()

    def get_array(self, name):
        n = self._lib.pencil_jit_array_size(self._h, name.encode())
        if n < 0:
            raise KeyError(name)
        vals, flags, ints = np.empty(n, np.float64), np.empty(n, np.uint8), np.empty(n, np.int64)
        self._lib.pencil_jit_get_array(self._h, name.encode(), vals.ctypes.data, flags.ctypes.data,
                                       ints.ctypes.data, n)
        check_status()
        return vals, ints, flags.astype(bool)

    def call(self, fn, args):
        from ._lib import pencil_arg as PencilArg, pencil_value as PencilValue
        from .interp import Arg
        arr = (PencilArg * max(1, len(args)))()
        keep = []
        for i, a in enumerate(args):
            if isinstance(a, Arg) and a.is_array:
                b = a.array_name.encode()
                keep.append(b)
                arr[i].kind, arr[i].array = 2, b
            elif isinstance(a, Arg):
                a = a.value
            if not (isinstance(args[i], Arg) and args[i].is_array):
                if isinstance(a, (int, np.integer)):
                    arr[i].kind, arr[i].i = 0, int(a)
                else:
                    arr[i].kind, arr[i].f = 1, float(a)
        ret = PencilValue()
        self._lib.pencil_jit_call(self._h, fn.encode(), len(args), arr, ctypes.byref(ret))
        check_status()
        return ret.i if ret.kind == 0 else ret.f

    def schedule(self, fn):
        buf = ctypes.create_string_buffer(64)
        n = self._lib.pencil_jit_schedule(self._h, fn.encode(), buf, 64)
        if n < 0:
            raise KeyError(fn)
        return buf.value.decode()

    @property
    def cuda_source(self):
        return self._lib.pencil_jit_cuda_source(self._h).decode()


def optiml_lower(construct):
    """OptiML construct (dict or JSON text; docs/op2-input.md) -> PENCIL unit text, as
    load_optiml_construct + lower_optiml (optiml.hpp:27-41).  Run it with ``JitUnit``."""
    lib = _lib.load()
    text = (construct if isinstance(construct, str) else json.dumps(construct)).encode()
    n = lib.pencil_optiml_lower(text, None, 0)
    if n < 0:
        check_status()
    buf = ctypes.create_string_buffer(n + 1)
    lib.pencil_optiml_lower(text, buf, n + 1)
    return buf.value.decode()


def _jit_access(self, fn):
    """Access summary of fn's array parameters: {name: ("r"|"w"|"rw"|"-", must_write_all)}."""
    buf = ctypes.create_string_buffer(4096)
    n = self._lib.pencil_jit_access(self._h, fn.encode(), buf, 4096)
    if n < 0:
        raise KeyError(fn)
    out = {}
    for item in filter(None, buf.value.decode().split(",")):
        name, mode = item.split("=")
        out[name] = (mode.rstrip("!"), mode.endswith("!"))
    return out


def _jit_call_host(self, fn, args):
    """Call on host numpy arrays; uploads/downloads planned from the access summary (written
    arrays are updated in place).  Returns (value, (h2d_bytes, d2h_bytes))."""
    from ._lib import pencil_arg as PencilArg, pencil_value as PencilValue
    n = len(args)
    arr = (PencilArg * max(1, n))()
    host = (ctypes.c_void_p * max(1, n))()
    dts = (ctypes.c_int * max(1, n))()
    cnt = (ctypes.c_longlong * max(1, n))()
    code = {np.dtype(np.int32): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2, np.dtype(np.uint8): 3}
    for i, a in enumerate(args):
        if isinstance(a, np.ndarray):
            if a.dtype not in code or not a.flags.c_contiguous:
                raise TypeError("host arrays must be contiguous int32/float32/float64/uint8")
            arr[i].kind = 2
            host[i], dts[i], cnt[i] = a.ctypes.data, code[a.dtype], a.size
        elif isinstance(a, (int, np.integer)):
            arr[i].kind, arr[i].i = 0, int(a)
        else:
            arr[i].kind, arr[i].f = 1, float(a)
    ret = PencilValue()
    self._lib.pencil_jit_call_host(self._h, fn.encode(), n, arr, host, dts, cnt, ctypes.byref(ret))
    check_status()
    h2d, d2h = ctypes.c_longlong(), ctypes.c_longlong()
    self._lib.pencil_jit_last_traffic(self._h, ctypes.byref(h2d), ctypes.byref(d2h))
    return (ret.i if ret.kind == 0 else ret.f), (h2d.value, d2h.value)


JitUnit.access = _jit_access
JitUnit.call_host = _jit_call_host


def _jit_enable_trace(self, on=True):
    """Interpreter::enable_trace (interp.hpp:45)."""
    self._lib.pencil_jit_enable_trace(self._h, int(bool(on)))
    check_status()


def _jit_trace(self):
    """Interpreter::trace (MemTrace list, interp.hpp:17-21): [(store name, [index], is_write)]."""
    n = self._lib.pencil_jit_trace_size(self._h)
    if n <= 0:
        return []
    names = (ctypes.c_char_p * n)()
    idx = np.empty(n, np.int64)
    w = np.empty(n, np.uint8)
    self._lib.pencil_jit_trace_get(self._h, 0, n, names, idx.ctypes.data, w.ctypes.data)
    check_status()
    return [(names[i].decode(), [int(idx[i])], bool(w[i])) for i in range(n)]


def _jit_set_array_values(self, name, values):
    """Interpreter::set_array with mixed int / float elements (python ints and floats)."""
    n = len(values)
    isd = np.array([isinstance(v, float) for v in values], np.uint8)
    ints = np.array([0 if isinstance(v, float) else int(v) for v in values], np.int64)
    dbls = np.array([float(v) if isinstance(v, float) else 0.0 for v in values], np.float64)
    self._lib.pencil_jit_set_array_values(self._h, name.encode(), ints.ctypes.data, dbls.ctypes.data,
                                          isd.ctypes.data, n)
    check_status()


JitUnit.enable_trace = _jit_enable_trace
JitUnit.trace = _jit_trace
JitUnit.set_array_values = _jit_set_array_values


def _jit_set_rand_sequence(self, values):
    """Interpreter::set_rand_sequence (interp.hpp:44): rand() pops these values first."""
    v = np.ascontiguousarray(values, dtype=np.int64)
    self._lib.pencil_jit_set_rand_sequence(self._h, v.ctypes.data, v.size)
    check_status()


JitUnit.set_rand_sequence = _jit_set_rand_sequence

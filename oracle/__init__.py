"""ORACLE / TEST INFRASTRUCTURE ONLY — the checker, never the product.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It exposes three reference tiers for the PENCIL kernel fixtures:

  * ``port``     — oracle/pencil_oracle.c: C restatement of pencil::Interpreter semantics
                   (fp64/int64, interpreter order), each function citing interp.cpp.
  * ``ref_run``  — oracle/_ref/ref_driver: the reference's own front end + Interpreter, compiled
                   from /root/reference sources by oracle/Makefile (pins the port).
  * ``emitted``  — oracle/_ref/libpencil_omp_{annot,outer}.so: C emitted by the reference's
                   emit_openmp for the fixtures, compiled -fopenmp (the reference CPU path).
"""
import ctypes
import glob
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
PORT_SO = os.path.join(HERE, "_build", "libpencil_oracle.so")
REF_DRIVER = os.path.join(REF_DIR, "ref_driver")
FIXTURES = os.path.join(os.path.dirname(HERE), "paper_1302_5586_b200", "pencil")

P = ctypes.c_void_p
_i, _d, _ll = ctypes.c_int, ctypes.c_double, ctypes.c_longlong

_PORT_SIGS = {
    "oracle_gemv": [_i, _i, _d, _d, P, P, P, P],
    "oracle_gemv_t": [_i, _i, _i, _i, _i, _d, _d, P, _ll, P, _ll, P, _ll, P],
    "oracle_dot": [_i, P, P, P],
    "oracle_axpy": [_i, _d, P, P, P],
    "oracle_spmv": [_i, _i, _i, P, P, P, P, P],
    "oracle_conv5x5_u8": [_i, _i, _i, P, P, P],
    "oracle_conv5x5_f32": [_i, _i, P, P, P, P],
    "oracle_gemm": [_i, _i, _i, _d, _d, P, P, P, P],
    "oracle_spmv_f32": [_i, _i, _i, P, P, P, P, P],
    "oracle_conv5x5_f32_f32": [_i, _i, P, P, P],
    "oracle_axpy_f32": [_i, ctypes.c_float, P, P],
}
_port = None


def build(with_reference=None):
    """Compile the port (always) and, when /root/reference is present, oracle/_ref."""
    if with_reference is None:
        with_reference = os.path.isdir("/root/reference/proj/core")
    targets = ["port"] + (["ref"] if with_reference else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build(with_reference=False)
        lib = ctypes.CDLL(PORT_SO)
        for name, args in _PORT_SIGS.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = _i
        _port = lib
    return _port


def _p(a):
    return a.ctypes.data


class OracleFault(RuntimeError):
    """The interpreter would raise PencilError("E-INTERP")."""


def _ok(r):
    if r:
        raise OracleFault("E-INTERP")


# ---- port wrappers: numpy in (fp32/int32), fp64/int64 out -------------------------------
def gemv(m, n, alpha, beta, A, x, y):
    out = np.empty(m, np.float64)
    _ok(port().oracle_gemv(m, n, alpha, beta, _p(A), _p(x), _p(y), _p(out)))
    return out


def gemv_t(m, n, lda, incx, incy, alpha, beta, A, x, y):
    out = np.empty(y.size, np.float64)
    _ok(port().oracle_gemv_t(m, n, lda, incx, incy, alpha, beta, _p(A), A.size, _p(x), x.size, _p(y), y.size,
                             _p(out)))
    return out


def dot(n, x, y):
    out = np.empty(1, np.float64)
    _ok(port().oracle_dot(n, _p(x), _p(y), _p(out)))
    return float(out[0])


def axpy(n, a, x, y):
    out = np.empty(n, np.float64)
    _ok(port().oracle_axpy(n, a, _p(x), _p(y), _p(out)))
    return out


def spmv(nrows, ncols, nnz, rowptr, col, val, x):
    out = np.empty(nrows, np.float64)
    _ok(port().oracle_spmv(nrows, ncols, nnz, _p(rowptr), _p(col), _p(val), _p(x), _p(out)))
    return out


def conv5x5_u8(h, w, scale, img, k):
    out = np.empty(h * w, np.int64)
    _ok(port().oracle_conv5x5_u8(h, w, scale, _p(img), _p(k), _p(out)))
    return out


def conv5x5_f32(h, w, img, k, out_in):
    out = np.empty(h * w, np.float64)
    _ok(port().oracle_conv5x5_f32(h, w, _p(img), _p(k), _p(out_in), _p(out)))
    return out


def gemm(m, n, k, alpha, beta, A, B, C):
    out = np.empty(m * n, np.float64)
    _ok(port().oracle_gemm(m, n, k, alpha, beta, _p(A), _p(B), _p(C), _p(out)))
    return out


# ---- fp32 semantics of the emitted C as written (source order, no contraction) ---------------------------
def spmv_f32(nrows, ncols, nnz, rowptr, col, val, x):
    out = np.empty(nrows, np.float32)
    _ok(port().oracle_spmv_f32(nrows, ncols, nnz, _p(rowptr), _p(col), _p(val), _p(x), _p(out)))
    return out


def conv5x5_f32_f32(h, w, img, k, out_in):
    out = out_in.copy()
    _ok(port().oracle_conv5x5_f32_f32(h, w, _p(img), _p(k), _p(out)))
    return out


def axpy_f32(n, a, x, y):
    out = y.copy()
    _ok(port().oracle_axpy_f32(n, a, _p(x), _p(out)))
    return out


# ---- the reference Interpreter itself (oracle/_ref/ref_driver run) -----------------------
def ref_run(fixture, fn, args):
    """Run `fn` of paper_1302_5586_b200/pencil/<fixture>.pencil.c in pencil::Interpreter.

    args: python int/float scalars or numpy int32/float32 arrays (parameter order).  Returns
    (ret, outs) where outs[i] is the fp64 / int64 content of array argument i after the call.
    Raises OracleFault when the interpreter raises E-INTERP."""
    if not os.path.exists(REF_DRIVER):
        raise FileNotFoundError(REF_DRIVER)
    src = os.path.join(FIXTURES, fixture + ".pencil.c")
    with tempfile.TemporaryDirectory() as td:
        lines, paths = [], {}
        for idx, a in enumerate(args):
            if isinstance(a, np.ndarray):
                path = os.path.join(td, f"a{idx}.bin")
                if a.dtype == np.float32:
                    lines.append(f"array f32 {path}")
                elif a.dtype == np.int32:
                    lines.append(f"array i32 {path}")
                else:
                    raise TypeError(a.dtype)
                a.tofile(path)
                paths[idx] = (path, a.dtype)
            elif isinstance(a, (int, np.integer)):
                lines.append(f"scalar int {int(a)}")
            else:
                lines.append(f"scalar float {float(a)!r}")
        p = subprocess.run([REF_DRIVER, "run", src, fn], input="\n".join(lines) + "\n", capture_output=True,
                           text=True)
        if p.returncode == 3:
            raise OracleFault(p.stdout.strip())
        if p.returncode != 0:
            raise RuntimeError(f"ref_driver failed: {p.stderr}{p.stdout}")
        ret = None
        for line in p.stdout.splitlines():
            if line.startswith("ret "):
                _, kind, v = line.split()
                ret = int(v) if kind == "int" else float(v)
        outs = {}
        for idx, (path, dt) in paths.items():
            outs[idx] = np.fromfile(path + ".out", dtype=np.float64 if dt == np.float32 else np.int64)
        return ret, outs


def ref_trace(source, fn, args):
    """Run `fn` of the unit text `source` in pencil::Interpreter with its MemTrace on
    (Interpreter::enable_trace / trace, interp.hpp:17-21, 45-46).  args as for ref_run.  Returns
    [(argument index, flat index, is_write)] for every recorded load / store of an array argument,
    in the interpreter's order."""
    if not os.path.exists(REF_DRIVER):
        raise FileNotFoundError(REF_DRIVER)
    with tempfile.TemporaryDirectory() as td:
        src = os.path.join(td, "unit.pencil.c")
        with open(src, "w") as f:
            f.write(source)
        lines = []
        for idx, a in enumerate(args):
            if isinstance(a, np.ndarray):
                path = os.path.join(td, f"a{idx}.bin")
                lines.append(f"array {'f32' if a.dtype == np.float32 else 'i32'} {path}")
                a.tofile(path)
            elif isinstance(a, (int, np.integer)):
                lines.append(f"scalar int {int(a)}")
            else:
                lines.append(f"scalar float {float(a)!r}")
        tpath = os.path.join(td, "trace.txt")
        p = subprocess.run([REF_DRIVER, "run", src, fn], input="\n".join(lines) + "\n", capture_output=True,
                           text=True, env=dict(os.environ, PENCIL_REF_TRACE=tpath))
        if p.returncode != 0:
            raise RuntimeError(f"ref_driver failed: {p.stderr}{p.stdout}")
        out = []
        with open(tpath) as f:
            for line in f:
                parts = line.split()
                if parts and parts[0].startswith("arg"):
                    out.append((int(parts[0][3:]), int(parts[1]), parts[-1] == "1"))
        return out


def ref_analyze(fixture, params=None, arrays=None, outer=False):
    import json
    src = os.path.join(FIXTURES, "outer" if outer else "", fixture + ".pencil.c")
    cmd = [REF_DRIVER, "analyze", src]
    for k, v in (params or {}).items():
        cmd += ["--param", f"{k}={v}"]
    for k, v in (arrays or {}).items():
        cmd += ["--array", f"{k}={','.join(str(t) for t in v)}"]
    p = subprocess.run(cmd, capture_output=True, text=True, check=True)
    return [json.loads(l) for l in p.stdout.splitlines() if l.strip()]


# ---- C emitted by the reference's emit_openmp (the reference CPU path) -------------------
_emitted = {}
_EMIT_SIGS = {
    "gemv": (None, [_i, _i, ctypes.c_float, ctypes.c_float, P, P, P]),
    "gemv_t": (None, [_i, _i, _i, _i, _i, ctypes.c_float, ctypes.c_float, P, P, P]),
    "dot": (ctypes.c_float, [_i, P, P]),
    "axpy": (None, [_i, ctypes.c_float, P, P]),
    "spmv_vec": (None, [_i, _i, _i, P, P, P, P, P]),
    "spmv_inline": (None, [_i, _i, _i, P, P, P, P, P]),
    "spmv": (None, [_i, _i, _i, P, P, P, P, P]),
    "conv5x5_u8": (None, [_i, _i, _i, P, P, P]),
    "conv5x5_f32": (None, [_i, _i, P, P, P]),
    "gemm": (None, [_i, _i, _i, ctypes.c_float, ctypes.c_float, P, P, P]),
}


def build_native():
    """The emitted outer-pragma C compiled for THIS host's CPU (gcc -O3 -march=native -fopenmp,
    fp contraction left to gcc) — the timing build of the CPU baseline (bench.py).  Compiled
    where it runs (the GPU box's host), from the emitted C under _ref/emitted/outer; the parity
    build (_ref/libpencil_omp_outer.so) keeps -march=x86-64-v3 -ffp-contract=off."""
    out = os.path.join(REF_DIR, "libpencil_omp_native.so")
    src = sorted(glob.glob(os.path.join(REF_DIR, "emitted", "outer", "*.c")))
    if not src:
        raise FileNotFoundError("no emitted C under oracle/_ref/emitted/outer (build() the oracle first)")
    defs = ["-DACCESS(x)=", "-DDEF(x)=(void)0", "-DUSE(x)=(void)0", "-DMAY_DEF(x)=(void)0"]
    subprocess.run(["gcc", "-std=gnu11", "-O3", "-march=native", "-fopenmp", "-fPIC", "-shared"] + defs + src +
                   ["-o", out], check=True, capture_output=True)
    return out


def emitted(variant="outer"):
    """ctypes handle of the emitted-OpenMP library ('outer': pragmas on outermost loops only —
    the fast CPU baseline; 'annot': every annotated loop, as the fixtures are written; 'native':
    'outer' compiled for this host's CPU, timing only, build_native)."""
    if variant not in _emitted:
        if variant == "native":
            build_native()
        path = os.path.join(REF_DIR, f"libpencil_omp_{variant}.so")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _EMIT_SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _emitted[variant] = lib
    return _emitted[variant]

"""GPU parity (run with -m gpu on a B200).  Every golden vector of tests/golden (outputs of the
reference's own pencil::Interpreter) is replayed through the CUDA path via three doors of the
C ABI — the Interpreter-mirror name dispatch, the drop-in with host arrays, the drop-in with
device arrays — and compared:

  * integer kernels (conv5x5_u8), integer-valued SpMV: bit-exact;
  * source-order kernels (spmv_inline, spmv, axpy, conv5x5_f32): bit-exact against the
    reference-emitted C semantics (oracle.*_f32) AND normwise against the interpreter;
  * reassociated reductions (gemv, gemv_t, dot, spmv_vec, gemm): normwise error
    max_i |y_i - ref_i| / sum_j |term_ij| <= TOL (the interpreter's fp64 result as ref);
  * interpreter faults (E-INTERP) must surface as PencilError('E-INTERP').
"""
import numpy as np
import pytest

import oracle
from conftest import golden_cases, normwise_err

pytestmark = pytest.mark.gpu
TOL = 1e-5  # normwise, fp32 reductions (north star: "1e-5 fp32, scaled by reduction length")

CASES = golden_cases()


def reduction_scale(fn, a):
    """sum of |terms| feeding each output (the normwise denominator); 0 where the output is a
    plain copy of its input (must then match exactly)."""
    f64 = lambda t: np.abs(np.asarray(t, np.float64))  # noqa: E731
    if fn == "gemv":
        m, n, al, be, A, x, y = a
        return abs(al) * (f64(A).reshape(m, n) @ f64(x) if n else np.zeros(m)) + abs(be) * f64(y)
    if fn == "gemv_t":
        m, n, lda, ix, iy, al, be, A, x, y = a
        s = np.zeros(y.size)
        if m:
            At = f64(A).reshape(m, lda)[:, :n]
            s[np.arange(n) * iy] = abs(al) * (f64(x)[np.arange(m) * ix] @ At) + abs(be) * f64(y)[np.arange(n) * iy]
        else:
            s[np.arange(n) * iy] = abs(be) * f64(y)[np.arange(n) * iy] + 1e-300
        return s
    if fn == "dot":
        return np.array([np.sum(f64(a[1]) * f64(a[2]))])
    if fn == "axpy":
        return abs(a[1]) * f64(a[2]) + f64(a[3])
    if fn in ("spmv_vec", "spmv_inline", "spmv"):
        nrows, ncols, nnz, rp, col, val, x, _ = a
        terms = f64(val) * f64(x)[col] if nnz else np.zeros(0)
        cs = np.concatenate([[0.0], np.cumsum(terms)])
        return cs[rp[1:]] - cs[rp[:-1]]
    if fn == "conv5x5_f32":
        h, w, img, k, out = a
        s = np.zeros(h * w)
        I = f64(img).reshape(h, w)
        K = f64(k).reshape(5, 5)
        acc = np.zeros((h, w))
        for di in range(5):
            for dj in range(5):
                if h >= 5 and w >= 5:
                    acc[2:h - 2, 2:w - 2] += K[di, dj] * I[di:h - 4 + di, dj:w - 4 + dj]
        s[:] = acc.reshape(-1)
        return s
    if fn == "gemm":
        m, n, k, al, be, A, B, C = a
        return (abs(al) * (f64(A).reshape(m, k) @ f64(B).reshape(k, n)) + abs(be) * f64(C).reshape(m, n)).reshape(-1)
    raise KeyError(fn)


OUT_INDEX = {"gemv": 6, "gemv_t": 9, "axpy": 3, "spmv_vec": 7, "spmv_inline": 7, "spmv": 7,
             "conv5x5_u8": 5, "conv5x5_f32": 4, "gemm": 7}


def check(case, got, ret=None):
    fn, a = case.fn, case.args
    if fn == "dot":
        err = normwise_err([ret], [case.ret], reduction_scale(fn, a))
        assert err <= TOL, (case.name, err)
        return
    idx = OUT_INDEX[fn]
    ref = case.outs[idx]
    got = np.asarray(got)
    if fn == "conv5x5_u8":
        assert np.array_equal(got.astype(np.int64), ref), case.name
        return
    if fn in ("spmv_inline", "spmv"):
        exact = oracle.spmv_f32(a[0], a[1], a[2], a[3], a[4], a[5], a[6])
        assert np.array_equal(got.view(np.uint32), exact.view(np.uint32)), case.name
    elif fn == "axpy":
        exact = oracle.axpy_f32(a[0], a[1], a[2], a[3])
        assert np.array_equal(got.view(np.uint32), exact.view(np.uint32)), case.name
    elif fn == "conv5x5_f32":
        exact = oracle.conv5x5_f32_f32(a[0], a[1], a[2], a[3], a[4])
        assert np.array_equal(got.view(np.uint32), exact.view(np.uint32)), case.name
    if "intvals" in case.name:  # every partial sum exact in fp32: index handling bit-exact
        assert np.array_equal(got.astype(np.float64), ref), case.name
    err = normwise_err(got, ref, reduction_scale(fn, a))
    assert err <= TOL, (case.name, err)


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_golden_via_interpreter_mirror(cuda, case):
    import paper_1302_5586_b200 as pb
    it = pb.CudaInterpreter(0)
    args = []
    for i, a in enumerate(case.args):
        if isinstance(a, np.ndarray):
            it.set_array(f"a{i}", a)
            args.append(pb.Arg.array(f"a{i}"))
        else:
            args.append(pb.Arg.scalar(a))
    if case.fault:
        with pytest.raises(pb.PencilError) as ei:
            it.call(case.fn, args)
        assert ei.value.code == "E-INTERP"
        return
    ret = it.call(case.fn, args)
    if case.fn == "dot":
        check(case, None, ret)
    else:
        check(case, it.get_array(f"a{OUT_INDEX[case.fn]}"))
    assert it.fp_reordered() == (case.fn in ("gemv", "gemv_t", "dot", "spmv_vec", "gemm"))


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_golden_via_dropin_host(cuda, case):
    import paper_1302_5586_b200 as pb
    a = [x.copy() if isinstance(x, np.ndarray) else x for x in case.args]
    fn = getattr(pb.dropin, case.fn)
    if case.fault:
        with pytest.raises(pb.PencilError) as ei:
            fn(*a)
        assert ei.value.code == "E-INTERP"
        return
    ret = fn(*a)
    if case.fn == "dot":
        check(case, None, ret)
    else:
        check(case, a[OUT_INDEX[case.fn]])


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_golden_via_dropin_device(cuda, case):
    import paper_1302_5586_b200 as pb
    torch = cuda
    a = [torch.from_numpy(x.copy()).cuda() if isinstance(x, np.ndarray) else x for x in case.args]
    fn = getattr(pb.dropin, case.fn)
    if case.fault:
        with pytest.raises(pb.PencilError):
            fn(*a)
        return
    ret = fn(*a)
    if case.fn == "dot":
        check(case, None, ret)
    else:
        check(case, a[OUT_INDEX[case.fn]].cpu().numpy())


def test_library_loaded_in_tree(cuda):
    import paper_1302_5586_b200 as pb
    lib = pb.load()
    assert pb.LIB_PATH.endswith("paper_1302_5586_b200/lib/libpencil_b200.so")
    with open("/proc/self/maps") as f:
        assert pb.LIB_PATH in f.read()
    assert lib.pencil_version().startswith(b"pencil-b200")

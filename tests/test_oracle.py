"""Oracle tests (CPU).  The C restatement (oracle/pencil_oracle.c) must reproduce the reference
Interpreter's outputs BIT FOR BIT on every golden vector (tests/golden/*.npz were produced by the
reference's own pencil::Interpreter through oracle/_ref/ref_driver), and the reference-emitted
OpenMP C must agree with both — exactly for integer and source-order kernels."""
import os

import numpy as np
import pytest

import oracle
from conftest import golden_cases


def run_port(c):
    a = c.args
    f = c.fn
    if f == "gemv":
        return {6: oracle.gemv(*a[:4], a[4], a[5], a[6])}
    if f == "gemv_t":
        return {9: oracle.gemv_t(*a[:7], a[7], a[8], a[9])}
    if f == "dot":
        return {"ret": oracle.dot(a[0], a[1], a[2])}
    if f == "axpy":
        return {3: oracle.axpy(a[0], a[1], a[2], a[3])}
    if f in ("spmv_vec", "spmv_inline", "spmv"):
        return {7: oracle.spmv(a[0], a[1], a[2], a[3], a[4], a[5], a[6])}
    if f == "conv5x5_u8":
        return {5: oracle.conv5x5_u8(a[0], a[1], a[2], a[3], a[4])}
    if f == "conv5x5_f32":
        return {4: oracle.conv5x5_f32(a[0], a[1], a[2], a[3], a[4])}
    if f == "gemm":
        return {7: oracle.gemm(*a[:5], a[5], a[6], a[7])}
    raise KeyError(f)


CASES = golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_port_bit_exact_vs_reference_interpreter(case):
    if case.fault:
        with pytest.raises(oracle.OracleFault):
            run_port(case)
        return
    got = run_port(case)
    for key, val in got.items():
        if key == "ret":
            assert val == case.ret  # fp64 value, bit-identical
            continue
        ref = case.outs[key]
        assert val.dtype == ref.dtype
        assert np.array_equal(val.view(np.uint64) if val.dtype == np.float64 else val,
                              ref.view(np.uint64) if ref.dtype == np.float64 else ref), case.name


def test_golden_set_covers_every_fixture_function():
    fns = {c.fn for c in CASES}
    assert fns >= {"gemv", "gemv_t", "dot", "axpy", "spmv_vec", "spmv_inline", "spmv", "conv5x5_u8",
                   "conv5x5_f32", "gemm"}
    assert any(c.fault for c in CASES)


def test_interpreter_faults_are_pinned():
    names = {c.name for c in CASES if c.fault}
    assert {"fault_spmv_col_oob", "fault_conv_u8_scale0"} <= names


# ---- the reference CPU path (C emitted by emit_openmp) against the pinned oracle ---------
needs_emitted = pytest.mark.skipif(
    not os.path.exists(os.path.join(oracle.REF_DIR, "libpencil_omp_outer.so")),
    reason="oracle/_ref not built (needs /root/reference at build time)")


@needs_emitted
@pytest.mark.parametrize("variant", ["outer", "annot"])
def test_emitted_c_matches_oracle(variant):
    lib = oracle.emitted(variant)
    for c in CASES:
        if c.fault:
            continue
        a = [x.copy() if isinstance(x, np.ndarray) else x for x in c.args]
        P = lambda t: t.ctypes.data  # noqa: E731
        if c.fn in ("spmv_vec", "spmv_inline", "spmv"):
            getattr(lib, c.fn)(a[0], a[1], a[2], P(a[3]), P(a[4]), P(a[5]), P(a[6]), P(a[7]))
            exact = oracle.spmv_f32(a[0], a[1], a[2], a[3], a[4], a[5], a[6])
            # source-order fp32 mul+add: the emitted C compiled as written
            assert np.array_equal(a[7].view(np.uint32), exact.view(np.uint32)), (variant, c.name)
        elif c.fn == "conv5x5_u8":
            lib.conv5x5_u8(a[0], a[1], a[2], P(a[3]), P(a[4]), P(a[5]))
            assert np.array_equal(a[5].astype(np.int64), c.outs[5]), (variant, c.name)
        elif c.fn == "conv5x5_f32":
            lib.conv5x5_f32(a[0], a[1], P(a[2]), P(a[3]), P(a[4]))
            exact = oracle.conv5x5_f32_f32(a[0], a[1], c.args[2], c.args[3], c.args[4])
            assert np.array_equal(a[4].view(np.uint32), exact.view(np.uint32)), (variant, c.name)
        elif c.fn == "axpy":
            lib.axpy(a[0], a[1], P(a[2]), P(a[3]))
            exact = oracle.axpy_f32(a[0], a[1], c.args[2], c.args[3])
            assert np.array_equal(a[3].view(np.uint32), exact.view(np.uint32)), (variant, c.name)
        elif c.fn == "gemv":
            lib.gemv(a[0], a[1], a[2], a[3], P(a[4]), P(a[5]), P(a[6]))
            ref = c.outs[6]
            scale = abs(a[2]) * (np.abs(c.args[4].reshape(a[0], a[1]).astype(np.float64)) @
                                 np.abs(c.args[5].astype(np.float64))) + abs(a[3]) * np.abs(c.args[6])
            err = np.abs(a[6] - ref)
            assert np.all(err <= 1e-5 * scale + (scale == 0) * 0), (variant, c.name)
        elif c.fn == "dot":
            r = lib.dot(a[0], P(a[1]), P(a[2]))
            scale = float(np.sum(np.abs(c.args[1].astype(np.float64) * c.args[2])))
            assert abs(r - c.ret) <= 1e-5 * scale, (variant, c.name)

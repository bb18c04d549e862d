"""Summary-driven data movement: access summaries of the fixtures (read / write /
must-write-in-full, through calls and through the ACCESS summary of spmv_row —
summaries.cpp:635-663) and host-array calls that upload only what is read and download only what
is written (pencil_jit_call_host).
"""
import os

import numpy as np
import pytest

from conftest import golden_cases

FIX = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1302_5586_b200", "pencil")


def unit(name):
    from paper_1302_5586_b200.op2 import JitUnit
    return JitUnit(open(os.path.join(FIX, name + ".pencil.c")).read())


EXPECTED = {
    ("gemv", "gemv"): {"A": ("r", False), "x": ("r", False), "y": ("rw", False)},
    ("axpy", "axpy"): {"x": ("r", False), "y": ("rw", False)},
    ("dot", "dot"): {"x": ("r", False), "y": ("r", False)},
    ("gemm", "gemm"): {"A": ("r", False), "B": ("r", False), "C": ("rw", False)},
    ("conv5x5", "conv5x5_f32"): {"img": ("r", False), "k": ("r", False), "out": ("w", False)},  # interior only
    ("conv5x5", "conv5x5_u8"): {"img": ("r", False), "k": ("r", False), "out": ("w", True)},  # every pixel
    ("spmv", "spmv_vec"): {"rowptr": ("r", False), "col": ("r", False), "val": ("r", False), "x": ("r", False),
                           "y": ("w", True)},
    # the driver writes y only through spmv_row, whose ACCESS summary says DEF(y[i]): must-written in full
    ("spmv", "spmv"): {"rowptr": ("r", False), "col": ("r", False), "val": ("r", False), "x": ("r", False),
                       "y": ("w", True)},
}


@pytest.mark.parametrize("fixture,fn", sorted(EXPECTED))
def test_access_summaries(fixture, fn):
    assert unit(fixture).access(fn) == EXPECTED[(fixture, fn)]


# small concrete bindings under which the reference computes the access sets
BINDINGS = {
    ("gemv", "gemv"): {"m": 2, "n": 3},
    ("gemv_t", "gemv_t"): {"m": 3, "n": 2, "lda": 4, "incx": 2, "incy": 3},
    ("axpy", "axpy"): {"n": 5},
    ("dot", "dot"): {"n": 5},
    ("gemm", "gemm"): {"m": 2, "n": 3, "k": 2},
    ("conv5x5", "conv5x5_u8"): {"h": 6, "w": 7},
    ("conv5x5", "conv5x5_f32"): {"h": 6, "w": 7},
    ("spmv", "spmv_vec"): {"nrows": 3, "ncols": 3, "nnz": 4},
    ("spmv", "spmv_inline"): {"nrows": 3, "ncols": 3, "nnz": 4},
    ("spmv", "spmv"): {"nrows": 3, "ncols": 3, "nnz": 4},
    ("spmv", "spmv_row"): {"nrows": 3, "ncols": 3, "nnz": 4, "i": 1},
}
CSR = {"rowptr": [0, 1, 3, 4], "col": [0, 0, 2, 1]}


def reference_access(fixture, fn, scalars):
    """The reference's summarize_call (summaries.cpp:635-648) of fn(params...) under `scalars`
    (oracle/_ref/ref_driver summarize): per array parameter, mode r / w / rw and whether the
    must-write set is the whole declared extent with no read (the data plan's "written in full,
    no upload needed")."""
    import json
    import subprocess
    import oracle
    cmd = [oracle.REF_DRIVER, "summarize", os.path.join(FIX, fixture + ".pencil.c"), fn]
    for k, v in scalars.items():
        cmd += ["--param", f"{k}={v}"]
    if fixture == "spmv":
        for k, v in CSR.items():
            cmd += ["--array", k + "=" + ",".join(map(str, v))]
    r = subprocess.run(cmd, capture_output=True, text=True, check=True)
    sig = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "signatures.json")))[fn]
    extents = {p.split(":")[0]: p.split(":")[3] for p in sig.split(";")[1:] if p.split(":")[1] == "array"}
    out = {}
    for line in r.stdout.splitlines():
        a = json.loads(line)
        n = eval(extents[a["array"]], {}, dict(scalars))  # extents are products / sums of scalars
        mode = ("r" if a["read"] else "") + ("w" if (a["must"] or a["may"]) else "")
        full = not a["read"] and not a["unknown"] and a["must"] == list(range(n))
        out[a["array"]] = (mode or "-", full)
    return out


@pytest.mark.parametrize("fixture,fn", sorted(BINDINGS))
def test_access_summaries_equal_reference_summarize_call(fixture, fn):
    """The product's summaries (pencil_jit_access: symbolic, used for every call) equal the
    reference's concrete summarize_call sets on a small binding, array by array — read / write
    mode and must-written-in-full."""
    import oracle
    if not os.path.exists(oracle.REF_DRIVER):
        pytest.skip("oracle/_ref not built")
    ours = unit(fixture).access(fn)
    ref = reference_access(fixture, fn, BINDINGS[(fixture, fn)])
    assert {k: v for k, v in ours.items() if v[0] != "-"} == {k: v for k, v in ref.items() if v[0] != "-"}


SPMV = [c for c in golden_cases("spmv") if c.fn == "spmv" and not c.fault]


@pytest.mark.gpu
@pytest.mark.parametrize("case", SPMV, ids=[c.name for c in SPMV])
def test_host_call_moves_only_what_the_summary_needs(cuda, case):
    u = unit("spmv")
    args = [a.copy() if isinstance(a, np.ndarray) else a for a in case.args]
    y = args[-1]
    y[:] = np.nan  # never uploaded: must be fully overwritten
    ret, (h2d, d2h) = u.call_host("spmv", args)
    ref = case.outs[len(args) - 1]
    assert np.array_equal(y.astype(np.float64), ref.astype(np.float32).astype(np.float64))
    inputs = sum(a.nbytes for a in args[3:-1])
    assert h2d == inputs and d2h == y.nbytes

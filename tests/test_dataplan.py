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
    ("spmv", "spmv_vec"): {"rowptr": ("r", False), "col": ("r", False), "val": ("r", False), "x": ("r", False),
                           "y": ("w", True)},
    # the driver writes y only through spmv_row, whose ACCESS summary says DEF(y[i]): must-written in full
    ("spmv", "spmv"): {"rowptr": ("r", False), "col": ("r", False), "val": ("r", False), "x": ("r", False),
                       "y": ("w", True)},
}


@pytest.mark.parametrize("fixture,fn", sorted(EXPECTED))
def test_access_summaries(fixture, fn):
    assert unit(fixture).access(fn) == EXPECTED[(fixture, fn)]


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

"""The C++ secondary boundary: pencil_b200::CudaInterpreter
(include/pencil_cuda_interpreter.hpp), compiled against the REFERENCE's interp.hpp / ast / printer
and linked with libpencil_b200.so (oracle/_ref/cuda_interp_check, built from oracle/Makefile).
The reference's own Interpreter known-answer cases (proj/tests/test_interp.cpp:8-108: arithmetic,
arrays shared through calls, loops, while, rand sequence + LCG, trace, float, OOB fault, unknown
function, step budget) and two fixture kernels run through the reference Interpreter and the CUDA
one side by side.  CPU: the restated cases pass on the reference itself.  GPU: they pass on the
CUDA interpreter too, with the same arrays, trace and PencilError codes."""
import os
import subprocess

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(os.path.dirname(oracle.REF_DRIVER), "cuda_interp_check")
FIX = os.path.join(ROOT, "paper_1302_5586_b200", "pencil")


def run():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/cuda_interp_check not built")
    r = subprocess.run([BIN, FIX], capture_output=True, text=True, timeout=600)
    return r, [l for l in r.stdout.splitlines() if l.startswith(("ok", "FAIL"))]


def test_known_answer_cases_pass_on_the_reference_interpreter():
    r, lines = run()
    ref = [l for l in lines if l.endswith("[reference]")]
    assert len(ref) == 14, r.stdout
    assert all(l.startswith("ok") for l in ref), r.stdout


@pytest.mark.gpu
def test_known_answer_cases_pass_on_the_cuda_interpreter(cuda):
    r, lines = run()
    assert r.returncode == 0, r.stdout + r.stderr
    cu = [l for l in lines if l.endswith("[cuda]")]
    assert len(cu) == 14 and all(l.startswith("ok") for l in cu), r.stdout

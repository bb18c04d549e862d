"""The reference's own Interpreter tests (tests/test_interp.cpp: arithmetic, arrays shared through
calls, loops and conditionals, while, rand sequence then LCG, floats, out-of-bounds store,
unknown function, step budget) replayed through the general mapper on the GPU."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def unit(src):
    from paper_1302_5586_b200.op2 import JitUnit
    return JitUnit(src)


def test_arithmetic_and_return(cuda):
    u = unit("int f(int a, int b)\n{\n  int r;\n  r = a * b + a / b - a % b;\n  return r;\n}\n")
    assert u.call("f", [7, 3]) == 7 * 3 + 7 // 3 - 7 % 3


def test_arrays_are_shared_through_calls(cuda):
    from paper_1302_5586_b200 import Arg
    u = unit("void set(int n, int A[restrict const static n])\n{\n  A[1] = 42;\n}\n"
             "void run(int n, int A[restrict const static n])\n{\n  set(n, A);\n  A[0] = A[1];\n}\n")
    u.set_array("mem", np.zeros(3, np.int32))
    u.call("run", [3, Arg.array("mem")])
    assert u.get_array("mem")[1][:2].tolist() == [42, 42]


def test_loops_and_conditionals(cuda):
    u = unit("int tri(int n)\n{\n  int s;\n  int i;\n  s = 0;\n"
             "  for (i = 1; i <= n; i++) {\n    if (i % 2 == 0) {\n      s += i;\n    }\n  }\n  return s;\n}\n")
    assert u.call("tri", [6]) == 2 + 4 + 6


def test_while_loop(cuda):
    u = unit("int halve(int n)\n{\n  int c;\n  c = 0;\n  while (n > 1) {\n    n = n / 2;\n    c += 1;\n  }\n"
             "  return c;\n}\n")
    assert u.call("halve", [16]) == 4


def test_rand_pops_sequence_then_lcg(cuda):
    from paper_1302_5586_b200 import Arg
    src = ("void take(int n, int A[restrict const static n])\n{\n  int i;\n"
           "  for (i = 0; i < n; i++) {\n    A[i] = rand();\n  }\n}\n")
    outs = []
    for _ in range(2):
        u = unit(src)
        u.set_array("A", np.zeros(5, np.int32))
        u.set_rand_sequence([9, 8])
        u.call("take", [5, Arg.array("A")])
        outs.append(u.get_array("A")[1].tolist())
    assert outs[0][:2] == [9, 8] and outs[0] == outs[1]
    # the fallback is the interpreter's LCG from its seed (interp.hpp:67)
    s, ref = 0x9e3779b97f4a7c15, []
    for _ in range(3):
        s = (s * 6364136223846793005 + 1442695040888963407) % (1 << 64)
        ref.append((s >> 33) & 0x7fffffff)
    assert outs[0][2:] == ref


def test_floating_point_values(cuda):
    u = unit("float scale(float x)\n{\n  return x * 0.5;\n}\n")
    assert u.call("scale", [3.0]) == 1.5


def test_out_of_bounds_store_faults(cuda):
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import Arg
    u = unit("void f(int n, int A[restrict const static n])\n{\n  A[n] = 1;\n}\n")
    u.set_array("A", np.zeros(2, np.int32))
    with pytest.raises(pb.PencilError) as e:
        u.call("f", [2, Arg.array("A")])
    assert e.value.code == "E-INTERP"


def test_unknown_function_faults(cuda):
    import paper_1302_5586_b200 as pb
    u = unit("void f(int n)\n{\n}\n")
    with pytest.raises(pb.PencilError) as e:
        u.call("nope", [])
    assert e.value.code == "E-INTERP"


def test_step_budget_stops_runaway_loops(cuda):
    import paper_1302_5586_b200 as pb
    u = unit("void spin(int n)\n{\n  while (n < 1) {\n    n = n - 1;\n  }\n}\n")
    with pytest.raises(pb.PencilError) as e:
        u.call("spin", [0])
    assert e.value.code == "E-INTERP" and "budget" in str(e.value)


def test_rand_sequence_survives_call_buffer_growth(cuda):
    """set_rand_sequence, then calls that grow the unit's call buffers (a reduction over many
    threads) before and between the rand() calls: the sequence must still be read intact, and
    a second sequence replaces the first (regression: buffer growth used to free it)."""
    import torch
    from paper_1302_5586_b200 import Arg
    src = ("void take(int n, int A[restrict const static n])\n{\n  int i;\n"
           "  for (i = 0; i < n; i++) {\n    A[i] = rand();\n  }\n}\n"
           "int big(int n, int B[restrict const static n])\n{\n  int i;\n  int s;\n  s = 0;\n"
           "  #pragma pencil reduction (+: s)\n  for (i = 0; i < n; i++) {\n    s += B[i];\n  }\n  return s;\n}\n")
    u = unit(src)
    seq = list(range(1000, 1300))
    u.set_rand_sequence(seq)
    u.set_array("B", np.ones(1 << 20, np.int32))
    assert u.call("big", [1 << 20, Arg.array("B")]) == 1 << 20
    junk = torch.full((1 << 22,), -7, dtype=torch.int64, device="cuda")  # reuse freed memory, if any
    torch.cuda.synchronize()
    u.set_array("A", np.zeros(300, np.int32))
    u.call("take", [300, Arg.array("A")])
    assert u.get_array("A")[1].tolist() == seq
    u.set_rand_sequence([5, 6, 7])
    u.call("take", [3, Arg.array("A")])
    assert u.get_array("A")[1][:3].tolist() == [5, 6, 7]
    del junk


def test_trace_records_reads_and_writes_in_order(cuda):
    """test_interp.cpp:64-80 through the Python surface of the JIT (enable_trace / trace)."""
    from paper_1302_5586_b200 import Arg
    u = unit("void copy(int n, int A[restrict const static n], int B[restrict const static n])\n"
             "{\n  A[0] = B[1];\n}\n")
    u.set_array("A", np.zeros(2, np.int32))
    u.set_array("B", np.array([5, 6], np.int32))
    u.enable_trace(True)
    u.call("copy", [2, Arg.array("A"), Arg.array("B")])
    assert u.trace() == [("B", [1], False), ("A", [0], True)]


def test_trace_of_a_parallel_loop_is_sequential(cuda):
    """With the trace on, an `independent` loop runs in the interpreter's order (one device thread):
    records i = 0, 1, 2, ... each a read of x[i] then a write of y[i]; mixed int / float values
    set with set_array_values keep their types."""
    from paper_1302_5586_b200 import Arg
    u = unit("void sc(int n, float x[restrict const static n], float y[restrict const static n])\n{\n"
             "  #pragma pencil independent\n  for (int i = 0; i < n; i++) {\n    y[i] = x[i] * 2;\n  }\n}\n")
    u.set_array_values("x", [1, 2.5, -3, 0.25])
    u.set_array("y", np.zeros(4, np.float32))
    u.enable_trace(True)
    u.call("sc", [4, Arg.array("x"), Arg.array("y")])
    exp = []
    for i in range(4):
        exp += [("x", [i], False), ("y", [i], True)]
    assert u.trace() == exp
    vals, ints, isd = u.get_array("y")
    assert vals.tolist() == [2.0, 5.0, -6.0, 0.5] and isd.tolist() == [False, True, False, True]
    u.enable_trace(False)
    u.call("sc", [4, Arg.array("x"), Arg.array("y")])
    assert len(u.trace()) == 8  # off: nothing recorded, earlier records kept


def test_binary_operands_in_the_reference_binarys_order(cuda):
    """The reference evaluates `a - b` as arith(op, eval(a), eval(b)), argument order unspecified in
    C++; its g++ build evaluates b first.  rand() draws expose the order: the GPU result must equal
    oracle/_ref/ref_driver's (the reference itself) for the LCG's first two draws."""
    import os
    import subprocess
    import tempfile
    import oracle
    if not os.path.exists(oracle.REF_DRIVER):
        pytest.skip("oracle/_ref not built")
    src = "int f(void)\n{\n  int r;\n  r = rand() - 2 * rand();\n  return r;\n}\n"
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "u.pencil.c")
        open(p, "w").write(src)
        r = subprocess.run([oracle.REF_DRIVER, "run", p, "f"], input="", capture_output=True, text=True)
    ref = int(r.stdout.split()[-1])
    assert unit(src).call("f", []) == ref

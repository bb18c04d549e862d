"""30 random PENCIL functions over float arrays and double scalars
(tests/golden/make_random_float_units.py) through the general mapper, bit-identical to the
REFERENCE Interpreter: fp64 operations in the interpreter's order (NVRTC --fmad=false), the
int/double typing rules, truncating integer division, conditionals and while loops on doubles.
No licensed reductions occur, so every schedule must reproduce the sequential bits."""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "random_float_units.json")))


def unhex(vals):
    return np.array([float.fromhex(v) for v in vals], np.float64)


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(CASES)))
def test_random_float_unit_matches_reference(cuda, k):
    from paper_1302_5586_b200 import Arg
    from paper_1302_5586_b200.op2 import JitUnit
    c = CASES[k]
    u = JitUnit(c["src"])
    for name in ("A", "B", "t"):
        u.set_array(name, np.asarray(c[name], np.float32))
    ret = u.call("f", [c["n"], Arg.array("A"), Arg.array("B"), Arg.array("t")])
    assert float(ret).hex() == c["ret"]
    for name in ("A", "B"):
        vals, ints, is_double = u.get_array(name)
        got = np.where(np.asarray(is_double, bool), np.asarray(vals, np.float64), np.asarray(ints, np.float64))
        want = unhex(c[name + "_out"])
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), name


def test_random_float_units_use_parallel_schedules():
    from paper_1302_5586_b200.op2 import JitUnit
    seen = set()
    for c in CASES:
        seen.update(JitUnit(c["src"]).schedule("f"))
    assert {"S", "P"} <= seen

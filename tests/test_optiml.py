"""OptiML constructs: lowered to PENCIL (pencil_optiml_lower) and run on the GPU by
the general mapper.

CPU: the documented error codes; the mapper's schedule equals the reference's documented analysis
outcome (docs/op2-input.md table); the lowered units pass the REFERENCE checker and its analyzer
gives those verdicts.
GPU: vector / gradient (batch, stochastic) results equal the REFERENCE Interpreter's on the same
unit (oracle/_ref/ref_driver run), bit for bit.
"""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

import oracle

CONSTRUCTS = {
    "sum": ({"kind": "sum", "lo": 1, "hi": 100, "body": "exp"}, "optiml_sum", "SR", "PARALLEL_WITH_REDUCTION"),
    "vector": ({"kind": "vector", "lo": 3, "hi": 1000, "init": 7}, "optiml_vector", "SP", "PARALLEL"),
    "untilconverged": ({"kind": "untilconverged", "threshold": 0.5}, "optiml_untilconverged", "S", "UNKNOWN"),
    "batch": ({"kind": "gradient", "variant": "batch"}, "optiml_gradient_batch", "SP", "ASSUMED_PARALLEL"),
    "stochastic": ({"kind": "gradient", "variant": "stochastic"}, "optiml_gradient_stochastic", "S", None),
}


def lower(c):
    from paper_1302_5586_b200.op2 import optiml_lower
    return optiml_lower(c)


@pytest.mark.parametrize("doc,code", [
    ({"kind": "sum", "lo": 5, "hi": 1}, "E-OPTIML-RANGE"),
    ({"kind": "nope"}, "E-OPTIML-SHAPE"),
    ({"kind": "gradient", "variant": "minibatch"}, "E-OPTIML-SHAPE"),
    ({"lo": 1}, "E-OPTIML-SHAPE"),
    ("[1, 2]", "E-OPTIML-SHAPE"),
])
def test_errors(doc, code):
    import paper_1302_5586_b200 as pb
    with pytest.raises(pb.PencilError) as e:
        lower(doc)
    assert e.value.code == code


@pytest.mark.parametrize("name", sorted(CONSTRUCTS))
def test_schedule_matches_documented_analysis(name):
    from paper_1302_5586_b200.op2 import JitUnit
    doc, fn, sched, verdict = CONSTRUCTS[name]
    src = lower(doc)
    assert JitUnit(src).schedule(fn) == sched
    if not os.path.exists(oracle.REF_DRIVER):
        pytest.skip("oracle/_ref not built")
    with tempfile.NamedTemporaryFile("w", suffix=".pencil.c", delete=False) as f:
        f.write(src)
    try:
        chk = subprocess.run([oracle.REF_DRIVER, "check", f.name], capture_output=True, text=True)
        assert chk.returncode == 0, chk.stdout + chk.stderr
        an = subprocess.run([oracle.REF_DRIVER, "analyze", f.name], capture_output=True, text=True)
    finally:
        os.unlink(f.name)
    reps = [json.loads(x) for x in an.stdout.splitlines() if x.strip()]
    if verdict is not None:
        assert [r["verdict"] for r in reps] == [verdict], an.stdout
    else:  # stochastic: sequential (UNKNOWN without a binding, SERIAL once bound)
        assert reps[0]["verdict"] in ("UNKNOWN", "SERIAL")


def _reference(src, fn, args):
    """Run `fn` of the unit text in the reference Interpreter (ref_driver run)."""
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "u.pencil.c")
        open(path, "w").write(src)
        lines, paths = [], {}
        for i, a in enumerate(args):
            if isinstance(a, np.ndarray):
                p = os.path.join(td, f"a{i}.bin")
                a.tofile(p)
                lines.append(f"array {'f32' if a.dtype == np.float32 else 'i32'} {p}")
                paths[i] = (p, a.dtype)
            else:
                lines.append(f"scalar {'int' if isinstance(a, int) else 'float'} {a!r}")
        r = subprocess.run([oracle.REF_DRIVER, "run", path, fn], input="\n".join(lines) + "\n",
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        return {i: np.fromfile(p + ".out", np.float64 if dt == np.float32 else np.int64)
                for i, (p, dt) in paths.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["vector", "batch", "stochastic"])
def test_constructs_on_gpu_equal_reference(cuda, name):
    """tests/golden/optiml/<name>.npz: the reference Interpreter's outputs (make_optiml_golden.py)."""
    from paper_1302_5586_b200 import Arg
    from paper_1302_5586_b200.op2 import JitUnit
    doc, fn, _, _ = CONSTRUCTS[name]
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "optiml", f"{name}.npz"))
    u = JitUnit(lower(doc))
    n = int(z["n"])
    cargs = [n]
    ins = sorted(k for k in z.files if k.startswith("in"))
    for k in ins:
        u.set_array(k, z[k])
        cargs.append(Arg.array(k))
    u.call(fn, cargs)
    for k in ins:
        ref = z["out" + k[2:]]
        vals, ints, isd = u.get_array(k)
        if ref.dtype == np.int64:
            assert np.array_equal(ints, ref)
        else:
            assert np.array_equal(vals.view(np.uint64), ref.view(np.uint64))

"""OptiML constructs: lowered to PENCIL (pencil_optiml_lower) and run on the GPU by
the general mapper.

CPU: the documented error codes; the mapper's schedule equals the reference's documented analysis
outcome (docs/op2-input.md table); the lowered units pass the REFERENCE checker and its analyzer
gives those verdicts.
GPU: vector / gradient (batch, stochastic) results equal the REFERENCE Interpreter's on the same
unit (oracle/_ref/ref_driver run), bit for bit; the sum (the reduction construct, exp body) within a
stated ulp bound of it.
Pinned to the reference's own OptiML module (core/src/optiml.cpp compiled into
oracle/_ref/ref_op2_driver): the lowered text equals lower_optiml's and the error codes match.
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


# --------------------------------------------- the reference's own OptiML module (ref_op2_driver)
REF_OP2 = os.path.join(os.path.dirname(oracle.REF_DRIVER), "ref_op2_driver")
SUM_RANGES = [(1, 100), (1, 1), (-50, 50), (0, 700), (-745, -700)]
LOWER_DOCS = [c[0] for c in CONSTRUCTS.values()] + \
    [{"kind": "sum", "lo": lo, "hi": hi, "body": "exp"} for lo, hi in SUM_RANGES] + \
    [{"kind": "vector", "lo": 0, "hi": 0, "init": -3}, {"kind": "untilconverged", "threshold": 1e-9}]


def ref_optiml(cmd, doc):
    if not os.path.exists(REF_OP2):
        pytest.skip("oracle/_ref not built")
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        f.write(doc if isinstance(doc, str) else json.dumps(doc))
    try:
        return subprocess.run([REF_OP2, cmd, f.name], capture_output=True, text=True)
    finally:
        os.unlink(f.name)


@pytest.mark.parametrize("doc", LOWER_DOCS, ids=[json.dumps(d, sort_keys=True) for d in LOWER_DOCS])
def test_lowering_equals_reference_lower_optiml(doc):
    """pencil_optiml_lower's unit is the reference's lower_optiml (optiml.cpp:94-139), compiled
    from the reference sources: equal in the reference printer's canonical form."""
    ref = ref_optiml("optiml-lower", doc)
    assert ref.returncode == 0, ref.stdout
    canon = ref_optiml("canon", lower(doc))
    assert canon.returncode == 0
    assert canon.stdout == ref.stdout


@pytest.mark.parametrize("doc,code", [
    ({"kind": "sum", "lo": 5, "hi": 1}, "E-OPTIML-RANGE"),
    ({"kind": "nope"}, "E-OPTIML-SHAPE"),
    ({"kind": "gradient", "variant": "minibatch"}, "E-OPTIML-SHAPE"),
    ({"lo": 1}, "E-OPTIML-SHAPE"),
    ("[1, 2]", "E-OPTIML-SHAPE"),
])
def test_error_codes_equal_reference(doc, code):
    r = ref_optiml("optiml-lower", doc)
    assert r.returncode == 3 and r.stdout.split()[1] == code, r.stdout


def returning_sum(src):
    """The lowered sum unit with x returned (lower_optiml's optiml_sum keeps x local, so neither
    the reference nor the GPU exposes it): `void optiml_sum(void)` -> `double`, `return x;` last."""
    head = "void optiml_sum(void)"
    assert head in src
    body_end = src.rindex("}")
    return src[:body_end].replace(head, "double optiml_sum(void)") + "  return x;\n}\n"


@pytest.mark.gpu
@pytest.mark.parametrize("lo,hi", SUM_RANGES)
def test_sum_on_gpu_within_ulp_bound_of_reference(cuda, lo, hi):
    """The reduction construct (x = f(lo); reduction(+: x) over i in (lo, hi]; f = exp) on the GPU
    against the reference Interpreter on the same unit.  Bound: the GPU's exp is within 1 ulp
    (CUDA double exp) and the licensed reduction reassociates the n = hi - lo + 1 terms, so
    |gpu - ref| <= (2n + 2) * 2^-53 * sum|exp(i)| — the standard recursive-summation bound
    (n - 1) eps sum|t_i| plus one ulp per term and the reference's own rounding."""
    from paper_1302_5586_b200.op2 import JitUnit
    src = returning_sum(lower({"kind": "sum", "lo": lo, "hi": hi, "body": "exp"}))
    ref = None
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "u.pencil.c")
        open(path, "w").write(src)
        r = subprocess.run([oracle.REF_DRIVER, "run", path, "optiml_sum"], input="", capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        ref = float(r.stdout.split()[-1])
    u = JitUnit(src)
    assert u.schedule("optiml_sum") == "SRS"  # serial init, the reduction loop, the return
    got = u.call("optiml_sum", [])
    n = hi - lo + 1
    mag = float(np.sum(np.exp(np.arange(lo, hi + 1, dtype=np.float64))))
    bound = (2 * n + 2) * 2.0 ** -53 * mag
    assert abs(got - ref) <= bound, (got, ref, abs(got - ref) / bound)

"""OP2 mesh loops: the reference's mesh model executed on the GPU.

CPU (no GPU needed): model validation with the reference's codes (tests/test_op2.cpp of the
reference: E-OP2-RANGE / -SHAPE / -KERNEL / -CONFLICT), the schedule chosen per par_loop, and
the product's lowering checked by the REFERENCE checker and analyzer (compliant; the increment
loop analyses as PARALLEL_WITH_REDUCTION on dcells, as test_op2.cpp "increment loops analyze
as reductions, never serial" requires).
GPU: every case of tests/golden/op2_cases.json (the reference Interpreter's results, generated
by make_op2_golden.py) bit-exact through Op2Model.run(), faults as E-INTERP, and a full-size
mesh against the numpy restatement.
"""
import copy
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

import oracle
from oracle import op2_ref

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "op2_cases.json")))


def model(doc):
    from paper_1302_5586_b200.op2 import Op2Model
    return Op2Model(doc)


def err_code(doc):
    import paper_1302_5586_b200 as pb
    with pytest.raises(pb.PencilError) as e:
        model(doc)
    return e.value.code


# ---------------------------------------------------------------- load / validate (CPU)
def test_mesh_loads_with_declared_shape():
    m = model(CASES["mesh"]["doc"])
    assert m.num_loops == 1
    assert m.dat("dcells").tolist() == [1, 2, 3]  # before any run: the document's data
    assert m.loop_info(0) == ("parallel", 1)


def test_map_entry_outside_target_set():
    d = copy.deepcopy(CASES["mesh"]["doc"])
    d["maps"][0]["table"] = [0, 1, 1, 5]
    assert err_code(d) == "E-OP2-RANGE"


def test_dat_with_wrong_number_of_values():
    d = copy.deepcopy(CASES["mesh"]["doc"])
    d["dats"][0]["data"] = [1, 2, 3, 4]
    assert err_code(d) == "E-OP2-SHAPE"


def test_arg_offset_outside_map_arity():
    d = copy.deepcopy(CASES["mesh"]["doc"])
    d["par_loops"][0]["args"][2]["offset"] = 2
    assert err_code(d) == "E-OP2-RANGE"


def test_kernel_with_mismatched_signature():
    d = copy.deepcopy(CASES["mesh"]["doc"])
    src = d["kernels"][0]["source"].replace(", int ic1", "").replace("dcells[ic1]", "dcells[ic0]")
    d["kernels"][0]["source"] = src
    assert err_code(d) == "E-OP2-KERNEL"


def test_dat_incremented_and_overwritten_conflicts():
    d = copy.deepcopy(CASES["mesh"]["doc"])
    d["par_loops"][0]["args"][1]["access"] = "OP_RW"
    assert err_code(d) == "E-OP2-CONFLICT"


@pytest.mark.parametrize("text,code", [
    ("[1, 2]", "E-OP2-SHAPE"),                                   # not an object
    ('{"sets": [{"name": "a", "size": -1}]}', "E-OP2-SHAPE"),
    ('{"sets": [{"name": "a", "size": 1}, {"name": "a", "size": 2}]}', "E-OP2-SHAPE"),
])
def test_malformed_documents(text, code):
    assert err_code(text) == code


def test_kernel_that_does_not_parse():
    d = copy.deepcopy(CASES["mesh"]["doc"])
    d["kernels"][0]["source"] = d["kernels"][0]["source"].replace("+=", "+== ")
    assert err_code(d) == "E-OP2-KERNEL"


@pytest.mark.parametrize("name,strategies", [
    ("mesh", ["parallel"]),
    ("random_increments", ["parallel"]),
    ("helper_function_alias", ["parallel"]),
    ("inc_dat_also_read_serial", ["serial"]),
    ("rand_serial", ["serial"]),
    ("multi_loop_levels", ["parallel", "parallel", "levels"]),
])
def test_schedule_per_par_loop(name, strategies):
    m = model(CASES[name]["doc"])
    assert [m.loop_info(i)[0] for i in range(m.num_loops)] == strategies


def _ref(cmd, src, *extra):
    if not os.path.exists(oracle.REF_DRIVER):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    with tempfile.NamedTemporaryFile("w", suffix=".pencil.c", delete=False) as f:
        f.write(src)
    try:
        return subprocess.run([oracle.REF_DRIVER, cmd, f.name, *extra], capture_output=True, text=True)
    finally:
        os.unlink(f.name)


def test_lowering_is_compliant_and_analyzes_as_reduction():
    doc = CASES["mesh"]["doc"]
    m = model(doc)
    low = m.lowered
    assert "void kernel_loop(int n_iter, int n_dedges, int n_dcells, int n_pecell," in low
    assert "#pragma pencil reduction (+: dcells)" in low
    assert "kernel(n_dedges, n_dcells, dedges, dcells, i, pecell[2 * i + 0], pecell[2 * i + 1]);" in low
    chk = _ref("check", low)
    assert chk.returncode == 0, chk.stdout + chk.stderr
    args = ["--param", "n_iter=2", "--param", "n_dedges=2", "--param", "n_dcells=3", "--param", "n_pecell=4",
            "--array", "pecell=0,1,1,2", "--array", "dcells=1,2,3", "--array", "dedges=10,20"]
    an = _ref("analyze", low, *args)
    reps = [json.loads(line) for line in an.stdout.splitlines() if line.strip()]
    drv = [r for r in reps if r["function"] == "kernel_loop"]
    assert len(drv) == 1 and drv[0]["verdict"] == "PARALLEL_WITH_REDUCTION", an.stdout
    assert drv[0]["reduction_vars"] == "dcells"


def test_product_lowering_runs_to_the_reference_result():
    """The product's lowered unit, executed by the reference Interpreter, gives the golden dats."""
    if not os.path.exists(oracle.REF_DRIVER):
        pytest.skip("oracle/_ref not built")
    doc = CASES["multi_loop_levels"]["doc"]
    src = model(doc).lowered
    # same op2_main wrapper as the oracle, but calling the product's `<kernel>_loop` drivers
    osrc, arrays, sizes = op2_ref.lower_unit(doc)
    main = osrc[osrc.index("void op2_main("):]
    for li, L in enumerate(doc["par_loops"]):
        main = main.replace(f"{L['kernel']}_loop{li}(", f"{L['kernel']}_loop(")
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "u.pencil.c")
        open(path, "w").write(src + "\n" + main)
        content = {d["name"]: d["data"] for d in doc["dats"]}
        content.update({mm["name"]: mm["table"] for mm in doc["maps"]})
        lines = [f"scalar int {n}" for n in sizes]
        for a in arrays:
            p = os.path.join(td, a + ".bin")
            np.asarray(content[a], np.int32).tofile(p)
            lines.append(f"array i32 {p}")
        r = subprocess.run([oracle.REF_DRIVER, "run", path, "op2_main"], input="\n".join(lines) + "\n",
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        for d in doc["dats"]:
            got = np.fromfile(os.path.join(td, d["name"] + ".bin.out"), np.int64)
            assert got.tolist() == CASES["multi_loop_levels"]["result"][d["name"]]


# ------------------------------------------- the reference's own OP2 module (oracle/_ref/ref_op2_driver)
REF_OP2 = os.path.join(os.path.dirname(oracle.REF_DRIVER), "ref_op2_driver")


def ref_op2(cmd, doc_or_text):
    if not os.path.exists(REF_OP2):
        pytest.skip("oracle/_ref not built")
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        f.write(doc_or_text if isinstance(doc_or_text, str) else json.dumps(doc_or_text))
    try:
        return subprocess.run([REF_OP2, cmd, f.name], capture_output=True, text=True)
    finally:
        os.unlink(f.name)


ALL_DOCS = {**{k: v for k, v in CASES.items()}, **{"random_" + k: v for k, v in
                                                    json.load(open(os.path.join(HERE, "golden", "op2_random.json"))).items()}}


@pytest.mark.parametrize("name", sorted(ALL_DOCS))
def test_lowering_equals_reference_lower_op2_model(name):
    """The product's lowered unit (pencil_op2_lowered) is the reference's lower_op2_model
    (op2.cpp:244-346) statement for statement: both in the reference printer's canonical form
    (pretty_print of the parsed unit), compiled from the reference sources."""
    doc = ALL_DOCS[name]["doc"]
    ref = ref_op2("op2-lower", doc)
    assert ref.returncode == 0, ref.stdout + ref.stderr
    ref_unit = "".join(l + "\n" for l in ref.stdout.splitlines() if not l.startswith("driver "))
    canon = ref_op2("canon", model(doc).lowered)
    assert canon.returncode == 0
    assert canon.stdout == ref_unit


@pytest.mark.parametrize("name", sorted(ALL_DOCS))
def test_golden_results_are_the_reference_interpret_op2_reference(name):
    """The golden dats (and faults) the GPU tests compare against are what the reference's own
    interpret_op2_reference (op2.cpp:388-429) computes for the model."""
    case = ALL_DOCS[name]
    r = ref_op2("op2-run", case["doc"])
    if "fault" in case:
        assert r.returncode == 3 and r.stdout.startswith("error E-INTERP"), r.stdout
        return
    assert r.returncode == 0, r.stdout + r.stderr
    got = json.loads(r.stdout)
    for k, v in case["result"].items():
        assert got[k] == v, k


@pytest.mark.parametrize("mutate,code", [
    (lambda d: d["maps"][0].__setitem__("table", [0, 1, 1, 5]), "E-OP2-RANGE"),
    (lambda d: d["dats"][0].__setitem__("data", [1, 2, 3, 4]), "E-OP2-SHAPE"),
    (lambda d: d["par_loops"][0]["args"][1].__setitem__("offset", 2), "E-OP2-RANGE"),
])
def test_validation_codes_equal_reference(mutate, code):
    """load_op2_model's stable codes (op2.hpp:79-81): the product and the reference agree."""
    d = copy.deepcopy(CASES["mesh"]["doc"])
    mutate(d)
    r = ref_op2("op2-lower", d)
    assert r.returncode == 3 and r.stdout.split()[1] == code, r.stdout
    assert err_code(d) == code


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_case_on_gpu(cuda, name):
    import paper_1302_5586_b200 as pb
    case = CASES[name]
    m = model(case["doc"])
    if "fault" in case:
        with pytest.raises(pb.PencilError) as e:
            m.run()
        assert e.value.code == "E-INTERP"
        return
    m.run()
    for k, v in case["result"].items():
        assert m.dat(k).tolist() == v, k


@pytest.mark.gpu
def test_run_twice_accumulates_and_set_dat_resets(cuda):
    doc = CASES["mesh"]["doc"]
    m = model(doc)
    m.run().run()
    assert m.dat("dcells").tolist() == [21, 62, 43]  # 11,32,23 + another pass of the increments
    m.set_dat("dcells", [1, 2, 3])
    m.run()
    assert m.dat("dcells").tolist() == [11, 32, 23]


@pytest.mark.gpu
def test_full_size_mesh_increments_vs_numpy(cuda):
    """2^21 cells, 2^22 edges, random edge->cell map: parallel atomics, bit-exact int64."""
    rng = np.random.default_rng(11)
    nc, ne = 1 << 21, 1 << 22
    table = rng.integers(0, nc, size=2 * ne, dtype=np.int64)
    dedges = rng.integers(-(1 << 40), 1 << 40, size=ne, dtype=np.int64)
    cells = rng.integers(-(1 << 40), 1 << 40, size=nc, dtype=np.int64)
    doc = copy.deepcopy(CASES["mesh"]["doc"])
    doc["sets"] = [{"name": "cells", "size": nc}, {"name": "edges", "size": ne}]
    doc["maps"][0]["table"] = table.tolist()
    doc["dats"][0]["data"] = cells.tolist()
    doc["dats"][1]["data"] = dedges.tolist()
    m = model(json.dumps(doc))
    m.run()
    ref = op2_ref.mesh_increment_numpy(cells, dedges, table)
    assert np.array_equal(m.dat("dcells"), ref)
    # dats of 4 MB and more set / read through the staging ring on the device side, into a reused array
    d2 = dedges[::-1].copy()
    m.set_dat("dcells", cells)
    m.set_dat("dedges", d2)
    m.run()
    out = np.full(nc, 7, np.int64)
    assert m.dat("dcells", out=out) is out
    assert np.array_equal(out, op2_ref.mesh_increment_numpy(cells, d2, table))
    with pytest.raises(ValueError):
        m.dat("dcells", out=np.empty(nc, np.int32))


RANDOM = json.load(open(os.path.join(HERE, "golden", "op2_random.json")))


def test_random_models_load_and_schedule():
    """The 24 random models (tests/golden/make_random_op2.py) load; their par_loops exercise the
    parallel-increment, direct and iteration-level strategies."""
    seen = set()
    for case in RANDOM.values():
        m = model(case["doc"])
        seen.update(m.loop_info(i)[0] for i in range(m.num_loops))
    assert {"parallel", "levels"} <= seen, seen


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(RANDOM))
def test_random_model_on_gpu(cuda, name):
    """Random mesh model vs the REFERENCE Interpreter on the documented lowering: bit-exact."""
    case = RANDOM[name]
    m = model(case["doc"])
    m.run()
    for k, v in case["result"].items():
        assert m.dat(k).tolist() == v, k


def test_openmp_array_reduction_cpu_form_matches_serial():
    """The CPU fix SURVEY §8f.1 names (emit_openmp's `reduction(+: dcells)` on an array parameter is
    not valid OpenMP): each driver loop as `parallel for reduction(+: d[0:n_d])` — bit-identical to
    the serial lowered C on a random mesh."""
    import ctypes
    import sys
    import tempfile
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import op2_probe
    from oracle import op2_ref
    doc = op2_probe.mesh_doc(1 << 12, 1 << 13)
    src, _, _ = op2_ref.openmp_lowered_c(doc)
    assert "#pragma omp parallel for reduction(+: dcells[0:n_dcells])" in src
    outs = []
    with tempfile.TemporaryDirectory() as td:
        for omp in (False, True):
            lib, arrays, sizes = op2_ref.compile_lowered_c(doc, td, openmp=omp)
            content = {d["name"]: np.asarray(d["data"], np.int32) for d in doc["dats"]}
            content.update({m["name"]: np.asarray(m["table"], np.int32) for m in doc["maps"]})
            lib.op2_main(*([ctypes.c_int(n) for n in sizes] + [ctypes.c_void_p(content[a].ctypes.data) for a in arrays]))
            outs.append(content["dcells"].copy())
    assert np.array_equal(outs[0], outs[1])

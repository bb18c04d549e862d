"""Generate tests/golden/op2_cases.json: OP2 mesh models and the REFERENCE Interpreter's results.

Run here (needs oracle/_ref/ref_driver, built from /root/reference by `make -C oracle`):
    python tests/golden/make_op2_golden.py
Each case = a model document (docs/op2-input.md format) + either the final dat contents after
`interpret_op2_reference` semantics (oracle/op2_ref.py runs the reference Interpreter on the
documented lowering) or the E-INTERP fault it raises.  Cases 1-4 restate the reference's own
unit tests (tests/test_op2.cpp: "reference execution of the mesh" -> dcells {11, 32, 23}, "an
edge joining a cell to itself increments it twice" -> {21, 22, 23}, "empty iteration set",
"increments commute across edge order").
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import OracleFault, op2_ref  # noqa: E402

KSIG = ("void kernel(int n_dedges, int n_dcells, int dedges[restrict const static n_dedges], "
        "int dcells[restrict const static n_dcells], int ie, int ic0, int ic1)\n")


def mesh(table=(0, 1, 1, 2), dedges=(10, 20), ncells=3, body=None):
    body = body or "{\n  dcells[ic1] += dedges[ie];\n  dcells[ic0] += dedges[ie];\n}\n"
    return {
        "sets": [{"name": "cells", "size": ncells}, {"name": "edges", "size": len(dedges)}],
        "maps": [{"name": "pecell", "from": "edges", "to": "cells", "arity": 2, "table": list(table)}],
        "dats": [{"name": "dcells", "set": "cells", "dim": 1, "data": list(range(1, ncells + 1))},
                 {"name": "dedges", "set": "edges", "dim": 1, "data": list(dedges)}],
        "kernels": [{"name": "kernel", "source": KSIG + body}],
        "par_loops": [{"kernel": "kernel", "set": "edges", "args": [
            {"dat": "dedges", "access": "OP_READ"},
            {"dat": "dcells", "map": "pecell", "offset": 0, "access": "OP_INC"},
            {"dat": "dcells", "map": "pecell", "offset": 1, "access": "OP_INC"}]}],
    }


def random_mesh(ncells, nedges, seed, body, access=("OP_READ", "OP_INC", "OP_INC")):
    rng = np.random.default_rng(seed)
    table = rng.integers(0, ncells, size=2 * nedges).tolist()
    dedges = rng.integers(-1000, 1000, size=nedges).tolist()
    m = mesh(table, dedges, ncells, body)
    m["dats"][0]["data"] = rng.integers(-50, 50, size=ncells).tolist()
    for a, acc in zip(m["par_loops"][0]["args"], access):
        a["access"] = acc
    return m


def multi_loop(seed):
    """Three par_loops: increments (parallel), a direct update (parallel), an indirect write
    with read-after-write chains through the map (iteration levels)."""
    rng = np.random.default_rng(seed)
    nn, ne = 300, 900
    t = rng.integers(0, nn, size=2 * ne).tolist()
    return {
        "sets": [{"name": "nodes", "size": nn}, {"name": "edges", "size": ne}],
        "maps": [{"name": "en", "from": "edges", "to": "nodes", "arity": 2, "table": t}],
        "dats": [{"name": "dn", "set": "nodes", "dim": 2, "data": rng.integers(-9, 9, size=2 * nn).tolist()},
                 {"name": "de", "set": "edges", "dim": 1, "data": rng.integers(1, 100, size=ne).tolist()}],
        "kernels": [
            {"name": "flux", "source":
                "void flux(int n_de, int n_dn, int de[restrict const static n_de], int dn[restrict const static n_dn], "
                "int e, int a, int b)\n{\n  int w;\n  w = de[e] * 3 - e % 5;\n  dn[2 * a] += w;\n  dn[2 * b + 1] -= w / 4;\n}\n"},
            {"name": "scale", "source":
                "void scale(int n_dn, int dn[restrict const static n_dn], int v)\n{\n  int k;\n"
                "  for (k = 0; k < 2; k++) {\n    if (dn[2 * v + k] > 0) dn[2 * v + k] = dn[2 * v + k] * 2 - 1;\n"
                "    else dn[2 * v + k] = -dn[2 * v + k] / 3;\n  }\n}\n"},
            {"name": "relax", "source":
                "void relax(int n_de, int n_dn, int de[restrict const static n_de], int dn[restrict const static n_dn], "
                "int e, int a, int b)\n{\n  dn[2 * a] = dn[2 * b] + de[e] % 7;\n}\n"},
        ],
        "par_loops": [
            {"kernel": "flux", "set": "edges", "args": [
                {"dat": "de", "access": "OP_READ"},
                {"dat": "dn", "map": "en", "offset": 0, "access": "OP_INC"},
                {"dat": "dn", "map": "en", "offset": 1, "access": "OP_INC"}]},
            {"kernel": "scale", "set": "nodes", "args": [{"dat": "dn", "access": "OP_RW"}]},
            {"kernel": "relax", "set": "edges", "args": [
                {"dat": "de", "access": "OP_READ"},
                {"dat": "dn", "map": "en", "offset": 0, "access": "OP_WRITE"},
                {"dat": "dn", "map": "en", "offset": 1, "access": "OP_READ"}]},
        ],
    }


def cases():
    out = {}
    out["mesh"] = mesh()
    out["mesh_self_loop"] = mesh(table=(0, 0, 1, 2))
    m = mesh()
    m["sets"][1]["size"] = 0
    m["maps"][0]["table"] = []
    m["dats"][1]["data"] = []
    out["mesh_empty_iteration_set"] = m
    out["mesh_commuted"] = mesh(table=(1, 2, 0, 1), dedges=(20, 10))
    out["random_increments"] = random_mesh(
        500, 2000, 1, "{\n  int v;\n  v = dedges[ie] * 2 + ie % 7;\n  dcells[ic0] += v;\n  dcells[ic1] -= v / 3;\n}\n")
    out["control_flow_and_doubles"] = random_mesh(
        64, 400, 2,
        "{\n  double w;\n  int k;\n  int acc;\n  int tmp[4];\n  w = 0.5 * dedges[ie];\n  acc = 0;\n"
        "  for (k = 0; k <= 3; k++) {\n    tmp[k] = k * ie - dedges[ie] % (k + 2);\n    acc += tmp[k];\n  }\n"
        "  k = 0;\n  while (k < 2 && acc > 0) {\n    acc = acc / 2;\n    k++;\n  }\n"
        "  if (w > 3.0 || !(ie % 3)) dcells[ic0] += acc + 1;\n  else dcells[ic1] += 2;\n}\n")
    out["helper_function_alias"] = random_mesh(
        40, 300, 3,
        "{\n  add2(n_dcells, dcells, ic0, dedges[ie]);\n  add2(n_dcells, dcells, ic1, sq(ie % 5));\n}\n"
        "void add2(int n, int a[restrict const static n], int k, int v)\n{\n  a[k] += v;\n}\n"
        "int sq(int x)\n{\n  return x * x;\n}\n")
    out["inc_dat_also_read_serial"] = random_mesh(
        50, 300, 4, "{\n  dcells[ic0] += dcells[ic1] % 5 + dedges[ie] % 3;\n}\n",
        access=("OP_READ", "OP_INC", "OP_READ"))
    out["rand_serial"] = random_mesh(30, 200, 5, "{\n  dcells[ic0] += rand() % 10;\n  dcells[ic1] += dedges[ie];\n}\n")
    out["multi_loop_levels"] = multi_loop(6)
    out["fault_out_of_bounds"] = mesh(body="{\n  dcells[ic1 + 2] += dedges[ie];\n}\n")
    out["fault_division_by_zero"] = mesh(body="{\n  dcells[ic1] += dedges[ie] / (ie - 1);\n}\n")
    return out


def main():
    res = {}
    for name, doc in cases().items():
        try:
            outs = op2_ref.reference_run(doc)
            res[name] = {"doc": doc, "result": {k: v.tolist() for k, v in outs.items()}}
        except OracleFault as e:
            res[name] = {"doc": doc, "fault": str(e)}
        print(name, "fault" if "fault" in res[name] else {k: v[:6] for k, v in res[name]["result"].items()})
    with open(os.path.join(HERE, "op2_cases.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

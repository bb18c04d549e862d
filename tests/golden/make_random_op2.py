"""Generate tests/golden/op2_random.json: 24 random OP2 mesh models (docs/op2-input.md format)
and the REFERENCE Interpreter's results on the documented lowering (oracle/op2_ref.py ->
oracle/_ref/ref_driver).  Each model has 1-3 par_loops drawn from: indirect increments through
an arity-2/3 map (OP_INC, several dats, dims 1-3), direct read-modify-write updates (OP_RW),
indirect writes with reads through the same map (OP_WRITE + OP_READ: iteration levels), and
kernels with local arrays, helper calls, conditionals and while loops.  Run here:
    python tests/golden/make_random_op2.py
"""
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import OracleFault, op2_ref  # noqa: E402


def arr(n):
    return f"int {n}[restrict const static n_{n}]"


def inc_loop(r, k, nn, ne, ar, dims):
    """edges -> nodes increments: dat 'e' (edges, dim 1) read directly, 'p' (nodes, dim dims['p'])
    incremented through map offsets."""
    offs = r.sample(range(ar), r.randint(1, ar))
    dp = dims["p"]
    idx = [f"c{o}" for o in offs]
    body = ["  int v;", "  int q;", f"  v = e[ie] * {r.randint(1, 5)} - ie % {r.randint(2, 9)};"]
    for o, c in zip(offs, idx):
        comp = r.randrange(dp)
        op = r.choice(["+=", "-="])
        expr = r.choice(["v", f"v / {r.randint(2, 5)}", f"v % {r.randint(3, 11)} + {c} % 3", "q"])
        if expr == "q":
            body.append(f"  q = 0;\n  while (q < {r.randint(1, 4)} && q < v % 5) {{\n    q = q + 1;\n  }}")
        body.append(f"  p[{dp} * {c} + {comp}] {op} {expr};")
    src = (f"void k{k}(int n_e, int n_p, {arr('e')}, {arr('p')}, int ie, " + ", ".join(f"int {c}" for c in idx) +
           ")\n{\n" + "\n".join(body) + "\n}\n")
    args = [{"dat": "e", "access": "OP_READ"}] + [{"dat": "p", "map": "m", "offset": o, "access": "OP_INC"}
                                                    for o in offs]
    return src, args, "edges"


def rw_loop(r, k, nn, ne, ar, dims):
    dp = dims["p"]
    src = (f"void k{k}(int n_p, {arr('p')}, int v)\n{{\n  int t;\n  int loc[3];\n"
           f"  for (t = 0; t < {dp}; t++) {{\n    loc[t % 3] = p[{dp} * v + t];\n"
           f"    if (loc[t % 3] > {r.randint(-5, 5)}) p[{dp} * v + t] = loc[t % 3] * 2 - {r.randint(0, 3)};\n"
           f"    else p[{dp} * v + t] = -loc[t % 3] / {r.randint(2, 4)} + helper(v);\n  }}\n}}\n"
           f"int helper(int x)\n{{\n  return x % {r.randint(3, 7)};\n}}\n")
    return src, [{"dat": "p", "access": "OP_RW"}], "nodes"


def write_loop(r, k, nn, ne, ar, dims):
    """indirect write through offset a, read through offset b of the same map (levels)"""
    a, b = r.sample(range(ar), 2)
    dq = dims["q"]
    src = (f"void k{k}(int n_e, int n_q, {arr('e')}, {arr('q')}, int ie, int ca, int cb)\n{{\n"
           f"  q[{dq} * ca] = q[{dq} * cb + {dq - 1}] + e[ie] % {r.randint(3, 13)};\n}}\n")
    args = [{"dat": "e", "access": "OP_READ"}, {"dat": "q", "map": "m", "offset": a, "access": "OP_WRITE"},
            {"dat": "q", "map": "m", "offset": b, "access": "OP_READ"}]
    return src, args, "edges"


def model(seed):
    r = random.Random(seed)
    rng = np.random.default_rng(seed)
    nn, ne, ar = r.choice([7, 50, 300, 1000]), r.choice([0, 1, 40, 500, 2500]), r.choice([2, 3])
    dims = {"p": r.randint(1, 3), "q": r.randint(1, 2)}
    gens = [inc_loop] + r.sample([inc_loop, rw_loop, write_loop], r.randint(0, 2))
    r.shuffle(gens)
    kernels, loops = [], []
    for k, g in enumerate(gens):
        src, args, st = g(r, k, nn, ne, ar, dims)
        kernels.append({"name": f"k{k}", "source": src})
        loops.append({"kernel": f"k{k}", "set": st, "args": args})
    return {
        "sets": [{"name": "nodes", "size": nn}, {"name": "edges", "size": ne}],
        "maps": [{"name": "m", "from": "edges", "to": "nodes", "arity": ar,
                  "table": rng.integers(0, nn, size=ar * ne).tolist()}],
        "dats": [{"name": "p", "set": "nodes", "dim": dims["p"], "data": rng.integers(-40, 40, size=dims["p"] * nn).tolist()},
                 {"name": "q", "set": "nodes", "dim": dims["q"], "data": rng.integers(-40, 40, size=dims["q"] * nn).tolist()},
                 {"name": "e", "set": "edges", "dim": 1, "data": rng.integers(-500, 500, size=ne).tolist()}],
        "kernels": kernels,
        "par_loops": loops,
    }


def main():
    res = {}
    for s in range(24):
        doc = model(7000 + s)
        try:
            outs = op2_ref.reference_run(doc)
            res[f"r{s}"] = {"doc": doc, "result": {k: v.tolist() for k, v in outs.items()}}
        except OracleFault as e:
            res[f"r{s}"] = {"doc": doc, "fault": str(e)}
        print(s, [l["kernel"] + ":" + l["set"] for l in doc["par_loops"]], "fault" if "fault" in res[f"r{s}"] else "ok")
    with open(os.path.join(HERE, "op2_random.json"), "w") as f:
        json.dump(res, f)


if __name__ == "__main__":
    main()

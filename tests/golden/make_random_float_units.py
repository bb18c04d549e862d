"""Generate tests/golden/random_float_units.json: random compliant PENCIL functions over float
arrays and double scalars, with the REFERENCE Interpreter's results (oracle/_ref/ref_driver run).
Companion of make_random_units.py for the interpreter's floating-point semantics (interp.cpp:
7-83: fp64 as soon as a double is involved, int64 otherwise, truncating integer `/`, comparisons
yielding ints, stores keeping the value's type).  Every block evaluates its floating-point
operations in an order the mapper must keep (independent loops, sequential recurrences, inner
sequential sums, conditionals, while loops, mixed int/double expressions) — no licensed
reductions, so the GPU results must be bit-identical.  Run here:
    python tests/golden/make_random_float_units.py
"""
import json
import os
import random
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

SIG = ("double f(int n, float A[restrict const static n], float B[restrict const static n], "
       "float t[restrict const static 16])\n")


def fc(r):
    return "%.3f" % r.uniform(0.1, 3.0)


def block_indep(r):
    c2, c3 = r.randint(1, 5), r.randint(0, 9)
    e = r.choice([f"A[i] * {fc(r)} + B[(i * {c2} + {c3}) % n] / {fc(r)}",
                  f"(A[i] - B[i]) * (A[i] + {fc(r)})",
                  f"A[i] / ({fc(r)} + B[i] * B[i]) + i / {r.randint(2, 5)}",
                  f"A[i] * (i % {r.randint(2, 7)}) - {fc(r)} * B[(i + {c3}) % n]"])
    body = f"A[i] = {e};"
    if r.random() < 0.5:
        body = (f"if (A[i] > B[i] * {fc(r)}) {{\n      A[i] = A[i] - {fc(r)};\n    }} else {{\n      {body}\n    }}")
    return f"  #pragma pencil independent\n  for (i = 0; i < n; i++) {{\n    {body}\n  }}\n"


def block_seq(r):
    return (f"  for (i = 1; i < n; i++) {{\n    B[i] = B[i - 1] * {fc(r)} - A[i] / {fc(r)} + "
            f"(i % {r.randint(2, 9)}) * 0.125;\n    if (B[i] > 1000.0 || B[i] < -1000.0) {{\n"
            f"      B[i] = B[i] / 1024.0;\n    }}\n  }}\n")


def block_nested(r):
    w = r.randint(2, 6)
    return (f"  #pragma pencil independent\n  for (i = 0; i < n; i++) {{\n    u = 0.0;\n"
            f"    for (j = 0; j < {w}; j++) {{\n      u += t[(i + j) % 16] * A[(i + j) % n] - j * {fc(r)};\n    }}\n"
            f"    B[i] = B[i] * {fc(r)} + u;\n  }}\n")


def block_sum(r):  # sequential (no pragma): the analyzer's verdict keeps it in order
    return (f"  for (i = 0; i < n; i++) {{\n    s = s + A[i] * {fc(r)} - B[i] / (i + 1);\n  }}\n")


def block_while(r):
    return (f"  u = s * s + {fc(r)};\n  while (u > 1.0) {{\n    u = u / {r.choice(['2.0', '3.0', '1.5'])};\n"
            f"    s = s + u * 0.5;\n  }}\n")


def program(r):
    blocks = [block_indep, block_seq, block_nested, block_sum, block_while]
    chosen = [b for b in blocks if r.random() < 0.7] or [block_indep]
    r.shuffle(chosen)
    body = "".join(b(r) for b in chosen)
    return (SIG + "{\n  int i;\n  int j;\n  double s;\n  double u;\n  s = " + fc(r) + ";\n  u = 0.0;\n" + body +
            "  return s + u;\n}\n")


def run_reference(src, n, A, B, t):
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "u.pencil.c")
        open(path, "w").write(src)
        lines = [f"scalar int {n}"]
        for name, a in (("A", A), ("B", B), ("t", t)):
            p = os.path.join(td, name + ".bin")
            a.astype(np.float32).tofile(p)
            lines.append(f"array f32 {p}")
        r = subprocess.run([oracle.REF_DRIVER, "run", path, "f"], input="\n".join(lines) + "\n",
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr + r.stdout
        ret = None
        for line in r.stdout.splitlines():
            if line.startswith("ret "):
                _, kind, v = line.split()
                ret = float(v) if kind == "float" else int(v)
        outs = [np.fromfile(os.path.join(td, k + ".bin.out"), np.float64) for k in ("A", "B")]
        return ret, outs


def main():
    cases = []
    for k in range(30):
        r = random.Random(5000 + k)
        src = program(r)
        n = r.choice([1, 7, 32, 100, 257, 1000])
        rng = np.random.default_rng(100 + k)
        A = rng.uniform(-2, 2, n).astype(np.float32)
        B = rng.uniform(-2, 2, n).astype(np.float32)
        t = rng.uniform(-1, 1, 16).astype(np.float32)
        ret, outs = run_reference(src, n, A, B, t)
        # doubles as hex so the JSON round trip is exact
        cases.append({"src": src, "n": n, "A": A.tolist(), "B": B.tolist(), "t": t.tolist(),
                      "ret": float(ret).hex(), "A_out": [float(v).hex() for v in outs[0]],
                      "B_out": [float(v).hex() for v in outs[1]]})
    with open(os.path.join(HERE, "random_float_units.json"), "w") as f:
        json.dump(cases, f)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()

"""Generate tests/golden/random_units.json: random compliant integer PENCIL functions and the
REFERENCE Interpreter's results on them (oracle/_ref/ref_driver run) — the mapper-generality
check in the spirit of the reference's acceptance criterion 8 (tests/acceptance.cpp:367-436:
random integer loops, interpreter vs lowered code).  Run here:
    python tests/golden/make_random_units.py
Each function mixes, at random, an `independent` loop (really independent: it writes A[i] and
reads A[i] and B), a `reduction (+: s)` loop, a sequential recurrence, nested loops with an
`independent` outer loop, a while loop and conditionals; divisors are kept non-zero.
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

SIG = ("int f(int n, int m, int A[restrict const static n], int B[restrict const static n], "
       "int t[restrict const static 16])\n")


def expr_a(r):
    c1, c2, c3 = r.randint(1, 7), r.randint(1, 5), r.randint(0, 9)
    op = r.choice(["+", "-", "*"])
    return f"(A[i] {op} B[(i * {c2} + {c3}) % n] * {c1}) % {r.randint(50, 997)}"


def block_indep(r):
    cond = r.random() < 0.5
    body = f"A[i] = {expr_a(r)};"
    if cond:
        body = f"if (A[i] % {r.randint(2, 5)} == {r.randint(0, 1)}) {{\n      A[i] = A[i] - {r.randint(1, 9)};\n    }} else {{\n      {body}\n    }}"
    return f"  #pragma pencil independent\n  for (i = 0; i < n; i++) {{\n    {body}\n  }}\n"


def block_red(r):
    k = r.randint(2, 4)
    return (f"  #pragma pencil reduction (+: s)\n  for (i = 0; i < n; i++) {{\n"
            f"    if (A[i] % {k} != 0) {{\n      s += A[i] * (i % {r.randint(2, 6)}) - B[i] / {r.randint(1, 5)};\n    }}\n  }}\n")


def block_seq(r):
    return (f"  for (i = 1; i < n; i++) {{\n    B[i] = B[i - 1] + A[i] / (m + {r.randint(1, 4)}) - "
            f"B[i] % {r.randint(2, 9)};\n  }}\n")


def block_nested(r):
    w = r.randint(2, 6)
    return (f"  #pragma pencil independent\n  for (i = 0; i < n; i++) {{\n    u = 0;\n"
            f"    for (j = 0; j < {w}; j++) {{\n      u += t[(i + j) % 16] * (j - {r.randint(0, 3)});\n    }}\n"
            f"    B[i] = B[i] - u % {r.randint(3, 11)};\n  }}\n")


def block_while(r):
    return (f"  u = m + {r.randint(1, 50)};\n  while (u > 1) {{\n    u = u / {r.randint(2, 3)};\n"
            f"    s = s + u * {r.randint(1, 4)};\n  }}\n")


def program(r):
    blocks = [block_indep, block_red, block_seq, block_nested, block_while]
    chosen = [b for b in blocks if r.random() < 0.7] or [block_indep]
    r.shuffle(chosen)
    body = "".join(b(r) for b in chosen)
    return (SIG + "{\n  int i;\n  int j;\n  int s;\n  int u;\n  s = " + str(r.randint(-5, 5)) + ";\n  u = 0;\n" + body +
            "  return s + u;\n}\n")


def run_reference(src, n, m, A, B, t):
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "u.pencil.c")
        open(path, "w").write(src)
        lines = [f"scalar int {n}", f"scalar int {m}"]
        for name, a in (("A", A), ("B", B), ("t", t)):
            p = os.path.join(td, name + ".bin")
            a.astype(np.int32).tofile(p)
            lines.append(f"array i32 {p}")
        r = subprocess.run([oracle.REF_DRIVER, "run", path, "f"], input="\n".join(lines) + "\n",
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr + r.stdout
        ret = None
        for line in r.stdout.splitlines():
            if line.startswith("ret "):
                ret = int(line.split()[2])
        outs = [np.fromfile(os.path.join(td, k + ".bin.out"), np.int64).tolist() for k in ("A", "B", "t")]
        return ret, outs


def main():
    cases = []
    for k in range(40):
        r = random.Random(1000 + k)
        src = program(r)
        n = r.choice([1, 7, 32, 100, 1000, 4099])
        m = r.randint(0, 20)
        rng = np.random.default_rng(k)
        A = rng.integers(-100, 100, n)
        B = rng.integers(-100, 100, n)
        t = rng.integers(-9, 9, 16)
        ret, outs = run_reference(src, n, m, A, B, t)
        cases.append({"src": src, "n": n, "m": m, "A": A.tolist(), "B": B.tolist(), "t": t.tolist(),
                      "ret": ret, "A_out": outs[0], "B_out": outs[1]})
    with open(os.path.join(HERE, "random_units.json"), "w") as f:
        json.dump(cases, f)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()

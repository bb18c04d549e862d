"""Generate tests/golden/optiml/<name>.npz: OptiML constructs lowered by pencil_optiml_lower and run
by the REFERENCE Interpreter (oracle/_ref/ref_driver run) — inputs and outputs for the GPU tests.
    python tests/golden/make_optiml_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from test_optiml import CONSTRUCTS, _reference, lower  # noqa: E402


def main():
    rng = np.random.default_rng(1)
    for name in ("vector", "batch", "stochastic"):
        doc, fn, _, _ = CONSTRUCTS[name]
        src = lower(doc)
        if name == "vector":
            n = 1000 - 3 + 1
            args = [n, np.zeros(n, np.int32)]
        else:
            n = 4096
            args = [n, rng.standard_normal(n).astype(np.float32), rng.standard_normal(n).astype(np.float32)]
        ref = _reference(src, fn, args)
        save = {"n": np.array(n)}
        for i, a in enumerate(args[1:], 1):
            save[f"in{i}"] = a
            save[f"out{i}"] = ref[i]
        np.savez(os.path.join(HERE, "optiml", f"{name}.npz"), **save)
        print(name, {k: v[:3] for k, v in ref.items()})


if __name__ == "__main__":
    main()

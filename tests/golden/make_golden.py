"""Generate the golden vectors of tests/golden/*.npz with the REFERENCE's own Interpreter.

Runs in the build container only (needs oracle/_ref/ref_driver, compiled from /root/reference
by oracle/Makefile).  For every case it feeds seeded inputs (paper_1302_5586_b200.synth, the
SURVEY §8d LCG) through pencil::Interpreter::call via ref_driver and stores inputs, scalar
arguments and the interpreter's fp64/int64 outputs.  The parity tests then check both the C
restatement (oracle/pencil_oracle.c, bit-exact) and the CUDA path (exact / normwise) against
these files on any machine, without /root/reference.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1302_5586_b200 import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(n, seed):
    return synth.f32(n, seed=seed)


def cases():
    c = []
    # ---- gemv (gemv.pencil.c)
    for (m, n, al, be, s) in [(37, 53, 1.5, 0.5, 1), (64, 256, 1.0, 0.0, 2), (1, 1, 2.0, 3.0, 3), (5, 0, 1.0, 2.0, 4)]:
        c.append((f"gemv_{m}x{n}", "gemv", "gemv",
                  [m, n, al, be, f32(m * n, s), f32(n, s + 100), f32(m, s + 200)]))
    # ---- gemv_t (VOBLA strided view)
    for (m, n, lda, ix, iy, al, be, s) in [(29, 41, 48, 2, 3, 0.75, -1.25, 5), (64, 64, 64, 1, 1, 1.0, 0.0, 6),
                                           (3, 7, 7, 5, 2, 1.0, 1.0, 7)]:
        c.append((f"gemv_t_{m}x{n}_lda{lda}_ix{ix}_iy{iy}", "gemv_t", "gemv_t",
                  [m, n, lda, ix, iy, al, be, f32(m * lda, s), f32(m * ix, s + 100), f32(n * iy, s + 200)]))
    # ---- dot / axpy
    for n, s in [(1000, 8), (1, 9), (0, 10), (4099, 11)]:
        c.append((f"dot_{n}", "dot", "dot", [n, f32(n, s), f32(n, s + 100)]))
    for n, a, s in [(1000, 2.5, 12), (7, -0.5, 13)]:
        c.append((f"axpy_{n}", "axpy", "axpy", [n, a, f32(n, s), f32(n, s + 100)]))
    # ---- spmv: three PENCIL spellings, same semantics in the interpreter
    rowptr, col, val, x, _ = synth.csr_powerlaw(300, avg_per_row=16.0, maxlen=200, seed=14)
    mats = {"powerlaw300": (rowptr, col, val, x)}
    # ragged edge cases: empty rows, a long row, leading/trailing empties
    lens = np.array([0, 1, 0, 0, 150, 3, 0, 2, 40, 0, 0, 1] + [0] * 5 + [5], dtype=np.int64)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    nz = int(rp[-1])
    rng_cols = (synth.u8_i32(nz, seed=15).astype(np.int64) * 7919 % 97).astype(np.int32)
    mats["ragged"] = (rp, np.sort(rng_cols), f32(nz, 16), f32(97, 17))
    # integer-valued entries: every partial sum is exact in fp32 (index handling bit-exact)
    iv = (synth.u8_i32(int(rowptr[-1]), seed=18) % 9 - 4).astype(np.float32)
    ix = (synth.u8_i32(300, seed=19) % 7 - 3).astype(np.float32)
    mats["intvals300"] = (rowptr, col, iv, ix)
    mats["empty"] = (np.zeros(6, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32), f32(4, 20))
    for name, (rp_, co_, va_, x_) in mats.items():
        nrows, ncols, nnz = rp_.size - 1, x_.size, co_.size
        for fn in ("spmv_vec", "spmv_inline", "spmv"):
            c.append((f"{fn}_{name}", "spmv", fn,
                      [nrows, ncols, nnz, rp_, co_, va_, x_, np.zeros(nrows, np.float32)]))
    # ---- conv5x5_u8 (int semantics)
    k_bin, k_sh = synth.BINOMIAL, synth.SHARPEN
    for (h, w, scale, k, tag, s) in [(67, 61, 256, k_bin, "binomial", 21), (67, 61, 1, k_sh, "sharpen", 22),
                                     (1, 1, 256, k_bin, "binomial", 23), (3, 2, 1, k_sh, "sharpen", 24),
                                     (5, 5, 256, k_bin, "binomial", 25), (9, 13, -3, k_bin, "negscale", 26),
                                     (8, 40, 7, k_sh, "sharpen_s7", 27)]:
        c.append((f"conv5x5_u8_{h}x{w}_{tag}", "conv5x5", "conv5x5_u8",
                  [h, w, scale, synth.u8_i32(h * w, seed=s), k.copy(), np.zeros(h * w, np.int32)]))
    # ---- conv5x5_f32 (interior only)
    kf = (k_bin.astype(np.float32) / 256.0).astype(np.float32)
    for (h, w, k, tag, s) in [(37, 45, kf, "binomial", 28), (37, 45, f32(25, 29), "random", 30),
                              (5, 5, kf, "binomial", 31), (4, 4, kf, "binomial", 32)]:
        c.append((f"conv5x5_f32_{h}x{w}_{tag}", "conv5x5", "conv5x5_f32",
                  [h, w, f32(h * w, s), k.copy(), f32(h * w, s + 100)]))
    # ---- gemm
    for (m, n, k, al, be, s) in [(33, 29, 17, 1.25, -0.5, 33), (16, 16, 16, 1.0, 0.0, 34), (1, 3, 2, 1.0, 1.0, 35)]:
        c.append((f"gemm_{m}x{n}x{k}", "gemm", "gemm",
                  [m, n, k, al, be, f32(m * k, s), f32(k * n, s + 100), f32(m * n, s + 200)]))
    return c


def fault_cases():
    rp = np.array([0, 2, 3], np.int32)
    return [
        ("fault_spmv_col_oob", "spmv", "spmv_inline",
         [2, 4, 3, rp, np.array([0, 4, 1], np.int32), f32(3, 40), f32(4, 41), np.zeros(2, np.float32)]),
        ("fault_conv_u8_scale0", "conv5x5", "conv5x5_u8",
         [3, 3, 0, synth.u8_i32(9, seed=42), synth.BINOMIAL.copy(), np.zeros(9, np.int32)]),
    ]


def save(name, fixture, fn, args, ret, outs, fault=False):
    spec = {"fixture": fixture, "fn": fn, "args": [], "ret": ret, "fault": fault}
    arrays = {}
    for i, a in enumerate(args):
        if isinstance(a, np.ndarray):
            spec["args"].append({"kind": "array", "dtype": str(a.dtype), "key": f"in{i}"})
            arrays[f"in{i}"] = a
            if i in outs:
                arrays[f"out{i}"] = outs[i]
        elif isinstance(a, (int, np.integer)):
            spec["args"].append({"kind": "int", "value": int(a)})
        else:
            spec["args"].append({"kind": "float", "value": float(a)})
    np.savez_compressed(os.path.join(OUT, name + ".npz"), spec=np.array(json.dumps(spec)), **arrays)


def main():
    n = 0
    for name, fixture, fn, args in cases():
        ret, outs = oracle.ref_run(fixture, fn, args)
        save(name, fixture, fn, args, ret, outs)
        n += 1
    for name, fixture, fn, args in fault_cases():
        try:
            oracle.ref_run(fixture, fn, args)
        except oracle.OracleFault:
            save(name, fixture, fn, args, None, {}, fault=True)
            n += 1
            continue
        raise SystemExit(f"{name}: the reference interpreter did not fault")
    # verdicts of every fixture as the reference analyzer reports them (mapper input)
    verdicts = {}
    for fx in ("gemv", "gemv_t", "dot", "axpy", "spmv", "conv5x5", "gemm"):
        verdicts[fx] = oracle.ref_analyze(fx)
    verdicts["spmv_bound"] = oracle.ref_analyze(
        "spmv", params={"nrows": 3, "ncols": 3, "nnz": 4}, arrays={"rowptr": [0, 1, 3, 4], "col": [0, 0, 2, 1]})
    with open(os.path.join(OUT, "verdicts.json"), "w") as f:
        json.dump(verdicts, f, indent=1, sort_keys=True)
    # parameter signatures as the reference parser reads them (the drop-in boundary)
    import subprocess
    sigs = {}
    for fx in ("gemv", "gemv_t", "dot", "axpy", "spmv", "conv5x5", "gemm"):
        out = subprocess.run([oracle.REF_DRIVER, "signature", os.path.join(oracle.FIXTURES, fx + ".pencil.c")],
                             capture_output=True, text=True, check=True).stdout
        for line in out.splitlines():
            name, sig = line.split("=", 1)
            sigs[name] = sig
    with open(os.path.join(OUT, "signatures.json"), "w") as f:
        json.dump(sigs, f, indent=1, sort_keys=True)
    print(f"wrote {n} golden cases + verdicts.json to {OUT}")


if __name__ == "__main__":
    main()

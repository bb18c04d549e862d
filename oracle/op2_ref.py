"""TEST INFRASTRUCTURE ONLY — the OP2 oracle: the reference Interpreter run on a mesh model.

The reference's own OP2 module (core/src/op2.cpp) needs nlohmann/json, absent here, so it is not
built.  Its semantics are `interpret_op2_reference` (op2.cpp:388-429): every par_loop in order,
the kernel called per iteration with (sizes of the distinct dats, the dats, one index per arg:
`i` or `map[arity*i + offset]`).  This module restates the documented lowering (append_driver,
op2.cpp:253-345; docs/op2-input.md "Lowering produces one driver per par_loop") in Python, adds
one `op2_main` that calls the drivers in order, and runs that unit through the REFERENCE
Interpreter (oracle/_ref/ref_driver `run`), so the outputs are the reference's own.

`mesh_increment_numpy` is the numpy restatement of the increment kernel used at full size
(beyond the interpreter's 100 M-step budget, interp.hpp:71).
"""
import os
import subprocess
import tempfile

import numpy as np

from . import REF_DRIVER, OracleFault


def _distinct(seq):
    out = []
    for s in seq:
        if s not in out:
            out.append(s)
    return out


def lower_unit(doc):
    """PENCIL text: the model's kernels, one `<kernel>_loop` driver per par_loop, and `op2_main`."""
    maps = {m["name"]: m for m in doc.get("maps", [])}
    dats = {d["name"]: d for d in doc.get("dats", [])}
    sets = {s["name"]: s for s in doc.get("sets", [])}
    parts = [k["source"] for k in doc.get("kernels", [])]
    calls = []
    for li, L in enumerate(doc.get("par_loops", [])):
        ds = _distinct(a["dat"] for a in L["args"])
        ms = _distinct(a["map"] for a in L["args"] if a.get("map"))
        fn = f"{L['kernel']}_loop{li}"
        params = ["int n_iter"] + [f"int n_{d}" for d in ds] + [f"int n_{m}" for m in ms]
        params += [f"int {d}[restrict const static n_{d}]" for d in ds]
        params += [f"int {m}[restrict const static n_{m}]" for m in ms]
        idx = []
        for a in L["args"]:
            if a.get("map"):
                idx.append(f"{a['map']}[{maps[a['map']]['arity']} * i + {a['offset']}]")
            else:
                idx.append("i")
        kargs = [f"n_{d}" for d in ds] + ds + idx
        parts.append(f"void {fn}({', '.join(params)})\n{{\n  int i;\n  for (i = 0; i < n_iter; i++) {{\n"
                     f"    {L['kernel']}({', '.join(kargs)});\n  }}\n}}\n")
        cargs = [str(sets[L["set"]]["size"])] + [str(len(dats[d]["data"])) for d in ds] + \
            [str(len(maps[m]["table"])) for m in ms] + ds + ms
        calls.append(f"  {fn}({', '.join(cargs)});")
    arrays = [d["name"] for d in doc.get("dats", [])] + [m["name"] for m in doc.get("maps", [])]
    sizes = [len(d["data"]) for d in doc.get("dats", [])] + [len(m["table"]) for m in doc.get("maps", [])]
    mparams = [f"int n_{a}" for a in arrays] + [f"int {a}[restrict const static n_{a}]" for a in arrays]
    parts.append(f"void op2_main({', '.join(mparams)})\n{{\n" + "\n".join(calls) + "\n}\n")
    return "\n".join(parts), arrays, sizes


def reference_run(doc):
    """Final dat contents after interpreting every par_loop (dict name -> int64 array)."""
    if not os.path.exists(REF_DRIVER):
        raise FileNotFoundError(REF_DRIVER)
    src, arrays, sizes = lower_unit(doc)
    content = {d["name"]: d["data"] for d in doc.get("dats", [])}
    content.update({m["name"]: m["table"] for m in doc.get("maps", [])})
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "model.pencil.c")
        with open(path, "w") as f:
            f.write(src)
        lines = [f"scalar int {n}" for n in sizes]
        for a in arrays:
            p = os.path.join(td, a + ".bin")
            np.asarray(content[a], dtype=np.int32).tofile(p)
            lines.append(f"array i32 {p}")
        r = subprocess.run([REF_DRIVER, "run", path, "op2_main"], input="\n".join(lines) + "\n",
                           capture_output=True, text=True)
        if r.returncode == 3:
            raise OracleFault(r.stdout.strip())
        if r.returncode != 0:
            raise RuntimeError(f"ref_driver failed: {r.stderr}{r.stdout}")
        return {d["name"]: np.fromfile(os.path.join(td, d["name"] + ".bin.out"), dtype=np.int64)
                for d in doc.get("dats", [])}


def mesh_increment_numpy(cells0, edges_val, table):
    """dcells[map[2e]] += dedges[e]; dcells[map[2e+1]] += dedges[e] for every edge e (int64)."""
    out = np.asarray(cells0, dtype=np.int64).copy()
    t = np.asarray(table, dtype=np.int64).reshape(-1, 2)
    v = np.asarray(edges_val, dtype=np.int64)
    np.add.at(out, t[:, 1], v)
    np.add.at(out, t[:, 0], v)
    return out


def openmp_lowered_c(doc):
    """The lowered unit with the CPU fix SURVEY §8f.1 names: each driver loop carries
    `#pragma omp parallel for` with an array-section reduction over the dats it increments
    (`reduction(+: d[0:n_d])`, OpenMP 4.5) — what emit_openmp's `reduction(+: dcells)` on an array
    parameter means but cannot express.  Loops that write a dat directly (OP_WRITE / OP_RW through
    the identity) stay parallel without a reduction; loops with an indirect non-INC write stay serial."""
    src, arrays, sizes = lower_unit(doc)
    for li, L in enumerate(doc.get("par_loops", [])):
        fn = f"{L['kernel']}_loop{li}"
        inc = _distinct(a["dat"] for a in L["args"] if a.get("access") == "OP_INC")
        ind_write = any(a.get("map") and a.get("access") in ("OP_WRITE", "OP_RW") for a in L["args"])
        if ind_write:
            continue
        red = (" reduction(+: " + ", ".join(f"{d}[0:n_{d}]" for d in inc) + ")") if inc else ""
        head = f"void {fn}("
        i = src.index(head)
        j = src.index("  for (i = 0; i < n_iter; i++) {", i)
        src = src[:j] + f"  #pragma omp parallel for{red}\n" + src[j:]
    return src, arrays, sizes


def compile_lowered_c(doc, outdir, openmp=False):
    """The model's lowering (kernels + drivers, as above) compiled as plain C with gcc -O3: the
    reference's CPU path for a mesh model.  emit_openmp would attach `reduction(+: dcells)` to
    the driver loop, which is not valid OpenMP for an array parameter ([P10]), so
    the C runs serially.  C `int` is 32-bit (the interpreter's values are int64): use inputs
    whose sums stay in range.  Returns a ctypes handle exposing `op2_main`."""
    import ctypes
    src, arrays, sizes = openmp_lowered_c(doc) if openmp else lower_unit(doc)
    path = os.path.join(outdir, "model_omp.c" if openmp else "model.c")
    with open(path, "w") as f:
        f.write(src)
    so = os.path.join(outdir, "model_omp.so" if openmp else "model.so")
    subprocess.run(["gcc", "-O3", "-march=x86-64-v3", "-std=gnu11", "-fPIC", "-shared", "-DACCESS(x)=",
                    "-DDEF(x)=(void)0", "-DUSE(x)=(void)0", "-DMAY_DEF(x)=(void)0"] + (["-fopenmp"] if openmp else [])
                   + ["-o", so, path], check=True)
    lib = ctypes.CDLL(so)
    lib.op2_main.restype = None
    return lib, arrays, sizes

"""The drop-in claim at the C level: one host program (tests/c/dropin_host.c), written against
the ABI the reference's emit_openmp prints, linked once against the reference's emitted OpenMP
code (oracle/_ref/libpencil_omp_outer.so — the CPU path being replaced) and once against
libpencil_b200.so.  Source-order and integer kernels must agree bit for bit; reassociated
reductions (gemv, gemv_t, dot, spmv_vec, gemm) within the normwise bound against fp64."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "dropin_host.c")
BUILD = os.path.join(ROOT, "tests", "c", "build")
OMP_LIB = os.path.join(ROOT, "oracle", "_ref", "libpencil_omp_outer.so")
B200_DIR = os.path.join(ROOT, "paper_1302_5586_b200", "lib")


def build(kind):
    os.makedirs(BUILD, exist_ok=True)
    exe = os.path.join(BUILD, "host_" + kind)
    cmd = ["gcc", "-O2", "-std=gnu11", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe]
    if kind == "omp":
        cmd += [OMP_LIB, "-Wl,-rpath," + os.path.dirname(OMP_LIB)]
    else:
        cmd += ["-DPENCIL_DROPIN_B200", "-L", B200_DIR, "-lpencil_b200", "-Wl,-rpath," + B200_DIR]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def run(exe, tmp_path):
    path = str(tmp_path / (os.path.basename(exe) + ".bin"))
    subprocess.run([exe, path], check=True, timeout=600)
    recs, raw = {}, open(path, "rb").read()
    o = 0
    while o < len(raw):
        name = raw[o:o + 16].split(b"\0")[0].decode()
        dt, n = np.frombuffer(raw, np.int32, 2, o + 16)
        t = {0: np.int32, 1: np.float32, 2: np.float64}[int(dt)]
        recs[name] = np.frombuffer(raw, t, int(n), o + 24).copy()
        o += 24 + int(n) * np.dtype(t).itemsize
    return recs


def normwise(got, ref64, terms):
    return float(np.max(np.abs(got.astype(np.float64) - ref64) / np.maximum(terms, 1e-300))) if got.size else 0.0


def references(r):
    """fp64 results + per-output sum of |terms| for the reassociated kernels."""
    out = {}
    m, n = 300, 257
    A = r["gemv.A"].reshape(m, n).astype(np.float64)
    x, y0 = r["gemv.x"].astype(np.float64), r["gemv.y0"].astype(np.float64)
    out["gemv.y"] = (1.5 * A @ x + 0.5 * y0, 1.5 * np.abs(A) @ np.abs(x) + 0.5 * np.abs(y0))
    tm, tn, lda, ix, iy = 65, 77, 80, 2, 3
    tA = r["gemvt.A"].reshape(tm, lda)[:, :tn].astype(np.float64)
    tx = r["gemvt.x"][::ix][:tm].astype(np.float64)
    ty0 = r["gemvt.y0"].astype(np.float64)
    ref = ty0.copy()
    ref[::iy][:tn] = tA.T @ tx + 0.25 * ty0[::iy][:tn]
    terms = np.abs(ty0).copy()
    terms[::iy][:tn] = np.abs(tA.T) @ np.abs(tx) + 0.25 * np.abs(ty0[::iy][:tn])
    out["gemvt.y"] = (ref, terms)
    dx, dy = r["dot.x"].astype(np.float64), r["dot.y"].astype(np.float64)
    out["dot.r"] = (np.array([dx @ dy]), np.array([np.abs(dx) @ np.abs(dy)]))
    rp, col, val, sx = r["spmv.rowptr"], r["spmv.col"], r["spmv.val"].astype(np.float64), r["spmv.x"].astype(np.float64)
    prod = val * sx[col]
    cs = np.concatenate([[0.0], np.cumsum(prod)])
    ca = np.concatenate([[0.0], np.cumsum(np.abs(prod))])
    out["spmv_vec.y"] = (cs[rp[1:]] - cs[rp[:-1]], ca[rp[1:]] - ca[rp[:-1]])
    gm, gn, gk = 64, 48, 40
    gA, gB = r["gemm.A"].reshape(gm, gk).astype(np.float64), r["gemm.B"].reshape(gk, gn).astype(np.float64)
    gC0 = r["gemm.C0"].reshape(gm, gn).astype(np.float64)
    out["gemm.C"] = ((gA @ gB + 0.5 * gC0).reshape(-1), (np.abs(gA) @ np.abs(gB) + 0.5 * np.abs(gC0)).reshape(-1))
    return out


INPUTS = ["gemv.A", "gemv.x", "gemv.y0", "gemvt.A", "gemvt.x", "gemvt.y0", "dot.x", "dot.y", "spmv.rowptr",
          "spmv.col", "spmv.val", "spmv.x", "conv.img", "convf.o0", "convf.img", "convf.k", "gemm.A", "gemm.B",
          "gemm.C0"]
EXACT = ["axpy.y", "spmv_inline.y", "spmv.y", "conv.u8", "conv.u8s", "convf.out"]


@pytest.fixture(scope="module")
def omp_results(tmp_path_factory):
    if not os.path.exists(OMP_LIB):
        pytest.skip("oracle/_ref not built")
    return run(build("omp"), tmp_path_factory.mktemp("omp"))


def test_host_program_links_against_both(omp_results):
    """CPU: the same source links against the emitted OpenMP library and against the B200
    library (the header's §1 prototypes are the emitted ABI); the reference build's results sit
    within the stated bounds of fp64."""
    build("b200")
    for name, (ref, terms) in references(omp_results).items():
        assert normwise(omp_results[name], ref, terms) <= 1e-5, name


@pytest.mark.gpu
def test_dropin_relink_matches_reference_build(omp_results, tmp_path):
    gpu = run(build("b200"), tmp_path)
    assert set(gpu) == set(omp_results)
    for name in EXACT:
        assert np.array_equal(gpu[name].view(np.uint32), omp_results[name].view(np.uint32)), name
    for name, (ref, terms) in references(gpu).items():
        assert normwise(gpu[name], ref, terms) <= 1e-5, name
    for name in INPUTS:  # same LCG on both sides
        assert np.array_equal(gpu[name], omp_results[name]), name

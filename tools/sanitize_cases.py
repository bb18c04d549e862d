"""Small-shape pass over every product kernel family, for compute-sanitizer (tools/sanitize.sh runs
it under memcheck, racecheck and synccheck, ONE tool per gpurun call — B200_PROFILING.md: several
tools in one call once left a GPU unusable).  Each case also checks its result against the oracle,
so the pass shows the kernels are clean AND still right under instrumentation.

usage: python tools/sanitize_cases.py        (prints one line per case; exit 1 on a mismatch)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1302_5586_b200 as pb  # noqa: E402
from paper_1302_5586_b200 import synth  # noqa: E402
from paper_1302_5586_b200.dist import band_halo_rows, shard_bands  # noqa: E402

dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
bad = []


def check(name, ok):
    print(("ok   " if ok else "FAIL ") + name, flush=True)
    if not ok:
        bad.append(name)


def bits(a):
    return np.asarray(a).view(np.uint32)


def main():
    torch.cuda.set_device(0)
    # SpMV: plan + flow kernel (aligned) + scalar-load kernel (unaligned) + fused dist stores
    rowptr, col, val, x, _ = synth.csr_powerlaw(3000, maxlen=700, seed=4)
    n, nnz = rowptr.size - 1, col.size
    ref = oracle.spmv_f32(n, n, nnz, rowptr, col, val, x)
    rp, xd = dev(rowptr), dev(x)
    for aligned in (True, False):
        sh = 0 if aligned else 1
        cd = torch.zeros(nnz + sh, dtype=torch.int32, device="cuda")[sh:]
        vd = torch.zeros(nnz + sh, device="cuda")[sh:]
        cd.copy_(torch.from_numpy(col))
        vd.copy_(torch.from_numpy(val))
        for mode in (0, 1):
            plan = pb.device.CsrPlan(n, n, nnz, rp, mode=mode)
            y = torch.empty(n, device="cuda")
            plan.spmv(rp, cd, vd, xd, y)
            tgt = torch.full((n + 64,), float("nan"), device="cuda")
            y2 = torch.empty(n, device="cuda")
            plan.spmv_dist(rp, cd, vd, xd, y2, [tgt.data_ptr() + 256])
            torch.cuda.synchronize()
            pb.device.sync_status()
            if mode == 0:
                check(f"spmv source order aligned={aligned}", np.array_equal(bits(y.cpu().numpy()), bits(ref)))
            r64 = oracle.spmv(n, n, nnz, rowptr, col, val, x)
            check(f"spmv mode {mode} aligned={aligned} normwise", np.max(np.abs(y.cpu().numpy() - r64)) < 1e-4)
            check(f"spmv_dist mode {mode} aligned={aligned}", torch.equal(tgt[64:].view(torch.int32), y2.view(torch.int32)))
            plan.close()
    # dense BLAS
    m, k = 300, 517
    A, xv, yv = synth.f32(m * k, 1), synth.f32(k, 2), synth.f32(m, 3)
    y = dev(yv.copy())
    pb.device.gemv(m, k, 1.5, 0.5, dev(A), dev(xv), y)
    check("gemv", np.max(np.abs(y.cpu().numpy() - oracle.gemv(m, k, 1.5, 0.5, A, xv, yv))) < 1e-3)
    mm, nn, lda = 200, 300, 304
    A2, xt, yt = synth.f32(mm * lda, 4), synth.f32(mm * 2, 5), synth.f32(nn * 3, 6)
    y = dev(yt.copy())
    pb.device.gemv_t(mm, nn, lda, 2, 3, 1.0, 0.25, dev(A2), dev(xt), y)
    check("gemv_t", np.max(np.abs(y.cpu().numpy() - oracle.gemv_t(mm, nn, lda, 2, 3, 1.0, 0.25, A2, xt, yt))) < 1e-3)
    nv = 100003
    a, b = synth.f32(nv, 7), synth.f32(nv, 8)
    r = torch.zeros(1, device="cuda")
    pb.device.dot(nv, dev(a), dev(b), r)
    check("dot", abs(float(r.item()) - oracle.dot(nv, a, b)) < 1e-3)
    yb = dev(b.copy())
    pb.device.axpy_ptr(nv, r, dev(a), yb)
    check("axpy(dot)", np.array_equal(bits(yb.cpu().numpy()), bits(oracle.axpy_f32(nv, np.float32(r.item()), a, b))))
    # stencils: every u8 / bytes / f32 variant, and the band kernels reading halos in place
    h, w = 70, 256
    img = synth.u8_i32(h * w, 9)
    for taps, scale, nm in ((synth.BINOMIAL, 256, "binomial"), (synth.SHARPEN, 1, "sharpen"),
                            (synth.f32(25, 3).view(np.int32) & 0x3f, 7, "25-tap")):
        ref = oracle.conv5x5_u8(h, w, scale, img, taps)
        out = torch.empty(h * w, dtype=torch.int32, device="cuda")
        pb.device.conv5x5_u8(h, w, scale, dev(img), taps, out)
        check(f"conv5x5_u8 {nm}", np.array_equal(out.cpu().numpy(), ref))
        o8 = torch.empty(h * w, dtype=torch.uint8, device="cuda")
        pb.device.conv5x5_u8_bytes(h, w, scale, dev(img.astype(np.uint8)), taps, o8)
        check(f"conv5x5_u8_bytes {nm}", np.array_equal(o8.cpu().numpy().astype(np.int64), ref))
    imgf = synth.f32(h * w, 10)
    for taps, nm in (((synth.BINOMIAL / 256.0).astype(np.float32), "pow2"), (synth.f32(25, 11), "generic")):
        out0 = synth.f32(h * w, 12)
        out = dev(out0.copy())
        pb.device.conv5x5_f32(h, w, dev(imgf), taps, out)
        check(f"conv5x5_f32 {nm}", np.array_equal(bits(out.cpu().numpy()), bits(oracle.conv5x5_f32_f32(h, w, imgf, taps, out0))))
    bnd = shard_bands(h, 3)
    rows = [int(bnd[q + 1] - bnd[q]) for q in range(3)]
    bands = [dev(img[int(bnd[q]) * w:int(bnd[q + 1]) * w]) for q in range(3)]
    whole = oracle.conv5x5_u8(h, w, 256, img, synth.BINOMIAL)
    ok = True
    for q in range(3):
        top, bot = band_halo_rows([t.data_ptr() for t in bands], rows, q, w, 4)
        out = torch.empty(rows[q] * w, dtype=torch.int32, device="cuda")
        pb.device.conv5x5_u8_band(rows[q], w, 256, bands[q], top, bot, synth.BINOMIAL, out)
        ok &= np.array_equal(out.cpu().numpy(), whole[int(bnd[q]) * w:int(bnd[q + 1]) * w])
    check("conv5x5_u8_band x3", ok)
    # gemm (tcgen05, ragged edges)
    gm, gn, gk = 257, 260, 100
    GA, GB, GC = synth.f32(gm * gk, 13), synth.f32(gk * gn, 14), synth.f32(gm * gn, 15)
    C = dev(GC.copy())
    pb.device.gemm(gm, gn, gk, 1.0, 0.5, dev(GA), dev(GB), C)
    refc = GA.reshape(gm, gk).astype(np.float64) @ GB.reshape(gk, gn) + 0.5 * GC.reshape(gm, gn)
    scale = np.abs(GA.reshape(gm, gk)).astype(np.float64) @ np.abs(GB.reshape(gk, gn)) + 0.5 * np.abs(GC.reshape(gm, gn))
    check("gemm 3xtf32", float(np.max(np.abs(C.cpu().numpy().reshape(gm, gn) - refc) / scale)) < 1e-5)
    # OP2 (atomics schedule) and a JIT unit
    import json
    from paper_1302_5586_b200.op2 import Op2Model
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "op2_cases.json")))
    for nm in ("mesh", "multi_loop_levels"):
        mo = Op2Model(cases[nm]["doc"])
        mo.run()
        check(f"op2 {nm}", all(mo.dat(kk).tolist() == v for kk, v in cases[nm]["result"].items()))
        mo.close()
    torch.cuda.synchronize()
    print("cases %d failed" % len(bad), flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

"""The general mapper (JitUnit) against the hand-written kernels on the same fixtures: how much the
interpreter-exact fp64/int64 path costs.  gemv 4096^2 (independent rows, inner reduction in
order) and spmv_vec at 2^20 rows (16 nnz/row), device-resident arrays, one call timed after a
warm-up call (the call includes the frame upload and the per-segment synchronisation).
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_5586_b200 as pb  # noqa: E402
from paper_1302_5586_b200 import Arg, synth  # noqa: E402
from paper_1302_5586_b200.op2 import JitUnit  # noqa: E402

FIX = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1302_5586_b200", "pencil")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


def main():
    out = {}
    m = n = 4096
    A, x, y = synth.f32(m * n), synth.f32(n, 3), np.zeros(m, np.float32)
    u = JitUnit(open(os.path.join(FIX, "gemv.pencil.c")).read())
    u.set_array("A", A)
    u.set_array("x", x)
    u.set_array("y", y)
    out["gemv_4096_jit_ms"] = timed(lambda: u.call("gemv", [m, n, 1.0, 0.0, Arg.array("A"), Arg.array("x"), Arg.array("y")]))
    Ad, xd, yd = (torch.from_numpy(a).cuda() for a in (A, x, y))
    out["gemv_4096_native_ms"] = timed(lambda: pb.device.gemv(m, n, 1.0, 0.0, Ad, xd, yd))
    rowptr, col, val, xs, _ = synth.csr_powerlaw(1 << 20)
    nr, nnz = rowptr.size - 1, col.size
    v = JitUnit(open(os.path.join(FIX, "spmv.pencil.c")).read())
    for k, a in (("rp", rowptr), ("col", col), ("val", val), ("x", xs), ("y", np.zeros(nr, np.float32))):
        v.set_array(k, a)
    out["spmv_2e20_jit_ms"] = timed(lambda: v.call("spmv_vec", [nr, nr, nnz] + [Arg.array(k) for k in ("rp", "col", "val", "x", "y")]))
    rp, cd, vd, xdd = (torch.from_numpy(a).cuda() for a in (rowptr, col, val, xs))
    ys = torch.empty(nr, device="cuda")
    plan = pb.device.CsrPlan(nr, nr, nnz, rp, mode=1)
    out["spmv_2e20_native_ms"] = timed(lambda: plan.spmv(rp, cd, vd, xdd, ys))
    print(json.dumps(out))


if __name__ == "__main__":
    main()

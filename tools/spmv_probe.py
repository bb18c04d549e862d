"""One headline SpMV (spmv_vec on the 2^24-row power-law matrix) and the row-free gather probe on the
same col / val / x, each after a warm-up and an L2 flush — the command the SpMV ncu captures profile.

usage: python tools/spmv_probe.py [mode]      (mode 1 = spmv_vec, 0 = spmv_inline)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1302_5586_b200 as pb  # noqa: E402
from paper_1302_5586_b200 import synth  # noqa: E402


def main():
    mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    torch.cuda.set_device(0)
    rowptr, col, val, x, _ = synth.csr_powerlaw(1 << 24)
    n, nnz = rowptr.size - 1, col.size
    rp, cd, vd, xd = (torch.from_numpy(a).cuda() for a in (rowptr, col, val, x))
    y = torch.empty(n, device="cuda")
    plan = pb.device.CsrPlan(n, n, nnz, rp, mode=mode)
    lib, st = pb.load(), torch.cuda.current_stream().cuda_stream
    res = torch.empty(148 * 8 * 256, device="cuda")
    for _ in range(3):
        pb.device.l2_flush()
        plan.spmv(rp, cd, vd, xd, y)
        pb.device.l2_flush()
        lib.pencil_micro_gather_val(st, nnz, cd.data_ptr(), vd.data_ptr(), xd.data_ptr(), res.data_ptr())
    torch.cuda.synchronize()
    pb.device.sync_status()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    pb.device.l2_flush()
    e[0].record()
    plan.spmv(rp, cd, vd, xd, y)
    e[1].record()
    pb.device.l2_flush()
    e[2].record()
    lib.pencil_micro_gather_val(st, nnz, cd.data_ptr(), vd.data_ptr(), xd.data_ptr(), res.data_ptr())
    e[3].record()
    torch.cuda.synchronize()
    print("spmv mode %d %.4f ms, gather probe %.4f ms" % (mode, e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])))


if __name__ == "__main__":
    main()

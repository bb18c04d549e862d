"""Headline matrix (2^24 rows, power-law, 16 nnz/row): the reassociating executor (spmv_vec) vs
the source-order one (spmv_inline / ACCESS spmv), device-resident, L2 flushed between reps."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_5586_b200 as pb  # noqa: E402
from paper_1302_5586_b200 import synth  # noqa: E402


def t(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        pb.device.l2_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(statistics.mean(ts), 4)


n = 1 << 24
rowptr, col, val, x, _ = synth.csr_powerlaw(n)
rp, cd, vd, xd = (torch.from_numpy(a).cuda() for a in (rowptr, col, val, x))
y = torch.empty(n, device="cuda")
out = {}
for mode, name in ((1, "spmv_vec (reassociated)"), (0, "spmv_inline (source order)")):  # noqa: E501
    plan = pb.device.CsrPlan(n, n, col.size, rp, mode=mode)
    out[name] = t(lambda: plan.spmv(rp, cd, vd, xd, y))
    out[name + " bits"] = int(y.view(torch.int32).to(torch.int64).sum())  # A/B builds: same bits
print(json.dumps(out))

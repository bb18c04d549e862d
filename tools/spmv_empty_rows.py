"""The headline matrix with an empty row inserted after every third row (2^24 non-empty rows,
~2.2 x 10^7 rows): plans with empty rows take the batch-and-fold executor (csr_flow_kernel).
Times both modes, device-resident, L2 flushed between reps."""
import json
import os
import statistics
import sys

import numpy as np
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


rowptr, col, val, x, _ = synth.csr_powerlaw(1 << 24)
n = rowptr.size - 1
lens = np.diff(rowptr)
nl = np.zeros(n + n // 3, np.int64)
pos = np.arange(n) + np.arange(n) // 3  # an empty row after every third row
nl[pos] = lens
rp2 = np.concatenate([[0], np.cumsum(nl)]).astype(np.int32)
n2 = rp2.size - 1
rp, cd, vd, xd = (torch.from_numpy(a).cuda() for a in (rp2, col, val, x))
y = torch.empty(n2, device="cuda")
out = {"rows": n2}
for mode, name in ((1, "spmv_vec"), (0, "spmv_inline")):
    plan = pb.device.CsrPlan(n2, x.size, col.size, rp, mode=mode)
    out[name] = t(lambda: plan.spmv(rp, cd, vd, xd, y))
print(json.dumps(out))

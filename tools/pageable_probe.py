"""Pageable-array drop-in calls (the staging ring): spmv_vec at 2^24 rows, axpy 2^28, conv5x5_u8
16384^2 on plain numpy arrays, median of 3 after a warm-up — A/B of staging builds
(PENCIL_B200_LIB).  usage: python tools/pageable_probe.py"""
import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_5586_b200 as pb  # noqa: E402
from paper_1302_5586_b200 import synth  # noqa: E402


def t(f, reps=3):
    f()
    ts = []
    for _ in range(reps):
        a = time.perf_counter()
        f()
        ts.append(time.perf_counter() - a)
    return statistics.median(ts)


out = {}
rowptr, col, val, x, _ = synth.csr_powerlaw(1 << 24)
nrows, nnz = rowptr.size - 1, col.size
y = np.zeros(nrows, np.float32)
s = t(lambda: pb.dropin.spmv_vec(nrows, nrows, nnz, rowptr, col, val, x, y))
out["spmv_vec GB/s"] = round((8 * nnz + 8 * nrows + 4 + 4 * nrows) / s / 1e9, 1)
del rowptr, col, val
n = 1 << 28
xa, ya = synth.f32(n, 1), synth.f32(n, 2)
s = t(lambda: pb.dropin.axpy(n, 1.5, xa, ya))
out["axpy GB/s"] = round(12 * n / s / 1e9, 1)
del xa, ya
h = w = 16384
img = synth.u8_i32(h * w)
o = np.empty(h * w, np.int32)
s = t(lambda: pb.dropin.conv5x5_u8(h, w, 256, img, synth.BINOMIAL, o))
out["conv5x5_u8 GB/s"] = round(8 * h * w / s / 1e9, 1)
print(json.dumps(out))

"""Time an OP2 edge->cell increment par_loop (the reference's mesh kernel) on a random mesh.

    python tools/op2_probe.py [log2_cells] [log2_edges]
Algorithmic bytes per edge: map row (2 x 4 B, int32 on the device) + dedges (8 B) + two 8-byte
increments (atomic read-modify-write at L2), plus one read + write of every cell value.
"""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_5586_b200 as pb  # noqa: E402
from paper_1302_5586_b200.op2 import Op2Model  # noqa: E402

KERNEL = ("void kernel(int n_dedges, int n_dcells, int dedges[restrict const static n_dedges], "
          "int dcells[restrict const static n_dcells], int ie, int ic0, int ic1)\n"
          "{\n  dcells[ic1] += dedges[ie];\n  dcells[ic0] += dedges[ie];\n}\n")


def mesh_doc(nc, ne, seed=1):
    rng = np.random.default_rng(seed)
    table = rng.integers(0, nc, size=2 * ne, dtype=np.int64)
    return {
        "sets": [{"name": "cells", "size": nc}, {"name": "edges", "size": ne}],
        "maps": [{"name": "pecell", "from": "edges", "to": "cells", "arity": 2, "table": table.tolist()}],
        "dats": [{"name": "dcells", "set": "cells", "dim": 1, "data": [0] * nc},
                 {"name": "dedges", "set": "edges", "dim": 1, "data": rng.integers(-999, 999, size=ne).tolist()}],
        "kernels": [{"name": "kernel", "source": KERNEL}],
        "par_loops": [{"kernel": "kernel", "set": "edges", "args": [
            {"dat": "dedges", "access": "OP_READ"},
            {"dat": "dcells", "map": "pecell", "offset": 0, "access": "OP_INC"},
            {"dat": "dcells", "map": "pecell", "offset": 1, "access": "OP_INC"}]}],
    }


def time_loop(m, steps=10, warmup=3):
    st = torch.cuda.ExternalStream(m.stream)
    ts = []
    with torch.cuda.stream(st):
        for it in range(warmup + steps):
            pb.device.l2_flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            m.run_loop_async(0)
            b.record()
            torch.cuda.synchronize()
            if it >= warmup:
                ts.append(a.elapsed_time(b))
    m.sync()
    return statistics.mean(ts)


def main():
    lc = int(sys.argv[1]) if len(sys.argv) > 1 else 22
    le = int(sys.argv[2]) if len(sys.argv) > 2 else 23
    nc, ne = 1 << lc, 1 << le
    t0 = time.time()
    doc = json.dumps(mesh_doc(nc, ne))
    t1 = time.time()
    m = Op2Model(doc)
    t2 = time.time()
    m.prepare()
    t3 = time.time()
    ms = time_loop(m)
    b = ne * (8 + 8 + 16) + nc * 16
    print(json.dumps({"cells": nc, "edges": ne, "ms": ms, "Gedges/s": ne / ms / 1e6, "GB/s": b / ms / 1e6,
                      "strategy": m.loop_info(0), "json_s": round(t1 - t0, 2), "load_s": round(t2 - t1, 2),
                      "prepare_s": round(t3 - t2, 2)}))


if __name__ == "__main__":
    main()

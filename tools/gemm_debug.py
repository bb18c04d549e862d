"""gemm layout debugging: error of the device gemm on integer-valued operands (lo halves zero: the
hi path and the operand layouts alone), on one-hot A (C rows must equal B rows) and on random fp32
operands; prints the first mismatches.  PENCIL_B200_LIB selects a variant build."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1302_5586_b200 as pb  # noqa: E402
from paper_1302_5586_b200 import synth  # noqa: E402


def run(m, n, k, A, B):
    C = torch.zeros(m * n, device="cuda")
    pb.device.gemm(m, n, k, 1.0, 0.0, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C)
    torch.cuda.synchronize()
    return C.cpu().numpy().reshape(m, n)


for (m, n, k) in [(256, 256, 16), (256, 256, 64), (300, 520, 40)]:
    i, p, j = np.arange(m)[:, None], np.arange(k)[None, :], np.arange(n)[None, :]
    A = (((i * 7 + p * 3) % 5) - 2).astype(np.float32)
    B = (((np.arange(k)[:, None] * 5 + j * 11) % 7) - 3).astype(np.float32)
    got, ref = run(m, n, k, A.ravel(), B.ravel()), A.astype(np.float64) @ B
    bad = np.argwhere(got != ref)
    print(f"int {m}x{n}x{k}: wrong {len(bad)} / {m * n}", bad[:6].tolist())
    oh = np.zeros((m, k), np.float32)
    oh[np.arange(m), np.arange(m) % k] = 1
    Bj = (np.arange(k)[:, None] * 100 + j % 100).astype(np.float32)
    got = run(m, n, k, oh.ravel(), Bj.ravel())
    ref = oh.astype(np.float64) @ Bj
    bad = np.argwhere(got != ref)
    print(f"onehot: wrong {len(bad)}", [(int(a), int(b), float(got[a, b]), float(ref[a, b])) for a, b in bad[:6]])
    Ar, Br = synth.f32(m * k, 1), synth.f32(k * n, 2)
    got = run(m, n, k, Ar, Br)
    A2, B2 = Ar.reshape(m, k).astype(np.float64), Br.reshape(k, n).astype(np.float64)
    err = np.max(np.abs(got - A2 @ B2) / (np.abs(A2) @ np.abs(B2)))
    print(f"random: normwise {err:.3e}")

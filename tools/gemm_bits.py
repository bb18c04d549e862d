"""Bit checksum of the device gemm on random fp32 operands (A/B builds that must agree bit for bit:
PENCIL_B200_LIB selects the variant).  usage: python tools/gemm_bits.py [m n k]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1302_5586_b200 as pb  # noqa: E402
from paper_1302_5586_b200 import synth  # noqa: E402

m, n, k = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (1536, 1280, 2064)
A = torch.from_numpy(synth.f32(m * k, 7)).cuda()
B = torch.from_numpy(synth.f32(k * n, 8) * np.float32(1e-3)).cuda()  # different binades than A
C = torch.zeros(m * n, device="cuda")
pb.device.gemm(m, n, k, 1.0, 0.0, A, B, C)
torch.cuda.synchronize()
bits = C.view(torch.int32).to(torch.int64)
print(m, n, k, int(bits.sum()), int((bits * torch.arange(bits.numel(), device="cuda")).sum() % (1 << 61)))

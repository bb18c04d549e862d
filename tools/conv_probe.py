"""Time the 5x5 stencil kernels at 16384^2 (device-resident, L2 flushed between reps)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_5586_b200 as pb
from paper_1302_5586_b200 import synth

def t(fn, reps=10):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        pb.device.l2_flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return round(min(ts), 4)

h = w = 16384
which = sys.argv[1:] or ["f32", "u8", "u8b"]
out = {}
if "f32" in which:
    img = torch.from_numpy(synth.f32(h * w)).cuda(); o = torch.zeros(h * w, device="cuda")
    kf = (synth.BINOMIAL.astype(np.float32) / 256.0).astype(np.float32)
    out["conv_f32_ms"] = t(lambda: pb.device.conv5x5_f32(h, w, img, kf, o))
    kg = synth.f32(25, 9)  # generic taps (not powers of two): the as-written kernel
    out["conv_f32_generic_ms"] = t(lambda: pb.device.conv5x5_f32(h, w, img, kg, o)); del img, o
# u8 / u8b: binomial (separable kernels) and sharpen (25-tap kernels); u8sharp / u8bsharp: sharpen only
if "u8" in which or "u8sharp" in which:
    img = torch.from_numpy(synth.u8_i32(h * w)).cuda(); o = torch.empty(h * w, dtype=torch.int32, device="cuda")
    if "u8" in which:
        out["conv_u8_i32_ms"] = t(lambda: pb.device.conv5x5_u8(h, w, 256, img, synth.BINOMIAL, o))
    out["conv_u8_i32_sharpen_ms"] = t(lambda: pb.device.conv5x5_u8(h, w, 1, img, synth.SHARPEN, o)); del img, o
if "u8b" in which or "u8bsharp" in which:
    img = torch.from_numpy(synth.u8(h * w)).cuda(); o = torch.empty(h * w, dtype=torch.uint8, device="cuda")
    if "u8b" in which:
        out["conv_u8_bytes_ms"] = t(lambda: pb.device.conv5x5_u8_bytes(h, w, 256, img, synth.BINOMIAL, o))
    out["conv_u8_bytes_sharpen_ms"] = t(lambda: pb.device.conv5x5_u8_bytes(h, w, 1, img, synth.SHARPEN, o))
print(json.dumps(out))

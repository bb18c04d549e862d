"""End-to-end timing of the pipelined host-array stencil drop-ins (conv5x5_u8 int32 / conv5x5_f32 at
16384^2, pinned and after pageable staged calls) with the bytes each call moved — the check behind
the bench lines' e2e numbers.  usage: python tools/e2e_stencil_probe.py"""
import sys, os, time, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1302_5586_b200 as pb
from paper_1302_5586_b200 import synth
h = w = 16384; npx = h * w
lib = pb.load()
def run(name, f, reps=5):
    f(); ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); ts.append((time.perf_counter() - t0) * 1e3)
    a, b = ctypes.c_longlong(), ctypes.c_longlong(); lib.pencil_last_transfer_bytes(ctypes.byref(a), ctypes.byref(b))
    print(name, [round(t, 1) for t in ts], a.value, b.value, flush=True)
himg = synth.u8_i32(npx)
i_ = torch.from_numpy(himg).pin_memory(); o_ = torch.from_numpy(np.empty(npx, np.int32)).pin_memory()
run("u8 binom", lambda: pb.dropin.conv5x5_u8(h, w, 256, i_, synth.BINOMIAL, o_))
run("u8 sharpen", lambda: pb.dropin.conv5x5_u8(h, w, 1, i_, synth.SHARPEN, o_))
f = synth.f32(npx); fi = torch.from_numpy(f).pin_memory(); fo = torch.from_numpy(np.zeros(npx, np.float32)).pin_memory()
kf = (synth.BINOMIAL / 256.0).astype(np.float32)
run("f32", lambda: pb.dropin.conv5x5_f32(h, w, fi, kf, fo))
run("u8 binom again", lambda: pb.dropin.conv5x5_u8(h, w, 256, i_, synth.BINOMIAL, o_))
# after pageable (staged) calls: does the staging pool slow the next pinned pipelined call?
n = 1 << 28
x, y = synth.f32(n, 1), synth.f32(n, 2)
run("axpy pageable", lambda: pb.dropin.axpy(n, 1.5, x, y), reps=3)
run("u8 binom after pageable", lambda: pb.dropin.conv5x5_u8(h, w, 256, i_, synth.BINOMIAL, o_))
hp, op = himg, np.empty(npx, np.int32)
run("u8 binom pageable", lambda: pb.dropin.conv5x5_u8(h, w, 256, hp, synth.BINOMIAL, op), reps=3)
run("u8 binom pinned after", lambda: pb.dropin.conv5x5_u8(h, w, 256, i_, synth.BINOMIAL, o_))
run("f32 pinned after", lambda: pb.dropin.conv5x5_f32(h, w, fi, kf, fo))

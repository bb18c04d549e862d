"""Time gemv 8192^2 / gemv_t 16384^2 strided / dot / axpy (device-resident, L2 flushed)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_5586_b200 as pb
from paper_1302_5586_b200 import synth

def t(fn, reps=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        pb.device.l2_flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort()
    return round(ts[len(ts) // 2], 4)

out = {}
m = n = 8192
A = torch.from_numpy(synth.f32(m * n)).cuda(); x = torch.from_numpy(synth.f32(n, 3)).cuda(); y = torch.zeros(m, device="cuda")
ms = t(lambda: pb.device.gemv(m, n, 1.0, 0.0, A, x, y)); b = 4 * (m * n + m + n)
out["gemv_8192"] = {"ms": ms, "GB/s": round(b / ms / 1e6, 1)}
print(json.dumps(out))
if len(sys.argv) > 1 and sys.argv[1] == "ref":
    # pure-read reference at the gemv size: dot over 2 x 2^25 floats = 268 MB
    n2 = 1 << 25
    xa = torch.from_numpy(synth.f32(n2, 5)).cuda(); ya = torch.from_numpy(synth.f32(n2, 6)).cuda(); r = torch.zeros(1, device="cuda")
    ms = t(lambda: pb.device.dot(n2, xa, ya, r))
    print(json.dumps({"dot_268MB": {"ms": ms, "GB/s": round(8 * n2 / ms / 1e6, 1)}}))

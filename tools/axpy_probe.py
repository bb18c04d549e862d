"""A/B timing of axpy variants (host scalar vs device scalar) on 2^28 vectors."""
import json, os, sys
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
    return min(ts), sum(ts) / len(ts)

n = 1 << 28
x = torch.from_numpy(synth.f32(n, 7)).cuda(); y = torch.from_numpy(synth.f32(n, 8)).cuda()
r = torch.full((1,), 0.5, device="cuda")
out = {}
out["axpy_host_scalar"] = t(lambda: pb.device.axpy(n, 0.5, x, y))
out["axpy_dev_scalar"] = t(lambda: pb.device.axpy_ptr(n, r, x, y))
out["dot"] = t(lambda: pb.device.dot(n, x, y, r))
out["torch_add_"] = t(lambda: y.add_(x, alpha=0.5))
pb.device.dot(n, x, y, r); torch.cuda.synchronize(); out["r_after_dot"] = float(r.item())
out["axpy_dev_scalar_after_dot"] = t(lambda: pb.device.axpy_ptr(n, r, x, y))
out["y_absmax"] = float(y.abs().max().item())
y2 = torch.from_numpy(synth.f32(n, 8)).cuda()
out["axpy_host_minus2751"] = t(lambda: pb.device.axpy(n, -2751.0, x, y2))
y3 = torch.from_numpy(synth.f32(n, 8)).cuda()
out["axpy_host_0.5_fresh"] = t(lambda: pb.device.axpy(n, 0.5, x, y3))
print(json.dumps(out))

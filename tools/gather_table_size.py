import json, sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1302_5586_b200 as pb
lib = pb.load()
st = torch.cuda.current_stream().cuda_stream
n = 1 << 28
out = {}
for lt in (20, 22, 23, 24, 25):
    ncols = 1 << lt
    table = torch.randn(ncols, device="cuda")
    idx = torch.randint(0, ncols, (n,), device="cuda", dtype=torch.int32)
    val = torch.randn(n, device="cuda")
    res = torch.empty(148 * 8 * 256, device="cuda")
    ts = []
    for r in range(8):
        pb.device.l2_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); lib.pencil_micro_gather_val(st, n, idx.data_ptr(), val.data_ptr(), table.data_ptr(), res.data_ptr()); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    out[f"table_{ncols*4>>20}MB"] = round(min(ts[2:]), 4)
    del table, idx, val
print(json.dumps(out))

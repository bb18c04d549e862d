"""Hardware probes used to set the roofline expectations in DESIGN.md (run on a B200):
random 4-byte gather rate out of a 64 MB table (the x[col[k]] access of SpMV) per load flavour,
and float4 copy bandwidth for HBM-resident and L2-resident buffers."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_5586_b200 as pb  # noqa: E402


def time_ms(fn, reps=10, flush=True):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        if flush:
            pb.device.l2_flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts), sum(ts) / len(ts)


def main():
    lib = pb.load()
    st = torch.cuda.current_stream().cuda_stream
    out = {"device": torch.cuda.get_device_name(0)}
    ncols = 1 << 24
    n = 1 << 28
    table = torch.randn(ncols, device="cuda")
    idx = torch.randint(0, ncols, (n,), device="cuda", dtype=torch.int32)
    res = torch.empty(148 * 8 * 256, device="cuda")
    for mode, name in enumerate(["ld.global", "ld.global.nc", "ld.global.cg", "ld.nc.L2::evict_last"]):
        best, avg = time_ms(lambda: lib.pencil_micro_gather(st, mode, n, idx.data_ptr(), table.data_ptr(), res.data_ptr()))
        out[f"gather_{name}"] = {"ms": best, "Ggathers/s": n / best / 1e6, "idx_GB/s": 4 * n / best / 1e6}
    # scaling: CTAs per SM (1,2,4) and one CTA per SM on all / half of the SMs
    for label, mode in [("1cta_per_sm", 1 | (1 << 4)), ("2cta_per_sm", 1 | (2 << 4)), ("4cta_per_sm", 1 | (4 << 4)),
                        ("1cta_bigsmem_148sm", 1 | (1 << 4) | (1 << 8)), ("1cta_bigsmem_74sm", 1 | (1 << 8) | (1 << 9))]:
        best, _ = time_ms(lambda: lib.pencil_micro_gather(st, mode, n, idx.data_ptr(), table.data_ptr(), res.data_ptr()))
        out[f"gather_scaling_{label}"] = {"ms": best, "Ggathers/s": n / best / 1e6}
    # the SpMV data path without rows: idx + val streams and the gather (practical SpMV ceiling)
    val = torch.randn(n, device="cuda")
    best, _ = time_ms(lambda: lib.pencil_micro_gather_val(st, n, idx.data_ptr(), val.data_ptr(), table.data_ptr(), res.data_ptr()))
    out["gather_val_stream"] = {"ms": best, "Ggathers/s": n / best / 1e6, "spmv_algo_GB/s": (8 * n + 12 * ncols) / best / 1e6}
    del val
    # sorted indices (perfect locality) for contrast
    idx_sorted, _ = torch.sort(idx)
    best, _ = time_ms(lambda: lib.pencil_micro_gather(st, 1, n, idx_sorted.data_ptr(), table.data_ptr(), res.data_ptr()))
    out["gather_sorted_idx"] = {"ms": best, "Ggathers/s": n / best / 1e6}
    del idx, idx_sorted
    for mb in [4096, 1024, 32]:
        nel = mb * (1 << 20) // 4
        a, b = torch.randn(nel, device="cuda"), torch.empty(nel, device="cuda")
        best, _ = time_ms(lambda: lib.pencil_micro_copy(st, nel, a.data_ptr(), b.data_ptr()), reps=20, flush=(mb > 64))
        out[f"copy_{mb}MiB"] = {"ms": best, "GB/s_rw": 8 * nel / best / 1e6}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the B200 PENCIL backend (contract: see DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload W]

Headline workload (BASELINE.json configs[1]): CSR SpMV fp32, synthetic power-law matrix with
2^24 rows, 16 nnz/row (SURVEY §8d generator, seed 42).  One step = one SpMV (spmv_vec) over the
device-resident matrix.  `value` = algorithmic bytes (8*nnz + 4*(nrows+1) + 4*nrows + 4*ncols)
per step / device time, whole job; `e2e` = the same metric through the drop-in C ABI with pinned
host buffers (H2D of the whole matrix + D2H of y inside the timed region).  The other configs
(gemv, VOBLA gemv_t+dot+axpy chain, 5x5 stencils u8/fp32, gemm) run as the `suite` object.

N>1 (torchrun, one process per GPU, NCCL): rows are sharded by non-zeros, x is all-gathered
every step (the data path's real exchange), value = global bytes / max-over-ranks time
(strong scaling).  `--impl reference` times the reference's CPU path: the C that the
reference's emit_openmp produced for the same PENCIL fixtures (oracle/_ref), all host cores.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "kernel GB/s & % HBM roofline (gemv/SpMV/stencil), gemm TFLOP/s; 1-8 B200"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
SPEC_HBM_GBS = 8000.0  # B200 HBM3e spec; the roofline `peak` is the measured copy rate
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def ncu_traffic(kernel):
    """DRAM read + write bytes per launch of `kernel` from the committed ncu capture
    (profiles/ncu_traffic.json, tools/traffic_capture.py); exact name, else the name without
    its template arguments; None when the kernel was not captured."""
    try:
        with open(NCU_SUMMARY) as f:
            t = json.load(f)
    except Exception:
        return None
    if kernel in t:
        return t[kernel]
    base = kernel.split("<")[0]
    cands = [v for k, v in t.items() if k.split("<")[0] == base]
    return cands[0] if len(cands) == 1 else None


# ------------------------------------------------------------------ clocks sampling
class Clocks:
    def __init__(self, index=0):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([t.strip() for t in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and "Active" in s[3 + i]
                          and "Not" not in s[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ workloads (ours)
def spmv_config(nrows, nnz, xm):
    """The headline workload (BASELINE.json configs[1]) — the same dict on both arms."""
    return {"workload": "CSR SpMV fp32 (spmv_vec), power-law rows 2^24 x 2^24, 16 nnz/row",
            "nrows": nrows, "ncols": nrows, "nnz": nnz, "alpha": 1.5, "xm": round(xm, 4), "maxlen": 4096, "seed": 42}


def spmv_bytes(nrows, ncols, nnz):
    return 8 * nnz + 4 * (nrows + 1) + 4 * nrows + 4 * ncols


class Timer:
    """Per-step CUDA events on torch's current stream (where the library launches)."""

    def __init__(self, torch, k):
        self.torch = torch
        self.s = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        self.e = [torch.cuda.Event(enable_timing=True) for _ in range(k)]

    def ms(self):
        return [a.elapsed_time(b) for a, b in zip(self.s, self.e)]


def run_steps(torch, step, k, w, flush, dist=None):
    for _ in range(w):
        step()
    torch.cuda.synchronize()
    t = Timer(torch, k)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(k):
        flush()  # L2 flush between steps, outside the per-step events
        t.s[i].record()
        step()
        t.e[i].record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    return t.ms()


def bench_spmv(args, torch, pb, rank, world, dist):
    from paper_1302_5586_b200 import synth
    nrows = 1 << 24
    rowptr, col, val, x, xm = synth.csr_powerlaw(nrows)
    nnz = int(col.size)
    flush = lambda: pb.device.l2_flush()  # noqa: E731
    if not args.dist_path:
        rp, cd, vd, xd = (torch.from_numpy(a).cuda() for a in (rowptr, col, val, x))
        y = torch.empty(nrows, device="cuda")
        plan = pb.device.CsrPlan(nrows, nrows, nnz, rp, mode=1)
        step = lambda: plan.spmv(rp, cd, vd, xd, y)  # noqa: E731
        ms = run_steps(torch, step, args.steps, args.warmup, flush)
        pb.device.sync_status()
        launches = args.steps * 3  # spmv + l2 flush (fill + discard) per step
        kernel_ms = statistics.mean(ms)
        # the measured ceiling of this matrix: the same col/val stream and x gathers without the
        # rows (k_micro.cu micro_gather_val), timed the same way, outside the timed SpMV steps
        lib, st = pb.load(), torch.cuda.current_stream().cuda_stream
        res_buf = torch.empty(148 * 8 * 256, device="cuda")
        ceil_ms = statistics.mean(run_steps(
            torch, lambda: lib.pencil_micro_gather_val(st, nnz, cd.data_ptr(), vd.data_ptr(), xd.data_ptr(),
                                                       res_buf.data_ptr()), max(3, args.steps // 2), 2, flush))
        # the same matrix in source order (spmv_inline / the ACCESS-summarised spmv: row sums folded
        # in order, bit-identical to the emitted C) — a suite line beside the headline
        plan0 = pb.device.CsrPlan(nrows, nrows, nnz, rp, mode=0)
        src_ms = statistics.mean(run_steps(torch, lambda: plan0.spmv(rp, cd, vd, xd, y), max(3, args.steps // 2), 2,
                                           flush))
        pb.device.sync_status()
        plan0.close()
    else:
        src_ms = None
        # one step of a row-sharded iterative SpMV: y = A x for the rank's rows, y gathered on
        # every rank (the next step's x) — fused into the SpMV kernel (NVLink / NVLS stores) or
        # SpMV + NCCL all-gather
        from paper_1302_5586_b200.dist import RowShardedCsr, FusedSpmvAllgather
        sh = RowShardedCsr(rowptr, col, val, rank, world)
        rp, cd, vd = (torch.from_numpy(a).cuda() for a in (sh.rowptr, sh.col, sh.val))
        x_local = sh.pad_local_x(torch.from_numpy(x[sh.r0:sh.r1]).cuda())
        xg = sh.allgather_x(x_local)  # the gathered x, resident
        y_pad = torch.zeros(sh.max_rows, device="cuda")
        y = y_pad[: sh.nrows]
        plan = pb.device.CsrPlan(sh.nrows, sh.ncols_padded, sh.nnz, rp, mode=1)
        mode = args.dist_mode if args.dist_backend == "nccl" else "nccl"
        if mode == "fused":
            try:
                fz = FusedSpmvAllgather(sh, torch.device("cuda", torch.cuda.current_device()))
                exchange = "fused SpMV->all-gather (%s)" % ("NVLS multicast stores" if fz.mc else "NVLink peer stores")
            except Exception as e:  # noqa: BLE001 — no symmetric memory here: the unfused step
                mode, why = "nccl", str(e).splitlines()[0][:120]
        # every step feeds the gathered y back as the next x (the iterative method the step
        # belongs to): the fused path through its ping-pong halves, the unfused one by swapping
        # two gathered buffers
        if mode == "fused":
            # one checked step before the timing: the fused result must equal SpMV + all-gather bit
            # for bit on every rank, else the bench takes the unfused step (and says why)
            fz.load(x_local)
            fz.step(plan, rp, cd, vd, None, y)
            got = fz.current().view(torch.int32).clone()
            y_ref = torch.zeros(sh.max_rows, device="cuda")
            plan.spmv(rp, cd, vd, xg, y_ref[: sh.nrows])
            ref = sh.allgather_x(y_ref).view(torch.int32)
            bad = torch.tensor([0 if torch.equal(got[: ref.numel()], ref) else 1], device="cuda")
            dist.all_reduce(bad)
            if int(bad.item()):
                mode, why = "nccl", "the fused step differed from SpMV + all-gather on %d rank(s)" % int(bad.item())
                exchange += " -> failed its check step"
            else:
                exchange += ", checked against SpMV + all-gather (bit-identical)"
                fz.load(x_local)  # restart the chain from x
        if mode == "fused":

            def step():
                fz.step(plan, rp, cd, vd, None, y)
        else:
            bufs = [xg, torch.empty(sh.ncols_padded, device="cuda")]
            exchange = "SpMV + %s all-gather of y" % args.dist_backend
            if args.dist_mode == "fused" and args.dist_backend == "nccl":
                exchange += " (fused path unavailable: %s)" % why

            def step():
                plan.spmv(rp, cd, vd, bufs[0], y)
                sh.allgather_x(y_pad, bufs[1])
                bufs.reverse()
        ms = run_steps(torch, step, args.steps, args.warmup, flush, dist)
        kernel_ms = statistics.mean(ms)
        launches = args.steps * (5 if mode == "fused" else 3)  # + the two symmetric-memory barriers
        e2e = None
        if not args.no_e2e:
            sh.total_nnz = nnz
            e2e = e2e_spmv_dist(args, torch, pb, sh, x, dist)
    algo = spmv_bytes(nrows, nrows, nnz)
    res = {"ms": kernel_ms, "bytes": algo, "launches": launches,
           "ceiling_ms": ceil_ms if not args.dist_path else None,
           "src_ms": src_ms if not args.dist_path else None,
           "config": dict(spmv_config(nrows, nnz, xm),
                          schedule="csr_seg_kernel, reassociated (persistent warps on 4096-nnz row-aligned "
                                   "tiles, 128-bit col/val streams, per-lane segments + warp segmented scan over "
                                   "the plan's row-start bitmap)",
                          l2="L2 flushed between steps outside the per-step events (256 MiB fill, then its lines "
                             "discarded: the step starts on a clean, empty L2); inputs 2.35 GB > L2")}
    if args.dist_path:
        res["config"]["exchange"] = exchange
        if e2e:
            res["e2e"] = e2e
    if rank == 0 and not args.dist_path and not args.no_e2e:
        res["e2e"] = e2e_spmv(args, torch, pb, rowptr, col, val, x)
        res["src_e2e"] = e2e_spmv(args, torch, pb, rowptr, col, val, x, fn="spmv_inline")
    if rank == 0 and not args.dist_path:
        res["src_cpu"] = {}
        hy = np.zeros(nrows, np.float32)  # kept alive across the calls (the C writes through its pointer)
        cpu_ref(args, res["src_cpu"], lambda L: L.spmv_inline(nrows, nrows, nnz, P(rowptr), P(col), P(val), P(x),
                                                               P(hy)), algo, "full matrix, spmv_inline")
    return res


def e2e_spmv(args, torch, pb, rowptr, col, val, x, fn="spmv_vec"):
    """drop-in C ABI on host buffers, H2D + plan + kernel + D2H per call (synchronous): pinned
    (the headline `e2e`) and pageable (plain numpy, as a C program relinked from the emitted
    OpenMP passes its malloc'd arrays) — median over the steps after one warm-up call."""
    nrows, nnz = rowptr.size - 1, col.size
    algo = spmv_bytes(nrows, nrows, nnz)

    def mk(pinned):
        hrp, hcol, hval, hx = (host_buf(torch, a, pinned) for a in (rowptr, col, val, x))
        hy = host_buf(torch, np.zeros(nrows, np.float32), pinned)
        return lambda: getattr(pb.dropin, fn)(nrows, nrows, nnz, hrp, hcol, hval, hx, hy)
    e = e2e_calls(torch, pb, mk, algo, "GB/s", "%s (drop-in C ABI on host arrays: pinned = the headline "
                  "value, pageable beside it)" % fn, reps=max(2, min(args.steps, 5)))
    if "ms_per_call" in e.get("pinned", {}):
        e["ms_per_call"] = e["pinned"]["ms_per_call"]
    return e


def e2e_spmv_dist(args, torch, pb, sh, x, dist):
    """N>1 end to end: each rank uploads its row block and its slice of x from pinned host memory
    over its own host link, the x slices are all-gathered (NVLink), the plan is built and the
    rank's rows multiplied, and its y rows come back to the host — the drop-in call's work,
    sharded.  Device-timed per rank (events around the whole call), max over ranks."""
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hrp, hcol, hval, hx = pin(sh.rowptr), pin(sh.col), pin(sh.val), pin(x[sh.r0:sh.r1])
    hy = torch.empty(sh.nrows, dtype=torch.float32).pin_memory()
    drp, dcol, dval = (torch.empty(a.numel(), dtype=a.dtype, device="cuda") for a in (hrp, hcol, hval))
    xpad = torch.zeros(sh.max_rows, device="cuda")
    xg = torch.empty(sh.ncols_padded, device="cuda")
    y = torch.empty(sh.nrows, device="cuda")
    plans = []

    def call():
        drp.copy_(hrp, non_blocking=True)
        dcol.copy_(hcol, non_blocking=True)
        dval.copy_(hval, non_blocking=True)
        xpad[: sh.nrows].copy_(hx, non_blocking=True)
        plan = pb.device.CsrPlan(sh.nrows, sh.ncols_padded, sh.nnz, drp, mode=1)  # per call, as the drop-in
        plans.append(plan)
        sh.allgather_x(xpad, xg)
        plan.spmv(drp, dcol, dval, xg, y)
        hy.copy_(y, non_blocking=True)

    ms = statistics.mean(run_steps(torch, call, max(2, min(args.steps, 5)), 2, lambda: None, dist))
    torch.cuda.synchronize()
    for p in plans:
        p.close()
    h2d = 4 * ((sh.nrows + 1) + 2 * sh.nnz + sh.nrows)
    t = torch.tensor([ms, float(h2d), 4.0 * sh.nrows], dtype=torch.float64, device=coll_dev(dist))
    tmax = t[:1].clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    ms = float(tmax.item())
    algo = spmv_bytes(len(x), len(x), int(sh.total_nnz))
    return {"value": algo / ms / 1e6, "unit": "GB/s", "ms_per_call": ms, "h2d_bytes_per_step": int(t[1].item()),
            "d2h_bytes_per_step": int(t[2].item()),
            "api": "row-sharded spmv_vec: per rank pinned-host row block + x slice -> its GPU, %s all-gather "
                   "of x, plan + SpMV, y rows -> host (device events around the call, max over ranks)"
                   % dist.get_backend()}


# 3xTF32 = three tf32 MMAs per fp32 product; dense tf32 runs at half the bf16 rate, so the
# measured-scaled 3xTF32 peak is bf16 / 6 (burst: the kernel timed alone; sustained: under the
# 1 kW power cap in a long loop) — MEASURED_PEAKS.json bf16_tflops / bf16_tflops_sustained
def tf32x3_peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]) / 6.0, float(p.get("bf16_tflops_sustained", p["bf16_tflops"])) / 6.0, "measured"
    except Exception:
        return 1590.0 / 6.0, 1400.0 / 6.0, "fallback"


def roofline(achieved, peak, unit, kernel, algo, bound="hbm", per="launch", **extra):
    r = {"bound": bound, "kernel": kernel, "achieved": achieved, "peak": peak, "unit": unit,
         "frac": achieved / peak if peak else None, "traffic": ncu_traffic(kernel)}
    r["algorithmic_bytes_per_%s" % per if bound == "hbm" else "algorithmic_flops_per_%s" % per] = algo
    if bound == "hbm":
        r["frac_spec"] = achieved / SPEC_HBM_GBS
    r.update(extra)
    return r


def bw_line(ms, nbytes, hbm, kernel, **extra):
    gbs = nbytes / ms / 1e6
    return dict({"ms": ms, "GB/s": gbs, "frac_hbm": gbs / hbm, "bytes": nbytes,
                 "roofline": roofline(gbs, hbm, "GB/s", kernel, nbytes)}, **extra)


def e2e_calls(torch, pb, make_call, metric_amount, unit, api, reps=3):
    """The line's metric end to end through the library's public call on HOST arrays:
    make_call(pinned) returns a no-argument call that runs the whole operation on pinned
    (page-locked) or pageable (plain numpy) host buffers — H2D of the inputs, the kernel(s), D2H
    of the outputs, synchronous.  Wall time around the call, median of `reps` after a warm-up;
    the bytes each call moved over the link come from pencil_last_transfer_bytes (or from the
    call itself when it copies through the device API: it returns (h2d, d2h))."""
    lib = pb.load()
    out = {"api": api}
    for kind in ("pinned", "pageable"):
        try:
            call = make_call(kind == "pinned")
            moved = call()
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                moved = call()
                ts.append(time.perf_counter() - t0)
            t = statistics.median(ts)
            if moved is None:
                h2d, d2h = ctypes.c_longlong(), ctypes.c_longlong()
                lib.pencil_last_transfer_bytes(ctypes.byref(h2d), ctypes.byref(d2h))
                moved = (h2d.value, d2h.value)
            out[kind] = {"value": metric_amount / t / (1e9 if unit in ("GB/s", "Gpix/s") else 1e12),
                         "unit": unit, "ms_per_call": t * 1e3, "ms_calls": [round(v * 1e3, 2) for v in ts],
                         "h2d_bytes_per_step": int(moved[0]), "d2h_bytes_per_step": int(moved[1])}
        except Exception as e:  # noqa: BLE001 — one door's failure must not take the suite down
            out[kind] = {"unavailable": str(e)[:200]}
    if "value" in out.get("pinned", {}):
        out.update({k: out["pinned"][k] for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step")})
    return out


def host_buf(torch, a, pinned):
    """a (numpy) as a host buffer the drop-in call reads: a pinned torch copy, or a itself."""
    return torch.from_numpy(a).pin_memory() if pinned else a


def suite(args, torch, pb, hbm):
    """Secondary configs of BASELINE.json, one line each: device-resident kernel time (value +
    roofline object) and the same metric end to end through the C ABI on host buffers (e2e:
    pinned and pageable), with the reference CPU path beside it."""
    from paper_1302_5586_b200 import synth
    out = {}
    k, w = max(3, args.suite_steps), 3
    flush = lambda: pb.device.l2_flush()  # noqa: E731
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    no_e2e = args.no_e2e

    # gemv 8192^2 (configs[0])
    m = n = 8192
    hA, hx = synth.f32(m * n), synth.f32(n, 42, m * n)
    A, x, y = dev(hA), dev(hx), torch.zeros(m, device="cuda")
    ms = statistics.mean(run_steps(torch, lambda: pb.device.gemv(m, n, 1.0, 0.0, A, x, y), k, w, flush))
    b = 4 * (m * n + n + m)
    out["gemv_8192"] = bw_line(ms, b, hbm, "gemv_kernel")
    if not no_e2e:
        def mk(pinned):
            hA_, hx_, hy_ = (host_buf(torch, a, pinned) for a in (hA, hx, np.zeros(m, np.float32)))
            return lambda: pb.dropin.gemv(m, n, 1.0, 0.0, hA_, hx_, hy_)
        out["gemv_8192"]["e2e"] = e2e_calls(torch, pb, mk, b, "GB/s", "gemv (drop-in C ABI, host arrays)")
    hy = np.zeros(m, np.float32)
    cpu_ref(args, out["gemv_8192"], lambda L: L.gemv(m, n, 1.0, 0.0, P(hA), P(hx), P(hy)), b, "full config")
    del A, hA

    # VOBLA chain: gemv_t 16384^2 (lda 16384, incx 2, incy 3) + dot + axpy on 2^28 vectors
    m = n = lda = 16384
    hA = synth.f32(m * lda)
    hxt, hyt = synth.f32(m * 2, 42, m * lda), synth.f32(n * 3, 42, m * lda + 2 * m)
    A, xt, yt = dev(hA), dev(hxt), dev(hyt)
    nv = 1 << 28
    hxv, hyv = synth.f32(nv, 7), synth.f32(nv, 8)
    xv, yv = dev(hxv), dev(hyv)
    r = torch.zeros(1, device="cuda")
    ms_t = statistics.mean(run_steps(torch, lambda: pb.device.gemv_t(m, n, lda, 2, 3, 1.0, 0.0, A, xt, yt), k, w, flush))
    ms_d = statistics.mean(run_steps(torch, lambda: pb.device.dot(nv, xv, yv, r), k, w, flush))
    ms_a = statistics.mean(run_steps(torch, lambda: pb.device.axpy_ptr(nv, r, xv, yv), k, w, flush))

    def chain():
        pb.device.gemv_t(m, n, lda, 2, 3, 1.0, 0.0, A, xt, yt)
        pb.device.dot(nv, xv, yv, r)
        pb.device.axpy_ptr(nv, r, xv, yv)
    ms_c = statistics.mean(run_steps(torch, chain, k, w, flush))
    bt, bd, ba = 4 * (m * n + m + n), 8 * nv, 12 * nv
    out["gemv_t_16384_strided"] = bw_line(ms_t, bt, hbm, "gemv_t_kernel", view="lda 16384, incx 2, incy 3")
    out["dot_2e28"] = bw_line(ms_d, bd, hbm, "dot_kernel")
    out["axpy_2e28"] = bw_line(ms_a, ba, hbm, "axpy_kernel", scalar="device (the dot result)")
    out["vobla_chain"] = bw_line(ms_c, bt + bd + ba, hbm, "gemv_t_kernel + dot_kernel + axpy_kernel",
                                 chain="gemv_t -> dot -> axpy(dot), scalar stays on the device")
    out["vobla_chain"]["roofline"]["traffic"] = None
    del A, xv, yv
    if not no_e2e:
        def mk_t(pinned):
            a_, x_, y_ = (host_buf(torch, q, pinned) for q in (hA, hxt, hyt.copy()))
            return lambda: pb.dropin.gemv_t(m, n, lda, 2, 3, 1.0, 0.0, a_, x_, y_)
        out["gemv_t_16384_strided"]["e2e"] = e2e_calls(torch, pb, mk_t, bt, "GB/s", "gemv_t (drop-in C ABI)")

        def mk_d(pinned):
            x_, y_ = host_buf(torch, hxv, pinned), host_buf(torch, hyv, pinned)

            def call():
                pb.dropin.dot(nv, x_, y_)
            return call
        out["dot_2e28"]["e2e"] = e2e_calls(torch, pb, mk_d, bd, "GB/s", "dot (drop-in C ABI, float returned)")

        def mk_a(pinned):
            x_, y_ = host_buf(torch, hxv, pinned), host_buf(torch, hyv.copy(), pinned)
            return lambda: pb.dropin.axpy(nv, 0.5, x_, y_)
        out["axpy_2e28"]["e2e"] = e2e_calls(torch, pb, mk_a, ba, "GB/s", "axpy (drop-in C ABI)")

        def mk_c(pinned):
            a_, xt_, yt_ = (host_buf(torch, q, pinned) for q in (hA, hxt, hyt.copy()))
            xv_, yv_ = host_buf(torch, hxv, pinned), host_buf(torch, hyv.copy(), pinned)
            lib = pb.load()

            def call():
                moved = [0, 0]

                def acc():
                    h2d, d2h = ctypes.c_longlong(), ctypes.c_longlong()
                    lib.pencil_last_transfer_bytes(ctypes.byref(h2d), ctypes.byref(d2h))
                    moved[0] += h2d.value
                    moved[1] += d2h.value
                pb.dropin.gemv_t(m, n, lda, 2, 3, 1.0, 0.0, a_, xt_, yt_)
                acc()
                d = pb.dropin.dot(nv, xv_, yv_)
                acc()
                pb.dropin.axpy(nv, d, xv_, yv_)
                acc()
                return moved
            return call
        out["vobla_chain"]["e2e"] = e2e_calls(torch, pb, mk_c, bt + bd + ba, "GB/s",
                                              "gemv_t, dot, axpy(dot) as three drop-in calls (the scalar returns to the host)")
    cpu_ref(args, out["gemv_t_16384_strided"],
            lambda L: L.gemv_t(m, n, lda, 2, 3, 1.0, 0.0, P(hA), P(hxt), P(hyt)), bt, "full config")
    cpu_ref(args, out["dot_2e28"], lambda L: L.dot(nv, P(hxv), P(hyv)), bd, "full config")
    cpu_ref(args, out["axpy_2e28"], lambda L: L.axpy(nv, 0.5, P(hxv), P(hyv)), ba, "full config")
    if "ms" in out["gemv_t_16384_strided"].get("cpu_baseline", {}):
        out["vobla_chain"]["cpu_baseline"] = dict(out["dot_2e28"]["cpu_baseline"], **{
            "ms": sum(out[q]["cpu_baseline"]["ms"] for q in ("gemv_t_16384_strided", "dot_2e28", "axpy_2e28")),
            "sample": "sum of the three calls above", "GB/s": None})
        out["vobla_chain"]["cpu_baseline"]["GB/s"] = (bt + bd + ba) / out["vobla_chain"]["cpu_baseline"]["ms"] / 1e6
    del hA, hxv, hyv

    # 5x5 stencils 16384^2
    h = w_ = 16384
    npx = h * w_
    himg = synth.u8_i32(npx)
    img_i = dev(himg)
    out_i = torch.empty(npx, dtype=torch.int32, device="cuda")
    b = 8 * npx
    for name, taps, scale, kern, desc in (
            ("conv5x5_u8_int32storage_16384", synth.BINOMIAL, 256, "stencil_ring_kernel<1, 1, 1, 0, 0>",
             "binomial (rank 1: separable kernel), scale 256"),
            ("conv5x5_u8_int32storage_16384_sharpen", synth.SHARPEN, 1, "stencil_ring_kernel<1, 1, 0, 1, 0>",
             "signed sharpen (diamond support: DIA kernel, 13 of 25 taps nonzero), scale 1")):
        ms = statistics.mean(run_steps(torch, lambda: pb.device.conv5x5_u8(h, w_, scale, img_i, taps, out_i),
                                       k, w, flush))
        out[name] = bw_line(ms, b, hbm, kern, taps=desc)
        if not no_e2e:
            def mk_u(pinned, taps=taps, scale=scale):
                i_, o_ = host_buf(torch, himg, pinned), host_buf(torch, np.empty(npx, np.int32), pinned)
                return lambda: pb.dropin.conv5x5_u8(h, w_, scale, i_, taps, o_)
            out[name]["e2e"] = e2e_calls(torch, pb, mk_u, b, "GB/s", "conv5x5_u8 (drop-in C ABI, int32 pixels)")
    img8 = img_i.to(torch.uint8)
    del img_i, out_i
    hout = np.empty(npx, np.int32)
    kb, ks = np.ascontiguousarray(synth.BINOMIAL, np.int32), np.ascontiguousarray(synth.SHARPEN, np.int32)
    cpu_ref(args, out["conv5x5_u8_int32storage_16384"], lambda L: L.conv5x5_u8(h, w_, 256, P(himg), P(kb), P(hout)),
            b, "full config")
    cpu_ref(args, out["conv5x5_u8_int32storage_16384_sharpen"],
            lambda L: L.conv5x5_u8(h, w_, 1, P(himg), P(ks), P(hout)), b, "full config")
    himg8 = himg.astype(np.uint8)
    del himg, hout
    out8 = torch.empty(npx, dtype=torch.uint8, device="cuda")
    b = 2 * npx
    for name, taps, scale, kern, desc in (
            ("conv5x5_u8_bytes_16384", synth.BINOMIAL, 256, "stencil_bytes_swar_kernel<16, 1, 1>",
             "binomial, scale 256 (16-bit SWAR sums, 16 px per lane)"),
            ("conv5x5_u8_bytes_16384_sharpen", synth.SHARPEN, 1, "stencil_bytes_swar2d_kernel<16, 1, 1, 1>",
             "signed sharpen (centre-positive, off-centre non-positive diamond taps: signed 2-D SWAR kernel), scale 1")):
        ms = statistics.mean(run_steps(torch, lambda: pb.device.conv5x5_u8_bytes(h, w_, scale, img8, taps, out8),
                                       k, w, flush))
        out[name] = bw_line(ms, b, hbm, kern, taps=desc, **{"Gpix/s": npx / ms / 1e6})
        if not no_e2e:
            # packed bytes have no emitted-C door (PENCIL has no uint8): the library's host-array entry
            def mk_b(pinned, taps=taps, scale=scale):
                i_, o_ = host_buf(torch, himg8, pinned), host_buf(torch, np.zeros(npx, np.uint8), pinned)
                return lambda: pb.dropin.conv5x5_u8_bytes(h, w_, scale, i_, taps, o_)
            out[name]["e2e"] = e2e_calls(torch, pb, mk_b, b, "GB/s",
                                         "pencil_conv5x5_u8_bytes (host arrays, library staging)")
    del img8, out8, himg8
    himgf = synth.f32(npx)
    imgf = dev(himgf)
    outf = torch.zeros(npx, device="cuda")
    b = 8 * npx
    kf = (synth.BINOMIAL.astype(np.float32) / 256.0).astype(np.float32)
    kg = synth.f32(25, 99)  # generic taps (uniform [-0.5, 0.5), not powers of two): as-written rounding
    for name, taps, kern, desc in (
            ("conv5x5_f32_16384", kf, "stencil_ring_kernel<0, 0, 0, 0, 1>",
             "binomial / 256 (16 power-of-two taps fused into one exact FMA each: PF 1)"),
            ("conv5x5_f32_16384_generic_taps", kg, "stencil_ring_kernel<0, 0, 0, 0, 0>",
             "25 generic fp32 taps (every product and sum rounds, as the emitted C)")):
        ms = statistics.mean(run_steps(torch, lambda: pb.device.conv5x5_f32(h, w_, imgf, taps, outf), k, w, flush))
        out[name] = bw_line(ms, b, hbm, kern, taps=desc)
        if not no_e2e:
            def mk_f(pinned, taps=taps):
                i_, o_ = host_buf(torch, himgf, pinned), host_buf(torch, np.zeros(npx, np.float32), pinned)
                return lambda: pb.dropin.conv5x5_f32(h, w_, i_, taps, o_)
            out[name]["e2e"] = e2e_calls(torch, pb, mk_f, b, "GB/s", "conv5x5_f32 (drop-in C ABI)")
    del imgf, outf
    houtf = np.zeros(npx, np.float32)
    cpu_ref(args, out["conv5x5_f32_16384"], lambda L: L.conv5x5_f32(h, w_, P(himgf), P(kf), P(houtf)), b,
            "full config")
    cpu_ref(args, out["conv5x5_f32_16384_generic_taps"], lambda L: L.conv5x5_f32(h, w_, P(himgf), P(kg), P(houtf)),
            b, "full config")
    del himgf, houtf

    # OP2 mesh loop: the reference's edge->cell increment kernel on a random mesh
    try:
        out["op2_mesh_inc_4M_cells_8M_edges"] = op2_line(args, torch, pb, k, w)
    except Exception as e:  # noqa: BLE001 — a suite line must not take the headline down
        out["op2_mesh_inc_4M_cells_8M_edges"] = {"unavailable": str(e)[:200]}

    # gemm 16384^3 via 3xTF32
    try:
        m = n = kk = 16384
        hA, hB = synth.f32(m * kk), synth.f32(kk * n, 43)
        A, B, C = dev(hA), dev(hB), torch.zeros(m * n, device="cuda")
        ms = statistics.mean(run_steps(torch, lambda: pb.device.gemm(m, n, kk, 1.0, 0.0, A, B, C), 5, 3, flush))
        flops = 2 * m * n * kk
        tf = flops / ms / 1e9
        burst, sustained, kind = tf32x3_peaks()
        out["gemm_16384_3xtf32"] = {
            "ms": ms, "TFLOP/s": tf,
            "roofline": roofline(tf, burst, "TFLOP/s", "gemm_3xtf32_kernel", flops, bound="tensor",
                                 peak_kind="%s: MEASURED_PEAKS bf16_tflops / 6 (3 tf32 MMAs per fp32 product, "
                                           "tf32 at half the bf16 rate), burst" % kind,
                                 frac_sustained=tf / sustained, peak_sustained=sustained,
                                 frac_spec=tf / 375.0, peak_spec="375 TFLOP/s (1.125 PF dense tf32 / 3)")}
        del A, B, C
        if not no_e2e:
            def mk_g(pinned):
                a_, b_, c_ = host_buf(torch, hA, pinned), host_buf(torch, hB, pinned), \
                    host_buf(torch, np.zeros(m * n, np.float32), pinned)
                return lambda: pb.dropin.gemm(m, n, kk, 1.0, 0.0, a_, b_, c_)
            out["gemm_16384_3xtf32"]["e2e"] = e2e_calls(torch, pb, mk_g, flops, "TFLOP/s", "gemm (drop-in C ABI)",
                                                        reps=1)
        del hA, hB
        # CPU beside it: the emitted triple loop at 1024^3 (16384^3 would take ~an hour), as a rate
        q = 1024
        ha, hb, hc = synth.f32(q * q), synth.f32(q * q, 43), np.zeros(q * q, np.float32)
        cpu_ref(args, out["gemm_16384_3xtf32"], lambda L: L.gemm(q, q, q, 1.0, 0.0, P(ha), P(hb), P(hc)),
                None, "1024^3 (rate extrapolated to the config)", reps=1, flops=2 * q ** 3)
    except pb.PencilError as e:
        out["gemm_16384_3xtf32"] = {"unavailable": str(e)}
    return out


def P(a):
    return a.ctypes.data


def host_cpu():
    """The host the CPU baselines run on: model name and logical CPUs."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


_CPU_LIB = {}


def cpu_lib():
    """The reference CPU path for timing: the C the reference's emit_openmp printed for the
    fixtures (outer-loop pragma), compiled on THIS host with gcc -O3 -march=native -fopenmp
    (oracle/Makefile `native`; the parity build keeps -march=x86-64-v3 -ffp-contract=off).
    Falls back to the portable build when the native one cannot be compiled here."""
    if "lib" not in _CPU_LIB:
        import oracle
        try:
            _CPU_LIB["lib"], _CPU_LIB["build"] = oracle.emitted("native"), "gcc -O3 -march=native -fopenmp"
        except Exception as e:  # noqa: BLE001
            _CPU_LIB["lib"] = oracle.emitted("outer")
            _CPU_LIB["build"] = "gcc -O3 -march=x86-64-v3 -fopenmp -ffp-contract=off (native build failed: %s)" % \
                str(e)[:80]
    return _CPU_LIB["lib"], _CPU_LIB["build"]


def cpu_ref(args, entry, call, nbytes, sample, reps=2, flops=None):
    """CPU beside a suite line: the reference's emit_openmp C (outer-loop pragma,
    oracle/_ref) on the same host inputs, all host threads, best of `reps` after one warm-up."""
    if args.no_cpu_baseline:
        return
    try:
        lib, build = cpu_lib()
        call(lib)
        best = float("inf")
        for _ in range(reps):
            t0 = time.perf_counter()
            call(lib)
            best = min(best, time.perf_counter() - t0)
        cb = {"ms": best * 1e3, "cores": os.cpu_count(), "kind": "reference", "host": host_cpu()["model"],
              "sample": sample + ": emit_openmp C (outer pragma), %s, best of %d" % (build, reps)}
        if nbytes:
            cb["GB/s"] = nbytes / best / 1e9
        if flops:
            cb["TFLOP/s"] = flops / best / 1e12
        entry["cpu_baseline"] = cb
    except Exception as e:  # noqa: BLE001 — a baseline must not take the suite down
        entry["cpu_baseline"] = {"unavailable": str(e)[:200]}


def op2_line(args, torch, pb, k, w):
    import json as _json
    import tempfile
    import ctypes
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import op2_probe
    from paper_1302_5586_b200.op2 import Op2Model
    nc, ne = 1 << 22, 1 << 23
    doc = op2_probe.mesh_doc(nc, ne)
    m = Op2Model(_json.dumps(doc))
    m.prepare()
    st = torch.cuda.ExternalStream(m.stream)
    with torch.cuda.stream(st):
        ms = statistics.mean(run_steps(torch, lambda: m.run_loop_async(0), k, w, lambda: pb.device.l2_flush()))
    m.sync()
    hbm, _, _ = peaks()
    # algorithmic bytes: the edge stream (2 map entries + one int64 edge value: 16 B per edge) and
    # the cell dat read and written once (16 B per cell); the increments themselves are L2 atomics
    # on the L2-resident 32 MB cell dat, which is what bounds the loop
    algo = ne * 16 + nc * 16
    res = {"ms": ms, "Gedges/s": ne / ms / 1e6, "GB/s": algo / ms / 1e6,
           "schedule": m.loop_info(0)[0], "data": "random edge->cell map (arity 2), int64 dats",
           "roofline": roofline(algo / ms / 1e6, hbm, "GB/s", "op2_loop_0", algo,
                                note="bound by L2 atomic throughput (2 x 8-byte atomic adds per edge into "
                                     "the L2-resident cell dat: %.0f G atomics/s), not by HBM" % (2 * ne / ms / 1e6)),
           "e2e": {"unavailable": "--no-e2e"}}
    if not args.no_e2e:
        # end to end through the model's host API: the loop's dats in from host arrays, the loop, the
        # incremented dat back (the mesh map stays resident from load, like a plan)
        host = {d["name"]: np.asarray(d["data"], np.int64) for d in doc["dats"]}
        cells_out = np.empty(nc, np.int64)

        def call():
            m.set_dat("dedges", host["dedges"])
            m.set_dat("dcells", host["dcells"])
            m.run()
            return m.dat("dcells", out=cells_out)
        call()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            call()
            ts.append(time.perf_counter() - t0)
        t = statistics.median(ts)
        res["e2e"] = {"value": algo / t / 1e9, "unit": "GB/s", "ms_per_call": t * 1e3,
                      "h2d_bytes_per_step": 8 * (ne + nc), "d2h_bytes_per_step": 8 * nc,
                      "api": "Op2Model.set_dat (dedges, dcells) + run + dat(dcells): pencil_op2_set_dat / "
                             "pencil_op2_run / pencil_op2_get_dat on pageable int64 host arrays; the map stays "
                             "resident from pencil_op2_load"}
    if not args.no_cpu_baseline:
        # CPU beside it: the model's lowering compiled as C (serial: the emitted reduction on an array
        # parameter is not valid OpenMP), one par_loop over the same mesh
        from oracle import op2_ref
        with tempfile.TemporaryDirectory() as td:
            lib, arrays, sizes = op2_ref.compile_lowered_c(doc, td)
            content = {d["name"]: np.asarray(d["data"], np.int32) for d in doc["dats"]}
            content.update({mm["name"]: np.asarray(mm["table"], np.int32) for mm in doc["maps"]})
            cargs = [ctypes.c_int(n) for n in sizes] + [ctypes.c_void_p(content[a].ctypes.data) for a in arrays]
            t0 = time.perf_counter()
            lib.op2_main(*cargs)
            cpu_s = time.perf_counter() - t0
        res["cpu_baseline"] = {"ms": cpu_s * 1e3, "Gedges/s": ne / cpu_s / 1e9, "cores": 1, "kind": "port",
                               "sample": "the model's lowered driver + kernel as C, gcc -O3, serial (the OpenMP "
                                         "form with an array-section reduction, oracle/op2_ref.openmp_lowered_c, "
                                         "is slower: a private copy of the cell dat per thread)"}
    m.close()
    return res


# ------------------------------------------------------------------ N>1 suite
def coll_dev(dist):
    """Where the small timing reductions live: the GPU under NCCL, host memory under gloo."""
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(torch, dist, v):
    t = torch.tensor([float(v)], dtype=torch.float64, device=coll_dev(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(torch, dist, v):
    t = torch.tensor([float(v)], dtype=torch.float64, device=coll_dev(dist))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def dist_line(torch, dist, ms_local, amount, unit, hbm_or_peak, kernel, per_rank_amount, extra=None, bound="hbm"):
    """One N>1 suite line: value = whole-job amount / max-over-ranks time; the roofline is per GPU
    (each rank's own bytes or flops over its own kernel time, the slowest rank reported)."""
    ms = max_over_ranks(torch, dist, ms_local)
    scale = 1e6 if unit in ("GB/s",) else 1e9
    ach_local = per_rank_amount / ms_local / scale
    ach = -max_over_ranks(torch, dist, -ach_local)  # the slowest rank
    line = {"ms": ms, unit: amount / ms / scale, "value": amount / ms / scale, "unit": unit,
            "roofline": {"bound": bound, "kernel": kernel, "achieved_per_gpu_min": ach, "peak": hbm_or_peak,
                         "unit": unit, "frac": ach / hbm_or_peak, "traffic": ncu_traffic(kernel)}}
    if extra:
        line.update(extra)
    return line


def suite_dist(args, torch, pb, rank, world, dist, hbm):
    """The sharded configs of SURVEY §8e at N GPUs (one process per GPU, max over ranks):
    gemm on the R x C tile grid (16384^3), the band-sharded 5x5 stencils with the halo read in
    place from the neighbours (16384^2, u8 int32 storage and f32), and row-sharded gemv 8192^2
    (x all-gather + local rows) captured in one CUDA graph.  Each line also carries the same
    work end to end (per-rank pinned-host inputs -> device -> outputs back, device-timed)."""
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200 import dist as pd
    out = {}
    k, w = max(3, args.suite_steps), 3
    flush = lambda: pb.device.l2_flush()  # noqa: E731
    fused_ok = args.dist_backend == "nccl"

    # gemm 16384^3 on the R x C grid: inputs replicated (no data-path collective)
    try:
        m = n = kk = 16384
        tg = pd.GemmTileGrid(m, n, kk, rank, world)
        hA, hB = synth.f32(m * kk), synth.f32(kk * n, 43)
        Ap = torch.from_numpy(hA.reshape(m, kk)[tg.m0:tg.m1].copy()).cuda().reshape(-1)
        Bp = torch.from_numpy(np.ascontiguousarray(hB.reshape(kk, n)[:, tg.n0:tg.n1])).cuda().reshape(-1)
        mt, nt = tg.m1 - tg.m0, tg.n1 - tg.n0
        Ct = torch.zeros(mt * nt, device="cuda")
        step = lambda: pb.device.gemm(mt, nt, kk, 1.0, 0.0, Ap, Bp, Ct)  # noqa: E731
        ms = statistics.mean(run_steps(torch, step, 5, 3, flush, dist))
        burst, sustained, _ = tf32x3_peaks()
        out["gemm_16384_3xtf32_grid"] = dist_line(
            torch, dist, ms, 2.0 * m * n * kk, "TFLOP/s", burst, "gemm_3xtf32_kernel", 2.0 * mt * nt * kk,
            {"grid": "%d x %d" % (tg.R, tg.C), "tile": "%d x %d" % (mt, nt),
             "collective": "none (A row panel + B column panel replicated per rank)"}, bound="tensor")
        if not args.no_e2e:
            pA, pB = torch.from_numpy(hA.reshape(m, kk)[tg.m0:tg.m1].copy()).pin_memory(), \
                torch.from_numpy(np.ascontiguousarray(hB.reshape(kk, n)[:, tg.n0:tg.n1])).pin_memory()
            pC = torch.empty(mt * nt).pin_memory()

            def call():
                Ap.copy_(pA.reshape(-1), non_blocking=True)
                Bp.copy_(pB.reshape(-1), non_blocking=True)
                pb.device.gemm(mt, nt, kk, 1.0, 0.0, Ap, Bp, Ct)
                pC.copy_(Ct, non_blocking=True)
            ms_e = statistics.mean(run_steps(torch, call, 2, 1, lambda: None, dist))
            out["gemm_16384_3xtf32_grid"]["e2e"] = {
                "value": 2.0 * m * n * kk / max_over_ranks(torch, dist, ms_e) / 1e9, "unit": "TFLOP/s",
                "ms_per_call": max_over_ranks(torch, dist, ms_e),
                "h2d_bytes_per_step": int(sum_over_ranks(torch, dist, 4 * (mt * kk + kk * nt))),
                "d2h_bytes_per_step": int(sum_over_ranks(torch, dist, 4 * mt * nt)),
                "api": "per rank: pinned A row panel + B column panel -> its GPU, pencil_gemm_dev, C tile -> host"}
        del Ap, Bp, Ct, hA, hB
    except Exception as e:  # noqa: BLE001
        out["gemm_16384_3xtf32_grid"] = {"unavailable": str(e)[:200]}

    # band-sharded 5x5 stencils 16384^2, halos read in place (FusedBandStencil) or exchanged (gloo)
    h = w_ = 16384
    for name, f32 in (("conv5x5_u8_bands_16384", False), ("conv5x5_f32_bands_16384", True)):
        try:
            img = synth.f32(h * w_) if f32 else synth.u8_i32(h * w_)
            dtype = torch.float32 if f32 else torch.int32
            kf = (synth.BINOMIAL / 256.0).astype(np.float32)
            fused, check = fused_ok, None
            if fused:
                fb = pd.FusedBandStencil(h, w_, rank, world, dtype, torch.device("cuda", torch.cuda.current_device()))
                fb.band().copy_(torch.from_numpy(img[fb.b0 * w_:fb.b1 * w_]))
                outb = torch.zeros(fb.nb * w_, dtype=dtype, device="cuda")
                step = (lambda: fb.step_f32(kf, outb)) if f32 else (lambda: fb.step_u8(256, synth.BINOMIAL, outb))
                rows, how = fb.nb, "fused: the band sweep reads the neighbours' edge rows over NVLink (cp.async from peer mappings)"
                # one checked step: the band must equal the same rows of the whole-image stencil
                step()
                full_in = torch.from_numpy(img).cuda()
                full_out = torch.zeros(h * w_, dtype=dtype, device="cuda")
                if f32:
                    pb.device.conv5x5_f32(h, w_, full_in, kf, full_out)
                else:
                    pb.device.conv5x5_u8(h, w_, 256, full_in, synth.BINOMIAL, full_out)
                same = torch.equal(outb.view(torch.int32), full_out[fb.b0 * w_:fb.b1 * w_].view(torch.int32))
                bad = torch.tensor([0 if same else 1], device="cuda")
                dist.all_reduce(bad)
                del full_in, full_out
                if int(bad.item()):
                    fused, check = False, "the fused band step differed from the whole-image stencil on %d rank(s)" % int(bad.item())
                    del fb, outb
                else:
                    check = "band == the same rows of the whole-image stencil, bit for bit (one step, every rank)"
            if not fused:
                band = pd.BandShardedImage(h, w_, rank, world)
                ext = torch.zeros(band.rows * w_, dtype=dtype, device="cuda")
                ext.view(band.rows, w_)[band.top:band.top + band.b1 - band.b0] = \
                    torch.from_numpy(img[band.b0 * w_:band.b1 * w_]).cuda().view(-1, w_)
                outb = torch.zeros(band.rows * w_, dtype=dtype, device="cuda")

                def step():
                    band.exchange_halos(ext.view(band.rows, w_))
                    if f32:
                        pb.device.conv5x5_f32(band.rows, w_, ext, kf, outb)
                    else:
                        pb.device.conv5x5_u8(band.rows, w_, 256, ext, synth.BINOMIAL, outb)
                rows, how = band.b1 - band.b0, "unfused: %s send/recv of 2 halo rows, then the stencil" % args.dist_backend
            ms = statistics.mean(run_steps(torch, step, k, w, flush, dist))
            extra = {"exchange": how, "taps": "binomial" + (" / 256" if f32 else ", scale 256")}
            if check:
                extra["check"] = check
            out[name] = dist_line(torch, dist, ms, 8.0 * h * w_, "GB/s", hbm,
                                  "stencil_band_kernel" if fused else "stencil_ring_kernel", 8.0 * rows * w_, extra)
            del img
        except Exception as e:  # noqa: BLE001
            out[name] = {"unavailable": str(e)[:200]}

    # VOBLA chain sharded (SURVEY §8e gemv_t / dot / axpy rows): gemv_t over this rank's column block
    # of the strided view (no collective), dot over its range of the 2^28 vectors + one all-reduce
    # of the partial (NCCL on the device scalar), axpy over the range with that scalar
    try:
        m = n = lda = 16384
        nv = 1 << 28
        g = pd.ColShardedGemvT(m, n, rank, world, lda=lda, incx=2, incy=3)
        A = torch.from_numpy(synth.f32(m * lda)).cuda()
        xt = torch.from_numpy(synth.f32(m * 2, 42, m * lda)).cuda()
        yt = torch.from_numpy(synth.f32(n * 3, 42, m * lda + 2 * m)).cuda()
        Av, yv_t = g.views(A, yt)
        lo, hi = pd.shard_range(nv, world, rank, align=4)
        xv = torch.from_numpy(synth.f32(hi - lo, 7, lo)).cuda()  # elements lo .. hi of the same streams
        yv = torch.from_numpy(synth.f32(hi - lo, 8, lo)).cuda()
        r = torch.zeros(1, device="cuda")
        nb = g.j1 - g.j0

        def chain():
            pb.device.gemv_t(m, nb, lda, 2, 3, 1.0, 0.0, Av, xt, yv_t)
            pb.device.dot(hi - lo, xv, yv, r)
            if world > 1 and dist.get_backend() == "nccl":
                dist.all_reduce(r)
            elif world > 1:
                rc = r.cpu()
                dist.all_reduce(rc)
                r.copy_(rc)
            pb.device.axpy_ptr(hi - lo, r, xv, yv)
        ms = statistics.mean(run_steps(torch, chain, k, w, flush, dist))
        bt, bd, ba = 4 * (m * n + m + n), 8 * nv, 12 * nv
        mine = 4 * (m * nb + m + nb) + 20 * (hi - lo)
        out["vobla_chain_ranks"] = dist_line(
            torch, dist, ms, bt + bd + ba, "GB/s", hbm, "gemv_t_kernel + dot_kernel + axpy_kernel", mine,
            {"split": "gemv_t column blocks of the strided view (%d columns here), dot / axpy ranges (%d elements), "
                      "one all-reduce of the dot partial (%s)" % (nb, hi - lo, dist.get_backend())})
        del A, xv, yv
    except Exception as e:  # noqa: BLE001
        out["vobla_chain_ranks"] = {"unavailable": str(e)[:200]}

    # gemv 8192^2 row-sharded: x all-gathered from its shards + the local rows, one CUDA graph
    try:
        m = n = 8192
        g = pd.RowShardedGemv(m, n, rank, world)
        hA, hx = synth.f32(m * n), synth.f32(n, 42, m * n)
        A_rows = torch.from_numpy(hA.reshape(m, n)[g.r0:g.r1].copy()).cuda().reshape(-1)
        lo, hi = pd.shard_range(n, world, rank, align=1)
        x_shard = torch.from_numpy(hx[lo:hi].copy()).cuda()
        y_rows = torch.zeros(g.r1 - g.r0, device="cuda")
        g.attach(torch.cuda.current_device(), y_rows)
        width = max(b - a for a, b in (pd.shard_range(n, world, r, align=1) for r in range(world)))
        xpad = torch.zeros(width, device="cuda")
        xg = torch.empty(width * world, device="cuda")
        bounds = [pd.shard_range(n, world, r, align=1) for r in range(world)]
        idx = torch.cat([torch.arange(b - a) + r * width for r, (a, b) in enumerate(bounds)]).cuda()
        xfull = torch.empty(n, device="cuda")

        def gemv_step():
            xpad[: hi - lo].copy_(x_shard)
            if world > 1 and dist.get_backend() == "nccl":
                dist.all_gather_into_tensor(xg, xpad)
            elif world > 1:
                pd._all_gather_list(list(xg.view(world, width).unbind(0)), xpad)
            else:
                xg.copy_(xpad)
            torch.index_select(xg, 0, idx, out=xfull)
            pb.device.gemv(g.r1 - g.r0, n, 1.0, 0.0, A_rows, xfull, y_rows)
        graph = None
        if dist.get_backend() == "nccl":
            try:
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    for _ in range(3):
                        gemv_step()
                torch.cuda.current_stream().wait_stream(s)
                torch.cuda.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    gemv_step()
            except Exception as e:  # noqa: BLE001 — capture refused: plain launches
                graph, why = None, str(e)[:100]
        step = graph.replay if graph is not None else gemv_step
        ms = statistics.mean(run_steps(torch, step, k, w, flush, dist))
        out["gemv_8192_rows"] = dist_line(
            torch, dist, ms, 4.0 * (m * n + n + m), "GB/s", hbm, "gemv_kernel", 4.0 * ((g.r1 - g.r0) * n + n + g.r1 - g.r0),
            {"step": "x all-gather (%s) + local rows" % dist.get_backend(),
             "launch": "one CUDA graph per step" if graph is not None else "plain launches"})
        del A_rows, hA
    except Exception as e:  # noqa: BLE001
        out["gemv_8192_rows"] = {"unavailable": str(e)[:200]}
    return out


# ------------------------------------------------------------------ reference arm (CPU)
def cpu_spmv(steps, warmup, rowptr, col, val, x):
    lib, _ = cpu_lib()
    nrows = rowptr.size - 1
    y = np.zeros(nrows, np.float32)
    P = lambda a: a.ctypes.data  # noqa: E731
    call = lambda: lib.spmv_vec(nrows, x.size, col.size, P(rowptr), P(col), P(val), P(x), P(y))  # noqa: E731
    for _ in range(warmup):
        call()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    return ts


def reference_arm(args):
    from paper_1302_5586_b200 import synth
    nrows = 1 << 24
    rowptr, col, val, x, xm = synth.csr_powerlaw(nrows)
    cores = os.cpu_count()
    # all host threads, whatever the launcher set (torchrun exports OMP_NUM_THREADS=1 per rank)
    cpu_lib()
    ctypes.CDLL("libgomp.so.1").omp_set_num_threads(cores)
    ts = cpu_spmv(args.steps, min(args.warmup, 3), rowptr, col, val, x)
    _, build = cpu_lib()
    t = statistics.mean(ts)
    algo = spmv_bytes(nrows, nrows, col.size)
    v = algo / t / 1e9
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(spmv_config(nrows, int(col.size), xm),
                           parallelism=f"openmp x{cores}"),
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores,
                             "kind": "reference", "host": host_cpu(),
                             "sample": "full matrix, one spmv_vec call per step: C emitted by the reference's "
                                       "emit_openmp (outer-loop pragma), %s" % build},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--suite-steps", type=int, default=10)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--force-dist", action="store_true",
                    help="take the N>1 code path (process group, shards, collectives) even at one rank")
    ap.add_argument("--dist-mode", default="fused", choices=["fused", "nccl"],
                    help="N>1 SpMV step: fused SpMV->all-gather kernel, or SpMV + NCCL all-gather")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl != "reference":
        # torchrun exports OMP_NUM_THREADS=1: the synthetic-input generator (OpenMP, outside every
        # timed region) gets its share of the host instead
        try:
            ctypes.CDLL("libgomp.so.1").omp_set_num_threads(max(1, (os.cpu_count() or 1) // world))
        except OSError:
            pass

    if args.impl == "reference":
        if rank == 0:
            os.environ.setdefault("OMP_PROC_BIND", "close")
            print(json.dumps(reference_arm(args)))
        return

    import torch
    import paper_1302_5586_b200 as pb
    # one process per GPU; with fewer GPUs than ranks (plumbing test: --dist-backend gloo) ranks
    # share devices — their kernels never wait on one another, only host-side collectives do
    dev = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist = None
    args.dist_path = world > 1 or args.force_dist
    if args.dist_path:
        import torch.distributed as tdist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        if args.dist_backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            tdist.init_process_group(args.dist_backend)
        dist = tdist
    hbm, tf, peak_kind = peaks()

    with Clocks(dev) as clk:
        res = bench_spmv(args, torch, pb, rank, world, dist)
        dsuite = suite_dist(args, torch, pb, rank, world, dist, hbm) if args.dist_path and not args.no_suite else None
    ms = res["ms"]
    if dist:
        t = torch.tensor([ms], device=coll_dev(dist))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = res["bytes"] / ms / 1e6  # GB/s, whole job (global matrix bytes / max-rank time)
    if rank == 0:
        kernel_gbs = res["bytes"] / res["ms"] / 1e6 if not args.dist_path else None
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(res["config"], parallelism=f"row-sharded x{world}" if args.dist_path else "single GPU"),
                "gpu_launches": res["launches"]}
        if not args.dist_path:
            line["roofline"] = {"bound": "hbm", "kernel": "csr_seg_kernel<0, 0, 0>", "achieved": kernel_gbs,
                                "peak": hbm, "unit": "GB/s", "frac": kernel_gbs / hbm,
                                "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else peak_kind,
                                "frac_spec": kernel_gbs / SPEC_HBM_GBS,
                                "algorithmic_bytes_per_launch": res["bytes"],
                                "traffic": ncu_traffic("csr_seg_kernel<0, 0, 0>"),
                                "measured_ceiling": {
                                    "kernel": "micro_gather_val: the same col/val stream + x gathers, no rows "
                                              "(random 4-byte gathers are L1->XBAR request-rate bound, DESIGN.md §3)",
                                    "ms": res["ceiling_ms"], "frac": res["ceiling_ms"] / res["ms"]}}
        line["clocks"] = clk.summary()
        if "e2e" in res:
            line["e2e"] = res["e2e"]
        if not args.dist_path and not args.no_cpu_baseline:
            try:
                from paper_1302_5586_b200 import synth
                rowptr, col, val, x, _ = synth.csr_powerlaw(1 << 24)
                ts = cpu_spmv(3, 1, rowptr, col, val, x)
                t = statistics.mean(ts)
                line["cpu_baseline"] = {"value": spmv_bytes(1 << 24, 1 << 24, col.size) / t / 1e9, "unit": "GB/s",
                                        "cores": os.cpu_count(), "kind": "reference", "host": host_cpu(),
                                        "sample": "full matrix x3 calls of the emit_openmp C (outer pragma), "
                                                  "%s, all host threads" % cpu_lib()[1]}
                # and on one thread (OMP_NUM_THREADS = 1 and = all cores)
                gomp = ctypes.CDLL("libgomp.so.1")
                gomp.omp_set_num_threads(1)
                t1 = min(cpu_spmv(1, 0, rowptr, col, val, x))
                gomp.omp_set_num_threads(os.cpu_count())
                line["cpu_baseline"]["value_1thread"] = spmv_bytes(1 << 24, 1 << 24, col.size) / t1 / 1e9
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "unavailable": str(e)[:200]}
        if dsuite is not None:
            line["suite"] = dsuite
        if not args.dist_path and not args.no_suite:
            line["suite"] = suite(args, torch, pb, hbm)
            if res.get("src_ms"):
                line["suite"] = dict({"spmv_inline_2e24": bw_line(
                    res["src_ms"], res["bytes"], hbm, "csr_seg_kernel<0, 1, 0>",
                    order="source order (spmv_inline / ACCESS spmv): each row folded in order, bit-identical to "
                          "the emitted C; row chains carried lane to lane",
                    measured_ceiling_ms=res["ceiling_ms"])}, **line["suite"])
                if res.get("src_e2e"):
                    line["suite"]["spmv_inline_2e24"]["e2e"] = res["src_e2e"]
                if res.get("src_cpu", {}).get("cpu_baseline"):
                    line["suite"]["spmv_inline_2e24"]["cpu_baseline"] = res["src_cpu"]["cpu_baseline"]
            # the measured peak is a copy test (read + write); read-mostly streams go past it, so
            # every bandwidth line also carries its fraction of the B200 spec (8 TB/s HBM3e)
            for v in line["suite"].values():
                if "frac_hbm" in v:
                    v["frac_spec"] = v["GB/s"] / SPEC_HBM_GBS
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

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
    try:
        with open(NCU_SUMMARY) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


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
    if world == 1:
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
    else:
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
            fz.load(x_local)

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
           "ceiling_ms": ceil_ms if world == 1 else None,
           "config": {"workload": "CSR SpMV fp32 (spmv_vec), power-law rows 2^24 x 2^24, 16 nnz/row",
                      "nrows": nrows, "ncols": nrows, "nnz": nnz, "alpha": 1.5, "xm": round(xm, 4),
                      "maxlen": 4096, "seed": 42, "schedule": "csr_flow_kernel, reassociated (persistent warps, 1024-nnz window tiles, continuous 128-bit col/val streams)",
                      "l2": "L2 flushed between steps outside the per-step events (256 MiB fill, then its lines discarded: the step starts on a clean, empty L2); inputs 2.35 GB > L2"}}
    if world > 1:
        res["config"]["exchange"] = exchange
        if e2e:
            res["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_e2e:
        res["e2e"] = e2e_spmv(args, torch, pb, rowptr, col, val, x)
    return res


def e2e_spmv(args, torch, pb, rowptr, col, val, x):
    """drop-in C ABI, pinned host buffers, H2D + kernel + D2H per call (synchronous)."""
    nrows, nnz = rowptr.size - 1, col.size
    pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
    hrp, hcol, hval, hx = pin(rowptr), pin(col), pin(val), pin(x)
    hy = torch.empty(nrows, dtype=torch.float32).pin_memory()
    call = lambda: pb.dropin.spmv_vec(nrows, nrows, nnz, hrp, hcol, hval, hx, hy)  # noqa: E731
    call()
    ts = []
    for _ in range(max(2, min(args.steps, 5))):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    algo = spmv_bytes(nrows, nrows, nnz)
    import ctypes
    h2d, d2h = ctypes.c_longlong(), ctypes.c_longlong()  # what the call moved over the link
    pb.load().pencil_last_transfer_bytes(ctypes.byref(h2d), ctypes.byref(d2h))
    return {"value": algo / t / 1e9, "unit": "GB/s", "ms_per_call": t * 1e3, "h2d_bytes_per_step": h2d.value,
            "d2h_bytes_per_step": d2h.value, "api": "spmv_vec (drop-in C ABI, pinned host arrays)"}


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
    t = torch.tensor([ms, float(h2d), 4.0 * sh.nrows], dtype=torch.float64, device="cuda")
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


def suite(args, torch, pb, hbm):
    """Secondary configs of BASELINE.json, one line each (device-resident inputs)."""
    from paper_1302_5586_b200 import synth
    out = {}
    k, w = max(3, args.suite_steps), 3
    flush = lambda: pb.device.l2_flush()  # noqa: E731
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731

    # gemv 8192^2 (configs[0])
    m = n = 8192
    hA, hx = synth.f32(m * n), synth.f32(n, 42, m * n)
    A, x, y = dev(hA), dev(hx), torch.zeros(m, device="cuda")
    ms = statistics.mean(run_steps(torch, lambda: pb.device.gemv(m, n, 1.0, 0.0, A, x, y), k, w, flush))
    b = 4 * (m * n + n + m)
    out["gemv_8192"] = {"ms": ms, "GB/s": b / ms / 1e6, "frac_hbm": b / ms / 1e6 / hbm, "bytes": b}
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
    out["gemv_t_16384_strided"] = {"ms": ms_t, "GB/s": bt / ms_t / 1e6, "frac_hbm": bt / ms_t / 1e6 / hbm}
    out["dot_2e28"] = {"ms": ms_d, "GB/s": bd / ms_d / 1e6, "frac_hbm": bd / ms_d / 1e6 / hbm}
    out["axpy_2e28"] = {"ms": ms_a, "GB/s": ba / ms_a / 1e6, "frac_hbm": ba / ms_a / 1e6 / hbm}
    out["vobla_chain"] = {"ms": ms_c, "GB/s": (bt + bd + ba) / ms_c / 1e6,
                          "frac_hbm": (bt + bd + ba) / ms_c / 1e6 / hbm, "bytes": bt + bd + ba}
    del A, xv, yv
    cpu_ref(args, out["gemv_t_16384_strided"],
            lambda L: L.gemv_t(m, n, lda, 2, 3, 1.0, 0.0, P(hA), P(hxt), P(hyt)), bt, "full config")
    cpu_ref(args, out["dot_2e28"], lambda L: L.dot(nv, P(hxv), P(hyv)), bd, "full config")
    cpu_ref(args, out["axpy_2e28"], lambda L: L.axpy(nv, 0.5, P(hxv), P(hyv)), ba, "full config")
    if "cpu_baseline" in out["gemv_t_16384_strided"]:
        out["vobla_chain"]["cpu_baseline"] = {
            "ms": sum(out[q]["cpu_baseline"]["ms"] for q in ("gemv_t_16384_strided", "dot_2e28", "axpy_2e28")),
            "cores": os.cpu_count(), "kind": "reference", "sample": "sum of the three calls above"}
    del hA, hxv, hyv

    # 5x5 stencils 16384^2
    h = w_ = 16384
    himg = synth.u8_i32(h * w_)
    img_i = dev(himg)
    out_i = torch.empty(h * w_, dtype=torch.int32, device="cuda")
    ms = statistics.mean(run_steps(torch, lambda: pb.device.conv5x5_u8(h, w_, 256, img_i, synth.BINOMIAL, out_i),
                                   k, w, flush))
    b = 8 * h * w_
    out["conv5x5_u8_int32storage_16384"] = {"ms": ms, "GB/s": b / ms / 1e6, "frac_hbm": b / ms / 1e6 / hbm,
                                            "taps": "binomial (rank 1: separable kernel), scale 256"}
    ms = statistics.mean(run_steps(torch, lambda: pb.device.conv5x5_u8(h, w_, 1, img_i, synth.SHARPEN, out_i),
                                   k, w, flush))
    out["conv5x5_u8_int32storage_16384_sharpen"] = {"ms": ms, "GB/s": b / ms / 1e6, "frac_hbm": b / ms / 1e6 / hbm,
                                                    "taps": "signed sharpen (diamond support: DIA kernel, 13 of 25 taps nonzero), scale 1"}
    img8 = img_i.to(torch.uint8)
    del img_i, out_i
    hout = np.empty(h * w_, np.int32)
    kb = np.ascontiguousarray(synth.BINOMIAL, np.int32)
    cpu_ref(args, out["conv5x5_u8_int32storage_16384"], lambda L: L.conv5x5_u8(h, w_, 256, P(himg), P(kb), P(hout)),
            b, "full config")
    del himg, hout
    out8 = torch.empty(h * w_, dtype=torch.uint8, device="cuda")
    ms = statistics.mean(run_steps(torch, lambda: pb.device.conv5x5_u8_bytes(h, w_, 256, img8, synth.BINOMIAL, out8),
                                   k, w, flush))
    b = 2 * h * w_
    out["conv5x5_u8_bytes_16384"] = {"ms": ms, "GB/s": b / ms / 1e6, "frac_hbm": b / ms / 1e6 / hbm,
                                     "Gpix/s": h * w_ / ms / 1e6, "taps": "binomial, scale 256",
                                     "kernel": "stencil_bytes_swar_kernel<16> (16-bit SWAR sums, 16 px per lane)"}
    ms = statistics.mean(run_steps(torch, lambda: pb.device.conv5x5_u8_bytes(h, w_, 1, img8, synth.SHARPEN, out8),
                                   k, w, flush))
    out["conv5x5_u8_bytes_16384_sharpen"] = {"ms": ms, "GB/s": b / ms / 1e6, "frac_hbm": b / ms / 1e6 / hbm,
                                             "Gpix/s": h * w_ / ms / 1e6, "taps": "signed sharpen (diamond support: DIA kernel), scale 1"}
    del img8, out8
    himgf = synth.f32(h * w_)
    imgf = dev(himgf)
    outf = torch.zeros(h * w_, device="cuda")
    kf = (synth.BINOMIAL.astype(np.float32) / 256.0).astype(np.float32)
    ms = statistics.mean(run_steps(torch, lambda: pb.device.conv5x5_f32(h, w_, imgf, kf, outf), k, w, flush))
    b = 8 * h * w_
    out["conv5x5_f32_16384"] = {"ms": ms, "GB/s": b / ms / 1e6, "frac_hbm": b / ms / 1e6 / hbm,
                                "taps": "binomial / 256",
                                "kernel": "stencil_ring_kernel<F32, PF 1> (16 power-of-two taps fused, exact)"}
    del imgf, outf
    houtf = np.zeros(h * w_, np.float32)
    cpu_ref(args, out["conv5x5_f32_16384"], lambda L: L.conv5x5_f32(h, w_, P(himgf), P(kf), P(houtf)), b,
            "full config")
    del himgf, houtf

    # OP2 mesh loop: the reference's edge->cell increment kernel on a random mesh
    try:
        out["op2_mesh_inc_4M_cells_8M_edges"] = op2_line(args, torch, pb, k, w)
    except Exception as e:  # noqa: BLE001 — a suite line must not take the headline down
        out["op2_mesh_inc_4M_cells_8M_edges"] = {"unavailable": str(e)[:200]}

    # gemm 16384^3 via 3xTF32
    try:
        m = n = kk = 16384
        A, B, C = dev(synth.f32(m * kk)), dev(synth.f32(kk * n, 43)), torch.zeros(m * n, device="cuda")
        ms = statistics.mean(run_steps(torch, lambda: pb.device.gemm(m, n, kk, 1.0, 0.0, A, B, C), 2, 1, flush))
        out["gemm_16384_3xtf32"] = {"ms": ms, "TFLOP/s": 2 * m * n * kk / ms / 1e9}
        del A, B, C
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


def cpu_ref(args, entry, call, nbytes, sample, reps=2, flops=None):
    """CPU beside a suite line: the reference's emit_openmp C (outer-loop pragma,
    oracle/_ref) on the same host inputs, all host threads, best of `reps` after one warm-up."""
    if args.no_cpu_baseline:
        return
    try:
        import oracle
        lib = oracle.emitted("outer")
        call(lib)
        best = float("inf")
        for _ in range(reps):
            t0 = time.perf_counter()
            call(lib)
            best = min(best, time.perf_counter() - t0)
        cb = {"ms": best * 1e3, "cores": os.cpu_count(), "kind": "reference",
              "sample": sample + ": emit_openmp C (outer pragma), gcc -O3 -fopenmp, best of %d" % reps}
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
    res = {"ms": ms, "Gedges/s": ne / ms / 1e6, "GB/s": (ne * 32 + nc * 16) / ms / 1e6,
           "schedule": m.loop_info(0)[0], "data": "random edge->cell map (arity 2), int64 dats"}
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
                               "sample": "the model's lowered driver + kernel as C, gcc -O3, serial"}
    m.close()
    return res


# ------------------------------------------------------------------ reference arm (CPU)
def cpu_spmv(steps, warmup, rowptr, col, val, x):
    import oracle
    lib = oracle.emitted("outer")
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
    rowptr, col, val, x, _ = synth.csr_powerlaw(nrows)
    cores = os.cpu_count()
    ts = cpu_spmv(args.steps, min(args.warmup, 3), rowptr, col, val, x)
    t = statistics.mean(ts)
    algo = spmv_bytes(nrows, nrows, col.size)
    v = algo / t / 1e9
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "CSR SpMV fp32 (spmv_vec), power-law rows 2^24 x 2^24, 16 nnz/row",
                       "nrows": nrows, "nnz": int(col.size), "parallelism": f"openmp x{os.environ.get('OMP_NUM_THREADS', cores)}"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": int(os.environ.get("OMP_NUM_THREADS", cores)),
                             "kind": "reference",
                             "sample": "full matrix, one spmv_vec call per step: C emitted by the reference's "
                                       "emit_openmp (outer-loop pragma), gcc -O3 -fopenmp"},
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
    ap.add_argument("--dist-mode", default="fused", choices=["fused", "nccl"],
                    help="N>1 SpMV step: fused SpMV->all-gather kernel, or SpMV + NCCL all-gather")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

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
    if world > 1:
        import torch.distributed as tdist
        if args.dist_backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            tdist.init_process_group(args.dist_backend)
        dist = tdist
    hbm, tf, peak_kind = peaks()

    with Clocks(dev) as clk:
        res = bench_spmv(args, torch, pb, rank, world, dist)
    ms = res["ms"]
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = res["bytes"] / ms / 1e6  # GB/s, whole job (global matrix bytes / max-rank time)
    if rank == 0:
        kernel_gbs = res["bytes"] / res["ms"] / 1e6 if world == 1 else None
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(res["config"], parallelism=f"row-sharded x{world}" if world > 1 else "single GPU"),
                "gpu_launches": res["launches"]}
        if world == 1:
            line["roofline"] = {"bound": "hbm", "kernel": "csr_flow_kernel", "achieved": kernel_gbs,
                                "peak": hbm, "unit": "GB/s", "frac": kernel_gbs / hbm,
                                "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else peak_kind,
                                "frac_spec": kernel_gbs / SPEC_HBM_GBS,
                                "algorithmic_bytes_per_launch": res["bytes"],
                                "traffic": ncu_traffic("csr_flow_kernel"),
                                "measured_ceiling": {
                                    "kernel": "micro_gather_val: the same col/val stream + x gathers, no rows "
                                              "(random 4-byte gathers are L1->XBAR request-rate bound, DESIGN.md §3)",
                                    "ms": res["ceiling_ms"], "frac": res["ceiling_ms"] / res["ms"]}}
        line["clocks"] = clk.summary()
        if "e2e" in res:
            line["e2e"] = res["e2e"]
        if world == 1 and not args.no_cpu_baseline:
            try:
                from paper_1302_5586_b200 import synth
                rowptr, col, val, x, _ = synth.csr_powerlaw(1 << 24)
                ts = cpu_spmv(3, 1, rowptr, col, val, x)
                t = statistics.mean(ts)
                line["cpu_baseline"] = {"value": spmv_bytes(1 << 24, 1 << 24, col.size) / t / 1e9, "unit": "GB/s",
                                        "cores": os.cpu_count(), "kind": "reference",
                                        "sample": "full matrix x3 calls of the emit_openmp C (outer pragma), "
                                                  "gcc -O3 -fopenmp, all host threads"}
                # and on one thread (OMP_NUM_THREADS = 1 and = all cores)
                gomp = ctypes.CDLL("libgomp.so.1")
                gomp.omp_set_num_threads(1)
                t1 = min(cpu_spmv(1, 0, rowptr, col, val, x))
                gomp.omp_set_num_threads(os.cpu_count())
                line["cpu_baseline"]["value_1thread"] = spmv_bytes(1 << 24, 1 << 24, col.size) / t1 / 1e9
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "unavailable": str(e)[:200]}
        if world == 1 and not args.no_suite:
            line["suite"] = suite(args, torch, pb, hbm)
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

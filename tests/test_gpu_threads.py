"""Re-entrancy (SURVEY §8b threading): the drop-in entry points called from several host
threads at once give the single-threaded results, and the error channel is per thread — a
thread whose call faults (E-INTERP) does not see, or leak its status into, the others' calls."""
import threading

import numpy as np
import pytest

import oracle
from paper_1302_5586_b200 import synth

pytestmark = pytest.mark.gpu


def test_concurrent_dropin_calls_match_sequential(cuda):
    import paper_1302_5586_b200 as pb
    rowptr, col, val, x, _ = synth.csr_powerlaw(30000, maxlen=500, seed=21)
    nrows, nnz = rowptr.size - 1, col.size
    m, n = 700, 513
    A, xv = synth.f32(m * n, 4), synth.f32(n, 5)
    h, w = 90, 132
    img = synth.u8_i32(h * w, seed=8)
    ref_spmv = np.zeros(nrows, np.float32)
    pb.dropin.spmv_inline(nrows, nrows, nnz, rowptr, col, val, x, ref_spmv)
    ref_conv = oracle.conv5x5_u8(h, w, 256, img, synth.BINOMIAL)
    ref_gemv = np.zeros(m, np.float32)
    pb.dropin.gemv(m, n, 1.0, 0.0, A, xv, ref_gemv)
    errors = []

    def worker(tid):
        try:
            for it in range(6):
                kind = (tid + it) % 3
                if kind == 0:
                    y = np.zeros(nrows, np.float32)
                    pb.dropin.spmv_inline(nrows, nrows, nnz, rowptr, col, val, x, y)
                    assert np.array_equal(y.view(np.uint32), ref_spmv.view(np.uint32))
                elif kind == 1:
                    out = np.zeros(h * w, np.int32)
                    pb.dropin.conv5x5_u8(h, w, 256, img, synth.BINOMIAL, out)
                    assert np.array_equal(out.astype(np.int64), ref_conv)
                else:
                    y = np.zeros(m, np.float32)
                    pb.dropin.gemv(m, n, 1.0, 0.0, A, xv, y)
                    assert np.array_equal(y.view(np.uint32), ref_gemv.view(np.uint32))
                assert pb.load().pencil_cuda_last_status() == 0
        except BaseException as e:  # noqa: BLE001
            errors.append((tid, repr(e)))

    ts = [threading.Thread(target=worker, args=(t,)) for t in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_fault_status_is_per_thread(cuda):
    import paper_1302_5586_b200 as pb
    rowptr = np.array([0, 2, 3], np.int32)
    bad_col = np.array([0, 99, 1], np.int32)  # column 99 >= ncols: E-INTERP
    val = np.ones(3, np.float32)
    x = np.ones(4, np.float32)
    results = {}
    go = threading.Barrier(2)

    def faulty():
        go.wait()
        try:
            pb.dropin.spmv_inline(2, 4, 3, rowptr, bad_col, val, x, np.zeros(2, np.float32))
            results["faulty"] = "no error"
        except pb.PencilError as e:
            results["faulty"] = e.code
        results["faulty_status"] = pb.load().pencil_cuda_last_status()

    def clean():
        go.wait()
        y = np.zeros(2, np.float32)
        for _ in range(20):
            pb.dropin.spmv_inline(2, 4, 3, rowptr, np.array([0, 1, 1], np.int32), val, x, y)
        results["clean_status"] = pb.load().pencil_cuda_last_status()
        results["clean_y"] = y.tolist()

    ts = [threading.Thread(target=faulty), threading.Thread(target=clean)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert results["faulty"] == "E-INTERP"
    assert results["faulty_status"] != 0
    assert results["clean_status"] == 0 and results["clean_y"] == [2.0, 1.0]


def test_conv_u8_repair_flag_is_per_stream(cuda):
    """Two streams interleave conv5x5_u8 launches, one on an image holding non-byte values
    (its launches need the exact repair pass), one on a byte image: the repair flag of one
    stream's launch must never be consumed or re-armed by the other's."""
    import torch
    import paper_1302_5586_b200 as pb
    h, w = 256, 512
    good = synth.u8_i32(h * w, seed=31)
    bad = good.copy()
    bad[::997] = 5000
    ref_good = oracle.conv5x5_u8(h, w, 256, good, synth.BINOMIAL)
    ref_bad = oracle.conv5x5_u8(h, w, 256, bad, synth.BINOMIAL)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    dg, db = torch.from_numpy(good).cuda(), torch.from_numpy(bad).cuda()
    outs_a = [torch.empty(h * w, dtype=torch.int32, device="cuda") for _ in range(8)]
    outs_b = [torch.empty(h * w, dtype=torch.int32, device="cuda") for _ in range(8)]
    torch.cuda.synchronize()
    for i in range(8):
        pb.device.conv5x5_u8(h, w, 256, db, synth.BINOMIAL, outs_a[i], stream=sa.cuda_stream)
        pb.device.conv5x5_u8(h, w, 256, dg, synth.BINOMIAL, outs_b[i], stream=sb.cuda_stream)
    torch.cuda.synchronize()
    for i in range(8):
        assert np.array_equal(outs_a[i].cpu().numpy().astype(np.int64), ref_bad), i
        assert np.array_equal(outs_b[i].cpu().numpy().astype(np.int64), ref_good), i


def test_two_streams_share_no_device_state(cuda):
    """Device API calls on two streams at once (re-entrant per (device, stream)):
    gemv_t launches with different shapes (their last-CTA counters), one CSR plan used on both
    streams (its tile tickets) — many launches queued on each before either is synchronized — give
    the single-stream results bit for bit; a fault raised on one stream is reported by that
    stream's sync_status only."""
    import torch
    import paper_1302_5586_b200 as pb
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    # gemv_t: two shapes, one launch interleaved on each stream
    shapes = [(1500, 3000, 3008, 2, 3), (2900, 1100, 1104, 1, 2)]
    data = []
    for q, (m, n, lda, incx, incy) in enumerate(shapes):
        A = torch.from_numpy(synth.f32(m * lda, 10 + q)).cuda()
        x = torch.from_numpy(synth.f32(m * incx, 20 + q)).cuda()
        y0 = torch.from_numpy(synth.f32(n * incy, 30 + q)).cuda()
        ref = y0.clone()
        pb.device.gemv_t(m, n, lda, incx, incy, 1.25, 0.5, A, x, ref)
        data.append((A, x, y0, ref))
    torch.cuda.synchronize()
    outs = [[], []]
    for it in range(8):
        for q, s in enumerate((s1, s2)):
            m, n, lda, incx, incy = shapes[q]
            A, x, y0, _ = data[q]
            with torch.cuda.stream(s):
                y = y0.clone()
                pb.device.gemv_t(m, n, lda, incx, incy, 1.25, 0.5, A, x, y)
                outs[q].append(y)
    torch.cuda.synchronize()
    for q in range(2):
        for y in outs[q]:
            assert torch.equal(y.view(torch.int32), data[q][3].view(torch.int32))
    # one CSR plan, both streams
    rowptr, col, val, x, _ = synth.csr_powerlaw(120000, maxlen=2000, seed=33)
    nrows, nnz = rowptr.size - 1, col.size
    rp, cd, vd, xd = (torch.from_numpy(a).cuda() for a in (rowptr, col, val, x))
    plan = pb.device.CsrPlan(nrows, nrows, nnz, rp, mode=0)
    ref = torch.empty(nrows, device="cuda")
    plan.spmv(rp, cd, vd, xd, ref)
    torch.cuda.synchronize()
    ys = []
    for it in range(6):
        for s in (s1, s2):
            with torch.cuda.stream(s):
                y = torch.full((nrows,), float("nan"), device="cuda")
                plan.spmv(rp, cd, vd, xd, y)
                ys.append(y)
    torch.cuda.synchronize()
    for y in ys:
        assert torch.equal(y.view(torch.int32), ref.view(torch.int32))
    # a fault on s1 (column out of range) is s1's alone
    bad = cd.clone()
    bad[5] = nrows + 7
    with torch.cuda.stream(s1):
        plan.spmv(rp, bad, vd, xd, torch.empty(nrows, device="cuda"))
    with torch.cuda.stream(s2):
        plan.spmv(rp, cd, vd, xd, torch.empty(nrows, device="cuda"))
    pb.device.sync_status(s2.cuda_stream)
    with pytest.raises(pb.PencilError):
        pb.device.sync_status(s1.cuda_stream)
    pb.device.sync_status(s1.cuda_stream)  # read and cleared


def test_interpreter_launches_the_mapped_kernel(cuda):
    """pencil_runtime_call launches the schedule's kernel: the CSR fixtures report the
    reassociating or the source-order executor by their inner loop's verdict."""
    import paper_1302_5586_b200 as pb
    rowptr, col, val, x, _ = synth.csr_powerlaw(5000, maxlen=300, seed=2)
    nrows, nnz = rowptr.size - 1, col.size
    it = pb.CudaInterpreter(0)
    for nm, a in (("rowptr", rowptr), ("col", col), ("val", val), ("x", x), ("y", np.zeros(nrows, np.float32))):
        it.set_array(nm, a)
    args = [pb.Arg.scalar(nrows), pb.Arg.scalar(nrows), pb.Arg.scalar(nnz)] + [pb.Arg.array(n) for n in
                                                                        ("rowptr", "col", "val", "x", "y")]
    for fn, kern in (("spmv_vec", "csr_tiles_reassoc"), ("spmv_inline", "csr_tiles_source_order"),
                     ("spmv", "csr_tiles_source_order")):
        it.call(fn, args)
        assert it.last_kernel() == kern
    ref = oracle.spmv_f32(nrows, nrows, nnz, rowptr, col, val, x)
    assert np.array_equal(it.get_array("y").view(np.uint32), ref.view(np.uint32))

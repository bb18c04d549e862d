"""Pageable host arrays through the drop-in ABI (csrc/hoststage.cpp): malloc'd / numpy memory of
4 MB and more goes through the multi-threaded pinned staging ring instead of the driver's
single-threaded bounce buffer.  Results must equal the pinned-memory calls bit for bit — whole
buffers, ragged sizes (not multiples of a chunk or of 64 bytes), the fp32 stencil's interior-only
copy-back (its border bytes untouched), the pipelined SpMV upload / y download — and concurrent
calls from several host threads must not mix their chunks."""
import threading

import numpy as np
import pytest

from paper_1302_5586_b200 import synth

pytestmark = pytest.mark.gpu


def pinned(torch, a):
    return torch.from_numpy(a).pin_memory()


def test_gemv_pageable_equals_pinned(cuda):
    import paper_1302_5586_b200 as pb
    torch = cuda
    m, n = 4099, 2053  # 33.7 MB of A: two ring chunks and a ragged tail
    A, x = synth.f32(m * n, 3), synth.f32(n, 4)
    y_pg = synth.f32(m, 5)
    y_pin = pinned(torch, y_pg.copy())
    pb.dropin.gemv(m, n, 1.5, 0.5, A, x, y_pg)
    pb.dropin.gemv(m, n, 1.5, 0.5, pinned(torch, A), pinned(torch, x), y_pin)
    assert np.array_equal(y_pg.view(np.uint32), y_pin.numpy().view(np.uint32))


def test_conv_f32_interior_copy_back_pageable(cuda):
    import paper_1302_5586_b200 as pb
    torch = cuda
    h, w = 2051, 2049
    img, k = synth.f32(h * w, 6), synth.f32(25, 7)
    out_pg = np.full(h * w, np.nan, np.float32)
    out_pin = pinned(torch, out_pg.copy())
    pb.dropin.conv5x5_f32(h, w, img, k, out_pg)
    pb.dropin.conv5x5_f32(h, w, pinned(torch, img), k, out_pin)
    assert np.array_equal(out_pg.view(np.uint32), out_pin.numpy().view(np.uint32))
    o = out_pg.reshape(h, w)
    border = np.ones((h, w), bool)
    border[2:h - 2, 2:w - 2] = False
    assert np.isnan(o[border]).all() and not np.isnan(o[~border]).any()


@pytest.mark.parametrize("fn", ["spmv_vec", "spmv_inline"])
def test_spmv_pipelined_pageable_equals_pinned(cuda, fn):
    import paper_1302_5586_b200 as pb
    torch = cuda
    rowptr, col, val, x, _ = synth.csr_powerlaw(1 << 20, seed=9)  # ~2^24 non-zeros: the pipelined path
    nrows, nnz = rowptr.size - 1, col.size
    y_pg = np.zeros(nrows, np.float32)
    y_pin = pinned(torch, np.zeros(nrows, np.float32))
    getattr(pb.dropin, fn)(nrows, nrows, nnz, rowptr, col, val, x, y_pg)
    getattr(pb.dropin, fn)(nrows, nrows, nnz, *(pinned(torch, a) for a in (rowptr, col, val, x)), y_pin)
    assert np.array_equal(y_pg.view(np.uint32), y_pin.numpy().view(np.uint32))


def test_concurrent_pageable_calls(cuda):
    import paper_1302_5586_b200 as pb
    m, n = 2048, 2560  # 21 MB of A per call
    A = [synth.f32(m * n, 10 + t) for t in range(4)]
    x = synth.f32(n, 20)
    refs = []
    for t in range(4):
        y = np.zeros(m, np.float32)
        pb.dropin.gemv(m, n, 1.0, 0.0, A[t], x, y)
        refs.append(y)
    errors = []

    def worker(t):
        try:
            for _ in range(4):
                y = np.zeros(m, np.float32)
                pb.dropin.gemv(m, n, 1.0, 0.0, A[t], x, y)
                assert np.array_equal(y.view(np.uint32), refs[t].view(np.uint32))
        except BaseException as e:  # noqa: BLE001
            errors.append((t, repr(e)))

    ts = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("taps,scale", [("BINOMIAL", 256), ("SHARPEN", 1)])
def test_conv_u8_bytes_host_entry(cuda, taps, scale):
    """pencil_conv5x5_u8_bytes on pageable numpy (staging ring: 8.4 MB), pinned and device arrays:
    bit-identical to the device API and to the oracle"""
    import oracle
    import paper_1302_5586_b200 as pb
    torch = cuda
    k = getattr(synth, taps)
    h, w = 2051, 4100
    img = synth.u8_i32(h * w, seed=31)
    img8 = img.astype(np.uint8)
    dev_out = torch.empty(h * w, dtype=torch.uint8, device="cuda")
    pb.device.conv5x5_u8_bytes(h, w, scale, torch.from_numpy(img8).cuda(), k, dev_out)
    ref = dev_out.cpu().numpy()
    out_pg = np.zeros(h * w, np.uint8)
    pb.dropin.conv5x5_u8_bytes(h, w, scale, img8, k, out_pg)
    assert np.array_equal(out_pg, ref)
    out_pin = torch.zeros(h * w, dtype=torch.uint8).pin_memory()
    pb.dropin.conv5x5_u8_bytes(h, w, scale, torch.from_numpy(img8).pin_memory(), k, out_pin)
    assert np.array_equal(out_pin.numpy(), ref)
    out_d = torch.zeros(h * w, dtype=torch.uint8, device="cuda")
    pb.dropin.conv5x5_u8_bytes(h, w, scale, torch.from_numpy(img8).cuda(), torch.from_numpy(
        np.ascontiguousarray(k, np.int32).reshape(-1)).cuda(), out_d)
    assert np.array_equal(out_d.cpu().numpy(), ref)
    # small case against the oracle (also below the staging threshold: the driver's copy)
    hs, ws = 37, 103
    imgs = synth.u8_i32(hs * ws, seed=5)
    o = np.zeros(hs * ws, np.uint8)
    pb.dropin.conv5x5_u8_bytes(hs, ws, scale, imgs.astype(np.uint8), k, o)
    assert np.array_equal(o.astype(np.int64), oracle.conv5x5_u8(hs, ws, scale, imgs, k))


def test_conv_u8_bytes_host_entry_errors(cuda):
    import paper_1302_5586_b200 as pb
    img = np.zeros(64, np.uint8)
    with pytest.raises(pb.PencilError) as e:
        pb.dropin.conv5x5_u8_bytes(8, 8, 0, img, synth.BINOMIAL, np.zeros(64, np.uint8))
    assert e.value.code == "E-INTERP"
    with pytest.raises(pb.PencilError) as e:
        pb.dropin.conv5x5_u8_bytes(-1, 8, 1, img, synth.BINOMIAL, np.zeros(64, np.uint8))
    assert e.value.code == "E-ARG"
    pb.dropin.conv5x5_u8_bytes(0, 8, 0, img, synth.BINOMIAL, np.zeros(64, np.uint8))  # empty: no-op


@pytest.mark.parametrize("pinned", [False, True])
def test_stencil_dropins_pipelined_equal_device_api(cuda, pinned):
    """conv5x5_u8 / conv5x5_f32 on host arrays of 64 MB and more run pipelined by row blocks (band
    sweeps over the resident image, uploads and downloads overlapping): bit-identical to the device
    API on the whole image — ragged last block, separable / diamond / generic taps, a non-byte pixel
    (the exact repair pass), fp32 power-of-two and generic taps with the border left untouched."""
    import paper_1302_5586_b200 as pb
    torch = cuda
    h, w = 4099, 4100  # 67 MB of int32 / fp32: ragged blocks of 513 rows
    host = (lambda a: torch.from_numpy(a).pin_memory()) if pinned else (lambda a: a)
    img = synth.u8_i32(h * w, seed=41)
    odd = img.copy()
    odd[h // 2 * w + 7] = 300  # not a byte: the exact repair pass
    odd[2051 * w + 100] = -5   # ... and one in the rows both blocks around row 2052 read
    for im, k, scale in ((img, synth.BINOMIAL, 256), (img, synth.SHARPEN, 1), (odd, synth.BINOMIAL, 256),
                         (img, synth.BINOMIAL * 3, 7)):
        dev = torch.empty(h * w, dtype=torch.int32, device="cuda")
        pb.device.conv5x5_u8(h, w, scale, torch.from_numpy(im).cuda(), k, dev)
        out = host(np.full(h * w, -1, np.int32))
        pb.dropin.conv5x5_u8(h, w, scale, host(im), k, out)
        got = out.numpy() if pinned else out
        assert np.array_equal(got, dev.cpu().numpy()), (scale, int(k[12]))
    f = synth.f32(h * w, 43)
    for k in ((synth.BINOMIAL / 256.0).astype(np.float32), synth.f32(25, 44)):
        dev = torch.full((h * w,), np.nan, device="cuda")
        pb.device.conv5x5_f32(h, w, torch.from_numpy(f).cuda(), k, dev)
        out = host(np.full(h * w, np.nan, np.float32))
        pb.dropin.conv5x5_f32(h, w, host(f), k, out)
        got = out.numpy() if pinned else out
        assert np.array_equal(got.view(np.uint32), dev.cpu().numpy().view(np.uint32))
        o = got.reshape(h, w)
        assert np.isnan(o[:2]).all() and np.isnan(o[-2:]).all() and np.isnan(o[:, :2]).all() and np.isnan(o[:, -2:]).all()


@pytest.mark.parametrize("pinned", [False, True])
def test_bytes_stencil_pipelined_equals_device_api(cuda, pinned):
    """pencil_conv5x5_u8_bytes on host arrays of 64 MB and more runs the SWAR kernels by row blocks
    (output rows [q0, q1) of the resident image): bit-identical to the whole-image device call —
    separable and signed / symmetric and skewed taps, 16- and 8-pixel lanes (w % 16 != 0), a ragged
    last block; taps without a SWAR form take the whole-image path."""
    import paper_1302_5586_b200 as pb
    torch = cuda
    host = (lambda a: torch.from_numpy(a).pin_memory()) if pinned else (lambda a: a)
    skew = np.outer([1, 3, 5, 2, 0], [2, 1, 4, 6, 3]).astype(np.int32).reshape(-1)
    asym = np.array([[0, 0, -1, 0, 0], [0, -2, -1, -3, 0], [-1, -3, 20, -2, 0],
                     [0, -1, -2, 0, 0], [0, 0, -4, 0, 0]], np.int32).reshape(-1)
    for h, w in ((8195, 8192), (8193, 8200)):
        img8 = synth.u8_i32(h * w, seed=h + w).astype(np.uint8)
        for k, scale in ((synth.BINOMIAL, 256), (synth.SHARPEN, 1), (skew, 256), (asym, 2), (synth.BINOMIAL * 40, 9)):
            dev = torch.empty(h * w, dtype=torch.uint8, device="cuda")
            pb.device.conv5x5_u8_bytes(h, w, scale, torch.from_numpy(img8).cuda(), k, dev)
            out = host(np.zeros(h * w, np.uint8))
            pb.dropin.conv5x5_u8_bytes(h, w, scale, host(img8), k, out)
            got = out.numpy() if pinned else out
            assert np.array_equal(got, dev.cpu().numpy()), (h, w, scale, int(k[12]))


@pytest.mark.parametrize("pinned", [False, True])
def test_axpy_pipelined_equals_emitted_c(cuda, pinned):
    """axpy on host arrays of 64 MB and more runs in chunks (upload / axpy / download overlapping):
    y bit-identical to the emitted C's a * x + y, ragged last chunk (n not a multiple of 4)."""
    import oracle
    import paper_1302_5586_b200 as pb
    torch = cuda
    n = (1 << 24) + 3
    x, y0 = synth.f32(n, 51), synth.f32(n, 52)
    ref = oracle.axpy_f32(n, np.float32(1.7), x, y0)
    host = (lambda a: torch.from_numpy(a).pin_memory()) if pinned else (lambda a: a)
    y = host(y0.copy())
    pb.dropin.axpy(n, 1.7, host(x), y)
    got = y.numpy() if pinned else y
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_f32_stencil_pipelined_tiny_pixels_across_block_edges(cuda):
    """The pipelined fp32 stencil (row blocks of 513 rows at h = 4099) with pixels whose fused
    power-of-two products would round (below 2^-126) straddling a block edge: each block's guard /
    repair pass keeps the result as written — bit-identical to the emitted C, border untouched."""
    import oracle
    import paper_1302_5586_b200 as pb
    h, w = 4099, 4100
    binom = (synth.BINOMIAL.astype(np.float32) / 256.0).astype(np.float32)
    img = synth.f32(h * w, seed=61).reshape(h, w)
    img[505:522, 90:150] = (img[505:522, 90:150] * np.float32(2.0 ** -118)).astype(np.float32)  # rows 513 +- 8
    img = img.reshape(-1)
    o0 = synth.f32(h * w, seed=62)
    out = o0.copy()
    pb.dropin.conv5x5_f32(h, w, img, binom, out)
    exact = oracle.conv5x5_f32_f32(h, w, img, binom, o0)
    assert np.array_equal(out.view(np.uint32), exact.view(np.uint32))

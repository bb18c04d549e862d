"""Array and view descriptors (include/pencil_b200.h §10).

CPU: the symbolic affine forms of every fixture access (coefficients may be scalar parameters, which
the reference's affine_form rejects, depanalysis.cpp:167-169), evaluated under bindings, generate
exactly the index sets the REFERENCE's summarize_call computes for the same binding
(oracle/_ref/ref_driver summarize); non-affine accesses (x[col[k]], a clamped img[r*w + c]) are
flagged; gemv_t's views and their slices; array descriptors' shard specs.
GPU: gemv_t through views (pencil_gemv_t_view_dev) and the column-sharded gemv_t of dist.py on
sliced views equal the plain call bit for bit; named arrays carry descriptors.
"""
import itertools
import json
import os
import subprocess

import numpy as np
import pytest

import oracle
from paper_1302_5586_b200 import synth

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = os.path.join(os.path.dirname(HERE), "paper_1302_5586_b200", "pencil")


def V():
    from paper_1302_5586_b200 import views
    return views


def test_symbolic_forms_of_the_strided_view():
    acc = V().affine_accesses(V().fixture_source("gemv_t"), "gemv_t", m=3, n=2, lda=4, incx=2, incy=3)
    forms = {(a["array"], a["write"]): (a["form"], a["stride"], [l[0] for l in a["loops"]]) for a in acc}
    assert forms[("A", False)] == ("j + i*lda", [1, 4], ["j", "i"])
    assert forms[("x", False)] == ("i*incx", [0, 2], ["j", "i"])
    assert forms[("y", True)] == ("j*incy", [3], ["j"])


def test_non_affine_accesses_are_flagged():
    sp = {a["array"]: a["affine"] for a in V().affine_accesses(V().fixture_source("spmv"), "spmv_vec",
                                                                  nrows=3, ncols=3, nnz=4)}
    assert sp["x"] is False and sp["col"] is True  # x[col[k]]: an indirection
    cv = [a for a in V().affine_accesses(V().fixture_source("conv5x5"), "conv5x5_u8", h=6, w=7, scale=1)
          if a["array"] == "img"]
    assert cv and not cv[0]["affine"]  # img[r * w + c] with r, c clamped locals
    f32 = [a for a in V().affine_accesses(V().fixture_source("conv5x5"), "conv5x5_f32", h=6, w=7)
           if a["array"] == "img"][0]
    assert f32["affine"] and f32["form"] == "i*w + j + di*w + dj - 2 - 2*w" and f32["offset"] == -16


BIND = {("gemv", "gemv"): {"m": 3, "n": 4}, ("gemv_t", "gemv_t"): {"m": 3, "n": 2, "lda": 5, "incx": 2, "incy": 3},
        ("axpy", "axpy"): {"n": 6}, ("dot", "dot"): {"n": 6}, ("gemm", "gemm"): {"m": 2, "n": 3, "k": 4},
        ("conv5x5", "conv5x5_f32"): {"h": 7, "w": 8}}


@pytest.mark.parametrize("fixture,fn", sorted(BIND))
def test_affine_index_sets_equal_reference_summarize_call(fixture, fn):
    """For every affine access: the indices offset + sum_d stride_d * v_d over the loop ranges equal
    the reference's concrete read / must-write set of that array (summarize_call under the same
    binding) — the views address exactly what the reference nest touches."""
    if not os.path.exists(oracle.REF_DRIVER):
        pytest.skip("oracle/_ref not built")
    b = BIND[(fixture, fn)]
    cmd = [oracle.REF_DRIVER, "summarize", os.path.join(FIX, fixture + ".pencil.c"), fn]
    for k, v in b.items():
        cmd += ["--param", f"{k}={v}"]
    ref = {j["array"]: j for j in map(json.loads, subprocess.run(cmd, capture_output=True, text=True,
                                                                   check=True).stdout.splitlines())}
    got = {}
    for a in V().affine_accesses(V().fixture_source(fixture), fn, **b):
        assert a["affine"], a
        ranges = [range(lo, hi) for _, lo, hi in a["loops"]]
        idx = {a["offset"] + sum(s * v for s, v in zip(a["stride"], vs)) for vs in itertools.product(*ranges)}
        key = (a["array"], "must" if a["write"] else "read")
        got[key] = got.get(key, set()) | idx
    for (arr, kind), idx in got.items():
        assert sorted(idx) == ref[arr][kind], (arr, kind)


def test_gemv_t_views_and_slices():
    A, x, y = V().gemv_t_views(30, 20, 24, 2, 3)
    assert (A.extent, A.stride, x.extent, x.stride, y.extent, y.stride) == ((30, 20), (24, 1), (30,), (2,), (20,), (3,))
    a, yy = A.slice(1, 5, 15), y.slice(0, 5, 15)
    assert (a.offset, a.extent, yy.offset, yy.extent) == (5, (30, 10), 15, (10,))
    import paper_1302_5586_b200 as pb
    with pytest.raises(pb.PencilError):
        A.slice(1, 5, 21)


def test_array_descriptor_shards():
    import paper_1302_5586_b200 as pb
    d = V().ArrayDesc(np.float32, 10, [0, 4, 4, 10])
    assert d.nshards == 3 and [d.owner(i) for i in (0, 3, 4, 9, 10)] == [0, 0, 2, 2, -1]
    assert d.shard(2)[:2] == (4, 10)
    d.attach(2, 0, 0x1000)
    assert d.shard(2)[2:] == (0, 0x1000)
    v = d.view(2)
    assert v.extent == (6,) and v.stride == (1,)
    with pytest.raises(pb.PencilError):
        V().ArrayDesc(np.float32, 10, [0, 6, 4, 10])  # not ordered
    with pytest.raises(pb.PencilError):
        V().ArrayDesc(np.float32, 10, [1, 10])  # does not start at 0


@pytest.mark.gpu
def test_gemv_t_through_views_and_column_shards(cuda):
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200.dist import ColShardedGemvT
    torch = cuda
    m, n, lda, incx, incy = 3000, 2100, 2112, 2, 3
    A, x, y = synth.f32(m * lda, 4), synth.f32(m * incx, 5), synth.f32(n * incy, 6)
    dA, dx = torch.from_numpy(A).cuda(), torch.from_numpy(x).cuda()
    ref = torch.from_numpy(y.copy()).cuda()
    pb.device.gemv_t(m, n, lda, incx, incy, 1.25, 0.5, dA, dx, ref)
    Av, xv, yv = V().gemv_t_views(m, n, lda, incx, incy)
    got = torch.from_numpy(y.copy()).cuda()
    V().gemv_t_view(1.25, 0.5, Av.on(dA), xv.on(dx), yv.on(got))
    assert torch.equal(got.view(torch.int32), ref.view(torch.int32))
    for world in (2, 3, 5):  # every rank's column block on sliced views, one GPU
        out = torch.from_numpy(y.copy()).cuda()
        for r in range(world):
            ColShardedGemvT(m, n, r, world, lda=lda, incx=incx, incy=incy).step(1.25, 0.5, dA, dx, out)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int32), ref.view(torch.int32)), world
    # a view the kernel cannot take (A with non-unit stride along j) is refused
    bad = V().View(__import__("paper_1302_5586_b200")._lib.pencil_view.from_buffer_copy(Av.c))
    bad.c.stride[1] = 2
    with pytest.raises(pb.PencilError):
        V().gemv_t_view(1.0, 0.0, bad.on(dA), xv.on(dx), yv.on(got))


@pytest.mark.gpu
def test_named_arrays_are_descriptors(cuda):
    import ctypes
    import paper_1302_5586_b200 as pb
    it = pb.CudaInterpreter(0)
    it.set_array("x", synth.f32(100, 3))
    lib = pb.load()
    h = lib.pencil_runtime_array_desc(it._rt, b"x")
    assert h
    dt, n, ns = ctypes.c_int(), ctypes.c_longlong(), ctypes.c_int()
    lib.pencil_array_info(h, ctypes.byref(dt), ctypes.byref(n), ctypes.byref(ns), None)
    assert (dt.value, n.value, ns.value) == (1, 100, 1)
    lo, hi, dev, ptr = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_int(), ctypes.c_void_p()
    lib.pencil_array_shard(h, 0, ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(dev), ctypes.byref(ptr))
    dptr = ctypes.c_void_p()
    lib.pencil_runtime_array_info(it._rt, b"x", None, None, ctypes.byref(dptr))
    assert (lo.value, hi.value, dev.value, ptr.value) == (0, 100, 0, dptr.value)

"""General mapper for PENCIL units (csrc/jit.cpp): any compliant unit on the GPU
with the reference Interpreter's value semantics.

CPU: schedules derived from the directives (independent -> parallel grid, reduction -> parallel
+ fixed-order combine, everything else serial) and load errors.
GPU: every golden vector of tests/golden (the reference Interpreter's fp64 / int64 outputs on the
fixtures) replayed through the JIT: bit-exact wherever no reduction is split across threads
(gemv, gemv_t, axpy, the three SpMV spellings, both stencils, gemm: their reductions are inner
loops, run in order inside one thread), within 1e-12 normwise for dot's top-level reduction, and
the interpreter's faults as E-INTERP; plus a unit exercising frames, local arrays, returns,
int/double dynamic typing, while loops and last-iteration scalar values.
"""
import os

import numpy as np
import pytest

from conftest import golden_cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "paper_1302_5586_b200", "pencil")


def unit(src):
    from paper_1302_5586_b200.op2 import JitUnit
    return JitUnit(src)


def fixture_src(name):
    return open(os.path.join(FIX, name + ".pencil.c")).read()


@pytest.mark.parametrize("fixture,fn,sched", [
    ("gemv", "gemv", "W"), ("gemv_t", "gemv_t", "W"), ("dot", "dot", "SRS"), ("axpy", "axpy", "P"),
    ("spmv", "spmv_vec", "W"), ("spmv", "spmv_inline", "P"), ("spmv", "spmv", "S"), ("gemm", "gemm", "2"),
    ("conv5x5", "conv5x5_u8", "2"), ("conv5x5", "conv5x5_f32", "2"),
])
def test_schedule_from_directives(fixture, fn, sched):
    assert unit(fixture_src(fixture)).schedule(fn) == sched


def test_unparsable_unit_is_rejected():
    import paper_1302_5586_b200 as pb
    with pytest.raises(pb.PencilError) as e:
        unit("void f(int n) { n = ; }")
    assert e.value.code == "E-ARG" and "E-SYNTAX" in str(e.value)


GOLD = [c for c in golden_cases() if c.fixture in ("gemv", "gemv_t", "dot", "axpy", "spmv", "conv5x5", "gemm")]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD, ids=[c.name for c in GOLD])
def test_golden_vectors_through_the_jit(cuda, case):
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200.interp import Arg
    u = unit(fixture_src(case.fixture))
    args = []
    for i, a in enumerate(case.args):
        if isinstance(a, np.ndarray):
            u.set_array(f"a{i}", a)
            args.append(Arg.array(f"a{i}"))
        else:
            args.append(a)
    if case.fault:
        with pytest.raises(pb.PencilError) as e:
            u.call(case.fn, args)
        assert e.value.code == "E-INTERP"
        return
    ret = u.call(case.fn, args)
    if case.fn == "dot":  # top-level reduction split across threads: re-associated fp64
        x, y = case.args[1].astype(np.float64), case.args[2].astype(np.float64)
        assert abs(ret - case.ret) <= 1e-12 * max(1e-300, float(np.sum(np.abs(x * y))))
    elif case.ret is not None:
        assert ret == case.ret
    scale = _reassociated_scale(case)
    for i, ref in case.outs.items():
        vals, ints, isd = u.get_array(f"a{i}")
        if ref.dtype == np.int64:
            assert np.array_equal(ints, ref), i
        elif scale is None or scale.shape != ref.shape:  # not split across lanes: bit-exact fp64
            assert np.array_equal(vals.view(np.uint64), ref.astype(np.float64).view(np.uint64)), i
        else:  # warp-split inner reduction (the pragma licenses re-association): normwise
            assert np.all(np.abs(vals - ref) <= 1e-12 * scale + 0.0), i


def _reassociated_scale(case):
    """Per-element magnitude of the reductions the mapper splits across a warp (schedule 'W'):
    gemv / gemv_t rows, spmv_vec rows; None for everything computed in source order."""
    a = case.args
    if case.fn == "gemv":
        m, n, alpha, beta, A, x, y = a
        return abs(alpha) * (np.abs(A.astype(np.float64).reshape(m, n)) @ np.abs(x.astype(np.float64))) + \
            abs(beta) * np.abs(y.astype(np.float64))
    if case.fn == "gemv_t":
        m, n, lda, incx, incy, alpha, beta, A, x, y = a
        sc = np.abs(y.astype(np.float64)) * abs(beta)
        if m > 0:
            At = np.abs(A.astype(np.float64)[: m * lda].reshape(m, lda)[:, :n])
            xs = np.abs(x.astype(np.float64)[np.arange(m) * incx])
            sc[np.arange(n) * incy] += abs(alpha) * (xs @ At)
        return sc
    if case.fn == "spmv_vec":
        nrows, ncols, nnz, rowptr, col, val, x, y = a
        t = np.abs(val.astype(np.float64)) * np.abs(x.astype(np.float64)[np.clip(col, 0, ncols - 1)])
        cs = np.concatenate([[0.0], np.cumsum(t)])
        rp = np.clip(rowptr, 0, nnz)
        return np.maximum(cs[rp[1:]] - cs[rp[:-1]], 0.0)
    return None


SEMANTICS = r"""
int helper(int n, int a[restrict const static n], int k)
{
  int t;
  t = a[k] * 2;
  a[k] = t;
  if (t > 10) return t / 3;
  return -t % 4;
}

double mix(int n, int a[restrict const static n], float b[restrict const static n], int out[restrict const static n])
{
  int i;
  int last;
  float f;
  double acc;
  int tmp[4];
  f = 3;
  acc = 0.0;
  last = -1;
  #pragma pencil independent
  for (i = 0; i < n; i++) {
    int w[2];
    w[0] = a[i] + i;
    w[1] = w[0] / 2;
    out[i] = w[1] - helper(n, a, i);
    b[i] = b[i] * 0.5 + f / 2;
    last = i * 10;
  }
  tmp[1] = last;
  #pragma pencil reduction (+: acc)
  for (i = 0; i < n; i++) {
    acc += out[i] + 0.25;
  }
  while (tmp[1] > 7) {
    tmp[1] = tmp[1] - 7;
  }
  out[0] = tmp[1];
  return acc + i;
}
"""


@pytest.mark.gpu
def test_interpreter_semantics_unit(cuda):
    from paper_1302_5586_b200.interp import Arg
    n = 257
    rng = np.random.default_rng(3)
    a = rng.integers(-20, 20, n).astype(np.int32)
    b = rng.standard_normal(n).astype(np.float32)
    u = unit(SEMANTICS)
    assert u.schedule("mix") == "SPSRS"
    u.set_array("a", a)
    u.set_array("b", b)
    u.set_array("out", np.zeros(n, np.int32))
    ret = u.call("mix", [n, Arg.array("a"), Arg.array("b"), Arg.array("out")])
    # python restatement of the interpreter's semantics (int64 / fp64, C-truncating / and %)
    def cdiv(x, y):
        q = abs(x) // abs(y)
        return q if (x >= 0) == (y >= 0) else -q

    def cmod(x, y):
        return x - cdiv(x, y) * y
    A, out = a.astype(np.int64).tolist(), [0] * n
    for i in range(n):
        w0 = A[i] + i
        w1 = cdiv(w0, 2)
        t = A[i] * 2
        A[i] = t
        h = cdiv(t, 3) if t > 10 else cmod(-t, 4)
        out[i] = w1 - h
    last = (n - 1) * 10
    acc = sum(o + 0.25 for o in out)
    t1 = last
    while t1 > 7:
        t1 -= 7
    out[0] = t1
    vals, ints, isd = u.get_array("a")
    assert ints.tolist() == A
    vals, ints, isd = u.get_array("out")
    assert ints.tolist() == out
    vals, ints, isd = u.get_array("b")
    ref_b = b.astype(np.float64) * 0.5 + 1  # int division 3 / 2 == 1
    assert np.array_equal(vals, ref_b) and isd.all()
    # after `for (i = 0; i < n; i++)` the interpreter leaves i = n - 1 (interp.cpp:207-217)
    assert abs(ret - (acc + n - 1)) <= 1e-9 * abs(acc + n)


REDUCTIONS = r"""
double red4(int n, int a[restrict const static n], float b[restrict const static n], int out[restrict const static 4])
{
  int i;
  int s;
  int p;
  int mx;
  double mn;
  s = 0;
  p = 1;
  mx = -1000000;
  mn = 1000000.0;
  #pragma pencil reduction (+: s)
  for (i = 0; i < n; i++) {
    s += a[i] * 3 - i % 7;
  }
  #pragma pencil reduction (*: p)
  for (i = 0; i < n; i++) {
    if (a[i] % 5 == 0) p *= -1;
  }
  #pragma pencil reduction (max: mx)
  for (i = 0; i < n; i++) {
    if (a[i] > mx) mx = a[i];
  }
  #pragma pencil reduction (min: mn)
  for (i = 0; i < n; i++) {
    if (b[i] < mn) mn = b[i];
  }
  out[0] = s;
  out[1] = p;
  out[2] = mx;
  return mn;
}

void oob(int n, int a[restrict const static n])
{
  int i;
  #pragma pencil independent
  for (i = 0; i < n; i++) {
    a[i + 1] = i;
  }
}

int divz(int n, int a[restrict const static n])
{
  int i;
  int t;
  t = 0;
  for (i = 0; i < n; i++) {
    t = t + 100 / (a[i] - 3);
  }
  return t;
}
"""


@pytest.mark.gpu
def test_reductions_and_faults(cuda):
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200.interp import Arg
    n = 100003
    rng = np.random.default_rng(9)
    a = rng.integers(-10000, 10000, n).astype(np.int32)
    b = rng.standard_normal(n).astype(np.float32)
    u = unit(REDUCTIONS)
    assert u.schedule("red4") == "SRRRRS"
    u.set_array("a", a)
    u.set_array("b", b)
    u.set_array("out", np.zeros(4, np.int32))
    mn = u.call("red4", [n, Arg.array("a"), Arg.array("b"), Arg.array("out")])
    _, ints, _ = u.get_array("out")
    i = np.arange(n)
    a64 = a.astype(np.int64)
    s_ref = int(np.sum(a64 * 3 - (i % 7)))
    p_ref = (-1) ** int(np.sum(np.fmod(a64, 5) == 0))
    assert ints[:3].tolist() == [s_ref, p_ref, int(a.max())]
    assert mn == float(b.astype(np.float64).min())  # min is exact whatever the order
    # a store past the end inside a parallel loop, and a division by zero: E-INTERP like the interpreter
    u.set_array("z", np.zeros(16, np.int32))
    with pytest.raises(pb.PencilError) as e:
        u.call("oob", [16, Arg.array("z")])
    assert e.value.code == "E-INTERP" and "store out of bounds" in str(e.value)
    u.set_array("d", np.array([1, 2, 3, 4], np.int32))
    with pytest.raises(pb.PencilError) as e:
        u.call("divz", [4, Arg.array("d")])
    assert e.value.code == "E-INTERP" and "division by zero" in str(e.value)


NESTED = r"""
int grid2(int m, int n, int out[restrict const static m * n])
{
  int i;
  int j;
  int last;
  last = -7;
  #pragma pencil independent
  for (i = 0; i < m; i++) {
    #pragma pencil independent
    for (j = 0; j < n; j++) {
      out[i * n + j] = i * 1000 + j;
      last = i + j;
    }
  }
  return i * 100000 + j * 100 + last;
}
"""


@pytest.mark.gpu
def test_nested_independent_loops_collapse_to_a_2d_grid(cuda):
    from paper_1302_5586_b200.interp import Arg
    u = unit(NESTED)
    assert u.schedule("grid2") == "S2S"
    m, n = 37, 53
    u.set_array("o", np.zeros(m * n, np.int32))
    ret = u.call("grid2", [m, n, Arg.array("o")])
    _, ints, _ = u.get_array("o")
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    assert np.array_equal(ints.reshape(m, n), ii * 1000 + jj)
    # after the loops: i = m-1, j = n-1 (interp.cpp:207-217), last = (m-1)+(n-1)
    assert ret == (m - 1) * 100000 + (n - 1) * 100 + (m - 1) + (n - 1)
    # inner range empty: the outer variable still advances, j and last keep their values
    u.set_array("o0", np.zeros(1, np.int32))
    ret = u.call("grid2", [5, 0, Arg.array("o0")])
    assert ret == 4 * 100000 + 0 * 100 - 7

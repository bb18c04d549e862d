"""Distribution plans: which arrays a split of a nest's parallel loop
shards, which need a halo, which must be replicated (all-gathered) and which reduction variables
need an all-reduce — derived from the index expressions and ACCESS summaries of the PENCIL source
(pencil_dist_plan, csrc/distplan.cpp), not written down per kernel.

Checked three ways: the plans of the fixtures are pinned; every class is validated against the
REFERENCE interpreter's own memory trace (Interpreter::enable_trace, interp.hpp:17-21, 45-46) of
single iterations of the loop (the loop header restricted to [d, d+1) in the source); and the
multi-GPU shard classes (dist.py) take their halo / gather decisions from the plans."""
import re

import numpy as np
import pytest

import oracle
from paper_1302_5586_b200 import views


def plan(fixture, fn, dim=0):
    return views.dist_plan(fixture, fn)["dims"][dim]


def cls(p, a):
    v = p["arrays"][a]
    return (v["mode"], v["kind"], v.get("stride"), tuple(v.get("halo", ())) or None, v.get("via"))


# --- pinned plans of the fixtures ---------------------------------------------------------------
EXPECTED = {
    ("gemv", "gemv", 0): ("i", "parallel", {"A": ("r", "block", "n", (0, 0), None), "x": ("r", "all", None, None, None),
                                            "y": ("rw", "block", "1", (0, 0), None)}, ["y"], [], ["x"]),
    ("gemv_t", "gemv_t", 0): ("j", "parallel", {"A": ("r", "view", "1", (0, 0), None),
                                                "x": ("r", "all", None, None, None),
                                                "y": ("rw", "block", "incy", (0, 0), None)}, ["y"], [], ["x"]),
    ("dot", "dot", 0): ("i", "reduction", {"x": ("r", "block", "1", (0, 0), None),
                                           "y": ("r", "block", "1", (0, 0), None)}, [], [], []),
    ("axpy", "axpy", 0): ("i", "analyzed", {"x": ("r", "block", "1", (0, 0), None),
                                            "y": ("rw", "block", "1", (0, 0), None)}, ["y"], [], []),
    ("spmv", "spmv_vec", 0): ("i", "parallel", {"rowptr": ("r", "block", "1", (0, 1), None),
                                                "col": ("r", "via", None, None, "rowptr"),
                                                "val": ("r", "via", None, None, "rowptr"),
                                                "x": ("r", "all", None, None, None),
                                                "y": ("w", "block", "1", (0, 0), None)}, ["y"], ["rowptr"], ["x"]),
    ("spmv", "spmv_inline", 0): ("i", "parallel", {"rowptr": ("r", "block", "1", (0, 1), None),
                                                   "col": ("r", "via", None, None, "rowptr"),
                                                   "val": ("r", "via", None, None, "rowptr"),
                                                   "x": ("r", "all", None, None, None),
                                                   "y": ("w", "block", "1", (0, 0), None)}, ["y"], ["rowptr"], ["x"]),
    # the ACCESS-summarised driver: its summary over-approximates col / val (USE(col[k]) for every
    # k), so the plan replicates them — the summary is the contract (summaries.cpp:635-648)
    ("spmv", "spmv", 0): ("i", "analyzed", {"rowptr": ("r", "block", "1", (0, 1), None),
                                            "col": ("r", "all", None, None, None),
                                            "val": ("r", "all", None, None, None),
                                            "x": ("r", "all", None, None, None),
                                            "y": ("w", "block", "1", (0, 0), None)},
                          ["y"], ["rowptr"], ["col", "val", "x"]),
    ("conv5x5", "conv5x5_u8", 0): ("i", "parallel", {"img": ("r", "block", "w", (-2, 2), None),
                                                     "k": ("r", "all", None, None, None),
                                                     "out": ("w", "block", "w", (0, 0), None)},
                                   ["out"], ["img"], ["k"]),
    ("conv5x5", "conv5x5_f32", 0): ("i", "parallel", {"img": ("r", "block", "w", (-2, 2), None),
                                                      "k": ("r", "all", None, None, None),
                                                      "out": ("w", "block", "w", (0, 0), None)},
                                    ["out"], ["img"], ["k"]),
    ("conv5x5", "conv5x5_f32", 1): ("j", "parallel", {"img": ("r", "view", "1", (-2, 2), None),
                                                      "k": ("r", "all", None, None, None),
                                                      "out": ("w", "view", "1", (0, 0), None)},
                                    ["out"], ["img"], ["k"]),
    ("gemm", "gemm", 0): ("i", "parallel", {"A": ("r", "block", "k", (0, 0), None),
                                            "B": ("r", "all", None, None, None),
                                            "C": ("rw", "block", "n", (0, 0), None)}, ["C"], [], ["B"]),
    # the 2-D tile grid: B column panels and C tiles are strided views along j
    ("gemm", "gemm", 1): ("j", "parallel", {"A": ("r", "all", None, None, None),
                                            "B": ("r", "view", "1", (0, 0), None),
                                            "C": ("rw", "view", "1", (0, 0), None)}, ["C"], [], ["A"]),
}


@pytest.mark.parametrize("key", sorted(EXPECTED), ids=lambda k: f"{k[1]}-d{k[2]}")
def test_fixture_plans(key):
    fixture, fn, dim = key
    var, kind, arrays, owned, halo, gather = EXPECTED[key]
    p = plan(fixture, fn, dim)
    assert (p["var"], p["kind"]) == (var, kind)
    assert {a: cls(p, a) for a in p["arrays"]} == arrays
    assert (sorted(p["owned"]), sorted(p["halo"]), sorted(p["replicated"]), p["conflicts"]) == \
        (sorted(owned), sorted(halo), sorted(gather), [])


def test_reductions_and_views():
    assert plan("dot", "dot")["reduce"] == ["s"]  # one all-reduce of the partial sums
    assert plan("gemv_t", "gemv_t")["arrays"]["A"]["inner"] == ["i:lda"]  # A(i, j) = A[i*lda + j]
    assert plan("gemm", "gemm", 1)["arrays"]["B"]["inner"] == ["p:n"]


# --- validation against the reference interpreter's trace --------------------------------------
def function_text(src, fn):
    """the unit with fn's distributed loop restricted to [d, d + 1): returns (prefix, header, rest)"""
    start = src.index(re.search(r"\b\w+\s+" + fn + r"\s*\(", src).group(0))
    m = re.compile(r"for \(int (\w+) = ([^;]+); \1 < ([^;]+); \1\+\+\)").search(src, start)
    return src[:m.start()], m, src[m.end():]


def one_iteration(fixture, fn, d):
    src = views.fixture_source(fixture)
    pre, m, post = function_text(src, fn)
    v = m.group(1)
    return pre + f"for (int {v} = {d}; {v} < {d} + 1; {v}++)" + post


def rng_args(fixture, fn):
    r = np.random.default_rng(3)
    f32 = lambda n: r.random(n, dtype=np.float32) - np.float32(0.5)  # noqa: E731
    if fixture == "gemv":
        m, n = 9, 7
        return {"m": m, "n": n}, [m, n, 1.5, 0.5, f32(m * n), f32(n), f32(m)], 4
    if fixture == "gemv_t":
        m, n, lda, incx, incy = 6, 5, 8, 2, 3
        return ({"m": m, "n": n, "lda": lda, "incx": incx, "incy": incy},
                [m, n, lda, incx, incy, 1.0, 0.5, f32(m * lda), f32(m * incx), f32(n * incy)], 3)
    if fixture == "dot":
        return {"n": 11}, [11, f32(11), f32(11)], 5
    if fixture == "axpy":
        return {"n": 11}, [11, 2.0, f32(11), f32(11)], 5
    if fixture == "spmv":
        lens = [2, 0, 3, 1, 4, 2, 1]
        rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        nnz, nc = int(rowptr[-1]), 6
        col = r.integers(0, nc, nnz).astype(np.int32)
        return ({"nrows": 7, "ncols": nc, "nnz": nnz, "rowptr": rowptr},
                [7, nc, nnz, rowptr, col, f32(nnz), f32(nc), f32(7)], 4)
    if fixture == "conv5x5":
        h, w = 9, 8
        if fn == "conv5x5_u8":
            img = r.integers(0, 256, h * w).astype(np.int32)
            return {"h": h, "w": w}, [h, w, 16, img, r.integers(-3, 4, 25).astype(np.int32),
                                      np.zeros(h * w, np.int32)], 4
        return {"h": h, "w": w}, [h, w, f32(h * w), f32(25), np.zeros(h * w, np.float32)], 4
    if fixture == "gemm":
        m, n, k = 5, 6, 4
        return {"m": m, "n": n, "k": k}, [m, n, k, 1.0, 0.5, f32(m * k), f32(k * n), f32(m * n)], 2
    raise KeyError(fixture)


def stride_value(expr, env):
    return int(eval(expr.replace("*", " * "), {}, dict(env)))  # noqa: S307 — the plan's own polynomial text


@pytest.mark.parametrize("fixture,fn", [("gemv", "gemv"), ("gemv_t", "gemv_t"), ("dot", "dot"), ("axpy", "axpy"),
                                        ("spmv", "spmv_vec"), ("spmv", "spmv_inline"), ("spmv", "spmv"),
                                        ("conv5x5", "conv5x5_u8"), ("conv5x5", "conv5x5_f32"), ("gemm", "gemm")])
def test_plan_against_reference_trace(fixture, fn):
    """every element one iteration d of the distributed loop touches (the reference interpreter's
    MemTrace) lies where the plan says: a block's rows d + h0 .. d + h1, a via-array's range
    rowptr[d] .. rowptr[d + 1], and stores only in the iteration's own block"""
    env, args, d = rng_args(fixture, fn)
    p = plan(fixture, fn)
    src = views.fixture_source(fixture)
    import inspect  # noqa: F401
    names = re.search(r"\b\w+\s+" + fn + r"\s*\(([^)]*)\)", src).group(1)
    params = [re.split(r"[\s\[*]+", q.strip())[1] for q in names.split(",")]
    lo = int(env.get("lo", 0))
    for it in sorted({d, d + 1, lo + (2 if fixture == "conv5x5" and fn == "conv5x5_f32" else 0)}):
        trace = oracle.ref_trace(one_iteration(fixture, fn, it), fn, args)
        assert trace, (fn, it)
        for argi, idx, wr in trace:
            name = params[argi]
            c = p["arrays"][name]
            if wr:
                assert name in p["owned"], (fn, name)
            if c["kind"] == "block":
                s = stride_value(c["stride"], env)
                row = idx // s
                lo_h, hi_h = c["halo"] if not wr else (0, 0)
                assert it + lo_h <= row <= it + hi_h, (fn, name, it, idx, c)
            elif c["kind"] == "via":
                rp = env[c["via"]]
                assert rp[it] <= idx < rp[it + 1], (fn, name, it, idx)
            elif c["kind"] == "view":
                s = stride_value(c["stride"], env)
                inner = [stride_value(q.split(":")[1], env) for q in c["inner"]]
                lo_h, hi_h = c["halo"]
                # idx = s * it + h + sum_q inner_q * k_q: the residue modulo the (single) inner stride
                assert len(inner) >= 1
                r_ = (idx - s * it) % inner[0]
                r_ = r_ - inner[0] if r_ > inner[0] // 2 else r_
                assert lo_h <= r_ // s <= hi_h, (fn, name, it, idx, c)


# --- synthetic units: halo widths, transposes, gathers, conflicts ------------------------------
UNIT = """
void stencil3(int n, float x[restrict const static n], float y[restrict const static n])
{
  #pragma pencil independent
  for (int i = 1; i < n - 1; i++) {
    y[i] = x[i - 1] + x[i] + x[i + 1];
  }
}
void transpose(int m, int n, float A[restrict const static m * n], float B[restrict const static n * m])
{
  #pragma pencil independent
  for (int i = 0; i < m; i++) {
    for (int j = 0; j < n; j++) {
      B[j * m + i] = A[i * n + j];
    }
  }
}
void gather(int n, int m, int idx[restrict const static n], float x[restrict const static m],
            float y[restrict const static n])
{
  #pragma pencil independent
  for (int i = 0; i < n; i++) {
    y[i] = x[idx[i]];
  }
}
void histogram(int n, int m, int key[restrict const static n], int h[restrict const static m])
{
  for (int i = 0; i < n; i++) {
    h[key[i]] += 1;
  }
}
void rows2(int m, int n, float A[restrict const static m * n], float y[restrict const static m])
{
  #pragma pencil independent
  for (int i = 0; i < m; i++) {
    float s;
    s = 0.0;
    for (int j = 0; j < n; j++) {
      s += A[i * n + j] + A[(i + 1) * n - 1 - j];
    }
    y[i] = s;
  }
}
"""


def test_synthetic_units():
    p = views.dist_plan(UNIT, "stencil3")["dims"][0]
    assert cls(p, "x") == ("r", "block", "1", (-1, 1), None) and p["halo"] == ["x"]
    p = views.dist_plan(UNIT, "transpose")["dims"][0]
    assert cls(p, "A") == ("r", "block", "n", (0, 0), None)
    assert p["arrays"]["B"]["kind"] == "view" and p["arrays"]["B"]["inner"] == ["j:m"]
    p = views.dist_plan(UNIT, "gather")["dims"][0]
    assert p["replicated"] == ["x"] and p["owned"] == ["y"] and cls(p, "idx") == ("r", "block", "1", (0, 0), None)
    p = views.dist_plan(UNIT, "histogram")["dims"][0]
    assert p["kind"] == "serial" and p["conflicts"] == ["h"]  # a scattered increment: not splittable as written
    p = views.dist_plan(UNIT, "rows2")["dims"][0]
    assert cls(p, "A") == ("r", "block", "n", (0, 0), None)  # both ends of row i stay in row i


# --- the shard classes follow the plans ---------------------------------------------------------
def test_shard_classes_follow_plans():
    from paper_1302_5586_b200 import dist
    assert dist.BandShardedImage.halo_rows() == 2  # conv5x5 img halo (-2, 2)
    assert dist.RowShardedCsr.gathered() == ["x"]  # spmv_vec: x replicated, col / val via rowptr
    assert dist.RowShardedGemv.gathered() == ["x"]
    assert dist.ColShardedGemvT.gathered() == ["x"]
    assert dist.GemmTileGrid.panels_needed() == {"A": "rows", "B": "cols"}
    assert dist.dot_allreduce_vars() == ["s"]


# --- random nests against the reference trace ---------------------------------------------------
def random_unit(rng, idx):
    """A random 2-deep nest: reads of A in rows i + a (a in [-2, 2]) at columns j + b, of a row
    vector B[j] (replicated), of a column vector c[i + e]; writes y[i*m + j] or z[i]."""
    reads, terms = [], []
    for t in range(int(rng.integers(1, 4))):
        a, b = int(rng.integers(-2, 3)), int(rng.integers(-1, 2))
        reads.append(("A", a, b))
        terms.append(f"A[(i + {a}) * m + j + {b}]")
    if rng.random() < 0.5:
        terms.append("B[j]")
    e = int(rng.integers(-1, 2))
    terms.append(f"c[i + {e}]")
    write_row = rng.random() < 0.5
    body = (f"      y[i * m + j] = {' + '.join(terms)};\n" if write_row else
            f"      s += {' + '.join(terms)};\n")
    src = f"""void f{idx}(int n, int m, float A[restrict const static n * m], float B[restrict const static m],
          float c[restrict const static n], float y[restrict const static n * m], float z[restrict const static n])
{{
  #pragma pencil independent
  for (int i = 2; i < n - 2; i++) {{
    float s;
    s = 0.0;
    for (int j = 1; j < m - 1; j++) {{
{body}    }}
    z[i] = s;
  }}
}}
"""
    a_lo = min(a for _, a, _ in reads)
    a_hi = max(a for _, a, _ in reads)
    return src, (a_lo, a_hi), e, "B[j]" in terms, write_row


@pytest.mark.parametrize("seed", range(12))
def test_random_nests_against_reference_trace(seed):
    rng = np.random.default_rng(100 + seed)
    src, (a_lo, a_hi), e, has_b, write_row = random_unit(rng, seed)
    fn = f"f{seed}"
    p = views.dist_plan(src, fn)["dims"][0]
    assert cls(p, "A")[:4] == ("r", "block", "m", (a_lo, a_hi))
    assert cls(p, "c")[:4] == ("r", "block", "1", (e, e))
    assert ("B" in p["replicated"]) == has_b
    assert p["owned"] == (["y", "z"] if write_row else ["z"])
    n, m = 9, 7
    f32 = lambda k: (rng.random(k, dtype=np.float32) - np.float32(0.5))  # noqa: E731
    args = [n, m, f32(n * m), f32(m), f32(n), np.zeros(n * m, np.float32), np.zeros(n, np.float32)]
    names = ["n", "m", "A", "B", "c", "y", "z"]
    for it in (2, 4, 6):
        unit = re.sub(r"for \(int i = 2; i < n - 2; i\+\+\)", f"for (int i = {it}; i < {it} + 1; i++)", src)
        for argi, idx, wr in oracle.ref_trace(unit, fn, args):
            name = names[argi]
            c = p["arrays"][name]
            if c["kind"] == "block":
                s = {"m": m, "1": 1}[c["stride"]]
                lo_h, hi_h = c["halo"]
                assert it + lo_h <= idx // s <= it + hi_h, (name, it, idx, c)
            if wr:
                assert name in p["owned"] and c["kind"] == "block" and idx // {"m": m, "1": 1}[c["stride"]] == it

"""One-process-per-GPU partitioning of the PENCIL nests, over torch.distributed
(NCCL on B200s, gloo for the CPU tests).  The data path per step:

  * CSR SpMV / gemv — row blocks balanced by non-zeros (pencil_shard_rows_by_nnz).  Each rank owns
    rows [r0, r1) of A and the same slice of x; x is gathered into a rank-padded buffer.  Column
    indices are remapped once, at setup, into the padded layout (col -> owner*max_rows + col -
    bounds[owner]) so no unpad copy runs per step.  The step of an iterative method (y = A x,
    y gathered as the next x) runs fused (FusedSpmvAllgather: the SpMV kernel stores its rows
    into every rank's buffer over NVLink / NVLS multicast) or as SpMV + NCCL all-gather.
  * 5x5 stencils — equal row bands; each rank exchanges 2 halo rows with each neighbour
    (send/recv) and runs the stencil on its band extended by the halos.
  * gemv — row blocks, x replicated (all-gathered from its shards when it starts sharded);
    gemv_t — column blocks of the strided view, no collective; dot — ranges + one all-reduce of
    fp64 partials; axpy — ranges, no collective; gemm — the R x C tile grid of
    pencil_shard_gemm_grid on replicated inputs, C tiles all-gathered on request.

The local compute is a callable so the same plumbing is exercised on CPU (gloo + the oracle)
and on GPUs (NCCL + the CUDA kernels).
"""
import ctypes

import numpy as np

from . import _lib


_PLANS = {}


def fixture_plan(fixture, fn, dim=0):
    """The distribution plan of a fixture's nest (views.dist_plan: derived from its index
    expressions and ACCESS summaries, csrc/distplan.cpp) — the shard classes below take their
    halo widths, replicated (all-gathered) arrays and reductions from it."""
    key = (fixture, fn, dim)
    if key not in _PLANS:
        from .views import dist_plan
        _PLANS[key] = dist_plan(fixture, fn)["dims"][dim]
    return _PLANS[key]


def _gloo():
    import torch.distributed as dist
    return dist.get_backend() != "nccl"


def _all_gather_list(out_rows, t):
    """all_gather into the rows of `out_rows` (a list of views).  gloo (CPU tests, one-GPU plumbing
    runs) moves no CUDA memory: device tensors go through host copies."""
    import torch.distributed as dist
    if t.is_cuda and _gloo():
        host = [r.cpu() for r in out_rows]
        dist.all_gather(host, t.cpu())
        for r, h in zip(out_rows, host):
            r.copy_(h)
        return
    dist.all_gather(out_rows, t)


def shard_rows_by_nnz(rowptr, nshards):
    lib = _lib.load()
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int32)
    bounds = np.zeros(nshards + 1, dtype=np.int32)
    st = lib.pencil_shard_rows_by_nnz(rowptr.ctypes.data, rowptr.size - 1, nshards, bounds.ctypes.data)
    if st:
        raise ValueError("pencil_shard_rows_by_nnz failed")
    return bounds


def shard_bands(h, nshards):
    lib = _lib.load()
    bounds = np.zeros(nshards + 1, dtype=np.int32)
    if lib.pencil_shard_bands(h, nshards, bounds.ctypes.data):
        raise ValueError("pencil_shard_bands failed")
    return bounds


def shard_gemm_grid(m, n, nshards):
    lib = _lib.load()
    r, c = ctypes.c_int(), ctypes.c_int()
    if lib.pencil_shard_gemm_grid(m, n, nshards, ctypes.byref(r), ctypes.byref(c)):
        raise ValueError("pencil_shard_gemm_grid failed")
    return r.value, c.value


class RowShardedCsr:
    """Local piece of a row-sharded square CSR matrix plus the x all-gather plumbing.  The plan of
    spmv_vec: y owned in row blocks, col / val sharded through rowptr (a one-row halo), x
    replicated — the arrays `gathered()` lists are all-gathered every step."""

    @staticmethod
    def gathered():
        p = fixture_plan("spmv", "spmv_vec")
        assert p["arrays"]["col"]["kind"] == "via" and p["arrays"]["val"]["kind"] == "via" and p["owned"] == ["y"]
        return p["replicated"]

    def __init__(self, rowptr, col, val, rank, world, bounds=None):
        self.rank, self.world = rank, world
        self.bounds = shard_rows_by_nnz(rowptr, world) if bounds is None else np.asarray(bounds, np.int32)
        r0, r1 = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.r0, self.r1 = r0, r1
        self.max_rows = int(np.max(self.bounds[1:] - self.bounds[:-1]))
        p0, p1 = int(rowptr[r0]), int(rowptr[r1])
        self.rowptr = (rowptr[r0:r1 + 1] - p0).astype(np.int32)
        c = col[p0:p1].astype(np.int64)
        owner = np.searchsorted(self.bounds, c, side="right") - 1
        self.col = (owner * self.max_rows + (c - self.bounds[owner])).astype(np.int32)
        self.val = val[p0:p1]
        self.nrows, self.nnz = r1 - r0, p1 - p0
        self.ncols_padded = self.max_rows * world

    def pad_local_x(self, x_local, like=None):
        """x_local (this rank's rows) into a max_rows buffer for the all-gather."""
        import torch
        buf = torch.zeros(self.max_rows, dtype=torch.float32, device=x_local.device)
        buf[: x_local.numel()] = x_local
        return buf

    def allgather_x(self, x_local_padded, out=None):
        import torch
        import torch.distributed as dist
        if out is None:
            out = torch.empty(self.ncols_padded, dtype=torch.float32, device=x_local_padded.device)
        if dist.get_backend() == "nccl":
            dist.all_gather_into_tensor(out, x_local_padded)
        else:  # gloo (CPU tests): list form
            _all_gather_list(list(out.view(self.world, self.max_rows).unbind(0)), x_local_padded)
        return out


def dist_targets(buffer_ptrs, offset, multicast_ptr, rank, max_rows):
    """Where rank `rank`'s row results go in the fused SpMV -> all-gather step: its slot
    [rank*max_rows, (rank+1)*max_rows) of every rank's gathered-vector buffer (the padded layout
    RowShardedCsr remaps columns into, so the result is the next step's x as is).  Returns
    (peer addresses, multicast address): one multimem store per row when the group has an NVLS
    multicast mapping, else one store per rank's peer mapping."""
    slot = 4 * rank * max_rows + offset
    if multicast_ptr:
        return [], multicast_ptr + slot
    return [int(b) + slot for b in buffer_ptrs], 0


def pingpong_targets(buffer_ptrs, offset, multicast_ptr, rank, max_rows, n):
    """dist_targets for both halves of a ping-pong pair of gathered-vector buffers laid out back
    to back (half h starts 4*h*n bytes after `offset`): [(peers, mc) of half 0, of half 1]."""
    return [dist_targets(buffer_ptrs, offset + 4 * h * n, multicast_ptr, rank, max_rows) for h in (0, 1)]


def step_halves(k):
    """(half the step reads x from, half it stores the gathered y into) for step k."""
    return k & 1, (k + 1) & 1


class FusedSpmvAllgather:
    """Row-sharded SpMV step whose result reaches every rank inside the SpMV kernel
    (pencil_spmv_dev_dist): each warp stores its finished rows to the rank's slot of every
    rank's gathered-vector buffer (torch symmetric memory: NVLink peer mappings, NVLS multicast
    when the switch offers it) while the rest of the matrix is still being multiplied, so the
    exchange overlaps the compute row batch by row batch.  The unfused equivalent is SpMV + NCCL
    all-gather of y (`RowShardedCsr.allgather_x`).

    The gathered vector is double-buffered: step k gathers x from half k & 1 and stores y into
    half (k + 1) & 1 of every rank, so the next step's x never overwrites entries a warp of this
    or another rank is still gathering (one buffer would be read and written by the same
    launch).  Each step is bracketed by symmetric-memory barriers on the stream: the one before
    orders the stores after every rank's last read of the target half (and after the caller's
    writes of x), the one after orders the consumers after every rank's stores.

        fz.load(x_local)                      # this rank's slice of x -> the first half
        for _ in range(iters):
            x = fz.step(plan, rowptr, col, val, None, y)   # returns the half the next step reads
    """

    def __init__(self, shard, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.sh = shard
        n = shard.ncols_padded
        self.mem = symm.empty(2 * n, dtype=torch.float32, device=device)
        self.mem.zero_()
        self.hdl = symm.rendezvous(self.mem, group or dist.group.WORLD)
        self.halves = (self.mem[:n], self.mem[n:])
        mc = int(self.hdl.multicast_ptr or 0)  # 0: no NVLS multicast mapping for this group
        base = int(self.hdl.buffer_ptrs[self.hdl.rank])
        offset = self.mem.data_ptr() - base
        self.targets = pingpong_targets(self.hdl.buffer_ptrs, offset, mc, shard.rank, shard.max_rows, n)
        self.mc = self.targets[0][1]
        self.peers = self.targets[0][0]
        self.k = 0

    def current(self):
        """The gathered x the next step reads (every rank's rows, padded layout)."""
        return self.halves[step_halves(self.k)[0]]

    def load(self, x_local_padded):
        """Gather every rank's x slice (max_rows elements, padded) into the half the next step reads."""
        self.sh.allgather_x(x_local_padded, self.current())
        return self.current()

    def step(self, plan, rowptr, col, val, x, y):
        """y = A_local x for this rank's rows (x = None: the gathered buffer of the previous step /
        load()); every rank's y lands in the other half.  Returns that half — the x of the next
        step — valid on every rank once this returns (stream order)."""
        src, dst = step_halves(self.k)
        xin = self.halves[src] if x is None else x
        d = self.halves[dst]
        lo, hi = d.data_ptr(), d.data_ptr() + 4 * d.numel()
        if lo < xin.data_ptr() + 4 * xin.numel() and xin.data_ptr() < hi:
            raise ValueError("x overlaps the half this step stores into; pass x=None to chain steps")
        peers, mc = self.targets[dst]
        self.hdl.barrier(channel=0)
        plan.spmv_dist(rowptr, col, val, xin, y, peers, mc)
        self.hdl.barrier(channel=0)
        self.k += 1
        return d


class BandShardedImage:
    """Row band of an h x w image with the halo rows a 5x5 stencil needs (2: the plan of
    conv5x5_u8 / conv5x5_f32 reads img in rows i - 2 .. i + 2)."""

    @staticmethod
    def halo_rows():
        h = 0
        for fn in ("conv5x5_u8", "conv5x5_f32"):
            lo, hi = fixture_plan("conv5x5", fn)["arrays"]["img"]["halo"]
            h = max(h, -lo, hi)
        return h

    def __init__(self, h, w, rank, world):
        self.HALO = self.halo_rows()
        self.h, self.w, self.rank, self.world = h, w, rank, world
        b = shard_bands(h, world)
        self.b0, self.b1 = int(b[rank]), int(b[rank + 1])
        self.top = self.HALO if rank > 0 else 0          # halo rows present above the band
        self.bot = self.HALO if rank < world - 1 else 0  # and below
        self.rows = self.b1 - self.b0 + self.top + self.bot

    def exchange_halos(self, ext):
        """ext: (rows, w) tensor = [top halo | own band | bottom halo]; fills the halos from the
        neighbours' edge rows (send own first/last 2 rows, receive theirs)."""
        import torch.distributed as dist
        H, reqs = self.HALO, []
        own0, own1 = self.top, self.top + (self.b1 - self.b0)
        host = ext.is_cuda and _gloo()  # gloo moves host memory only
        mv = (lambda t: t.cpu()) if host else (lambda t: t)  # noqa: E731
        if self.rank > 0:
            reqs.append(dist.isend(mv(ext[own0:own0 + H].contiguous()), self.rank - 1))
            top = mv(ext[0:H].clone())
            reqs.append(dist.irecv(top, self.rank - 1))
        if self.rank < self.world - 1:
            reqs.append(dist.isend(mv(ext[own1 - H:own1].contiguous()), self.rank + 1))
            bot = mv(ext[own1:own1 + H].clone())
            reqs.append(dist.irecv(bot, self.rank + 1))
        for r in reqs:
            r.wait()
        if self.rank > 0:
            ext[0:H] = top
        if self.rank < self.world - 1:
            ext[own1:own1 + H] = bot
        return ext


def band_halo_rows(band_ptrs, rows, rank, w, esize):
    """Device addresses of rows -2, -1 (top) and h, h + 1 (bot) of `rank`'s band, h = rows[rank]:
    band_ptrs[q] is the address of rank q's band (rows[q] rows of w elements of esize bytes).  The
    neighbours' edge rows, or the band's own first / last row at the image's top / bottom
    (clamp-to-edge, the conv5x5_u8 edge rule; the fp32 stencil never reads them)."""
    world = len(rows)
    if world > 1 and min(rows) < 2:
        raise ValueError("every band needs >= 2 rows for a 2-row halo")
    row = lambda q, r: int(band_ptrs[q]) + int(r) * w * esize  # noqa: E731
    h = int(rows[rank])
    top = (row(rank - 1, rows[rank - 1] - 2), row(rank - 1, rows[rank - 1] - 1)) if rank > 0 else (row(rank, 0),) * 2
    bot = (row(rank + 1, 0), row(rank + 1, 1)) if rank < world - 1 else (row(rank, h - 1),) * 2
    return top, bot


def band_interior(h, b0, b1):
    """Band-relative output rows [lo, hi) of the fp32 stencil (image interior rows 2 .. h-3) for
    the band of global rows [b0, b1)."""
    lo = max(0, 2 - b0)
    return lo, max(lo, min(b1, h - 2) - b0)


class FusedBandStencil:
    """Band-sharded 5x5 stencil step with the halo exchange fused into the sweep: every rank's
    band lives in torch symmetric memory and the kernel's ring loader reads the two rows above
    and below the band straight out of the neighbours' buffers over NVLink (cp.async from their
    peer mappings: pencil_conv5x5_*_band_dev), so a step is one launch per rank with no halo
    copy.  A symmetric-memory barrier orders it after every rank's band writes, and one after it
    lets the caller overwrite its band (the next iteration's input).  The unfused equivalent is
    BandShardedImage.exchange_halos + the stencil on a halo-extended buffer."""

    def __init__(self, h, w, rank, world, dtype, device, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        b = shard_bands(h, world)
        self.h, self.w, self.rank, self.world = h, w, rank, world
        self.b0, self.b1 = int(b[rank]), int(b[rank + 1])
        self.rows = [int(b[q + 1] - b[q]) for q in range(world)]
        self.nb = self.rows[rank]
        self.buf = symm.empty(max(self.rows) * w, dtype=dtype, device=device)
        self.hdl = symm.rendezvous(self.buf, group or dist.group.WORLD)
        base = int(self.hdl.buffer_ptrs[self.hdl.rank])
        offset = self.buf.data_ptr() - base
        ptrs = [int(p) + offset for p in self.hdl.buffer_ptrs]
        self.top, self.bot = band_halo_rows(ptrs, self.rows, rank, w, self.buf.element_size())
        self.out_lo, self.out_hi = band_interior(h, self.b0, self.b1)

    def band(self):
        """This rank's band (nb x w, flattened): write the input rows here."""
        return self.buf[: self.nb * self.w]

    def step_u8(self, scale, k, out):
        from . import device
        self.hdl.barrier(channel=0)
        device.conv5x5_u8_band(self.nb, self.w, scale, self.buf, self.top, self.bot, k, out)
        self.hdl.barrier(channel=0)
        return out

    def step_f32(self, k, out):
        from . import device
        self.hdl.barrier(channel=0)
        device.conv5x5_f32_band(self.nb, self.w, self.out_lo, self.out_hi, self.buf, self.top, self.bot, k, out)
        self.hdl.barrier(channel=0)
        return out


# ---------------------------------------------------------------- dense BLAS
def shard_range(n, world, rank, align=4):
    """Contiguous [lo, hi) of n elements for `rank`, interior boundaries multiples of `align`
    (keeps every shard's base 16-byte aligned for the float4 kernels)."""
    units = (n + align - 1) // align
    lo = min(n, (units * rank // world) * align)
    hi = min(n, (units * (rank + 1) // world) * align) if rank < world - 1 else n
    return lo, hi


def allgather_vector(local, n, world, rank, align=4):
    """Replicate a vector whose rank shards are shard_range(n, world, r, align): one all-gather of
    rank-padded pieces, then the padding is dropped.  Returns the full length-n tensor."""
    import torch
    import torch.distributed as dist
    bounds = [shard_range(n, world, r, align) for r in range(world)]
    width = max(hi - lo for lo, hi in bounds)
    pad = torch.zeros(width, dtype=local.dtype, device=local.device)
    pad[: local.numel()] = local
    out = torch.empty(width * world, dtype=local.dtype, device=local.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, pad)
    else:
        _all_gather_list(list(out.view(world, width).unbind(0)), pad)
    parts = out.view(world, width)
    return torch.cat([parts[r, : hi - lo] for r, (lo, hi) in enumerate(bounds)])


class RowShardedGemv:
    """gemv (i PARALLEL over rows): rank owns rows [r0, r1) of A and of y; x is replicated (or
    all-gathered from its shards with `allgather_vector`).  No collective on y: each rank's
    rows are final; `gather_y` assembles them when a caller wants the whole vector.  The row
    partition is an array descriptor (include/pencil_b200.h §10): y's shard spec."""

    @staticmethod
    def gathered():
        return fixture_plan("gemv", "gemv")["replicated"]

    def __init__(self, m, n, rank, world):
        from .views import ArrayDesc
        self.m, self.n, self.rank, self.world = m, n, rank, world
        self.y_desc = ArrayDesc(np.float32, m, [shard_range(m, world, r, align=1)[0] for r in range(world)] + [m])
        self.r0, self.r1 = self.y_desc.shard(rank)[:2]

    def attach(self, device, y_rows):
        """Record this rank's y rows (device memory) in the descriptor."""
        self.y_desc.attach(self.rank, device, y_rows)

    def step(self, local_gemv, alpha, beta, A_rows, x, y_rows):
        """local_gemv(m, n, alpha, beta, A, x, y): the CUDA kernel (pb.device.gemv) or a checker."""
        return local_gemv(self.r1 - self.r0, self.n, alpha, beta, A_rows, x, y_rows)

    def gather_y(self, y_rows):
        return allgather_vector(y_rows, self.m, self.world, self.rank, align=1)


class ColShardedGemvT:
    """gemv_t (VOBLA transposed view, j PARALLEL over columns): rank owns columns [j0, j1); every
    rank reads all m rows of its column block and the replicated x, and writes y[j*incy] for its j
    only.  No collective.  The rank's work is expressed in view descriptors: the fixture's views
    (from the affine forms of A[i*lda + j], x[i*incx], y[j*incy], pencil_gemv_t_views) sliced to
    the column block (pencil_view_slice) — A at offset j0, y at offset j0*incy."""

    @staticmethod
    def gathered():
        p = fixture_plan("gemv_t", "gemv_t")
        assert p["arrays"]["A"]["kind"] == "view" and p["owned"] == ["y"]  # column blocks of the strided view
        return p["replicated"]

    def __init__(self, m, n, rank, world, lda=None, incx=1, incy=1):
        from . import views as V
        self.m, self.n, self.rank, self.world = m, n, rank, world
        self.j0, self.j1 = shard_range(n, world, rank, align=4)
        lda = n if lda is None else lda
        A, x, y = V.gemv_t_views(m, n, lda, incx, incy)
        self.A, self.x, self.y = A.slice(1, self.j0, self.j1), x, y.slice(0, self.j0, self.j1)

    def views(self, A_flat, y_flat, incy=None):
        """(A view, y view) of this rank's column block inside the caller's flat arrays (host
        arrays: the elements from the views' offsets on)."""
        return A_flat[self.A.offset:], y_flat[self.y.offset:]

    def step(self, alpha, beta, A, x, y, stream=None):
        """The rank's columns on the device: A, x, y are the full flat device arrays."""
        from . import views as V
        V.gemv_t_view(alpha, beta, self.A.on(A), self.x.on(x), self.y.on(y), stream)


def dot_allreduce_vars():
    """The reduction variables of dot's loop (its plan): one all-reduce of their partials."""
    return fixture_plan("dot", "dot")["reduce"]


def dot_sharded(local_dot, x_local, y_local):
    """dot (i PARALLEL_WITH_REDUCTION): local partial on this rank's range, then one all-reduce.
    The partials are summed in fp64 (rank order fixed by the collective) and rounded once."""
    import torch
    import torch.distributed as dist
    dev = "cpu" if _gloo() else x_local.device
    part = torch.tensor([float(local_dot(x_local, y_local))], dtype=torch.float64, device=dev)
    dist.all_reduce(part)
    return float(part.item())


class GemmTileGrid:
    """gemm (i, j independent; p reduction kept local): the R x C process grid of
    pencil_shard_gemm_grid; rank (ri, ci) computes the C tile rows [m0, m1) x cols [n0, n1) from
    A's row panel and B's column panel (inputs replicated: no data-path collective; `gather_c`
    assembles C on every rank when asked)."""

    @staticmethod
    def panels_needed():
        """Per operand, the piece a tile needs, from the plans of gemm's i and j dimensions: A is
        sharded along i (row panel) and replicated along j, B the other way (column panel)."""
        pi, pj = fixture_plan("gemm", "gemm", 0), fixture_plan("gemm", "gemm", 1)
        out = {}
        for a in ("A", "B"):
            ki, kj = pi["arrays"][a]["kind"], pj["arrays"][a]["kind"]
            out[a] = "rows" if ki == "block" and kj == "all" else "cols" if ki == "all" and kj == "view" else "all"
        return out

    def __init__(self, m, n, k, rank, world):
        self.m, self.n, self.k, self.rank, self.world = m, n, k, rank, world
        self.R, self.C = shard_gemm_grid(m, n, world)
        self.ri, self.ci = divmod(rank, self.C)
        self.m0, self.m1 = shard_range(m, self.R, self.ri, align=1)
        self.n0, self.n1 = shard_range(n, self.C, self.ci, align=4)

    def panels(self, A, B):
        """(A row panel, B column panel made contiguous) for this rank's tile."""
        Ap = A.reshape(self.m, self.k)[self.m0:self.m1].reshape(-1)
        Bp = B.reshape(self.k, self.n)[:, self.n0:self.n1]
        Bp = Bp.contiguous().reshape(-1) if hasattr(Bp, "contiguous") else Bp.copy().reshape(-1)
        return Ap, Bp

    def step(self, local_gemm, alpha, beta, Ap, Bp, C_tile):
        return local_gemm(self.m1 - self.m0, self.n1 - self.n0, self.k, alpha, beta, Ap, Bp, C_tile)

    def step_views(self, gemm_strided, alpha, beta, A, B, C):
        """The rank's tile on views of the replicated operands (no panel copies): A's row panel
        (rows m0.., pitch k), B's column panel (columns n0.., pitch n) and C's tile (pitch n) —
        the plan's split: A a block along i, B a view along j (views.dist_plan("gemm", "gemm"))."""
        m, n, k = self.m, self.n, self.k
        return gemm_strided(self.m1 - self.m0, self.n1 - self.n0, k, alpha, beta, A[self.m0 * k:], k,
                            B[self.n0:], n, C[self.m0 * n + self.n0:], n)

    def gather_c(self, c_tile):
        """All-gather every rank's tile (padded to the largest) and assemble the m x n matrix."""
        import torch
        import torch.distributed as dist
        tiles = [(shard_range(self.m, self.R, r // self.C, 1), shard_range(self.n, self.C, r % self.C, 4))
                 for r in range(self.world)]
        width = max((a1 - a0) * (b1 - b0) for (a0, a1), (b0, b1) in tiles)
        pad = torch.zeros(width, dtype=c_tile.dtype, device=c_tile.device)
        pad[: c_tile.numel()] = c_tile.reshape(-1)
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        _all_gather_list(parts, pad)
        out = torch.empty(self.m, self.n, dtype=c_tile.dtype, device=c_tile.device)
        for r, ((a0, a1), (b0, b1)) in enumerate(tiles):
            out[a0:a1, b0:b1] = parts[r][: (a1 - a0) * (b1 - b0)].view(a1 - a0, b1 - b0)
        return out

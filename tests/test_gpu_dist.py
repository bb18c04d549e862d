"""The N>1 data path of bench.py on the real stack, at world size 1 (this run has one GPU): NCCL
process group, RowShardedCsr (rank-padded x all-gather + column remap) feeding the CUDA SpMV
through a CsrPlan, the band-sharded stencil with its halo buffers, and the dense shards — each
against the single-process CUDA result.  The multi-rank exchange itself is covered by the gloo
tests (test_dist_cpu.py, world 2 and 4)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl(cuda):
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


def test_row_sharded_spmv_over_nccl(nccl):
    import torch
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200.dist import RowShardedCsr
    rowptr, col, val, x, _ = synth.csr_powerlaw(200000, maxlen=2048, seed=5)
    nrows, nnz = rowptr.size - 1, col.size
    sh = RowShardedCsr(rowptr, col, val, 0, 1)
    rp, cd, vd = (torch.from_numpy(a).cuda() for a in (sh.rowptr, sh.col, sh.val))
    xl = sh.pad_local_x(torch.from_numpy(x[sh.r0:sh.r1]).cuda())
    xg = sh.allgather_x(xl)
    y = torch.empty(sh.nrows, device="cuda")
    plan = pb.device.CsrPlan(sh.nrows, sh.ncols_padded, sh.nnz, rp, mode=0)
    plan.spmv(rp, cd, vd, xg, y)
    pb.device.sync_status()
    ref = torch.empty(nrows, device="cuda")
    rp0 = torch.from_numpy(rowptr).cuda()
    pb.device.CsrPlan(nrows, nrows, nnz, rp0, mode=0).spmv(rp0, torch.from_numpy(col).cuda(),
                                                          torch.from_numpy(val).cuda(), torch.from_numpy(x).cuda(), ref)
    assert torch.equal(y.view(torch.int32), ref.view(torch.int32))


def test_dense_shards_over_nccl(nccl):
    import torch
    import paper_1302_5586_b200 as pb
    from paper_1302_5586_b200 import synth
    from paper_1302_5586_b200 import dist as pd
    n = 4096 + 13
    x = torch.from_numpy(synth.f32(n, 3)).cuda()
    lo, hi = pd.shard_range(n, 1, 0)
    full = pd.allgather_vector(x[lo:hi].contiguous(), n, 1, 0)
    assert torch.equal(full, x)
    r = torch.zeros(1, device="cuda")
    d = pd.dot_sharded(lambda a, b: (pb.device.dot(a.numel(), a, b, r), float(r.item()))[1], x, x)
    pb.device.dot(n, x, x, r)
    assert d == float(r.item())
    m, k, nn = 96, 64, 160
    A, B, C = synth.f32(m * k, 1), synth.f32(k * nn, 2), synth.f32(m * nn, 3)
    tg = pd.GemmTileGrid(m, nn, k, 0, 1)
    Ap, Bp = tg.panels(torch.from_numpy(A), torch.from_numpy(B))
    Ct = torch.from_numpy(C.copy()).cuda()
    tg.step(lambda mm, n2, kk, a, b, AA, BB, CC: pb.device.gemm(mm, n2, kk, a, b, AA, BB, CC), 1.0, 0.5,
            Ap.cuda(), Bp.cuda(), Ct)
    out = tg.gather_c(Ct)
    ref = torch.from_numpy(C.copy()).cuda()
    pb.device.gemm(m, nn, k, 1.0, 0.5, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), ref)
    assert torch.equal(out.reshape(-1), ref)

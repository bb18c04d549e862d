"""Cost of the fused SpMV -> all-gather stores on one GPU (bench workload, 2^24 rows): plain
SpMV vs pencil_spmv_dev_dist with 1 / 7 local target buffers (stand-ins for peer mappings:
same store count, HBM instead of NVLink), and the symmetric-memory step at world 1."""
import os
import socket
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_5586_b200 as pb  # noqa: E402
from paper_1302_5586_b200 import synth  # noqa: E402


def timeit(fn, k=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(k):
        pb.device.l2_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.mean(ts)


def main():
    n = 1 << 24
    rowptr, col, val, x, _ = synth.csr_powerlaw(n)
    rp, cd, vd, xd = (torch.from_numpy(a).cuda() for a in (rowptr, col, val, x))
    y = torch.empty(n, device="cuda")
    plan = pb.device.CsrPlan(n, n, col.size, rp, mode=1)
    print("plain spmv            %.4f ms" % timeit(lambda: plan.spmv(rp, cd, vd, xd, y)))
    bufs = [torch.empty(n, device="cuda") for _ in range(7)]
    for np_ in (1, 7):
        peers = [b.data_ptr() for b in bufs[:np_]]
        print("spmv_dist %d targets   %.4f ms" % (np_, timeit(lambda: plan.spmv_dist(rp, cd, vd, xd, y, peers))))
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(s.getsockname()[1])
    s.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_1302_5586_b200.dist import RowShardedCsr, FusedSpmvAllgather
    sh = RowShardedCsr(rowptr, col, val, 0, 1)
    fz = FusedSpmvAllgather(sh, torch.device("cuda", 0))
    print("symmetric memory: multicast=%s peers=%d" % (bool(fz.mc), len(fz.peers)))
    print("fused step (world 1)  %.4f ms" % timeit(lambda: fz.step(plan, rp, cd, vd, xd, y)))
    yg = torch.empty(n, device="cuda")
    print("spmv + nccl allgather %.4f ms" % timeit(lambda: (plan.spmv(rp, cd, vd, xd, y), sh.allgather_x(y, yg))))
    pb.device.sync_status()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Several processes on ONE GPU running the fused squaring exchange of
apsp_by_squaring_sharded across process boundaries: the D / D_next buffers
are mapped between the processes with CUDA IPC (torch.multiprocessing
tensor sharing — symmetric memory refuses ranks that share a device), gloo
carries the host-side flag all-reduce, and every rank's GEMM stores its rows
into the other processes' D_next through btas_gemm_peers.  No kernel waits on
another process's kernel (the step barrier is the host-side all-reduce), so
sharing one GPU is safe.  Checked against the single-process solve."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def worker(rank, world, n, inboxes, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29573", BTAS_EXCHANGE="peer")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200.apsp import _closure_base
    from paper_1701_04733_b200.graphs import random_graph_matrix
    from paper_1701_04733_b200.sharded import apsp_by_squaring_sharded

    keep = []

    def ipc_buffers(shape, dtype, dev, group, world_):
        bufs = [torch.empty(shape, dtype=dtype, device=dev) for _ in range(2)]
        for q in range(world_):
            if q != rank:
                inboxes[q].put((rank, bufs))
        got = dict(inboxes[rank].get(timeout=120) for _ in range(world_ - 1))
        keep.append(got)  # the mapped peer tensors must outlive the solve
        ptrs = [[got[q][i].data_ptr() for q in range(world_) if q != rank] for i in range(2)]
        torch.cuda.synchronize()
        dist.barrier()
        return bufs, ptrs

    for n_, p, wr, seed in ((n, 0.3, (1, 100), 1234), (700, 0.05, (1, 60), 55), (257, 0.5, (-2, 40), 9)):
        adj = random_graph_matrix(n_, p, wr, seed, dtype=torch.int32)
        res = apsp_by_squaring_sharded(_closure_base(adj).data.contiguous(), integer=True,
                                       peer_buffers=ipc_buffers)
        want = bt.apsp_by_squaring(adj)
        ok = res.multiplications_performed == want.multiplications_performed and \
            res.negative_cycle == want.negative_cycle and \
            (want.negative_cycle or torch.equal(res.distances, want.distances.dist.data))
        results.put((rank, n_, res.exchange, bool(ok), res.multiplications_performed))
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
    ctx = mp.get_context("spawn")
    inboxes = [ctx.Queue() for _ in range(world)]
    results = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, world, n, inboxes, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    out = sorted(results.get(timeout=10) for _ in range(3 * world))
    print(out)
    assert all(ok and ex == "peer" for _, _, ex, ok, _ in out), out
    print(f"{world}-process peer-store exchange OK")

"""floyd_warshall_distributed across real processes: 2-3 processes on ONE GPU,
gloo for the collectives, both panel distributions: the broadcast, and the
fused one where the owner's OWNER-stage kernels store the panels into the other
processes' workspaces (mapped with CUDA IPC).  Every wait is host-mediated,
so no kernel waits on another process's kernel.  Checked against the
single-process solve."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def worker(rank, world, inboxes, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29581")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200.graphs import random_graph_matrix
    from paper_1701_04733_b200.sharded import floyd_warshall_distributed

    keep = []

    def ipc_workspaces(nbytes, dev, group, world_):
        """two workspaces per rank, mapped into every other process (CUDA IPC)"""
        bufs = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
        for q in range(world_):
            if q != rank:
                inboxes[q].put((rank, bufs))
        got = dict(inboxes[rank].get(timeout=120) for _ in range(world_ - 1))
        keep.append(got)
        torch.cuda.synchronize()
        dist.barrier()
        return bufs, [[got[q][i].data_ptr() for q in range(world_) if q != rank] for i in range(2)]

    for fused in (False, True):
        for n, p, wr, seed, dt in ((700, 0.5, (1, 100), 1, torch.int32), (333, 0.05, (0, 60), 2, torch.float32),
                                   (517, 0.3, (-1, 40), 3, torch.int32), (130, 0.4, (1, 9), 4, torch.float64)):
            adj = random_graph_matrix(n, p, wr, seed, dtype=dt)
            got = floyd_warshall_distributed(adj, peer_workspaces=ipc_workspaces if fused else None)
            want = bt.floyd_warshall(adj)
            ok = got.negative_cycle == want.negative_cycle and (want.negative_cycle or got.distances.dist ==
                                                                  want.distances.dist)
            results.put((rank, fused, n, str(dt), bool(ok)))
            dist.barrier()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ctx = mp.get_context("spawn")
    inboxes = [ctx.Queue() for _ in range(world)]
    results = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, world, inboxes, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    out = sorted(results.get(timeout=10) for _ in range(8 * world))
    print(out)
    assert all(ok for *_, ok in out), out
    print(f"{world}-process distributed Floyd-Warshall OK")

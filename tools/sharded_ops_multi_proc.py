"""Several processes on ONE GPU running the row-sharded matmul of
sharded.matmul_sharded with the fused peer-store all-gather across process
boundaries: the output buffer is mapped between the processes with CUDA IPC
(symmetric memory refuses ranks that share a device), gloo carries the
saturation all-reduce that doubles as the barrier.  Also the NCCL-less
matvec_distributed on gloo (host all-gather).  Checked against the
single-process matmul / matvec."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def worker(rank, world, inboxes, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29577", BTAS_EXCHANGE="peer")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np

    import paper_1701_04733_b200 as bt
    from paper_1701_04733_b200.sharded import matmul_sharded

    keep = []

    def ipc_buffers(shape, dtype, dev, group, world_, count=1):
        bufs = [torch.empty(shape, dtype=dtype, device=dev) for _ in range(count)]
        for q in range(world_):
            if q != rank:
                inboxes[q].put((rank, bufs))
        got = dict(inboxes[rank].get(timeout=120) for _ in range(world_ - 1))
        keep.append(got)
        ptrs = [[got[q][i].data_ptr() for q in range(world_) if q != rank] for i in range(count)]
        torch.cuda.synchronize()
        dist.barrier()
        return bufs, ptrs

    rng = np.random.default_rng(77)
    MIN = bt.SemiringKind.MIN_PLUS
    for dtype in (torch.int32, torch.float32, torch.float64):
        for m, k, n in ((1000, 700, 900), (257, 129, 300)):
            xs = rng.integers(-1000, 1000, (m, k)).astype(float)
            ys = rng.integers(-1000, 1000, (k, n)).astype(float)
            xs[rng.random((m, k)) < 0.25] = np.inf
            ys[rng.random((k, n)) < 0.25] = np.inf
            x = bt.TropicalMatrix(MIN, xs, dtype=dtype)
            y = bt.TropicalMatrix(MIN, ys, dtype=dtype)
            out, sat = matmul_sharded(x.data, y.data, MIN, True, peer_buffers=ipc_buffers)
            want = bt.matmul(x, y)
            results.put((rank, str(dtype), m, bool(torch.equal(out, want.data)) and not sat))
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
    out = sorted(results.get(timeout=10) for _ in range(6 * world))
    print(out)
    assert all(ok for *_, ok in out), out
    print(f"{world}-process sharded matmul OK")

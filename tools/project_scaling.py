"""Projected P-GPU scaling of the C4 squaring (n = 65536 f32) from ONE GPU:
times the work of one rank of the row-sharded step — its n/P-row block of
D (x) D with the fused all-gather's peer stores into P-1 other row buffers
(same-GPU buffers here, NVLink on a P-GPU box) and the fixpoint compare — and
compares P x that with the single-GPU product.  A projection, not a
multi-GPU measurement: NVLink store bandwidth (P-1)/P n^2 4 B per step
(~15 GB at P = 8, < 20 ms at 900 GB/s) and the 12-byte flag all-reduce are
not on this device."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix  # noqa: E402
from paper_1701_04733_b200.matrix import _gemm  # noqa: E402
from paper_1701_04733_b200.sharded import partition  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
MIN = bt.SemiringKind.MIN_PLUS
adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.float32)
d = adj.data


def timed(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


out = {"n": n}
full = torch.empty_like(d)
t1 = timed(lambda: _gemm(d, d, MIN, True, out=full, cprev=d))
out["single_gpu_product_ms"] = round(t1, 1)
del full
torch.cuda.empty_cache()
for world in (2, 4, 8):
    chunk, spans = partition(n, world)
    r0, r1 = spans[0]
    rows = torch.empty((r1 - r0, n), dtype=d.dtype, device=d.device)
    peers = [torch.empty((r1 - r0, n), dtype=d.dtype, device=d.device) for _ in range(world - 1)]
    tp = timed(lambda: _gemm(d[r0:r1], d, MIN, True, out=rows, cprev=d[r0:r1], peers=[p.data_ptr() for p in peers]))
    out[f"P{world}"] = {"rank_block_rows": r1 - r0, "rank_step_ms": round(tp, 1),
                        "projected_speedup": round(t1 / tp, 2), "peer_stores": world - 1}
    del rows, peers
    torch.cuda.empty_cache()
print(json.dumps(out))

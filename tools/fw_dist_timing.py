"""Device time of the row-sharded FW stage sequence (virtual ranks run one
after another on one GPU, so the sum equals what P GPUs do in total) vs
btas_fw at the same n: the lookahead groups should keep the distributed
program within ~15 % of the single-GPU one."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix  # noqa: E402
from paper_1701_04733_b200.sharded import floyd_warshall_emulated  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.int32)


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        r = fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, r


t1, want = timed(lambda: bt.floyd_warshall(adj))
print(f"btas_fw n={n}: {t1:.1f} ms", flush=True)
for world in (2, 4, 8):
    for fused in (False, True):
        tp, got = timed(lambda: floyd_warshall_emulated(adj, world, fused=fused))
        same = got.distances.dist == want.distances.dist
        print(f"emulated P={world} fused={fused}: {tp:.1f} ms ({tp / t1:.3f} x btas_fw) identical={same}", flush=True)

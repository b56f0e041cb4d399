"""Floyd-Warshall (blocked) vs repeated squaring (general GEMM loop) at
mid sizes, non-negative integer weights (where both give the same bytes):
the crossover for floyd_warshall's squaring shortcut."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["BTAS_APSP_SMALL_MAX_N"] = "1024"
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200.graphs import random_graph_matrix  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        r = fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, r


for n in (1100, 1536, 2048, 3072, 4096, 6144):
    for p in (0.5, 0.05, 0.005):
        for dt in (torch.int32, torch.float32):
            adj = random_graph_matrix(n, p, (1, 100), n + int(p * 1000), dtype=dt)
            tf, fw = timed(lambda: bt.floyd_warshall(adj))
            ts, sq = timed(lambda: bt.apsp_by_squaring(adj))
            same = fw.distances.dist == sq.distances.dist
            print(f"n={n} p={p} {str(dt)[6:]}: fw {tf:.3f} ms  squaring {ts:.3f} ms ({sq.multiplications_performed} "
                  f"products)  same={same}", flush=True)

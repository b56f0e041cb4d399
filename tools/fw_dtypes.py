"""FW and squaring time per storage dtype (the reference API's default is float64)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
for dt in (torch.int32, torch.float32, torch.float64):
    adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=dt)
    for name, fn in (("fw", bt.floyd_warshall), ("squaring", bt.apsp_by_squaring)):
        fn(adj)
        torch.cuda.synchronize()
        t = time.perf_counter()
        rep = fn(adj)
        torch.cuda.synchronize()
        s = time.perf_counter() - t
        print(f"{str(dt):14s} {name:9s} n={n}: {s*1e3:9.1f} ms  mults={rep.multiplications_performed}", flush=True)

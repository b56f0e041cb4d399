"""C1 (n = 512 squaring) solves for an ncu launch list: host time per solve
vs the kernels it launches."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.float32)
for _ in range(3):
    bt.apsp_by_squaring(adj)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(reps):
    rep = bt.apsp_by_squaring(adj)
torch.cuda.synchronize()
print(f"n={n}: {(time.perf_counter() - t) / reps * 1e3:.3f} ms per solve (host wall), mults={rep.multiplications_performed}")

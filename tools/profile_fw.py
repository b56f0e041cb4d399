"""One blocked Floyd-Warshall solve (int32, p=0.5, weights 1..100) for ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200.graphs import random_graph_matrix  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
adj = random_graph_matrix(n, 0.5, (1, 100), 1, dtype=torch.int32)
rep = bt.floyd_warshall(adj)
torch.cuda.synchronize()
print("ok", rep.negative_cycle)

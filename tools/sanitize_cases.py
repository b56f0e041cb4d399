"""Small cases of the round-2 kernels for compute-sanitizer memcheck:
fused verifier (both GEMM verify modes + base pass), predecessor product
(packed-key and compare-and-select kernels), bounded / screened matvec,
lookahead-group distributed FW (virtual ranks, both distributions), f64
ternary GEMM, ragged shapes everywhere."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200.graphs import random_graph_matrix  # noqa: E402
from paper_1701_04733_b200.sharded import floyd_warshall_emulated  # noqa: E402

MIN, MAX = bt.SemiringKind.MIN_PLUS, bt.SemiringKind.MAX_PLUS
rng = np.random.default_rng(1)
for dtype in (torch.int32, torch.float32, torch.float64):
    for n in (1, 37, 301):
        adj = random_graph_matrix(n, 0.3, (1, 40), n, dtype=dtype)
        rep = bt.floyd_warshall(adj)
        assert bt.find_apsp_violation(adj, rep.distances) is None
        bad = rep.distances.dist.data.clone()
        bad[n // 2, n // 2] = 1
        assert bt.find_apsp_violation(adj, bt.DistanceMatrix(n, bt.TropicalMatrix._wrap(MIN, bad, True))) is not None
        p = bt.predecessors(adj, rep)
        big = random_graph_matrix(n, 0.3, (5000, 9000), n, dtype=dtype)  # compare-and-select kernel
        bt.predecessors(big)
        if n > 1:
            for world in (2, 3):
                got = floyd_warshall_emulated(adj, world, fused=world == 3)
                assert got.distances.dist == rep.distances.dist
    a = rng.integers(-100, 100, (333, 1024)).astype(float)
    a[rng.random(a.shape) < 0.2] = math.inf
    A = bt.TropicalMatrix(MAX, a, dtype=dtype)
    for b in (1, 3, 7):
        V = bt.TropicalMatrix(MAX, rng.integers(-100, 100, (b, 1024)).astype(float), dtype=dtype)
        assert torch.equal(bt.matvec_batched(A, V), bt.matvec_batched(A, V.data))
x = bt.TropicalMatrix(MIN, rng.uniform(-5, 5, (129, 77)))
y = bt.TropicalMatrix(MIN, rng.uniform(-5, 5, (77, 200)))
bt.matmul(x, y)
torch.cuda.synchronize()
print("sanitize cases ok")

"""Short driver for ncu captures of the round-2 kernels (one mode per run):
  verify   n=16384 squaring solve, then find_apsp_violation (btas_verify_base
           + two btas_gemm_verify products, EPI = kEpiCmp|kEpiVerify = 10)
  argmin   n=16384 Floyd-Warshall, then predecessors (MixArg kernel)
  matvec8  n=65536 max-plus f32, 8 vectors with known bounds (screen-free
           matvec_wide_kernel), 5 calls
"""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix  # noqa: E402

mode = sys.argv[1]
dev = torch.device("cuda", 0)
if mode == "verify":
    n = 16384
    adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.float32)
    dm = bt.apsp_by_squaring(adj).distances
    assert bt.find_apsp_violation(adj, dm) is None
elif mode == "argmin":
    n = 16384
    adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.int32)
    rep = bt.floyd_warshall(adj)
    p = bt.predecessors(adj, rep)
    assert int((p < 0).sum()) == n
elif mode == "matvec8":
    n = 65536
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    MAX = bt.SemiringKind.MAX_PLUS

    def make(r, c):
        s = torch.randint(-1000, 1001, (r, c), generator=g, device=dev, dtype=torch.int32).to(torch.float32)
        s[torch.rand((r, c), generator=g, device=dev) < 0.1] = math.inf
        return bt.TropicalMatrix(MAX, s, dtype=torch.float32, device=dev)

    A, V = make(n, n), make(8, n)
    for _ in range(5):
        bt.matvec_batched(A, V)
torch.cuda.synchronize()
print(f"{mode} ok")

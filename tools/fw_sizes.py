"""Blocked FW device time across sizes (int32, p = 0.5, weights 1..100;
the squaring shortcut disabled so the blocked program runs)."""
import os
import sys
from pathlib import Path

import torch

os.environ["BTAS_FW_SQUARING_MAX_N"] = "0"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix  # noqa: E402

for n in [int(v) for v in (sys.argv[1:] or ["2048", "4096", "8192", "16384", "32768"])]:
    adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.int32)
    bt.floyd_warshall(adj)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3 if n >= 16384 else 10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        bt.floyd_warshall(adj)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"FW n={n}: {min(ts):.3f} ms (min of {len(ts)}), {float(n) ** 3 / (min(ts) * 1e-3) / 1e12:.2f} T/s", flush=True)

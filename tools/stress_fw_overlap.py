"""The overlapped phase-1 FW schedule at its real threshold (n = 16384, 128
pivot blocks) on random instances across weight ranges that keep the s16x2
gate on, flip it inside groups, or keep it off: FW bytes == squaring bytes
and == the serial schedule (BTAS_FW_OVERLAP_P1_MIN_BLOCKS very large)."""
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200.graphs import random_graph_matrix  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
t0 = time.time()
cases = bad = 0
for seed in range(4):
    for p, wr in ((0.3, (1, 100)), (0.02, (1, 3000)), (0.02, (1, 6000)), (0.01, (1, 40000))):
        for dtype in (torch.int32, torch.float32):
            adj = random_graph_matrix(n, p, wr, 9000 + seed, dtype=dtype)
            os.environ.pop("BTAS_FW_OVERLAP_P1_MIN_BLOCKS", None)
            fw = bt.floyd_warshall(adj)
            os.environ["BTAS_FW_OVERLAP_P1_MIN_BLOCKS"] = "1000000000"
            serial = bt.floyd_warshall(adj)
            os.environ.pop("BTAS_FW_OVERLAP_P1_MIN_BLOCKS", None)
            sq = bt.apsp_by_squaring(adj)
            ok = fw.distances.dist == serial.distances.dist == sq.distances.dist and not fw.negative_cycle
            cases += 1
            bad += 0 if ok else 1
            if not ok:
                print("MISMATCH", seed, p, wr, dtype, flush=True)
print(f"fw overlap stress n={n}: {cases} cases, {bad} mismatches in {time.time() - t0:.0f} s")

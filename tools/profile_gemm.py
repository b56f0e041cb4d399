"""One GEMM per kernel path at the bench size, for ncu captures.

python tools/profile_gemm.py [n]  ->  s16x2 (i32 in [-1000,1000]),
fast32 VIADDMNMX (i32 in [-1e6,1e6]), fast32 FADD2+FMNMX3 (real f32).
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1701_04733_b200 as bt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dev = torch.device("cuda", 0)
for dtype, real, lo in ((torch.int32, False, 1000), (torch.int32, False, 10**6), (torch.float32, True, 1000)):
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    mats = []
    for _ in range(2):
        if real:
            sym = torch.rand((n, n), generator=g, device=dev) * 2000 - 1000
        else:
            sym = torch.randint(-lo, lo + 1, (n, n), generator=g, device=dev, dtype=torch.int32).float()
        sym[torch.rand((n, n), generator=g, device=dev) < 0.25] = float("inf")
        mats.append(bt.TropicalMatrix(bt.SemiringKind.MIN_PLUS, sym, dtype=dtype, device=dev))
    bt.matmul(mats[0], mats[1])
    torch.cuda.synchronize()
    del mats
print("ok")

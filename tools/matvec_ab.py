"""A/B of the matvec kernels with and without the overflow screen (one
process, alternating, CUDA events): n = 65536 max-plus f32, B = 1..8."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(5)
MAX = bt.SemiringKind.MAX_PLUS


def make(r, c):
    s = torch.randint(-1000, 1001, (r, c), generator=g, device=dev, dtype=torch.int32).to(torch.float32)
    s[torch.rand((r, c), generator=g, device=dev) < 0.1] = math.inf
    return bt.TropicalMatrix(MAX, s, dtype=torch.float32, device=dev)


A = make(n, n)
for B in (1, 2, 3, 4, 5, 6, 8):
    V = make(B, n)
    res = {}
    for name, fn in (("screen", lambda: bt.matvec_batched(A, V.data)), ("free", lambda: bt.matvec_batched(A, V))):
        for _ in range(3):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(40):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 40
        res[name] = (n * n + 2 * B * n) * 4 / (ms * 1e-3) / 1e9
    print(f"B={B} screen {res['screen']:.0f} GB/s  free {res['free']:.0f} GB/s", flush=True)

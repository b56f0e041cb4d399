"""Min-plus products at the Floyd-Warshall bulk-pass shape (M = N = n,
short K, accumulate in place) against the plain product, kernel time by CUDA
events: how much of the bulk pass's gap to the C2 kernel is per-tile
overhead (short K) and how much the accumulate epilogue.

usage: python tools/gemm_k_sweep.py [n] [K,K,...] [reps] [plain,acc,cmp]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200 import _lib  # noqa: E402
from paper_1701_04733_b200.matrix import _gemm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
ks = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1024,2048,4096").split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
modes = (sys.argv[4] if len(sys.argv) > 4 else "plain,acc").split(",")
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(3)
MIN = bt.SemiringKind.MIN_PLUS
p = _lib.probe_ceiling(2)
peak = p["pairs_per_clk_sm"] * torch.cuda.get_device_properties(0).multi_processor_count * 1965e6 / 1e12
c = torch.randint(0, 2000, (n, n), generator=g, device=dev, dtype=torch.int32)
for K in ks:
    a = torch.randint(1, 100, (n, K), generator=g, device=dev, dtype=torch.int32)
    b = torch.randint(1, 100, (K, n), generator=g, device=dev, dtype=torch.int32)
    for mode in modes:
        out = c.clone() if mode == "acc" else torch.empty_like(c)
        z = out if mode == "acc" else None
        cp = c if mode == "cmp" else None
        _gemm(a, b, MIN, True, out=out, z=z, cprev=cp)
        torch.cuda.synchronize()
        _lib.gemm_timing(True)
        for _ in range(reps):
            _gemm(a, b, MIN, True, out=out, z=z, cprev=cp)
        torch.cuda.synchronize()
        kms, kc = _lib.gemm_timing_read()
        _lib.gemm_timing(False)
        per = kms / reps
        tps = float(n) * n * K / (per * 1e-3) / 1e12
        print(f"n={n} K={K} {mode:5s}: kernel {per:.3f} ms = {tps:.2f} T/s ({tps / peak:.3f} of {peak:.2f})",
              flush=True)

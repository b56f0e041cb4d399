"""Developer probe: PCIe copy rates alone and concurrent with the GEMM."""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench, paper_1701_04733_b200 as bt  # noqa: E401

n = 16384
dev = torch.device("cuda", 0)
x, xs = bench.gemm_inputs(n, torch.int32, dev, 1)
y, ys = bench.gemm_inputs(n, torch.int32, dev, 2)
hx = xs.cpu().pin_memory()
hout = torch.empty((n, n), dtype=torch.int32).pin_memory()
dbuf = torch.empty((n, n), dtype=torch.float32, device=dev)
def t(f, k=3):
    f(); torch.cuda.synchronize(); s = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - s) / k * 1e3
print("h2d 1GiB ms", t(lambda: dbuf.copy_(hx, non_blocking=True)))
print("d2h 1GiB ms", t(lambda: hout.copy_(x.data, non_blocking=True)))
print("gemm ms", t(lambda: bt.matmul(x, y)))
print("TropicalMatrix(host) ms", t(lambda: bt.TropicalMatrix(bt.SemiringKind.MIN_PLUS, hx, dtype=torch.int32, device=dev)))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1):
        bt.matmul(x, y)
    with torch.cuda.stream(s2):
        for _ in range(4):
            dbuf.copy_(hx, non_blocking=True)
            hout.copy_(x.data, non_blocking=True)
print("gemm || 4x(h2d+d2h) ms", t(both))

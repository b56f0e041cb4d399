"""Developer probe: per-stream event timeline of bench.e2e_gemm's pipeline."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1701_04733_b200 as bt  # noqa: E402

n = 16384
dev = torch.device("cuda", 0)
x, xs = bench.gemm_inputs(n, torch.int32, dev, 1)
y, ys = bench.gemm_inputs(n, torch.int32, dev, 2)
hx, hy = xs.cpu().pin_memory(), ys.cpu().pin_memory()
hout = [torch.empty((n, n), dtype=torch.int32).pin_memory() for _ in range(2)]
MIN = bt.SemiringKind.MIN_PLUS
s_in, s_comp, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run(k, log):
    t0 = ev()
    t0.record()
    marks = []
    host = []
    for i in range(k):
        h0 = time.perf_counter()
        with torch.cuda.stream(s_in):
            a = ev(); a.record()
            dx = hx.to(dev, non_blocking=True)
            dy = hy.to(dev, non_blocking=True)
            b = ev(); b.record()
            X = bt.TropicalMatrix(MIN, dx, dtype=torch.int32, device=dev)
            Y = bt.TropicalMatrix(MIN, dy, dtype=torch.int32, device=dev)
            c = ev(); c.record()
        h1 = time.perf_counter()
        s_comp.wait_stream(s_in)
        with torch.cuda.stream(s_comp):
            X.data.record_stream(s_comp); Y.data.record_stream(s_comp)
            d = ev(); d.record()
            Z = bt.matmul(X, Y)
            e = ev(); e.record()
        s_out.wait_stream(s_comp)
        with torch.cuda.stream(s_out):
            Z.data.record_stream(s_out)
            f = ev(); f.record()
            hout[i % 2].copy_(Z.data, non_blocking=True)
            g = ev(); g.record()
        host.append((h1 - h0) * 1e3)
        marks.append((a, b, c, d, e, f, g))
    torch.cuda.synchronize()
    if log:
        for i, m in enumerate(marks):
            ts = [t0.elapsed_time(x) for x in m]
            print(f"step {i}: h2d {ts[0]:8.1f}-{ts[1]:8.1f}  ingest -{ts[2]:8.1f}  gemm {ts[3]:8.1f}-{ts[4]:8.1f}"
                  f"  d2h {ts[5]:8.1f}-{ts[6]:8.1f}  host_in {host[i]:6.1f} ms")


run(2, False)
s = time.perf_counter()
run(8, True)
print("ms/step", (time.perf_counter() - s) / 8 * 1e3)

"""One n = 65536 min-plus product (the C4 squaring step, s16x2 path) timed
with CUDA events: kernel efficiency at the largest size."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200 import _lib  # noqa: E402
from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix  # noqa: E402
from paper_1701_04733_b200.matrix import _gemm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.float32)
d = adj.data
out = torch.empty_like(d)
_gemm(d, d, bt.SemiringKind.MIN_PLUS, True, out=out, cprev=d)
torch.cuda.synchronize()
_lib.gemm_timing(True)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
_gemm(d, d, bt.SemiringKind.MIN_PLUS, True, out=out, cprev=d)
e.record()
torch.cuda.synchronize()
kms, kc = _lib.gemm_timing_read()
_lib.gemm_timing(False)
p = _lib.probe_ceiling(2)
peak = p["pairs_per_clk_sm"] * torch.cuda.get_device_properties(0).multi_processor_count * 1965e6 / 1e12
print(f"n={n}: step {s.elapsed_time(e):.1f} ms, kernel {kms:.1f} ms = {float(n) ** 3 / (kms * 1e-3) / 1e12:.2f} T/s "
      f"({float(n) ** 3 / (kms * 1e-3) / 1e12 / peak:.3f} of {peak:.2f})")

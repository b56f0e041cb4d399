"""One-rank run of the row-sharded squaring at full size through the
symmetric-memory (peer-store) exchange: memory fit, timing and the distance
checksum of bench.py's apsp_c4 (identical for every rank count)."""
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix  # noqa: E402
from paper_1701_04733_b200.sharded import apsp_by_squaring_distributed  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
os.environ.setdefault("BTAS_EXCHANGE", "peer")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.float32, device=dev)
torch.cuda.synchronize()
t = time.perf_counter()
rep = apsp_by_squaring_distributed(adj)
torch.cuda.synchronize()
secs = time.perf_counter() - t
d = rep.distances.dist.data
checksum = 0
for r0 in range(0, n, 4096):
    blk = d[r0:r0 + 4096]
    blk = torch.where(torch.isfinite(blk), blk, torch.full_like(blk, -1)).to(torch.int64)
    checksum = (checksum + int(blk.sum().item())) % (1 << 61)
print(f"n={n} exchange={os.environ['BTAS_EXCHANGE']} secs={secs:.2f} mults={rep.multiplications_performed} "
      f"negative={rep.negative_cycle} checksum={checksum} max_mem_GB={torch.cuda.max_memory_allocated() / 1e9:.1f}")
dist.destroy_process_group()

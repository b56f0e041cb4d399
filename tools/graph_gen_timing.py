"""Time the on-device instance generator against the host restatement."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix, random_graph_matrix_host

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
host_n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
for dt in (torch.float32, torch.int32):
    random_graph_matrix(1024, 0.5, (1, 100), 1, dtype=dt)
    torch.cuda.synchronize()
    t = time.perf_counter()
    m = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=dt)
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t
    t = time.perf_counter()
    h = random_graph_matrix_host(host_n, 0.5, (1, 100), instance_seed(1, host_n), dtype=dt)
    torch.cuda.synchronize()
    host_s = time.perf_counter() - t
    print(f"{dt} device n={n}: {dev_s*1e3:.1f} ms ({n*n/dev_s/1e9:.1f} G entries/s); "
          f"host n={host_n}: {host_s*1e3:.1f} ms ({host_n*host_n/host_s/1e9:.3f} G entries/s)", flush=True)

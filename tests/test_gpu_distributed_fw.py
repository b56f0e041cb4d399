"""Row-sharded Floyd-Warshall (lookahead groups, btas_fw_dist_group).

Only one GPU is available to this build, so P > 1 runs as virtual ranks
executed in sequence on one device (the broadcast becomes a device copy) —
the exact per-rank stage sequence and slab indexing of the multi-GPU path —
and the NCCL path itself runs with a one-rank process group.  Every result
must be byte-identical to the single-GPU solve (and therefore to the
reference)."""

import math

import numpy as np
import pytest
import torch

import paper_1701_04733_b200 as bt
from paper_1701_04733_b200.graphs import random_graph_matrix
from paper_1701_04733_b200.sharded import floyd_warshall_distributed, floyd_warshall_emulated

from gpu_helpers import DTYPES, MIN

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("fused", [False, True])
def test_emulated_ranks_match_single_gpu(cuda, dtype, world, fused):
    """fused=True: the owner's OWNER-stage kernels store the panels straight into the
    other virtual ranks' double-buffered workspaces (btas_fw_dist_group_peers)."""
    for n, p, wr, seed in ((700, 0.5, (1, 100), 1), (333, 0.05, (0, 60), 2), (130, 0.4, (-1, 40), 3), (1, 0.5, (1, 2), 4)):
        adj = random_graph_matrix(n, p, wr, seed, dtype=dtype)
        want = bt.floyd_warshall(adj)
        got = floyd_warshall_emulated(adj, world, fused=fused)
        assert got.negative_cycle == want.negative_cycle
        if not want.negative_cycle:
            assert got.distances.dist == want.distances.dist, (n, world)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_emulated_groups_larger_graphs(cuda, world):
    """Slabs of many pivot blocks: full lookahead groups of 8 plus ragged
    tails inside each slab (n = 2500 and 8192), both distributions."""
    for n, dtype in ((2500, torch.int32), (8192, torch.int32), (2500, torch.float32)):
        adj = random_graph_matrix(n, 0.5, (1, 100), 77 + n, dtype=dtype)
        want = bt.floyd_warshall(adj)
        for fused in (False, True):
            got = floyd_warshall_emulated(adj, world, fused=fused)
            assert got.distances.dist == want.distances.dist and not got.negative_cycle, (n, world, fused)


def test_emulated_negative_cycles_and_masked(cuda, golden):
    g = golden("negcycle.npz")
    for case in range(0, 200, 9):
        sym = np.asarray(g[f"adj{case}"], dtype=np.float64)
        sym[np.isinf(sym)] = math.inf
        adj = bt.TropicalMatrix(MIN, sym, dtype=torch.int32)
        assert floyd_warshall_emulated(adj, 2).negative_cycle == bool(g["meta"][case][1])
        assert floyd_warshall_emulated(adj, 3, fused=True).negative_cycle == bool(g["meta"][case][1])
    rng = np.random.default_rng(8)
    n = 300
    sym = rng.integers(1, 10**7, (n, n)).astype(float)
    sym[rng.random((n, n)) < 0.6] = math.inf
    np.fill_diagonal(sym, 0)
    adj = bt.TropicalMatrix(MIN, sym, dtype=torch.int32)
    bt.reset_saturation()
    want = bt.floyd_warshall(adj)
    sat = bt.saturation_seen()
    bt.reset_saturation()
    got = floyd_warshall_emulated(adj, 3)
    assert got.distances.dist == want.distances.dist and bt.saturation_seen() == sat


def test_nccl_single_rank(cuda):
    import torch.distributed as dist

    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1, device_id=cuda)
        created = True
    try:
        for dtype in DTYPES:
            adj = random_graph_matrix(517, 0.3, (1, 100), 9, dtype=dtype)
            want = bt.floyd_warshall(adj)
            got = floyd_warshall_distributed(adj)
            assert got.distances.dist == want.distances.dist and got.negative_cycle == want.negative_cycle
    finally:
        if created:
            dist.destroy_process_group()


def test_distributed_fw_across_processes(cuda):
    """floyd_warshall_distributed with 2 real processes on this GPU (gloo
    carries the pivot-panel broadcast and reductions): identical to the
    single-process solve (tools/fw_multi_proc.py)."""
    import subprocess
    import sys
    from pathlib import Path

    tool = Path(__file__).resolve().parent.parent / "tools" / "fw_multi_proc.py"
    res = subprocess.run([sys.executable, str(tool), "2"], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "2-process distributed Floyd-Warshall OK" in res.stdout

"""The multi-GPU programs pinned to the REFERENCE, not to the single-GPU
solve: the row-sharded Floyd-Warshall (NCCL-broadcast and fused peer-store
panel distributions) and the row-sharded squaring with the all-gather fused
into the GEMM epilogue, run as P virtual ranks on one GPU (the exact per-rank
stage sequence, slab indexing and peer addresses of the multi-GPU path), are
compared byte for byte with the reference's own outputs (tests/golden, made
by the real btas package: apsp.py:93-178) — distances, multiplication counts
and negative-cycle flags — for P in {2, 3, 8}."""

import numpy as np
import pytest
import torch

import paper_1701_04733_b200 as bt
from paper_1701_04733_b200.graphs import dense_rows
from paper_1701_04733_b200.sharded import apsp_by_squaring_emulated, floyd_warshall_emulated

from gpu_helpers import DTYPES, MIN, f64bytes, symbolic

pytestmark = pytest.mark.gpu

WORLDS = (2, 3, 8)


def _np(t):
    return bt.TropicalMatrix._wrap(MIN, t, True).to_numpy()


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("world", WORLDS)
def test_sharded_programs_match_reference_apsp_goldens(cuda, golden, dtype, world):
    """test_acceptance.py:155-175's 700 digraphs (every 4th for the 4-byte
    storages): both FW distributions and the fused squaring equal the
    reference bytes and counts on every virtual rank."""
    g = golden("apsp_small.npz")
    meta = g["meta"]
    step = 1 if dtype == torch.float64 else 4
    for case in range(0, len(meta), step):
        adj = bt.TropicalMatrix(MIN, symbolic(g[f"adj{case}"]), dtype=dtype)
        for fused in (False, True):
            fw = floyd_warshall_emulated(adj, world, fused=fused)
            assert fw.negative_cycle == bool(meta[case][2]), (case, fused)
            if not fw.negative_cycle:
                assert fw.distances.dist.to_numpy().tobytes() == f64bytes(g[f"fw{case}"]), (case, fused)
        rep, per_rank = apsp_by_squaring_emulated(adj, world)
        assert rep.negative_cycle == bool(meta[case][3]), case
        assert rep.multiplications_performed == meta[case][1], case
        if not rep.negative_cycle:
            for d in per_rank:
                assert _np(d).tobytes() == f64bytes(g[f"sq{case}"]), case


@pytest.mark.parametrize("world", WORLDS)
def test_sharded_programs_match_reference_negative_cycles(cuda, golden, world):
    """test_acceptance.py:178-193 (weights in [-3, 10]): the flags of the
    reference; distances wherever it has no negative cycle."""
    g = golden("negcycle.npz")
    meta = g["meta"]
    for case in range(0, len(meta), 2):
        sym = symbolic(g[f"adj{case}"])
        for dtype in (torch.float64, torch.int32):
            adj = bt.TropicalMatrix(MIN, sym, dtype=dtype)
            fw = floyd_warshall_emulated(adj, world, fused=bool(case % 4))
            rep, per_rank = apsp_by_squaring_emulated(adj, world)
            # meta: (n, fw negative, squaring negative, multiplications)
            assert fw.negative_cycle == bool(meta[case][1]), case
            assert rep.negative_cycle == bool(meta[case][2]), case
            if not fw.negative_cycle:
                assert fw.distances.dist.to_numpy().tobytes() == f64bytes(g[f"fw{case}"]), case
                assert rep.multiplications_performed == meta[case][3], case
                for d in per_rank:
                    assert _np(d).tobytes() == f64bytes(g[f"sq{case}"]), case


@pytest.mark.parametrize("world", WORLDS)
def test_sharded_programs_match_reference_c1(cuda, golden, world):
    """Config C1 (n = 512, the reference's own full solve): bytes and the
    reference's multiplication count on every virtual rank; FW digest."""
    import hashlib

    g = golden("c1_apsp512.npz")
    sym = np.concatenate([b for _, b in dense_rows(512, 0.5, (1, 100), int(g["seed"][0]))])
    for dtype in (torch.float32, torch.int32, torch.float64):
        adj = bt.TropicalMatrix(MIN, sym, dtype=dtype)
        rep, per_rank = apsp_by_squaring_emulated(adj, world)
        assert rep.multiplications_performed == int(g["meta"][0]) and not rep.negative_cycle
        for d in per_rank:
            assert _np(d).tobytes() == f64bytes(g["sq"])
        for fused in (False, True):
            fw = floyd_warshall_emulated(adj, world, fused=fused)
            dig = hashlib.sha256(np.ascontiguousarray(fw.distances.dist.to_numpy()).tobytes()).hexdigest()
            assert dig == str(g["fw_digest"][0]) and not fw.negative_cycle

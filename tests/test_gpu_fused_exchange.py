"""GEMM with peer stores (btas_gemm_peers) — the fused all-gather of the
row-sharded squaring.

Only one GPU is available to this build, so the "peers" are other buffers on
the same device: every peer must receive exactly the bytes the local output
receives, for every dtype, both epilogue variants and ragged shapes.  The
whole fused squaring loop then runs as virtual ranks on one GPU
(apsp_by_squaring_emulated), with the same peer addresses the multi-GPU path
computes from the symmetric-memory mapping, and must equal the single-GPU
result (and so the reference) byte for byte on every virtual rank."""

import ctypes

import numpy as np
import pytest
import torch

import paper_1701_04733_b200 as bt
from paper_1701_04733_b200 import _lib
from paper_1701_04733_b200.graphs import random_graph_matrix
from paper_1701_04733_b200.matrix import _gemm
from paper_1701_04733_b200.sharded import apsp_by_squaring_emulated

from gpu_helpers import DTYPES, MAX, MIN, rand_sym

pytestmark = pytest.mark.gpu


def _mats(rng, kind, dtype, m, n, k, integer):
    a = bt.TropicalMatrix(kind, rand_sym(rng, m, k, integer=integer), dtype=dtype)
    b = bt.TropicalMatrix(kind, rand_sym(rng, k, n, integer=integer), dtype=dtype)
    return a, b


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("kind", [MIN, MAX])
@pytest.mark.parametrize("shape", [(128, 256, 128), (300, 190, 77), (1, 1, 1), (129, 517, 260)])
def test_peer_stores_equal_local_output(cuda, dtype, kind, shape):
    m, n, k = shape
    rng = np.random.default_rng(m * 7 + n + k)
    a, b = _mats(rng, kind, dtype, m, n, k, integer=True)
    want, wflags = _gemm(a.data, b.data, kind, a.integer)
    for n_peers in (1, 3, 7):
        out = torch.full_like(want, 7)
        peers = [torch.full((m, n), 5, dtype=want.dtype, device=want.device) for _ in range(n_peers)]
        got, flags = _gemm(a.data, b.data, kind, a.integer, out=out, peers=[p.data_ptr() for p in peers])
        assert torch.equal(got, want)
        for p in peers:
            assert torch.equal(p, want)
        assert int(flags[_lib.FLAG_SATURATED]) == int(wflags[_lib.FLAG_SATURATED])


@pytest.mark.parametrize("dtype", DTYPES)
def test_peer_stores_with_fixpoint_compare(cuda, dtype):
    """kEpiCmp|kEpiPeers: the changed flag must match the plain compare path."""
    rng = np.random.default_rng(3)
    n = 260
    sym = rand_sym(rng, n, n, lo=0, hi=50, p_inf=0.5)
    np.fill_diagonal(sym, 0)
    d = bt.TropicalMatrix(MIN, sym, dtype=dtype)
    # d ⊗ d changes d; the closure does not change
    closed = bt.apsp_by_squaring(d).distances.dist
    for mat, changed in ((d, 1), (closed, 0)):
        x = mat.data
        want, wf = _gemm(x, x, MIN, mat.integer, cprev=x)
        peer = torch.empty_like(want)
        got, f = _gemm(x, x, MIN, mat.integer, cprev=x, out=torch.empty_like(want), peers=[peer.data_ptr()])
        assert torch.equal(got, want) and torch.equal(peer, want)
        assert int(f[_lib.FLAG_CHANGED]) == int(wf[_lib.FLAG_CHANGED]) == changed


def test_peer_store_strided_rows(cuda):
    """Peers share the output's leading dimension: a row window of a taller
    buffer (the sharded layout) is written in place, the rest untouched."""
    rng = np.random.default_rng(5)
    a, b = _mats(rng, MIN, torch.int32, 256, 300, 200, True)
    want, _ = _gemm(a.data, b.data, MIN, True)
    big = torch.full((1024, 300), -3, dtype=torch.int32, device=want.device)
    local = torch.full((1024, 300), -4, dtype=torch.int32, device=want.device)
    r0 = 384
    _gemm(a.data, b.data, MIN, True, out=local[r0:r0 + 256], peers=[big.data_ptr() + r0 * 300 * 4])
    assert torch.equal(big[r0:r0 + 256], want) and torch.equal(local[r0:r0 + 256], want)
    assert bool((big[:r0] == -3).all()) and bool((big[r0 + 256:] == -3).all())


def test_peer_count_limit_and_accumulate_rejected(cuda):
    rng = np.random.default_rng(6)
    a, b = _mats(rng, MIN, torch.int32, 64, 64, 64, True)
    outs = [torch.empty((64, 64), dtype=torch.int32, device=a.data.device) for _ in range(8)]
    with pytest.raises(_lib.BtasStatusError):
        _gemm(a.data, b.data, MIN, True, peers=[o.data_ptr() for o in outs])
    with pytest.raises(ValueError):
        _gemm(a.data, b.data, MIN, True, z=outs[0], peers=[outs[1].data_ptr()])
    arr = (ctypes.c_void_p * 1)(None)
    rc = _lib.load().btas_gemm_peers(_lib.I32, _lib.MIN_PLUS, 1, a.data.data_ptr(), 64, b.data.data_ptr(), 64,
                                     outs[0].data_ptr(), 64, 64, 64, 64, None, 0, arr, 1, None, None, 0, None)
    assert rc == _lib.ERR_INVALID


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("world", [2, 3, 8])
def test_fused_squaring_virtual_ranks(cuda, dtype, world):
    for n, p, wr, seed in ((700, 0.3, (1, 100), 11), (333, 0.05, (0, 60), 12), (130, 0.4, (-1, 40), 13),
                           (1, 0.5, (1, 2), 14), (2, 1.0, (1, 3), 15)):
        adj = random_graph_matrix(n, p, wr, seed, dtype=dtype)
        want = bt.apsp_by_squaring(adj)
        got, per_rank = apsp_by_squaring_emulated(adj, world)
        assert got.negative_cycle == want.negative_cycle, (n, world)
        assert got.multiplications_performed == want.multiplications_performed
        if not want.negative_cycle:
            assert got.distances.dist == want.distances.dist, (n, world)
            for d in per_rank:
                assert torch.equal(d, per_rank[0])


def test_fused_squaring_negative_cycles(cuda, golden):
    import math

    g = golden("negcycle.npz")
    for case in range(0, 200, 11):
        sym = np.asarray(g[f"adj{case}"], dtype=np.float64)
        sym[np.isinf(sym)] = math.inf
        adj = bt.TropicalMatrix(MIN, sym, dtype=torch.int32)
        rep, _ = apsp_by_squaring_emulated(adj, 3)
        assert rep.negative_cycle == bool(g["meta"][case][1])


def test_fused_exchange_across_processes(cuda):
    """The fused exchange across real process boundaries: 2 processes on
    this GPU, D / D_next mapped between them with CUDA IPC, gloo for the
    host-side flag all-reduce, each rank's GEMM storing its rows into the
    other process's D_next (tools/symm_two_proc.py)."""
    import subprocess
    import sys
    from pathlib import Path

    tool = Path(__file__).resolve().parent.parent / "tools" / "symm_two_proc.py"
    res = subprocess.run([sys.executable, str(tool), "2", "1100"], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "2-process peer-store exchange OK" in res.stdout

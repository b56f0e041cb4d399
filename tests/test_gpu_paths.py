"""Path reconstruction (an extension — the reference
returns distances only): the predecessor product (btas_gemm_argmin) against
the oracle's definition, and shortest paths walked from it reproduce the
distances."""

import math

import numpy as np
import pytest
import torch

import paper_1701_04733_b200 as bt
from paper_1701_04733_b200.graphs import dense_rows, random_graph_matrix
from oracle import tropical as ot

from gpu_helpers import DTYPES, MIN, symbolic

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", DTYPES)
def test_predecessors_match_oracle(cuda, dtype):
    for n, p, wr, seed in ((1, 0.5, (1, 9), 1), (2, 1.0, (1, 9), 2), (37, 0.3, (0, 5), 3), (130, 0.1, (1, 100), 4),
                           (300, 0.5, (1, 3), 5), (257, 0.02, (0, 20), 6), (90, 0.3, (1000, 20000), 7)):
        adj = random_graph_matrix(n, p, wr, seed, dtype=dtype)
        rep = bt.floyd_warshall(adj)
        pred = bt.predecessors(adj, rep)
        sym = np.concatenate([b for _, b in dense_rows(n, p, wr, seed)])
        want = ot.predecessors(ot.orient(ot.MIN, sym), rep.distances.dist.to_numpy())
        assert np.array_equal(pred.cpu().numpy(), want), (n, p, wr)
        assert bt.predecessors(adj, bt.apsp_by_squaring(adj)).equal(pred)


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32])
def test_shortest_paths_reproduce_distances(cuda, dtype):
    """Positive weights: every walked path exists edge by edge and its weight
    is the distance (n = 2000, 300 sampled pairs incl. unreachable ones)."""
    n = 2000
    adj = random_graph_matrix(n, 0.001, (1, 100), 11, dtype=dtype)
    rep = bt.floyd_warshall(adj)
    pred = bt.predecessors(adj, rep)
    a = adj.to_numpy()
    d = rep.distances.dist.to_numpy()
    rng = np.random.default_rng(2)
    unreachable = 0
    for i, j in rng.integers(0, n, (300, 2)):
        path = bt.shortest_path(pred, int(i), int(j))
        if path is None:
            assert math.isinf(d[i, j])
            unreachable += 1
            continue
        assert path[0] == i and path[-1] == j and len(path) <= n
        w = sum(a[u, v] for u, v in zip(path, path[1:]))
        assert w == d[i, j], (i, j)
    assert 0 < unreachable < 300
    with pytest.raises(ValueError):
        bt.predecessors(bt.TropicalMatrix(MIN, [[0, -2], [1, 0]]))


def test_predecessors_at_scale(cuda):
    """n = 16384 int32 (the C2 size): path weights equal the distances on
    sampled pairs; the product runs through the tiled argmin GEMM."""
    n = 16384
    adj = random_graph_matrix(n, 0.5, (1, 100), 99, dtype=torch.int32)
    rep = bt.floyd_warshall(adj)
    pred = bt.predecessors(adj, rep)
    d = rep.distances.dist.data
    a = adj.data
    rng = np.random.default_rng(3)
    for i, j in rng.integers(0, n, (64, 2)):
        path = bt.shortest_path(pred, int(i), int(j))
        w = sum(int(a[u, v]) for u, v in zip(path, path[1:]))
        assert w == int(d[i, j])
    assert int((pred < 0).sum()) == n  # only the diagonal: the graph is strongly connected


@pytest.mark.parametrize("dtype", DTYPES)
def test_argmin_key_path_equals_compare_path(cuda, dtype):
    """btas_gemm_argmin's packed (value << 16 | k) key kernel (small integer
    operands) and its compare-and-select kernel (operand bound unknown)
    produce the same first-argmin indices."""
    from paper_1701_04733_b200 import _lib
    from paper_1701_04733_b200.matrix import _dtype_code, _workspace

    n = 700
    adj = random_graph_matrix(n, 0.4, (0, 50), 8, dtype=dtype)
    d = bt.floyd_warshall(adj).distances.dist.data
    b = adj.data.clone()
    b.diagonal().fill_(_lib.I32_INF if dtype == torch.int32 else math.inf)
    code = _dtype_code(dtype)
    ws = _workspace.get(d.device, _lib.load().btas_gemm_workspace_bytes(code, n, n, n))
    out = []
    for bound in (4000.0, -1.0):
        idx = torch.empty((n, n), dtype=torch.int32, device=d.device)
        _lib.call("btas_gemm_argmin", code, 1, bound, d.data_ptr(), n, b.data_ptr(), n, d.data_ptr(), n, n, n, n, 0,
                  idx.data_ptr(), n, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
        out.append(idx)
    assert torch.equal(out[0], out[1])


def test_predecessors_edge_cases(cuda):
    """n = 1, an edgeless graph, negative weights without a negative cycle,
    argument errors."""
    one = bt.TropicalMatrix(MIN, [[0]], dtype=torch.int32)
    assert bt.predecessors(one).cpu().tolist() == [[-1]]
    assert bt.shortest_path(bt.predecessors(one), 0, 0) == [0]
    empty = bt.TropicalMatrix.filled(MIN, 5, 5, dtype=torch.float32)
    p = bt.predecessors(empty)
    assert bool((p == -1).all()) and bt.shortest_path(p, 0, 4) is None
    neg = bt.TropicalMatrix(MIN, [[0, 4, math.inf], [math.inf, 0, -2], [1, math.inf, 0]], dtype=torch.float64)
    rep = bt.floyd_warshall(neg)
    assert not rep.negative_cycle
    p = bt.predecessors(neg, rep)
    assert bt.shortest_path(p, 0, 2) == [0, 1, 2] and bt.shortest_path(p, 2, 1) == [2, 0, 1]
    with pytest.raises(TypeError):
        bt.predecessors(neg, "not a report")
    with pytest.raises(bt.DtypeMismatch):
        bt.predecessors(bt.TropicalMatrix(MIN, [[0, 1], [1, 0]], dtype=torch.int32),
                        bt.DistanceMatrix(2, bt.TropicalMatrix(MIN, [[0, 1], [1, 0]], dtype=torch.float32)))
    with pytest.raises(IndexError):
        bt.shortest_path(p, 0, 7)


def test_verifier_mixed_dtypes_and_errors(cuda):
    """A float32 result checked against an int32 adjacency compares in
    float64; shape / kind errors as the reference raises them."""
    adj = random_graph_matrix(60, 0.3, (1, 20), 3, dtype=torch.int32)
    d32 = bt.TropicalMatrix(MIN, bt.floyd_warshall(adj).distances.dist.to_lists(), dtype=torch.float32)
    assert bt.find_apsp_violation(adj, bt.DistanceMatrix(60, d32)) is None
    with pytest.raises(bt.DimensionMismatch):
        bt.find_apsp_violation(adj, bt.DistanceMatrix(2, bt.identity_matrix(MIN, 2)))
    with pytest.raises(TypeError):
        bt.find_apsp_violation([[0]], bt.DistanceMatrix(1, bt.identity_matrix(MIN, 1)))

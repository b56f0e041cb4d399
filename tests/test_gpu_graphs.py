"""On-device instance generator (btas_graph_* / graphs.random_graph_matrix)
against the host restatement (dense_rows: numpy's own PCG64 draws, pinned to
the reference's random_graph + graph_to_matrix in test_oracle.py) — byte
equality of the stored matrix and the same integer flag, for every weight
draw family numpy's Generator uses: constant, 32-bit-buffered Lemire (with
its rare and its frequent rejections), raw 32-bit, 64-bit Lemire and uniform
reals (raw 64-bit words need a range no float weight_range can spell)."""

import math

import pytest
import torch

from paper_1701_04733_b200.graphs import instance_seed, random_graph_matrix, random_graph_matrix_host

pytestmark = pytest.mark.gpu

RANGES = [
    (1, 100),  # the benchmark family
    (7, 7),  # constant: integers(7, 8) draws nothing
    (-3, 10),
    (0, 2**31),  # Lemire32 rejecting about half the words
    (-(2**31), 2**31 - 1),  # raw 32-bit words
    (0, 2**32),  # 64-bit Lemire
    (-(2**40), 2**40 + 12345),
    (-(2**62), 2**62),  # 64-bit Lemire, about half the words rejected
    (0.5, 7.25),  # uniform reals
    (-1e3, 1e3 + 0.5),
    (2.5, 2.5),  # uniform with zero scale still draws
]


def _same(a, b):
    assert a.data.dtype == b.data.dtype and a.data.shape == b.data.shape
    assert torch.equal(a.data.view(torch.uint8) if a.data.dtype != torch.float64 else a.data.view(torch.int64),
                       b.data.view(torch.uint8) if b.data.dtype != torch.float64 else b.data.view(torch.int64))
    assert a.integer == b.integer


@pytest.mark.parametrize("wr", RANGES, ids=[str(r) for r in RANGES])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_device_generator_matches_host(cuda, wr, dtype):
    for n, p, seed in ((1, 0.5, 1), (2, 1.0, 2), (3, 0.5, 3), (33, 0.3, 4), (130, 0.05, 5), (700, 0.5, 6),
                       (1100, 1.0, 7), (257, 0.0, 8)):
        got = random_graph_matrix(n, p, wr, seed, dtype=dtype)
        want = random_graph_matrix_host(n, p, wr, seed, dtype=dtype)
        _same(got, want)


def test_device_generator_int32(cuda):
    for n, p, wr, seed in ((513, 0.5, (1, 100), 11), (64, 0.9, (-(2**27), 2**27), 12), (300, 0.2, (5, 5), 13)):
        _same(random_graph_matrix(n, p, wr, seed, dtype=torch.int32),
              random_graph_matrix_host(n, p, wr, seed, dtype=torch.int32))
    for gen in (random_graph_matrix, random_graph_matrix_host):
        with pytest.raises(ValueError):
            gen(40, 0.5, (0, 2**29), 3, dtype=torch.int32)
        with pytest.raises(ValueError):
            gen(40, 0.5, (0.5, 2.5), 3, dtype=torch.int32)
    # no edges: a real weight range still fits int32
    _same(random_graph_matrix(40, 0.0, (0.5, 2.5), 3, dtype=torch.int32),
          random_graph_matrix_host(40, 0.0, (0.5, 2.5), 3, dtype=torch.int32))


def test_device_generator_edge_probabilities(cuda):
    """p at the exact 2^-53 grid: presence is (u >> 11) < ceil(p 2^53)."""
    for p in (2.0**-53, 0.5 + 2.0**-53, 1.0 - 2.0**-53, 0.3, 1e-300):
        _same(random_graph_matrix(200, p, (1, 9), 21, dtype=torch.float32),
              random_graph_matrix_host(200, p, (1, 9), 21, dtype=torch.float32))


def test_device_generator_large(cuda):
    """Several thousand CTAs of every stage; the weight stream starts past
    n(n-1) presence doubles at a non-multiple of the chunk size."""
    n = 6001
    got = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.float32)
    want = random_graph_matrix_host(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.float32)
    _same(got, want)


def test_validation_errors(cuda):
    with pytest.raises(ValueError):
        random_graph_matrix(0, 0.5, (1, 2), 1)
    with pytest.raises(ValueError):
        random_graph_matrix(4, 1.5, (1, 2), 1)
    with pytest.raises(ValueError):
        random_graph_matrix(4, 0.5, (3, 2), 1)
    with pytest.raises(ValueError):
        random_graph_matrix(4, 0.5, (1, math.inf), 1)
    # huge floats are integral: numpy's integers() rejects bounds beyond int64
    for gen in (random_graph_matrix, random_graph_matrix_host):
        with pytest.raises(ValueError):
            gen(4, 0.5, (-1.5e308, 1.5e308), 1)


def _digest(t):
    import hashlib

    import numpy as np

    return hashlib.sha256(np.ascontiguousarray(t, dtype=np.float64).tobytes()).hexdigest()


def test_device_generator_reference_digests(cuda, golden):
    """float64 storage of the device generator == the reference's bytes."""
    for name in ("generator.npz", "generator_families.npz"):
        g = golden(name)
        for i in range(len(g["n"])):
            n, p, wr, seed = int(g["n"][i]), float(g["p"][i]), (g["lo"][i], g["hi"][i]), int(g["seed"][i])
            adj = random_graph_matrix(n, p, wr, seed, dtype=torch.float64)
            assert _digest(adj.to_numpy()) == str(g["digest"][i]), (name, i)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.int32])
def test_edge_list_matches_reference(cuda, golden, dtype):
    import numpy as np

    from oracle import graphs as og
    from paper_1701_04733_b200.graphs import edges_to_matrix

    g = golden("edgelist.npz")
    for case in range(int(g["count"][0])):
        n = int(g[f"n{case}"][0])
        src, dst, w = g[f"src{case}"], g[f"dst{case}"], g[f"w{case}"]
        want = np.asarray(g[f"out{case}"], dtype=np.float64)
        integral = bool(g[f"integer{case}"][0])
        if dtype == torch.int32 and not integral:
            with pytest.raises(ValueError):
                edges_to_matrix(n, src, dst, w, dtype=dtype)
            continue
        got = edges_to_matrix(n, src, dst, w, dtype=dtype)
        if dtype == torch.float64:
            assert got.to_numpy().tobytes() == want.tobytes(), case
            assert got.integer == integral
        else:
            assert got.to_numpy().tobytes() == want.astype(np.float32).astype(np.float64).tobytes(), case
        # torch inputs on the device take the same path
        t = edges_to_matrix(n, torch.as_tensor(src, device="cuda"), torch.as_tensor(dst, device="cuda"),
                            torch.as_tensor(w, device="cuda"), dtype=dtype)
        assert torch.equal(t.data, got.data)
        assert og.graph_to_matrix_edges(n, src, dst, w).astype(np.float64).tobytes() == want.tobytes()


def test_edge_list_errors_and_graph_objects(cuda):
    import numpy as np

    from paper_1701_04733_b200.graphs import edges_to_matrix, graph_to_matrix
    from oracle.graphs import graph_to_matrix_edges

    with pytest.raises(ValueError, match=r"edge \(0, 3\) out of range for n=3"):
        edges_to_matrix(3, [0, 0], [1, 3], [1.0, 2.0])
    with pytest.raises(ValueError, match=r"edge \(1, 1\) weight must be finite"):
        edges_to_matrix(3, [0, 1], [1, 1], [1.0, math.inf])
    with pytest.raises(ValueError):
        edges_to_matrix(0, [], [], [])
    with pytest.raises(ValueError):
        edges_to_matrix(3, [0], [1, 2], [1.0])

    class G:  # duck-typed reference Graph
        n = 4
        edges = ((0, 1, 5.0), (0, 1, 3.0), (2, 2, -1.0), (3, 0, -0.0), (1, 1, 7.0))

    got = graph_to_matrix(G(), dtype=torch.float64)
    want = graph_to_matrix_edges(4, [0, 0, 2, 3, 1], [1, 1, 2, 0, 1], [5.0, 3.0, -1.0, -0.0, 7.0])
    assert got.to_numpy().tobytes() == want.tobytes() and got.integer

    class E:
        n = 2
        edges = ()

    assert graph_to_matrix(E(), dtype=torch.int32).to_numpy().tobytes() == \
        np.array([[0.0, math.inf], [math.inf, 0.0]]).tobytes()
    # the edge list of a generated instance rebuilds the same matrix
    adj = random_graph_matrix(300, 0.2, (-5, 40), 77, dtype=torch.float32)
    d = adj.data
    mask = torch.isfinite(d) & ~torch.eye(300, dtype=torch.bool, device=d.device)
    s, t = mask.nonzero(as_tuple=True)
    back = edges_to_matrix(300, s, t, d[s, t].double(), dtype=torch.float32)
    assert torch.equal(back.data, d) and back.integer == adj.integer


def test_graph_objects_on_the_device(cuda):
    """graph_to_matrix(random_graph(...)) takes the device generator;
    matrix_to_graph inverts graph_to_matrix (graph_io.py:168-187)."""
    import paper_1701_04733_b200 as bt

    for n, p, wr, seed in ((257, 0.3, (1, 100), 5), (40, 0.9, (-3, 8), 6), (1, 0.5, (1, 2), 7)):
        rg = bt.random_graph(n, p, wr, seed)
        a = bt.graph_to_matrix(rg, dtype=torch.float64)
        assert a == random_graph_matrix(n, p, wr, seed, dtype=torch.float64)
        b = bt.graph_to_matrix(bt.Graph(n, rg.edges), dtype=torch.float64)  # the edge-list route
        assert a == b
        assert bt.matrix_to_graph(a) == rg
    with pytest.raises(ValueError):
        bt.matrix_to_graph(bt.TropicalMatrix(bt.SemiringKind.MAX_PLUS, [[0.0]]))

"""Property-based GPU parity (hypothesis): random shapes, kinds, storage
dtypes and value mixes — including Infinity-heavy and overflow-prone
operands — checked byte for byte against the pinned NumPy oracle, plus the
semiring laws the reference's test-suite states (test_matrix.py:57-120)."""

import math

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1701_04733_b200 as bt
from oracle import tropical as ot

from gpu_helpers import MAX, MIN, STORAGE, kname

pytestmark = pytest.mark.gpu

DTYPES = [torch.float64, torch.float32, torch.int32]


@st.composite
def operands(draw, max_dim=40):
    m = draw(st.integers(1, max_dim))
    k = draw(st.integers(1, max_dim))
    n = draw(st.integers(1, max_dim))
    dtype = draw(st.sampled_from(DTYPES))
    kind = draw(st.sampled_from([MIN, MAX]))
    p_inf = draw(st.sampled_from([0.0, 0.25, 0.9, 1.0]))
    # value regimes: tiny (s16 path), wide (32-bit path), near the storage limit
    regime = draw(st.sampled_from(["small", "wide", "edge"]))
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    if dtype == torch.int32:
        hi = {"small": 100, "wide": 10**6, "edge": 2**28 - 1}[regime]
    elif dtype == torch.float32:
        hi = {"small": 100, "wide": 10**6, "edge": 3.0e38}[regime]
    else:
        hi = {"small": 100, "wide": 10**9, "edge": 1.5e308}[regime]

    def draw_mat(r, c):
        if regime == "edge":
            a = rng.uniform(-1.0, 1.0, (r, c)) * hi
            if dtype == torch.int32:
                a = np.trunc(a)
            elif dtype == torch.float32:
                a = a.astype(np.float32).astype(np.float64)
        else:
            a = rng.integers(-hi, hi + 1, (r, c)).astype(np.float64)
        a[rng.random((r, c)) < p_inf] = math.inf
        return a

    return kind, dtype, draw_mat(m, k), draw_mat(k, n)


@settings(max_examples=150, deadline=None)
@given(operands())
def test_matmul_matches_oracle(cuda, ops):
    kind, dtype, xs, ys = ops
    x = bt.TropicalMatrix(kind, xs, dtype=dtype)
    y = bt.TropicalMatrix(kind, ys, dtype=dtype)
    integer = x.integer and y.integer
    bt.reset_saturation()
    got = bt.matmul(x, y).to_numpy()
    want, sat = ot.matmul(ot.orient(kname(kind), xs), ot.orient(kname(kind), ys), kname(kind), STORAGE[dtype],
                          integer)
    assert got.tobytes() == want.tobytes()
    assert bt.saturation_seen() == sat


@settings(max_examples=60, deadline=None)
@given(operands(max_dim=24))
def test_matvec_and_ewadd_match_oracle(cuda, ops):
    kind, dtype, xs, ys = ops
    a = bt.TropicalMatrix(kind, xs, dtype=dtype)
    v = bt.TropicalVector(kind, ys[:, 0], dtype=dtype)
    integer = a.integer and v.integer
    bt.reset_saturation()
    got = bt.matvec(a, v).to_numpy()
    want, sat = ot.matvec(ot.orient(kname(kind), xs), ot.orient(kname(kind), ys[:, 0]), kname(kind),
                          STORAGE[dtype], integer)
    assert got.tobytes() == want.tobytes() and bt.saturation_seen() == sat
    b = bt.TropicalMatrix(kind, xs[::-1].copy(), dtype=dtype)
    assert bt.ew_add(a, b).to_numpy().tobytes() == \
        ot.ew_add(ot.orient(kname(kind), xs), ot.orient(kname(kind), xs[::-1]), kname(kind)).tobytes()


@settings(max_examples=40, deadline=None)
@given(st.integers(2, 24), st.sampled_from(DTYPES), st.integers(0, 2**31 - 1), st.sampled_from([MIN, MAX]))
def test_semiring_laws_on_matrices(cuda, n, dtype, seed, kind):
    """Identity neutrality, associativity, ⊕-distributivity, and (min-plus,
    zero diagonal) monotone powers — the laws of test_matrix.py."""
    rng = np.random.default_rng(seed)

    def mat():
        a = rng.integers(-50, 101, (n, n)).astype(float)
        a[rng.random((n, n)) < 0.3] = math.inf
        return bt.TropicalMatrix(kind, a, dtype=dtype)

    a, b, c = mat(), mat(), mat()
    ident = bt.identity_matrix(kind, n, dtype=dtype)
    assert bt.matmul(ident, a) == a and bt.matmul(a, ident) == a
    assert bt.matmul(bt.matmul(a, b), c) == bt.matmul(a, bt.matmul(b, c))
    assert bt.matmul(a, bt.ew_add(b, c)) == bt.ew_add(bt.matmul(a, b), bt.matmul(a, c))
    assert bt.matmul(a, b, accumulate_into=c) == bt.ew_add(bt.matmul(a, b), c)


@settings(max_examples=40, deadline=None)
@given(st.integers(1, 90), st.floats(0.0, 1.0), st.integers(0, 2**31 - 1), st.sampled_from(DTYPES),
       st.sampled_from([(0, 100), (1, 5), (-2, 30)]))
def test_apsp_routes_agree_with_oracle(cuda, n, p, seed, dtype, wr):
    from paper_1701_04733_b200.graphs import dense_rows, random_graph_matrix

    adj = random_graph_matrix(n, p, wr, seed, dtype=dtype)
    sym = np.concatenate([blk for _, blk in dense_rows(n, p, wr, seed)])
    want, neg, mults, _ = ot.apsp_by_squaring(sym, STORAGE[dtype], True)
    sq = bt.apsp_by_squaring(adj)
    fw = bt.floyd_warshall(adj)
    assert sq.negative_cycle == neg == fw.negative_cycle
    assert sq.multiplications_performed == mults
    if not neg:
        assert sq.distances.dist.to_numpy().tobytes() == want.tobytes()
        assert fw.distances.dist == sq.distances.dist
        assert bt.verify_apsp_strict(adj, fw.distances)


def test_strict_verifier_rejects_fixpoints_below_the_closure(cuda):
    """The reference verifier accepts an all-zero matrix on a non-negative
    graph; the strict variant does not."""
    three = bt.TropicalMatrix(MIN, [[0, 1, 5], [math.inf, 0, 2], [math.inf, math.inf, 0]])
    zeros = bt.TropicalMatrix.filled(MIN, 3, 3, 0)
    assert bt.verify_apsp(three, bt.DistanceMatrix.from_matrix(zeros))  # reference behaviour
    assert not bt.verify_apsp_strict(three, bt.DistanceMatrix.from_matrix(zeros))
    good = bt.floyd_warshall(three).distances
    assert bt.verify_apsp_strict(three, good)
    msg = bt.find_apsp_violation_strict(three, bt.DistanceMatrix.from_matrix(zeros))
    assert "closure" in msg


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 300), st.sampled_from([0.0, 0.01, 0.3, 0.5, 1.0]),
       st.sampled_from([(1, 100), (0, 0), (-5, 7), (0, 2**31), (-(2**33), 2**33), (0.25, 9.5), (3.5, 3.5)]),
       st.integers(0, 2**63 - 1), st.sampled_from([torch.float64, torch.float32]))
def test_instance_generator_matches_host(cuda, n, p, wr, seed, dtype):
    """random_graph_matrix (device PCG64 stream) == the host restatement over
    random sizes, probabilities, weight families and seeds."""
    from paper_1701_04733_b200.graphs import random_graph_matrix, random_graph_matrix_host

    got = random_graph_matrix(n, p, wr, seed, dtype=dtype)
    want = random_graph_matrix_host(n, p, wr, seed, dtype=dtype)
    assert torch.equal(got.data.view(torch.uint8) if dtype == torch.float32 else got.data.view(torch.int64),
                       want.data.view(torch.uint8) if dtype == torch.float32 else want.data.view(torch.int64))
    assert got.integer == want.integer


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 40), st.integers(0, 400), st.integers(0, 2**31 - 1), st.sampled_from(DTYPES))
def test_edge_list_matches_oracle(cuda, n, m, seed, dtype):
    from oracle.graphs import graph_to_matrix_edges
    from paper_1701_04733_b200.graphs import edges_to_matrix

    rng = np.random.default_rng(seed)
    src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
    w = rng.integers(-20, 60, m).astype(np.float64)
    w[rng.random(m) < 0.1] = -0.0
    got = edges_to_matrix(n, src, dst, w, dtype=dtype)
    want = graph_to_matrix_edges(n, src, dst, w)
    assert got.to_numpy().tobytes() == want.tobytes()

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

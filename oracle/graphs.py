"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference instance
builders (btas/graph_io.py), the checker of the device generator and of the
edge-list scatter.  Pinned against tests/golden/{generator,generator_families,
edgelist}.npz, which the real reference produced (tests/golden/make_golden.py).
"""

from __future__ import annotations

import math

import numpy as np


def graph_to_matrix_edges(n: int, src, dst, weight) -> np.ndarray:
    """Graph normalisation (graph_io.py:64-83: duplicates keep the minimum,
    -0.0 -> 0.0, finite weights, indices in range) followed by graph_to_matrix
    (graph_io.py:158-165: inf, diagonal 0, ``if arr[s, d] > w: arr[s, d] = w``).
    Returns the symbolic float64 matrix."""
    src = np.asarray(src, dtype=np.int64).reshape(-1)
    dst = np.asarray(dst, dtype=np.int64).reshape(-1)
    w = np.asarray(weight, dtype=np.float64).reshape(-1)
    if not (len(src) == len(dst) == len(w)):
        raise ValueError("src, dst and weight must have the same length")
    bad = (src < 0) | (src >= n) | (dst < 0) | (dst >= n)
    if bad.any():
        e = int(np.argmax(bad))
        raise ValueError(f"edge ({src[e]}, {dst[e]}) out of range for n={n}")
    if not np.isfinite(w).all():
        e = int(np.argmax(~np.isfinite(w)))
        raise ValueError(f"edge ({src[e]}, {dst[e]}) weight must be finite, got {w[e]!r}")
    w = w + 0.0  # -0.0 -> +0.0
    arr = np.full((n, n), math.inf)
    np.fill_diagonal(arr, 0.0)
    np.minimum.at(arr, (src, dst), w)
    return arr


def random_graph_dense(n: int, p: float, weight_range, seed: int) -> np.ndarray:
    """random_graph + graph_to_matrix (graph_io.py:273-304, 158-165) in one
    shot: one PCG64 stream, n(n-1) presence doubles in row-major pair order,
    then one weight draw per present edge (integers(low, high+1) when both
    bounds are integral, else uniform(low, high)).  Symbolic float64 matrix."""
    low, high = float(weight_range[0]), float(weight_range[1])
    rng = np.random.Generator(np.random.PCG64(int(seed) & 0xFFFF_FFFF_FFFF_FFFF))
    present = rng.random(n * (n - 1)) < float(p)
    k = int(present.sum())
    if low.is_integer() and high.is_integer():
        w = rng.integers(int(low), int(high) + 1, size=k).astype(np.float64)
    else:
        w = rng.uniform(low, high, size=k)
    off = np.full(n * (n - 1), math.inf)
    off[present] = w
    arr = np.zeros((n, n))
    mask = ~np.eye(n, dtype=bool)
    arr[mask] = off  # row-major over the off-diagonal pairs
    return arr

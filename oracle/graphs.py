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


# ---------------------------------------------------------------------------
# row blocks of very large instances (n = 65536: n(n-1) = 4.3e9 presence
# doubles, ~2.1e9 weight draws) without walking the streams on one core
# ---------------------------------------------------------------------------
_SEG = 1 << 22  # stream units per worker task


def _threads(threads):
    import os

    return threads or len(os.sched_getaffinity(0))


def _count_present(seed: int, start: int, stop: int, p: float, threads=None) -> int:
    """#{t in [start, stop): presence double t < p} over the reference's
    presence stream (one ``Generator.random()`` double per ordered pair,
    graph_io.py:296-298), counted in parallel from PCG64.advance'd copies.
    numpy's own ``random()`` produces the doubles."""
    from concurrent.futures import ThreadPoolExecutor

    def seg(s0):
        bg = np.random.PCG64(seed)
        bg.advance(s0)
        g = np.random.Generator(bg)
        m = min(_SEG, stop - s0)
        return int(np.count_nonzero(g.random(m) < p))

    with ThreadPoolExecutor(_threads(threads)) as ex:
        return sum(ex.map(seg, range(start, stop, _SEG)))


def _lemire32_accept(raw: np.ndarray, rng: int) -> np.ndarray:
    """Accepted mask of numpy's buffered bounded Lemire draw (numpy 2.3.5
    ``random_buffered_bounded_lemire_uint32``, the path of
    ``Generator.integers(low, high + 1)`` for ranges below 2^32 - 1) over the
    32-bit words of raw 64-bit outputs, low half first (numpy's
    ``next_uint32`` buffering).  A word is rejected iff the low 32 bits of
    word * (rng + 1) fall below (2^32 - (rng + 1)) mod (rng + 1); acceptance
    is per word, so counts over disjoint segments add up."""
    words = raw.view(np.uint32).astype(np.uint64)  # little-endian: low half first
    excl = np.uint64(rng + 1)
    thresh = np.uint64(((1 << 32) - (rng + 1)) % (rng + 1))
    return ((words * excl) & np.uint64(0xFFFFFFFF)) >= thresh


def _locate_draw(seed: int, wstart: int, index: int, rng: int, threads=None) -> "tuple[int, int]":
    """(64-bit unit, half) of the weight stream holding accepted draw number
    ``index`` (0-based) of the stream that starts at unit ``wstart``."""
    from concurrent.futures import ThreadPoolExecutor

    def count(s0):
        bg = np.random.PCG64(seed)
        bg.advance(s0)
        return int(np.count_nonzero(_lemire32_accept(bg.random_raw(_SEG), rng)))

    # accepted draws per unit are ~2, so index/2 units suffice, plus slack
    nthr = _threads(threads)
    base, need = wstart, index
    with ThreadPoolExecutor(nthr) as ex:
        while True:
            starts = [base + i * _SEG for i in range(nthr)]
            counts = list(ex.map(count, starts))
            for s0, c in zip(starts, counts):
                if need < c:
                    bg = np.random.PCG64(seed)
                    bg.advance(s0)
                    acc = np.flatnonzero(_lemire32_accept(bg.random_raw(_SEG), rng))
                    w = int(acc[need])
                    return s0 + w // 2, w % 2
                need -= c
            base = starts[-1] + _SEG


def instance_rows(n: int, p: float, weight_range, seed: int, r0: int, r1: int, threads=None) -> np.ndarray:
    """Rows [r0, r1) of graph_to_matrix(random_graph(n, p, weight_range,
    seed)) (graph_io.py:273-304, 158-165) for integer weight ranges, without
    generating the rows before r0 one by one: the presence doubles before the
    block are counted in parallel, the weight stream is positioned at the
    first draw of the block, and numpy's own Generator then produces the
    block's presence doubles and weights.  Symbolic float64 rows (diagonal 0,
    absent +inf); equals the same rows of ``random_graph_dense``."""
    low, high = float(weight_range[0]), float(weight_range[1])
    if not (low.is_integer() and high.is_integer()) or high - low >= 0xFFFFFFFF:
        raise NotImplementedError("instance_rows covers integer weight ranges narrower than 2^32 - 1")
    seed = int(seed) & 0xFFFF_FFFF_FFFF_FFFF
    pairs = n * (n - 1)
    start, stop = r0 * (n - 1), r1 * (n - 1)
    before = _count_present(seed, 0, start, float(p), threads) if start else 0
    pres_bg = np.random.PCG64(seed)
    pres_bg.advance(start)
    present = np.random.Generator(pres_bg).random(stop - start) < float(p)
    rng = int(high) - int(low)
    wbg = np.random.PCG64(seed)
    if rng == 0:
        w = np.full(int(present.sum()), low)
    else:
        unit, half = _locate_draw(seed, pairs, before, rng, threads) if before else (pairs, 0)
        if half == 0:
            wbg.advance(unit)
        else:  # the block's first draw is the buffered high half of `unit`
            wbg.advance(unit)
            raw = int(wbg.random_raw())
            st = wbg.state
            st["has_uint32"], st["uinteger"] = 1, raw >> 32
            wbg.state = st
        w = np.random.Generator(wbg).integers(int(low), int(high) + 1, size=int(present.sum())).astype(np.float64)
    off = np.full(stop - start, math.inf)
    off[present] = w
    off = off.reshape(r1 - r0, n - 1)
    block = np.empty((r1 - r0, n))
    for a in range(r1 - r0):
        i = r0 + a
        block[a, :i] = off[a, :i]
        block[a, i] = 0.0
        block[a, i + 1 :] = off[a, i:]
    return block

"""Seeded random dense digraphs straight into device storage.

A vectorised, chunked restatement of the reference instance generator
``random_graph`` + ``graph_to_matrix`` (btas/graph_io.py:273-304,158-165) and
of ``instance_seed`` (btas/bench.py:153-156): the same PCG64 streams in the
same order, so the matrix is bit-identical to
``graph_to_matrix(random_graph(n, p, weight_range, seed))`` — but built in
row chunks (no n(n-1) Python tuples, no n x n float64 host array), which is
what makes n = 32768 / 65536 instances practical.

Stream layout of the reference: first one ``random()`` double per ordered
off-diagonal pair (row-major), then one weight draw per present edge.  The
weight stream is reproduced by advancing a second PCG64 past the n(n-1)
presence doubles.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .matrix import (
    TropicalMatrix,
    _dtype_code,
    _kind_code,
    _new_stats,
    _ptr,
    _read_stats,
    _resolve_device,
    _stream,
    get_default_dtype,
)
from .semiring import SemiringKind


def instance_seed(seed: int, n: int) -> int:
    """Per-size instance seed (reference bench.py:153-156)."""
    seq = np.random.SeedSequence(int(seed) & 0xFFFF_FFFF_FFFF_FFFF, spawn_key=(int(n),))
    return int(seq.generate_state(1, np.uint64)[0])


def _check(n, p, weight_range):
    if not isinstance(n, int) or n < 1:
        raise ValueError(f"vertex count must be a positive integer, got {n!r}")
    p = float(p)
    if math.isnan(p) or not 0.0 <= p <= 1.0:
        raise ValueError(f"edge probability must lie in [0, 1], got {p!r}")
    low, high = float(weight_range[0]), float(weight_range[1])
    if not (math.isfinite(low) and math.isfinite(high)) or low > high:
        raise ValueError(f"weight range must be finite with low <= high, got {weight_range!r}")
    return p, low, high


def dense_rows(n: int, p: float, weight_range, seed: int, chunk_rows: int = 1024):
    """Yield (row0, symbolic float64 block) for consecutive row blocks of the
    reference instance: diagonal 0, absent edges +inf (graph_to_matrix)."""
    p, low, high = _check(n, p, weight_range)
    s = int(seed) & 0xFFFF_FFFF_FFFF_FFFF
    presence = np.random.Generator(np.random.PCG64(s))
    wbits = np.random.PCG64(s)
    wbits.advance(n * (n - 1))  # past the presence doubles
    weights = np.random.Generator(wbits)
    integral = low.is_integer() and high.is_integer()
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        rows = r1 - r0
        present = presence.random(rows * (n - 1)) < p
        cnt = int(present.sum())
        if integral:
            w = weights.integers(int(low), int(high) + 1, size=cnt).astype(np.float64)
        else:
            w = weights.uniform(low, high, size=cnt)
        off = np.full(rows * (n - 1), math.inf)
        off[present] = w
        block = np.empty((rows, n), dtype=np.float64)
        # scatter the off-diagonal entries around the zero diagonal
        off = off.reshape(rows, n - 1)
        for a in range(rows):
            i = r0 + a
            block[a, :i] = off[a, :i]
            block[a, i] = 0.0
            block[a, i + 1 :] = off[a, i:]
        yield r0, block


def random_graph_matrix(n: int, p: float, weight_range, seed: int, *, dtype: "torch.dtype | None" = None,
                        device=None, chunk_rows: int = 1024) -> TropicalMatrix:
    """The reference instance as a min-plus TropicalMatrix on the GPU."""
    dt = dtype if dtype is not None else get_default_dtype()
    dev = _resolve_device(device)
    out = torch.empty((n, n), dtype=dt, device=dev)
    stats = _new_stats(dev)
    kind = SemiringKind.MIN_PLUS
    for r0, block in dense_rows(n, p, weight_range, seed, chunk_rows):
        src = torch.from_numpy(block).to(dev)
        dst = out[r0 : r0 + block.shape[0]]
        _lib.call("btas_ingest", _kind_code(kind), _lib.F64, _ptr(src), src.numel(), _dtype_code(dt), _ptr(dst),
                  _ptr(stats), _stream(dev))
    st = _read_stats(stats)
    if st.out_of_range:
        raise ValueError(f"instance weights do not fit {dt} storage")
    integer = dt == torch.int32 or (st.non_integral == 0 and st.over_limit == 0)
    return TropicalMatrix._wrap(kind, out, integer)

"""Seeded random dense digraphs straight into device storage.

``random_graph_matrix`` generates the instance on the GPU (btas_graph_*
kernels, csrc/btas_graph.cu); ``dense_rows`` / ``random_graph_matrix_host``
are the host restatement used as its independent check.

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

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .matrix import (
    TropicalMatrix,
    _device_ctx,
    _dtype_code,
    _host_read,
    _kind_code,
    _new_stats,
    _ptr,
    _read_stats,
    _resolve_device,
    _stats_bound,
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


def pcg64_state(seed: int) -> "_lib.Pcg64":
    """numpy's PCG64(seed) state after SeedSequence seeding (graph_io.py:289)."""
    st = np.random.PCG64(int(seed) & 0xFFFF_FFFF_FFFF_FFFF).state["state"]
    m64 = (1 << 64) - 1
    return _lib.Pcg64(st["state"] >> 64, st["state"] & m64, st["inc"] >> 64, st["inc"] & m64)


def _weight_plan(low: float, high: float):
    """(mode, range, int offset, float low, scale) of the reference weight draw
    (graph_io.py:300-303): integers(low, high + 1) or uniform(low, high)."""
    if low.is_integer() and high.is_integer():
        lo, hi = int(low), int(high)
        if lo < -(1 << 63) or hi + 1 > (1 << 63):
            raise ValueError(f"integer weight range ({low!r}, {high!r}) exceeds int64")
        rng = hi - lo
        return (_lib.WEIGHTS_CONST if rng == 0 else _lib.WEIGHTS_BOUNDED), rng, lo, 0.0, 0.0
    scale = high - low
    if not math.isfinite(scale):
        raise OverflowError("Range exceeds valid bounds")  # numpy Generator.uniform
    return _lib.WEIGHTS_UNIFORM, 0, 0, low, scale


def random_graph_matrix(n: int, p: float, weight_range, seed: int, *, dtype: "torch.dtype | None" = None,
                        device=None) -> TropicalMatrix:
    """The reference instance ``graph_to_matrix(random_graph(n, p, weight_range,
    seed))`` generated on the GPU (see _random_graph_matrix)."""
    dev = _resolve_device(device)
    with _device_ctx(dev):
        return _random_graph_matrix(n, p, weight_range, seed, dtype=dtype, device=dev)


def _random_graph_matrix(n: int, p: float, weight_range, seed: int, *, dtype: "torch.dtype | None" = None,
                         device=None) -> TropicalMatrix:
    """The reference instance ``graph_to_matrix(random_graph(n, p, weight_range,
    seed))`` generated on the GPU (include/btas_cuda.h btas_graph_*): presence
    draws, weight draws and the dense fill run as CUDA kernels over the same
    PCG64 stream, so the matrix is bit-identical to the reference's (and to
    ``dense_rows``) with no host-side O(n^2) work.  Two small host reads:
    the edge count and the accepted-draw count."""
    p, low, high = _check(n, p, weight_range)
    dt = dtype if dtype is not None else get_default_dtype()
    dev = _resolve_device(device)
    code = _dtype_code(dt)
    rng = pcg64_state(seed)
    thr = math.ceil(p * 2.0**53)  # u >> 11 < thr  <=>  (u >> 11) * 2^-53 < p  (exact)
    mode, wrange, off, flow, scale = _weight_plan(low, high)
    lib = _lib.load()
    ws = torch.empty(max(1, lib.btas_graph_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    edges_t = torch.zeros(1, dtype=torch.int64, device=dev)
    s = _stream(dev)
    _lib.call("btas_graph_presence", ctypes.byref(rng), n, thr, _ptr(ws), ws.numel(), _ptr(edges_t), s)
    edges = int(_host_read(edges_t)[0])
    draws = None
    if mode != _lib.WEIGHTS_CONST and edges > 0:
        if mode == _lib.WEIGHTS_UNIFORM:
            draws, per_unit, accept = torch.empty(edges, dtype=torch.float64, device=dev), 1, 1.0
        elif wrange < 0xFFFF_FFFF:
            draws, per_unit = torch.empty(edges, dtype=torch.int32, device=dev), 2
            accept = 1.0 - ((0xFFFF_FFFF - wrange) % (wrange + 1)) / 2.0**32
        elif wrange == 0xFFFF_FFFF:
            draws, per_unit, accept = torch.empty(edges, dtype=torch.int32, device=dev), 2, 1.0
        else:
            draws, per_unit = torch.empty(edges, dtype=torch.int64, device=dev), 1
            accept = 1.0 - ((0xFFFF_FFFF_FFFF_FFFF - wrange) % (wrange + 1)) / 2.0**64
        acc_t = torch.zeros(1, dtype=torch.int64, device=dev)
        unit0, accepted = 0, 0
        cap = n * (n - 1) + (1 << 20)
        while accepted < edges:
            need = edges - accepted
            units = min(cap, math.ceil(need / (per_unit * accept) * 1.001) + 4096)
            _lib.call("btas_graph_draw", ctypes.byref(rng), n, mode, wrange, flow, scale, edges, unit0, units,
                      _ptr(draws), _ptr(ws), ws.numel(), _ptr(acc_t), s)
            unit0 += units
            accepted = int(_host_read(acc_t)[0])
    out = torch.empty((n, n), dtype=dt, device=dev)
    stats = _new_stats(dev)
    _lib.call("btas_graph_fill", code, ctypes.byref(rng), n, thr, mode, wrange, off,
              _ptr(draws) if draws is not None else None, _ptr(out), n, _ptr(ws), ws.numel(), _ptr(stats), s)
    st = _read_stats(stats)
    if st.out_of_range:
        raise ValueError(f"instance weights do not fit {dt} storage")
    integer = dt == torch.int32 or (st.non_integral == 0 and st.over_limit == 0)
    # the validation-free fill of exactly representable integer weights
    # leaves the statistics empty; its entries are 0, Infinity or in [low, high]
    bound = _stats_bound(st) if st.finite_count else max(abs(low), abs(high))
    return TropicalMatrix._wrap(SemiringKind.MIN_PLUS, out, integer, bound)


def random_graph_matrix_host(n: int, p: float, weight_range, seed: int, *, dtype: "torch.dtype | None" = None,
                             device=None, chunk_rows: int = 1024) -> TropicalMatrix:
    """The same instance through the host restatement ``dense_rows`` (numpy's
    own PCG64) and btas_ingest: the independent check of the device generator."""
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
    return TropicalMatrix._wrap(kind, out, integer, _stats_bound(st))


def edges_to_matrix(n: int, src, dst, weight, *, dtype: "torch.dtype | None" = None, device=None) -> TropicalMatrix:
    """graph_to_matrix of an edge list; see _edges_to_matrix."""
    if not isinstance(n, int) or n < 1:
        raise ValueError(f"vertex count must be a positive integer, got {n!r}")
    dev = _resolve_device(device)
    with _device_ctx(dev):
        return _edges_to_matrix(n, src, dst, weight, dtype=dtype, device=dev)


def _edges_to_matrix(n: int, src, dst, weight, *, dtype: "torch.dtype | None" = None, device=None) -> TropicalMatrix:
    """``graph_to_matrix`` (graph_io.py:158-165) of an edge list given as three
    equal-length arrays (numpy or torch; src/dst integer, weight float):
    +inf off the diagonal, 0 on it, duplicates keep the minimum weight and a
    negative self-loop lowers the diagonal (Graph normalisation,
    graph_io.py:64-83).  One init, one atomic min-scatter and one decode
    kernel (btas_edges_to_matrix); errors are raised with the reference's
    messages for the first offending edge."""
    if not isinstance(n, int) or n < 1:
        raise ValueError(f"vertex count must be a positive integer, got {n!r}")
    dt = dtype if dtype is not None else get_default_dtype()
    dev = _resolve_device(device)

    def dev_arr(a, tdt):
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(a)))
        return t.to(device=dev, dtype=tdt).contiguous().reshape(-1)

    s_t, d_t, w_t = dev_arr(src, torch.int64), dev_arr(dst, torch.int64), dev_arr(weight, torch.float64)
    m = s_t.numel()
    if d_t.numel() != m or w_t.numel() != m:
        raise ValueError("src, dst and weight must have the same length")
    out = torch.empty((n, n), dtype=dt, device=dev)
    err = torch.empty(3, dtype=torch.int64, device=dev)
    s = _stream(dev)
    _lib.call("btas_edges_to_matrix", _dtype_code(dt), n, _ptr(s_t), _ptr(d_t), _ptr(w_t), m, _ptr(out), n,
              _ptr(err), s)
    stats = _new_stats(dev)
    _lib.call("btas_scan", _dtype_code(dt), _ptr(out), out.numel(), _ptr(stats), s)
    e_index, e_weight, e_range = (int(v) for v in _host_read(err))
    if min(e_index, e_weight) < m:
        e = min(e_index, e_weight)
        a, b = int(s_t[e].item()), int(d_t[e].item())
        if e == e_index:
            raise ValueError(f"edge ({a}, {b}) out of range for n={n}")
        raise ValueError(f"edge ({a}, {b}) weight must be finite, got {float(w_t[e].item())!r}")
    if e_range < m:
        if dt == torch.int32:
            raise ValueError(f"int32 storage needs integral entries with magnitude below {_lib.I32_LIMIT}")
        raise ValueError(f"entries do not fit {dt} storage")
    st = _read_stats(stats)
    integer = dt == torch.int32 or (st.non_integral == 0 and st.over_limit == 0)
    return TropicalMatrix._wrap(SemiringKind.MIN_PLUS, out, integer, _stats_bound(st))


def graph_to_matrix(g, *, dtype: "torch.dtype | None" = None, device=None) -> TropicalMatrix:
    """graph_io.graph_to_matrix (graph_io.py:158-165) for a ``Graph`` (ours or
    the reference's: anything with ``.n`` and ``.edges`` = ((src, dst,
    weight), ...)).  A ``random_graph`` recipe is generated on the GPU."""
    if isinstance(g, RandomGraph):
        n, p, wr, seed = g.recipe
        return random_graph_matrix(n, p, wr, seed, dtype=dtype, device=device)
    edges = tuple(g.edges)
    if edges:
        arr = np.asarray([(float(a), float(b), float(w)) for a, b, w in edges], dtype=np.float64)
        src, dst, w = arr[:, 0].astype(np.int64), arr[:, 1].astype(np.int64), arr[:, 2]
    else:
        src = dst = np.zeros(0, dtype=np.int64)
        w = np.zeros(0, dtype=np.float64)
    return edges_to_matrix(int(g.n), src, dst, w, dtype=dtype, device=device)


# ---------------------------------------------------------------------------
# graph objects (reference graph_io.py:55-87, 168-187, 273-304)
# ---------------------------------------------------------------------------
class Graph:
    """Directed weighted graph with finite weights (reference graph_io.Graph,
    graph_io.py:55-87): duplicates of one (src, dst) keep the minimum weight,
    -0.0 becomes 0.0, and the edges are sorted by (src, dst), so equal graphs
    compare equal.  Immutable."""

    __slots__ = ("n", "_edges")

    def __init__(self, n: int, edges=()):
        if not isinstance(n, int) or n < 1:
            raise ValueError(f"vertex count must be a positive integer, got {n!r}")
        best: "dict[tuple[int, int], float]" = {}
        for src, dst, weight in edges:
            if not (0 <= src < n) or not (0 <= dst < n):
                raise ValueError(f"edge ({src}, {dst}) out of range for n={n}")
            w = float(weight)
            if math.isnan(w) or math.isinf(w):
                raise ValueError(f"edge ({src}, {dst}) weight must be finite, got {w!r}")
            if w == 0.0:
                w = 0.0
            key = (int(src), int(dst))
            if key not in best or w < best[key]:
                best[key] = w
        object.__setattr__(self, "n", n)
        object.__setattr__(self, "_edges", tuple((a, b, best[(a, b)]) for a, b in sorted(best)))

    def __setattr__(self, name, value):
        raise AttributeError("Graph is immutable")

    @property
    def edges(self) -> "tuple[tuple[int, int, float], ...]":
        return self._edges

    @property
    def edge_count(self) -> int:
        return len(self.edges)

    def __eq__(self, other) -> bool:
        if not hasattr(other, "n") or not hasattr(other, "edges"):
            return NotImplemented
        return self.n == other.n and tuple(self.edges) == tuple(other.edges)

    def __hash__(self) -> int:
        return hash((self.n, self.edges))

    def __repr__(self) -> str:
        return f"Graph(n={self.n}, edge_count={self.edge_count})"


class RandomGraph(Graph):
    """``random_graph(n, p, weight_range, seed)`` (graph_io.py:273-304) kept as
    its recipe: ``graph_to_matrix`` builds the matrix on the GPU straight from
    the PCG64 stream (no edge list at all); ``.edges`` materialises the
    reference's tuple on first use (host, vectorised)."""

    __slots__ = ("recipe",)

    def __init__(self, n: int, p: float, weight_range, seed: int):
        p, low, high = _check(n, p, weight_range)
        object.__setattr__(self, "n", n)
        object.__setattr__(self, "_edges", None)
        object.__setattr__(self, "recipe", (n, p, (weight_range[0], weight_range[1]), int(seed)))

    @property
    def edges(self) -> "tuple[tuple[int, int, float], ...]":
        if self._edges is None:
            n, p, wr, seed = self.recipe
            out = []
            for r0, block in dense_rows(n, p, wr, seed):
                rows, cols = np.nonzero(np.isfinite(block))
                vals = block[rows, cols]
                keep = (rows + r0) != cols
                out.extend(zip((rows[keep] + r0).tolist(), cols[keep].tolist(), vals[keep].tolist()))
            object.__setattr__(self, "_edges", tuple(out))
        return self._edges


def random_graph(n: int, edge_probability: float, weight_range, seed: int) -> RandomGraph:
    """Seed-deterministic random digraph (reference graph_io.py:273-304); see
    RandomGraph.  graph_to_matrix(random_graph(...)) is generated on the GPU."""
    return RandomGraph(n, edge_probability, weight_range, seed)


def matrix_to_graph(m: TropicalMatrix) -> Graph:
    """Inverse of graph_to_matrix (reference graph_io.py:168-187): finite
    off-diagonal entries become edges; diagonal entries only when negative."""
    if m.kind is not SemiringKind.MIN_PLUS:
        raise ValueError("only min-plus matrices describe graphs")
    if m.n_rows != m.n_cols:
        raise ValueError(f"adjacency matrix must be square, got {m.shape}")
    a = m.to_numpy()
    keep = np.isfinite(a)
    diag = np.eye(a.shape[0], dtype=bool)
    keep &= ~diag | (a < 0.0)
    rows, cols = np.nonzero(keep)
    return Graph(m.n_rows, zip(rows.tolist(), cols.tolist(), a[rows, cols].tolist()))

"""NumPy restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

Every function follows the reference algorithm it names (file:line under
/root/reference/pkg/src/btas/), operating on *oriented* float64 arrays (the
reference's own storage form, matrix.py:3-7) and returning oriented float64
arrays plus the saturation bit, so results compare bytewise with the
reference's ``.data`` and with the GPU storage converted to float64.

``storage`` selects the element type whose arithmetic is restated:
  "f64"  the reference itself (candidate a+b in float64; integer limit 2^53)
  "f32"  float32 storage: candidate rounded once to float32 (for float32
         operands the float64 sum is exact or double rounding is innocuous,
         53 >= 2*24+2, so this equals the float32 FADD); integer limit 2^53,
         float overflow = float32 overflow
  "i32"  int32 storage: exact integers, saturation limit 2^28 (always)
"""

from __future__ import annotations

import math

import numpy as np

MIN, MAX = "minplus", "maxplus"
INT_LIMIT = {"f64": float(2**53), "f32": float(2**53), "i32": float(2**28)}


def eps(kind: str) -> float:
    """Oriented Infinity (reference matrix.py:74-75)."""
    return math.inf if kind == MIN else -math.inf


def combine(kind: str):
    """⊕ ufunc (reference matrix.py:78-79)."""
    return np.minimum if kind == MIN else np.maximum


def orient(kind: str, symbolic) -> np.ndarray:
    """Symbolic form (math.inf = Infinity) -> oriented float64 (matrix.py:82-95)."""
    arr = np.array(symbolic, dtype=np.float64) + 0.0
    if kind == MAX:
        arr[arr == math.inf] = -math.inf
    return arr


def to_storage(arr: np.ndarray, storage: str) -> np.ndarray:
    """Round oriented float64 values to the storage element type (as float64)."""
    if storage == "f32":
        with np.errstate(over="ignore"):
            return arr.astype(np.float32).astype(np.float64)
    return arr


def _limit(storage: str, integer: bool) -> float:
    if storage == "i32":
        return INT_LIMIT["i32"]
    return INT_LIMIT[storage] if integer else math.inf


def saturation_possible(x: np.ndarray, y: np.ndarray, storage: str, integer: bool) -> bool:
    """The exact screen of _saturation_limit (matrix.py:297-312): no candidate
    can overflow when max|x_fin| + max|y_fin| stays under the limit."""
    bound = 0.0
    for op in (x, y):
        fin = op[np.isfinite(op)]
        bound += float(np.max(np.abs(fin))) if fin.size else 0.0
    limit = _limit(storage, integer)
    if not math.isinf(limit):
        return bound >= limit
    return math.isinf(float(to_storage(np.array([bound]), storage)[0]))


def product_tile(x: np.ndarray, y: np.ndarray, kind: str, storage: str, integer: bool, screen: bool = True):
    """One output block of the tropical product with the masked-overflow rule
    of _product_tile (matrix.py:315-346): candidates x[r,k] + y[k,c],
    finite (x) finite sums that overflow / reach the integer limit -> ε.
    ``screen=False`` skips the mask (the caller proved no overflow)."""
    with np.errstate(over="ignore", invalid="ignore"):
        block = x[:, :, None] + y[None, :, :]
    block = to_storage(block, storage)
    if not screen:
        return combine(kind).reduce(block, axis=1), False
    limit = _limit(storage, integer)
    bad = np.isinf(block) if math.isinf(limit) else (np.abs(block) >= limit)
    saturated = False
    if bad.any():
        bad &= np.isfinite(x)[:, :, None]
        bad &= np.isfinite(y)[None, :, :]
        if bad.any():
            block[bad] = eps(kind)
            saturated = True
    return combine(kind).reduce(block, axis=1), saturated


def matmul(x: np.ndarray, y: np.ndarray, kind: str, storage: str = "f64", integer: bool = False,
           acc: "np.ndarray | None" = None, tile_rows: int = 16, tile_cols: int = 256, workers: int = 1):
    """Tropical product over output tiles, k never split (matrix.py:349-400).
    ``workers`` > 1 fans the tiles over a thread pool exactly like the
    reference (matrix.py:284-294,393-397; NumPy releases the GIL).
    Returns (oriented float64 result, saturated)."""
    assert x.shape[1] == y.shape[0]
    m, n = x.shape[0], y.shape[1]
    out = np.empty((m, n), dtype=np.float64)
    spans = [(r0, c0) for r0 in range(0, m, tile_rows) for c0 in range(0, n, tile_cols)]
    screen = saturation_possible(x, y, storage, integer)

    def run(span):
        r0, c0 = span
        blk, sat = product_tile(x[r0 : r0 + tile_rows], y[:, c0 : c0 + tile_cols], kind, storage, integer, screen)
        out[r0 : r0 + tile_rows, c0 : c0 + tile_cols] = blk
        return sat

    if workers > 1 and len(spans) > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=workers) as pool:
            saturated = any(pool.map(run, spans))
    else:
        saturated = any([run(s) for s in spans])
    if acc is not None:
        combine(kind)(out, acc, out=out)
    return out, saturated


def matvec(a: np.ndarray, v: np.ndarray, kind: str, storage: str = "f64", integer: bool = False):
    """out(i) = ⊕_k a(i,k) ⊗ v(k), always masking overflow (matrix.py:403-425)."""
    with np.errstate(over="ignore"):
        block = a + v[None, :]
    block = to_storage(block, storage)
    limit = _limit(storage, integer)
    bad = np.isinf(block) if math.isinf(limit) else np.abs(block) >= limit
    bad &= np.isfinite(a)
    bad &= np.isfinite(v)[None, :]
    saturated = bool(bad.any())
    if saturated:
        block[bad] = eps(kind)
    return combine(kind).reduce(block, axis=1), saturated


def ew_add(a: np.ndarray, b: np.ndarray, kind: str) -> np.ndarray:
    """Elementwise ⊕ (matrix.py:271-277)."""
    return combine(kind)(a, b)


def identity(kind: str, n: int) -> np.ndarray:
    """0 diagonal, ε elsewhere (matrix.py:257-263)."""
    arr = np.full((n, n), eps(kind))
    np.fill_diagonal(arr, 0.0)
    return arr


def matrix_power(a: np.ndarray, p: int, kind: str, storage: str = "f64", integer: bool = False):
    """LSB-first binary exponentiation (matrix.py:428-448)."""
    result, base, e, sat = None, a, p, False
    while True:
        if e & 1:
            if result is None:
                result = base
            else:
                result, s = matmul(result, base, kind, storage, integer)
                sat |= s
        e >>= 1
        if not e:
            return result, sat
        base, s = matmul(base, base, kind, storage, integer)
        sat |= s


def closure_base(adj: np.ndarray) -> np.ndarray:
    """I ⊕ A (apsp.py:80-90)."""
    base = np.array(adj)
    np.fill_diagonal(base, np.minimum(np.diagonal(base), 0.0))
    return base


def fw_limit(storage: str, integer: bool) -> float:
    if storage == "i32":
        return INT_LIMIT["i32"]
    if integer:
        return INT_LIMIT[storage]
    return float(np.finfo(np.float32).max) if storage == "f32" else math.inf


def floyd_warshall(adj: np.ndarray, storage: str = "f64", integer: bool = False):
    """Sequential k-rounds with the reference's screen / masked rounds
    (apsp.py:93-133).  Returns (distances, negative_cycle, saturated)."""
    n = adj.shape[0]
    d = closure_base(adj)
    finite = d[np.isfinite(d)]
    max_abs = float(np.max(np.abs(finite))) if finite.size else 0.0
    limit = fw_limit(storage, integer)
    saturated = False
    masked = not (2.0 * (n + 1) * max_abs < limit)
    for k in range(n):
        with np.errstate(over="ignore", invalid="ignore"):
            cand = np.add.outer(d[:, k], d[k, :])
        cand = to_storage(cand, storage)
        if masked:
            lim = limit if storage != "f32" or integer else math.inf
            bad = np.isinf(cand) if math.isinf(lim) else np.abs(cand) >= lim
            bad &= np.isfinite(d[:, k])[:, None]
            bad &= np.isfinite(d[k, :])[None, :]
            if bad.any():
                cand[bad] = math.inf
                saturated = True
        np.minimum(d, cand, out=d)
    return d, bool((np.diagonal(d) < 0.0).any()), saturated


def apsp_by_squaring(adj: np.ndarray, storage: str = "f64", integer: bool = False):
    """(I ⊕ A)^(n-1) by squaring with fixpoint exit and negative-cycle probe
    (apsp.py:136-178).  Returns (distances, negative_cycle, multiplications,
    saturated)."""
    n = adj.shape[0]
    base = closure_base(adj)
    mults, fixpoint, sat = 0, False, False
    if n == 1:
        d = identity(MIN, 1)
    else:
        d, power = base, 1
        while power < n - 1:
            sq, s = matmul(d, d, MIN, storage, integer)
            sat |= s
            mults += 1
            if sq.tobytes() == d.tobytes():
                fixpoint = True
                break
            d, power = sq, power * 2
    if fixpoint:
        neg = bool((np.diagonal(d) < 0.0).any())
    else:
        probe, s = matmul(d, base, MIN, storage, integer)
        sat |= s
        neg = probe.tobytes() != d.tobytes() or bool((np.diagonal(probe) < 0.0).any())
    return d, neg, mults, sat


def closure_rows(adj: np.ndarray, rows, storage: str = "f64", integer: bool = False, max_iter: int = 10_000,
                 gemm=None):
    """Sampled-row closure oracle: rows R of (I ⊕ A)* by
    iterating R <- R ⊗ (I ⊕ A) from R = base[rows] until R stops changing
    (Bellman-Ford by rows).  Equals the corresponding rows of the closure
    when there is no negative cycle.  ``gemm`` may be a faster restatement
    with the matmul signature (e.g. the C oracle)."""
    gemm = gemm or (lambda a, b: matmul(a, b, MIN, storage, integer)[0])
    base = closure_base(adj)
    r = base[np.asarray(rows)]
    for _ in range(max_iter):
        nxt = gemm(r, base)
        if nxt.tobytes() == r.tobytes():
            return r
        r = nxt
    raise RuntimeError("closure rows did not converge (negative cycle?)")


def predecessors(adj: np.ndarray, dist: np.ndarray) -> np.ndarray:
    """Predecessor matrix restated (the GPU extension's definition; the
    reference has no path output): P[i, j] = the smallest k != j with
    dist[i, k] + adj[k, j] == dist[i, j], -1 if i == j or none / infinite.
    Oriented min-plus float64 inputs, exact integer weights."""
    n = adj.shape[0]
    a = np.array(adj, dtype=np.float64)
    np.fill_diagonal(a, math.inf)
    out = np.full((n, n), -1, dtype=np.int32)
    for i in range(n):
        with np.errstate(invalid="ignore"):
            cand = dist[i][:, None] + a  # [k, j]
        best = cand.min(axis=0)
        k = np.argmin(cand, axis=0)  # first minimum
        ok = np.isfinite(best) & (best == dist[i])
        ok[i] = False
        out[i, ok] = k[ok]
    return out

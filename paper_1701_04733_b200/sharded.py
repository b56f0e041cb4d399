"""Row-sharded repeated-squaring APSP over several GPUs (one process per GPU).

Extends ``apsp_by_squaring`` (reference apsp.py:136-178) to P ranks of a
``torch.distributed`` group (NCCL over NVLink/NVSwitch on B200):

  * every rank holds the full D (n x n) and its own row block of D_next;
    rows are padded to P equal chunks of ``chunk`` rows (a multiple of the
    128-row GEMM tile) so the exchange is a single in-place all-gather;
  * step: D_next[rows_r] = D[rows_r] ⊗ D  with the fixpoint compare against
    D[rows_r] fused in the GEMM epilogue, then  all_gather(D_next)  and one
    all_reduce(MAX) of the {changed, diag<0, saturated} flag words;
  * rows are independent, so D is byte-identical for every P (and to the
    single-GPU result) and the multiplication count is the same.

The exchange volume per step is (P-1)/P * n^2 * 4 bytes per rank (≈15 GB at
n = 65536 fp32, ≈20 ms over NVLink 5) against ≈n^3/P pairs of compute, so
the all-gather is <2 % of a step; it is issued on the compute stream.

``gemm_rows`` is injectable so the host-side logic (partition, collectives,
loop control, probe) is testable with the gloo backend on CPU
(tests/test_sharded.py); the default is the CUDA tropical GEMM.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

from . import _lib

FLAG_WORDS = 3  # changed, diag_neg, saturated


@dataclass
class ShardedResult:
    distances: torch.Tensor  # full n x n oriented storage (every rank)
    negative_cycle: bool
    multiplications_performed: int
    saturated: bool


def apsp_by_squaring_distributed(adj, group=None):
    """``apsp_by_squaring`` (reference apsp.py:136-178) row-sharded over the
    ranks of ``group`` (one process per GPU, NCCL).  Every rank passes the
    same adjacency matrix and receives the full ApspReport; distances,
    multiplication count and negative-cycle flag equal the single-GPU
    result byte for byte."""
    from .apsp import Algorithm, ApspReport, DistanceMatrix, _closure_base, _require_square_minplus
    from .matrix import TropicalMatrix
    from .semiring import _note_saturation

    n = _require_square_minplus(adj)
    base = _closure_base(adj)
    res = apsp_by_squaring_sharded(base.data.contiguous(), group=group,
                                   gemm_rows=_cuda_gemm_rows(True, base.integer), integer=base.integer)
    if res.saturated:
        _note_saturation()
    dist_m = TropicalMatrix._wrap(adj.kind, res.distances.contiguous(), base.integer)
    return ApspReport(distances=DistanceMatrix(n, dist_m), algorithm=Algorithm.REPEATED_SQUARING,
                      negative_cycle=res.negative_cycle, multiplications_performed=res.multiplications_performed)


def partition(n: int, world: int, align: int = 128) -> "tuple[int, list[tuple[int, int]]]":
    """Equal, tile-aligned row chunks: returns (chunk, [(r0, r1) per rank]).
    Ranks past the end get empty ranges."""
    per = -(-n // world)
    chunk = -(-per // align) * align
    spans = []
    for r in range(world):
        r0 = min(n, r * chunk)
        spans.append((r0, min(n, r0 + chunk)))
    return chunk, spans


def _cuda_gemm_rows(kind_min: bool, integer: bool) -> Callable:
    from .matrix import _gemm
    from .semiring import SemiringKind

    kind = SemiringKind.MIN_PLUS if kind_min else SemiringKind.MAX_PLUS

    def gemm_rows(a_rows: torch.Tensor, b: torch.Tensor, cprev: torch.Tensor, out: torch.Tensor):
        _, flags = _gemm(a_rows, b, kind, integer, out=out, cprev=cprev)
        return torch.stack([flags[_lib.FLAG_CHANGED], flags[_lib.FLAG_DIAG_NEG], flags[_lib.FLAG_SATURATED]])

    return gemm_rows


def _diag_rows(d_rows: torch.Tensor, r0: int) -> torch.Tensor:
    """any(d[i, i] < 0) over this rank's rows, as an int flag tensor."""
    m = d_rows.shape[0]
    if m == 0:
        return torch.zeros((), dtype=torch.int32, device=d_rows.device)
    idx = torch.arange(m, device=d_rows.device)
    diag = d_rows[idx, idx + r0]
    return (diag < 0).any().to(torch.int32)


def apsp_by_squaring_sharded(base: torch.Tensor, group=None, gemm_rows: "Callable | None" = None,
                             integer: bool = True, align: int = 128) -> ShardedResult:
    """Closure of the closure base ``base`` (n x n oriented min-plus storage,
    identical on every rank) by repeated squaring, row-sharded over the
    group.  Mirrors apsp.py:136-178 step for step (fixpoint exit, counted
    detecting square, uncounted probe)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = base.shape[0]
    dev = base.device
    gemm_rows = gemm_rows or _cuda_gemm_rows(True, integer)
    chunk, spans = partition(n, world, align)
    r0, r1 = spans[rank]

    bufs = [torch.empty((world * chunk, n), dtype=base.dtype, device=dev) for _ in range(2)]
    bufs[0][:n].copy_(base)
    cur = 0
    mults, fixpoint, sat = 0, False, False
    if n == 1:
        d = torch.zeros((1, 1), dtype=base.dtype, device=dev)  # identity of size 1
        res_d = d
    else:
        power = 1
        while power < n - 1:
            d, nxt = bufs[cur], bufs[1 - cur]
            flags = gemm_rows(d[r0:r1], d[:n], d[r0:r1], nxt[r0:r1]) if r1 > r0 else \
                torch.zeros(FLAG_WORDS, dtype=torch.int32, device=dev)
            my_chunk = nxt[rank * chunk : (rank + 1) * chunk]
            dist.all_gather_into_tensor(nxt, my_chunk, group=group)
            flags = flags.to(torch.int32)
            dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
            f = flags.cpu().tolist()
            mults += 1
            sat |= bool(f[2])
            if not f[0]:
                fixpoint = True
                break
            cur = 1 - cur
            power *= 2
        res_d = bufs[cur][:n]
    if fixpoint:
        neg = _diag_rows(res_d[r0:r1], r0).reshape(1)
        dist.all_reduce(neg, op=dist.ReduceOp.MAX, group=group)
        negative = bool(neg.item())
    elif n == 1:
        b = base.reshape(1, 1)
        negative = bool((b < 0).any().item())  # probe I ⊗ base = base; != I iff base[0,0] < 0
    else:
        probe_out = torch.empty((max(r1 - r0, 0), n), dtype=base.dtype, device=dev)
        flags = gemm_rows(res_d[r0:r1], base, res_d[r0:r1], probe_out) if r1 > r0 else \
            torch.zeros(FLAG_WORDS, dtype=torch.int32, device=dev)
        flags = flags.to(torch.int32).clone()
        # the kernel's diagonal test sees block-local rows; test the true
        # diagonal of this row block here
        flags[1] = _diag_rows(probe_out, r0)
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
        f = flags.cpu().tolist()
        sat |= bool(f[2])
        negative = bool(f[0]) or bool(f[1])
    return ShardedResult(res_d, negative, mults, sat)

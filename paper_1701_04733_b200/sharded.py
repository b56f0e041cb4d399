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
the all-gather is <2 % of a step.

Two exchanges are implemented:
  * "peer" (default on NCCL when symmetric memory is available): D and D_next
    live in torch symmetric memory (every rank maps every peer's buffers
    over NVLink); btas_gemm_peers writes each finished output tile into the
    rank's own D_next AND into the same rows of every peer's D_next from the
    GEMM epilogue, so the all-gather disappears into the tile stores and
    overlaps the compute tile by tile.  The flag all_reduce that ends every
    step doubles as the barrier: a rank enters it only after its GEMM (which
    ends with a system-scope fence) has completed, and it starts the next
    step — which overwrites the buffer its peers read in this one — only
    after every rank has entered it.
  * "nccl": GEMM into the local rows, then all_gather_into_tensor.

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
from .matrix import _host_read

FLAG_WORDS = 3  # changed, diag_neg, saturated


@dataclass
class ShardedResult:
    distances: torch.Tensor  # full n x n oriented storage (every rank)
    negative_cycle: bool
    multiplications_performed: int
    saturated: bool
    exchange: str = "nccl"


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
    res = apsp_by_squaring_sharded(base.data.contiguous(), group=group, integer=base.integer)
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

    def gemm_rows(a_rows: torch.Tensor, b: torch.Tensor, cprev: torch.Tensor, out: torch.Tensor, peers=None):
        _, flags = _gemm(a_rows, b, kind, integer, out=out, cprev=cprev, peers=peers)
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


def _peer_buffers(shape, dtype, dev, group, world, count=2):
    """``count`` symmetric-memory buffers and, per buffer, the base addresses
    of the other ranks' copies; None when symmetric memory is unavailable."""
    try:
        import torch.distributed._symmetric_memory as symm_mem

        bufs, ptrs = [], []
        me = dist.get_rank(group)
        for _ in range(count):
            t = symm_mem.empty(*shape, dtype=dtype, device=dev)
            h = symm_mem.rendezvous(t, group if group is not None else dist.group.WORLD)
            addrs = [int(a) for a in h.buffer_ptrs]
            if len(addrs) != world or addrs[me] != t.data_ptr():
                return None
            bufs.append(t)
            ptrs.append([a for q, a in enumerate(addrs) if q != me])
        return bufs, ptrs
    except Exception as exc:  # no NVLink P2P / no symmetric-memory backend
        import os
        import sys

        if os.environ.get("BTAS_DEBUG"):
            print(f"[btas] symmetric memory unavailable: {type(exc).__name__}: {exc}", file=sys.stderr)
        return None


def _want_peer_exchange(group, world: int, dev: torch.device) -> bool:
    import os

    # auto: fused when there is someone to exchange with (NCCL groups);
    # peer: always, on any backend (the one-rank and same-GPU multi-process
    # tests of the symmetric-memory plumbing); nccl: never
    mode = os.environ.get("BTAS_EXCHANGE", "auto")
    if mode == "nccl" or world - 1 > 7 or dev.type != "cuda" or (world < 2 and mode != "peer"):
        return False
    return mode == "peer" or dist.get_backend(group) == "nccl"


def apsp_by_squaring_sharded(base: torch.Tensor, group=None, gemm_rows: "Callable | None" = None,
                             integer: bool = True, align: int = 128,
                             peer_buffers: "Callable | None" = None) -> ShardedResult:
    """Closure of the closure base ``base`` (n x n oriented min-plus storage,
    identical on every rank) by repeated squaring, row-sharded over the
    group.  Mirrors apsp.py:136-178 step for step (fixpoint exit, counted
    detecting square, uncounted probe).  With the default CUDA ``gemm_rows``
    on NCCL the exchange is fused into the GEMM epilogue (see module doc).
    ``peer_buffers(shape, dtype, device, group, world)`` may replace the
    symmetric-memory allocation (it returns the two local buffers and, per
    buffer, the other ranks' base addresses): the multi-process tests map
    buffers between processes on one GPU with CUDA IPC this way."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = base.shape[0]
    dev = base.device
    fused_ok = gemm_rows is None and _want_peer_exchange(group, world, dev)
    gemm_rows = gemm_rows or _cuda_gemm_rows(True, integer)
    chunk, spans = partition(n, world, align)
    r0, r1 = spans[rank]

    alloc = peer_buffers or _peer_buffers
    peer = alloc((world * chunk, n), base.dtype, dev, group, world) if fused_ok else None
    if fused_ok:  # every rank must take the same exchange
        ok = torch.tensor([1 if peer is not None else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if not int(_host_read(ok)[0]):
            peer = None
    if peer is not None:
        bufs, peer_ptrs = peer
        row_off = r0 * n * base.element_size()
    else:
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
            if peer is not None:
                # my rows land in every peer's D_next from the epilogue
                peers = [a + row_off for a in peer_ptrs[1 - cur]]
                flags = gemm_rows(d[r0:r1], d[:n], d[r0:r1], nxt[r0:r1], peers=peers) if r1 > r0 else \
                    torch.zeros(FLAG_WORDS, dtype=torch.int32, device=dev)
            else:
                flags = gemm_rows(d[r0:r1], d[:n], d[r0:r1], nxt[r0:r1]) if r1 > r0 else \
                    torch.zeros(FLAG_WORDS, dtype=torch.int32, device=dev)
                my_chunk = nxt[rank * chunk : (rank + 1) * chunk]
                dist.all_gather_into_tensor(nxt, my_chunk, group=group)
            flags = flags.to(torch.int32)
            dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
            f = _host_read(flags).tolist()
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
        f = _host_read(flags).tolist()
        sat |= bool(f[2])
        negative = bool(f[0]) or bool(f[1])
    return ShardedResult(res_d, negative, mults, sat, "peer" if peer is not None else "nccl")


def apsp_by_squaring_emulated(adj, world: int):
    """The fused peer-store squaring of ``apsp_by_squaring_sharded`` with
    ``world`` virtual ranks on ONE GPU, run one after another on one stream:
    each virtual rank owns its own D / D_next pair and its GEMM stores its
    rows into every other virtual rank's D_next through btas_gemm_peers,
    exactly the addresses the multi-GPU path uses.  Used by the GPU tests to
    check the fused exchange bit for bit; returns (ApspReport, per-rank D)."""
    from .apsp import Algorithm, ApspReport, DistanceMatrix, _closure_base, _require_square_minplus
    from .matrix import TropicalMatrix

    n = _require_square_minplus(adj)
    base = _closure_base(adj)
    b = base.data.contiguous()
    dev = b.device
    gemm_rows = _cuda_gemm_rows(True, base.integer)
    chunk, spans = partition(n, world)
    bufs = [[torch.empty((world * chunk, n), dtype=b.dtype, device=dev) for _ in range(2)] for _ in range(world)]
    for r in range(world):
        bufs[r][0][:n].copy_(b)
    esz = b.element_size()
    cur, mults, fixpoint, sat = 0, 0, False, False
    power = 1
    while n > 1 and power < n - 1:
        flags = torch.zeros(FLAG_WORDS, dtype=torch.int32, device=dev)
        for r, (r0, r1) in enumerate(spans):
            if r1 <= r0:
                continue
            d, nxt = bufs[r][cur], bufs[r][1 - cur]
            peers = [bufs[q][1 - cur].data_ptr() + r0 * n * esz for q in range(world) if q != r]
            flags = torch.maximum(flags, gemm_rows(d[r0:r1], d[:n], d[r0:r1], nxt[r0:r1], peers=peers).to(torch.int32))
        f = _host_read(flags).tolist()
        mults += 1
        sat |= bool(f[2])
        if not f[0]:
            fixpoint = True
            break
        cur = 1 - cur
        power *= 2
    per_rank = [bufs[r][cur][:n] for r in range(world)]
    d = per_rank[0]
    if n == 1:
        negative = bool((b < 0).any().item())  # probe I ⊗ base = base
        d = torch.zeros_like(b)  # identity of size 1
        per_rank = [d] * world
    elif fixpoint:
        negative = any(bool(_diag_rows(d[r0:r1], r0).item()) for r0, r1 in spans if r1 > r0)
    else:
        negative = False
        for r0, r1 in spans:
            if r1 <= r0:
                continue
            probe = torch.empty((r1 - r0, n), dtype=b.dtype, device=dev)
            fl = gemm_rows(d[r0:r1], b, d[r0:r1], probe)
            negative |= bool(fl[0].item()) or bool(_diag_rows(probe, r0).item())
            sat |= bool(fl[2].item())
    if sat:
        from .semiring import _note_saturation

        _note_saturation()
    dist_m = TropicalMatrix._wrap(adj.kind, d.contiguous(), base.integer)
    rep = ApspReport(distances=DistanceMatrix(n, dist_m), algorithm=Algorithm.REPEATED_SQUARING,
                     negative_cycle=negative, multiplications_performed=mults)
    return rep, per_rank


# ---------------------------------------------------------------------------
# row-sharded matmul / matvec (GEMM and matvec rows)
# ---------------------------------------------------------------------------
def _cuda_gemm_plain(kind, integer: bool) -> Callable:
    from .matrix import _gemm

    def gemm_rows(a_rows, b, out, z_rows=None, peers=None):
        _, flags = _gemm(a_rows, b, kind, integer, out=out, z=z_rows, peers=peers)
        return flags[_lib.FLAG_SATURATED].reshape(1).to(torch.int32)

    return gemm_rows


def matmul_sharded(x: torch.Tensor, y: torch.Tensor, kind, integer: bool, z: "torch.Tensor | None" = None,
                   group=None, gemm_rows: "Callable | None" = None, align: int = 128,
                   peer_buffers: "Callable | None" = None) -> "tuple[torch.Tensor, bool]":
    """Rows of ``x ⊗ y [⊕ z]`` (oriented storage, the same operands on every
    rank) split over the ranks of ``group``: rank r computes rows
    [r*chunk, (r+1)*chunk) against the replicated ``y`` and every rank ends
    with the full product.  Rows are independent (k is never split), so the
    product is byte-identical to the single-GPU matmul for any P.  On NCCL
    groups with symmetric memory the exchange is fused into the GEMM
    epilogue (peer stores of each finished tile into every rank's copy);
    otherwise NCCL all_gather.  Returns (product, saturated on any rank)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m, n = x.shape[0], y.shape[1]
    dev = x.device
    fused_ok = gemm_rows is None and z is None and _want_peer_exchange(group, world, dev)
    gemm_rows = gemm_rows or _cuda_gemm_plain(kind, integer)
    chunk, spans = partition(m, world, align)
    r0, r1 = spans[rank]
    peer = (peer_buffers or _peer_buffers)((world * chunk, n), x.dtype, dev, group, world, 1) if fused_ok else None
    if fused_ok:  # every rank must take the same exchange
        ok = torch.tensor([1 if peer is not None else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if not int(_host_read(ok)[0]):
            peer = None
    if peer is not None:
        bufs, peer_ptrs = peer
        full = bufs[0]
        peers = [a + r0 * n * x.element_size() for a in peer_ptrs[0]]
        sat = gemm_rows(x[r0:r1], y, full[r0:r1], peers=peers) if r1 > r0 else \
            torch.zeros(1, dtype=torch.int32, device=dev)
    else:
        full = torch.empty((world * chunk, n), dtype=x.dtype, device=dev)
        sat = gemm_rows(x[r0:r1], y, full[r0:r1], z_rows=None if z is None else z[r0:r1]) if r1 > r0 else \
            torch.zeros(1, dtype=torch.int32, device=dev)
        dist.all_gather_into_tensor(full, full[rank * chunk : (rank + 1) * chunk], group=group)
    # the flag all-reduce doubles as the barrier after the peers' stores
    sat = sat.to(torch.int32).reshape(1).clone()
    dist.all_reduce(sat, op=dist.ReduceOp.MAX, group=group)
    saturated = bool(int(_host_read(sat)[0]))
    out = full[:m]
    return (out if world * chunk == m and peer is None else out.clone()), saturated


def matmul_distributed(x, y, accumulate_into=None, group=None):
    """``matmul`` (reference matrix.py:349-400) row-sharded over the ranks of
    ``group`` (one process per GPU): same arguments and result on every
    rank, byte-identical to the single-GPU product; the saturation flag is
    set on every rank when any rank saturated."""
    from .matrix import (DimensionMismatch, TropicalMatrix, _check_same_kind, _check_same_storage, _max_bound,
                         _rowmajor, _sum_bound)
    from .semiring import _note_saturation

    _check_same_kind(x, y)
    if x.n_cols != y.n_rows:
        raise DimensionMismatch(f"matmul inner dimensions differ: {x.shape} x {y.shape}")
    _check_same_storage(x, y)
    integer = x.integer and y.integer
    z = None
    if accumulate_into is not None:
        _check_same_kind(x, accumulate_into)
        if accumulate_into.shape != (x.n_rows, y.n_cols):
            raise DimensionMismatch(
                f"accumulate_into shape {accumulate_into.shape} does not match output {(x.n_rows, y.n_cols)}")
        _check_same_storage(x, accumulate_into)
        integer = integer and accumulate_into.integer
        z = _rowmajor(accumulate_into.data)
    out, sat = matmul_sharded(_rowmajor(x.data), _rowmajor(y.data), x.kind, integer, z=z, group=group)
    if sat:
        _note_saturation()
    bound = _sum_bound(x.abs_bound, y.abs_bound)
    if accumulate_into is not None:
        bound = _max_bound(bound, accumulate_into.abs_bound)
    return TropicalMatrix._wrap(x.kind, out, integer, bound)


def matvec_distributed(a, v, group=None):
    """``matvec`` (reference matrix.py:403-425) with the rows of ``a`` split
    over the ranks: each rank streams only its rows of A from HBM (the
    HBM-bound pass scales with P) and the n-element result is all-gathered.
    Same result on every rank, byte-identical to matvec."""
    from .matrix import (DimensionMismatch, TropicalVector, _check_same_kind, _check_same_storage, _matvec,
                         _rowmajor, _sum_bound)
    from .semiring import _note_saturation

    _check_same_kind(a, v)
    if a.n_cols != len(v):
        raise DimensionMismatch(f"matvec dimensions differ: {a.shape} x {len(v)}")
    _check_same_storage(a, v)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m = a.n_rows
    dev = a.device
    chunk, spans = partition(m, world, 1)
    r0, r1 = spans[rank]
    integer = a.integer and v.integer
    full = torch.empty((world * chunk,), dtype=a.dtype, device=dev)
    sat = torch.zeros(1, dtype=torch.int32, device=dev)
    if r1 > r0:
        out, flags = _matvec(_rowmajor(a.data)[r0:r1], v.data.reshape(1, -1), a.kind, integer,
                             _sum_bound(a.abs_bound, v.abs_bound))
        full[r0:r1].copy_(out.reshape(-1))
        sat = flags[_lib.FLAG_SATURATED].reshape(1).clone()
    dist.all_gather_into_tensor(full, full[rank * chunk : (rank + 1) * chunk], group=group)
    dist.all_reduce(sat, op=dist.ReduceOp.MAX, group=group)
    if int(_host_read(sat)[0]):
        _note_saturation()
    return TropicalVector._wrap(a.kind, full[:m].clone(), integer, _sum_bound(a.abs_bound, v.abs_bound))


# ---------------------------------------------------------------------------
# row-sharded Floyd-Warshall (pivot-panel broadcast)
# ---------------------------------------------------------------------------
FW_STAGE_INIT, FW_STAGE_DIAG, FW_STAGE_OWNER, FW_STAGE_REST = 0, 4, 5, 6


class _FwRank:
    """One rank's slab, workspace(s) and flag words for btas_fw_dist_group.
    With the fused broadcast the rank holds two workspaces, alternated by the
    parity of the lookahead group (``alloc(nbytes)`` may place them in
    memory the peers can map)."""

    def __init__(self, rank, r0, rows, slab, code, n, dev, nbuf=1, alloc=None):
        import ctypes

        self.rank, self.r0, self.rows, self.slab = rank, r0, rows, slab
        off, nb = ctypes.c_size_t(), ctypes.c_size_t()
        total = _lib.load().btas_fw_dist_workspace_bytes(code, n, rows, ctypes.byref(off), ctypes.byref(nb))
        self.total, self.region_off, self.region_bytes = total, off.value, nb.value
        self.wss = [alloc(total) if alloc is not None else torch.empty(total, dtype=torch.uint8, device=dev)
                    for _ in range(nbuf)]
        self.flags = torch.zeros(_lib.NUM_FLAGS, dtype=torch.int32, device=dev)

    def ws(self, gi: int) -> torch.Tensor:
        return self.wss[gi % len(self.wss)]

    def region(self, gi: int = 0) -> torch.Tensor:
        return self.ws(gi)[self.region_off : self.region_off + self.region_bytes]


def fw_groups(n: int, b: int, chunk: int, look: int) -> "list[tuple[int, int, int]]":
    """Lookahead groups of the row-sharded FW: (first pivot block, blocks,
    owner rank) — up to ``look`` consecutive pivot blocks of ``b`` rows, never
    spanning two ranks' slabs of ``chunk`` rows."""
    nblk = -(-n // b)
    out, kb = [], 0
    while kb < nblk:
        owner = (kb * b) // chunk
        slab_end = -(-min(n, (owner + 1) * chunk) // b)  # first block past the owner's rows
        m = max(1, min(look, slab_end - kb, nblk - kb))
        out.append((kb, m, owner))
        kb += m
    return out


def _fw_rows_run(ranks, code, integer, n, ld, masked, min_fin, b, chunk, bcast, peers=None):
    """The group sequence of btas_fw_dist_group (include/btas_cuda.h) over
    the given local ranks; ``bcast(owner, ranks, gi)`` moves the owner's
    broadcast region of group ``gi`` to every rank.  With ``peers(gi, rank)
    -> [addresses]`` the owner's OWNER stage stores its region into the
    peers' regions itself (btas_fw_dist_group_peers) and ``bcast`` is only
    the barrier (also called once with owner -1 after the INIT stages)."""
    import ctypes

    from .matrix import _ptr, _stream

    look = int(_lib.load().btas_fw_dist_group_size(code))

    def stage(rk, s, kb0=0, m=1, gi=0):
        ws = rk.ws(gi)
        ptr = _ptr(rk.slab) if rk.rows > 0 else None
        args = (code, 1 if integer else 0, s, ptr, ld, n, rk.r0, rk.rows, kb0, m, 1 if masked else 0, min_fin,
                _ptr(rk.flags), _ptr(ws), ws.numel())
        pr = peers(gi, rk.rank) if (peers is not None and s == FW_STAGE_OWNER) else None
        if pr:
            arr = (ctypes.c_void_p * len(pr))(*pr)
            _lib.call("btas_fw_dist_group_peers", *args, arr, len(pr), _stream(ws.device))
        else:
            _lib.call("btas_fw_dist_group", *args, _stream(ws.device))

    for rk in ranks:
        for i in range(len(rk.wss)):
            stage(rk, FW_STAGE_INIT, gi=i)
    if peers is not None:
        # the peers' INIT (padding fill of their regions) must finish before
        # any owner stores a panel into them
        bcast(-1, ranks, -1)
    for gi, (kb0, m, owner) in enumerate(fw_groups(n, b, chunk, look)):
        for rk in ranks:
            if rk.rank == owner:
                stage(rk, FW_STAGE_OWNER, kb0, m, gi)
        bcast(owner, ranks, gi)
        for rk in ranks:
            stage(rk, FW_STAGE_REST, kb0, m, gi)
    for rk in ranks:
        stage(rk, FW_STAGE_DIAG)


def _fw_setup(adj):
    from .apsp import _closure_base, _fw_limit, _require_square_minplus
    from .matrix import _dtype_code

    n = _require_square_minplus(adj)
    base = _closure_base(adj)
    code = _dtype_code(base.dtype)
    b = 64 if base.dtype == torch.float64 else 128
    return n, base, code, b, _fw_limit(adj)


def _slab_stats(slab, code):
    """(max |finite|, min finite) of a slab as float64 device scalars (+inf/−inf if empty)."""
    from .matrix import _new_stats, _ptr, _read_stats, _stream

    dev = slab.device
    if slab.numel() == 0:
        return torch.tensor([0.0, float("inf")], dtype=torch.float64, device=dev)
    st = _new_stats(dev)
    _lib.call("btas_scan", code, _ptr(slab), slab.numel(), _ptr(st), _stream(dev))
    s = _read_stats(st)
    if s.finite_count == 0:
        return torch.tensor([0.0, float("inf")], dtype=torch.float64, device=dev)
    return torch.tensor([_lib.key_to_float(s.max_abs_key), _lib.key_to_float(s.min_key)], dtype=torch.float64,
                        device=dev)


def _fw_report(adj, d, negative):
    from .apsp import Algorithm, ApspReport, DistanceMatrix
    from .matrix import TropicalMatrix

    n = adj.n_rows
    m = TropicalMatrix._wrap(adj.kind, d, adj.integer)
    return ApspReport(distances=DistanceMatrix(n, m), algorithm=Algorithm.FLOYD_WARSHALL,
                      negative_cycle=negative, multiplications_performed=0)


def floyd_warshall_distributed(adj, group=None, peer_workspaces=None):
    """``floyd_warshall`` (reference apsp.py:93-133) with D row-sharded over
    the ranks of ``group`` (one process per GPU), with the single-GPU
    lookahead: pivot blocks go in groups of up to 8 (4-byte storage) inside
    one rank's slab (fw_groups); per group the owner runs the pivot tiles and
    row panels of all its blocks, every rank receives the group's pivot-row
    snapshots and packed row-panel snapshots once, computes its column panels
    and updates its rows with the whole group in one GEMM pass (K = 8b).

    On NCCL groups the panel distribution is **fused into the owner's
    kernels**: the workspaces live in symmetric memory and the owner's
    kernels store every snapshot into the peers' broadcast regions as they
    produce it (btas_fw_dist_group_peers); a one-word all-reduce per group
    then orders the peers' REST stage after it, and two workspaces alternate
    by group parity so the next owner never overwrites a region a peer is
    still reading.  Otherwise (``BTAS_EXCHANGE=nccl``, no symmetric memory)
    the owner's region goes out with one NCCL broadcast per group.
    ``peer_workspaces(nbytes, device, group, world)`` may replace the
    symmetric-memory allocation (multi-process tests on one GPU map the
    workspaces with CUDA IPC).  Every rank passes the same adjacency and
    receives the full result; the negative-cycle flag, and the distances of
    every graph without a negative cycle, are byte-identical to the
    single-GPU ``floyd_warshall`` for any number of ranks."""
    from .semiring import _note_saturation

    n, base, code, b, limit = _fw_setup(adj)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    chunk, spans = partition(n, world)
    r0, r1 = spans[rank]
    d = base.data
    dev = d.device
    ld = d.stride(0)
    st = _slab_stats(d[r0:r1], code)
    mx = st[:1].clone()
    mn = st[1:].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=group)
    max_abs, min_fin = float(mx.item()), float(mn.item())
    masked = not (2.0 * (n + 1) * max_abs < limit)

    fused = peer_workspaces is not None or _want_peer_exchange(group, world, dev)
    rk, peer_ptrs = None, None
    if fused:
        probe = _FwRank(rank, r0, r1 - r0, d[r0:r1], code, n, dev, nbuf=0)
        got = (peer_workspaces(probe.total, dev, group, world) if peer_workspaces is not None
               else _peer_buffers((probe.total,), torch.uint8, dev, group, world))
        ok = torch.tensor([1 if got is not None else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)  # every rank takes the same route
        if int(_host_read(ok)[0]) and got is not None:
            bufs, bases = got
            it = iter(bufs)
            rk = _FwRank(rank, r0, r1 - r0, d[r0:r1], code, n, dev, nbuf=2, alloc=lambda nbytes: next(it))
            peer_ptrs = [[a + rk.region_off for a in per_buf] for per_buf in bases]
    if rk is None:
        rk = _FwRank(rank, r0, r1 - r0, d[r0:r1], code, n, dev)

    if peer_ptrs is not None:
        token = torch.zeros(1, dtype=torch.int32, device=dev)

        def bcast(owner, ranks, gi):  # the owner's kernels already stored the panels into the peers
            dist.all_reduce(token, op=dist.ReduceOp.MAX, group=group)

        def peers(gi, r):
            return peer_ptrs[gi % 2]
    else:
        def bcast(owner, ranks, gi):
            dist.broadcast(ranks[0].region(gi), src=dist.get_global_rank(group, owner) if group is not None else owner,
                           group=group)

        peers = None

    _fw_rows_run([rk], code, base.integer, n, ld, masked, min_fin, b, chunk, bcast, peers)
    flags = rk.flags.clone()
    dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
    # gather the row slabs into the full distance matrix on every rank
    full = torch.empty((world * chunk, n), dtype=d.dtype, device=dev)
    mine = full[rank * chunk : (rank + 1) * chunk]
    if r1 > r0:
        mine[: r1 - r0].copy_(d[r0:r1])
    dist.all_gather_into_tensor(full, mine, group=group)
    f = _host_read(flags).tolist()
    if f[_lib.FLAG_SATURATED]:
        _note_saturation()
    return _fw_report(adj, full[:n].contiguous() if world * chunk != n else full, bool(f[_lib.FLAG_DIAG_NEG]))


def floyd_warshall_emulated(adj, world: int, fused: bool = False):
    """The row-sharded program of ``floyd_warshall_distributed`` with
    ``world`` virtual ranks executed in sequence on ONE GPU (slabs are row
    ranges of one matrix).  ``fused=False``: the broadcast is a device copy;
    ``fused=True``: the owner's OWNER-stage kernels store the panels into the other
    virtual ranks' (double-buffered) workspaces at exactly the addresses the
    multi-GPU path uses.  The result must equal the single-GPU solve."""
    from .semiring import _note_saturation

    n, base, code, b, limit = _fw_setup(adj)
    chunk, spans = partition(n, world)
    d = base.data
    ld = d.stride(0)
    st = [_slab_stats(d[r0:r1], code) for r0, r1 in spans]
    max_abs = max(float(s[0]) for s in st)
    min_fin = min(float(s[1]) for s in st)
    masked = not (2.0 * (n + 1) * max_abs < limit)
    nbuf = 2 if fused else 1
    ranks = [_FwRank(r, r0, r1 - r0, d[r0:r1], code, n, d.device, nbuf=nbuf) for r, (r0, r1) in enumerate(spans)]

    if fused:
        def bcast(owner, rks, gi):
            pass

        def peers(gi, r):
            return [rk.region(gi).data_ptr() for rk in ranks if rk.rank != r]
    else:
        def bcast(owner, rks, gi):
            src = rks[owner].region(gi)
            for rk in rks:
                if rk.rank != owner:
                    rk.region(gi).copy_(src)

        peers = None

    _fw_rows_run(ranks, code, base.integer, n, ld, masked, min_fin, b, chunk, bcast, peers)
    f = torch.stack([rk.flags for rk in ranks]).amax(dim=0).cpu().tolist()
    if f[_lib.FLAG_SATURATED]:
        _note_saturation()
    return _fw_report(adj, d, bool(f[_lib.FLAG_DIAG_NEG]))

"""Host-side logic of the row-sharded squaring APSP, world_size 2 over gloo
on CPU (the GPU path uses the same code with NCCL and the CUDA GEMM).

The per-rank row-block product is injected (the pinned NumPy oracle); the
test checks partitioning, the in-place all-gather, the flag all-reduce, the
fixpoint/probe control flow and that the result is byte-identical to the
single-process reference restatement for every rank."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tropical as ot
from paper_1701_04733_b200.graphs import dense_rows
from paper_1701_04733_b200.sharded import apsp_by_squaring_sharded, partition


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_gemm_rows(a_rows, b, cprev, out):
    c, sat = ot.matmul(a_rows.numpy(), b.numpy(), ot.MIN, "f64", True)
    out.copy_(torch.from_numpy(c))
    changed = int(c.tobytes() != cprev.numpy().tobytes())
    return torch.tensor([changed, 0, int(sat)], dtype=torch.int32)


def _cases():
    out = []
    for n, p, wr, seed in ((5, 0.5, (1, 100), 1), (64, 0.3, (0, 100), 2), (130, 0.05, (1, 20), 3),
                           (40, 0.4, (-3, 10), 4), (2, 1.0, (1, 5), 5), (1, 0.5, (1, 5), 6)):
        out.append(np.concatenate([b for _, b in dense_rows(n, p, wr, seed)]))
    one_loop = np.array([[-1.0]])
    out.append(one_loop)
    return out


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for idx, adj in enumerate(_cases()):
            base = torch.from_numpy(ot.closure_base(adj))
            res = apsp_by_squaring_sharded(base, gemm_rows=_oracle_gemm_rows, align=8)
            results[(rank, idx)] = (res.distances.numpy().tobytes(), res.negative_cycle,
                                    res.multiplications_performed, res.saturated)
    finally:
        dist.destroy_process_group()


def test_partition():
    chunk, spans = partition(65536, 8)
    assert chunk == 8192 and spans[-1] == (57344, 65536)
    chunk, spans = partition(130, 2)
    assert chunk == 128 and spans == [(0, 128), (128, 130)]
    chunk, spans = partition(100, 4)
    assert chunk == 128 and spans == [(0, 100), (100, 100), (100, 100), (100, 100)]


@pytest.mark.timeout(300)
def test_sharded_squaring_gloo_world2():
    world = 2
    port = _free_port()
    manager = mp.get_context("spawn").Manager()
    results = manager.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    for idx, adj in enumerate(_cases()):
        want, neg, mults, sat = ot.apsp_by_squaring(adj, "f64", True)
        for rank in range(world):
            got, gneg, gm, gsat = results[(rank, idx)]
            assert gneg == neg and gm == mults, (idx, rank)
            if not neg:
                assert got == want.tobytes(), (idx, rank)


def _oracle_gemm_plain(a_rows, b, out, z_rows=None, peers=None):
    c, sat = ot.matmul(a_rows.numpy(), b.numpy(), ot.MIN, "f64", True, acc=None if z_rows is None else z_rows.numpy())
    out.copy_(torch.from_numpy(c))
    return torch.tensor([int(sat)], dtype=torch.int32)


def _matmul_cases():
    rng = np.random.default_rng(21)
    out = []
    for m, k, n in ((1, 1, 1), (5, 7, 3), (130, 40, 17), (9, 300, 250)):
        x = rng.integers(-50, 100, (m, k)).astype(float)
        y = rng.integers(-50, 100, (k, n)).astype(float)
        z = rng.integers(-50, 100, (m, n)).astype(float)
        for a in (x, y, z):
            a[rng.random(a.shape) < 0.25] = math.inf
        out.append((x, y, z))
    big = 2.0**53 - 1  # one saturating product on one rank only
    out.append((np.array([[big], [1.0]]), np.array([[big]]), np.zeros((2, 1))))
    return out


def _matmul_worker(rank, world, port, results):
    from paper_1701_04733_b200.sharded import matmul_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for idx, (x, y, z) in enumerate(_matmul_cases()):
            for acc in (False, True):
                xt, yt = torch.from_numpy(ot.orient(ot.MIN, x)), torch.from_numpy(ot.orient(ot.MIN, y))
                zt = torch.from_numpy(ot.orient(ot.MIN, z)) if acc else None
                out, sat = matmul_sharded(xt, yt, None, True, z=zt, gemm_rows=_oracle_gemm_plain, align=1)
                results[(rank, idx, acc)] = (out.numpy().tobytes(), sat)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_matmul_gloo_world2():
    """matmul_sharded (row blocks + all-gather + saturation all-reduce) on two
    gloo ranks: every rank holds the full product, byte-identical to the
    single-process restatement of btas.matmul, saturation seen everywhere."""
    world = 2
    port = _free_port()
    manager = mp.get_context("spawn").Manager()
    results = manager.dict()
    mp.spawn(_matmul_worker, args=(world, port, results), nprocs=world, join=True)
    for idx, (x, y, z) in enumerate(_matmul_cases()):
        for acc in (False, True):
            want, sat = ot.matmul(ot.orient(ot.MIN, x), ot.orient(ot.MIN, y), ot.MIN, "f64", True,
                                  acc=ot.orient(ot.MIN, z) if acc else None)
            for rank in range(world):
                got, gsat = results[(rank, idx, acc)]
                assert got == want.tobytes() and gsat == sat, (idx, acc, rank)


def test_fw_groups_never_span_slabs():
    from paper_1701_04733_b200.sharded import fw_groups

    for n, world in ((65536, 8), (32768, 3), (1000, 2), (129, 2), (1, 1), (4097, 5)):
        chunk, spans = partition(n, world)
        groups = fw_groups(n, 128, chunk, 8)
        kb = 0
        for kb0, m, owner in groups:
            assert kb0 == kb and 1 <= m <= 8
            r0, r1 = spans[owner]
            assert r0 <= kb0 * 128 < r1 and min(n, (kb0 + m) * 128) <= r1
            kb += m
        assert kb == -(-n // 128)
    assert len(fw_groups(65536, 128, 8192, 8)) == 64

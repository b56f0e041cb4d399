"""Row-sharded matmul / matvec (SURVEY §8(e) GEMM and matvec rows): the
NCCL and fused peer-store exchanges on a one-rank group, and the fused
exchange across real process boundaries on this GPU (CUDA IPC).  Results
equal the single-GPU products (and so the reference) byte for byte."""

import numpy as np
import pytest
import torch

import paper_1701_04733_b200 as bt
from paper_1701_04733_b200.sharded import matmul_distributed, matvec_distributed

from gpu_helpers import DTYPES, MAX, MIN, rand_sym

pytestmark = pytest.mark.gpu


@pytest.fixture
def one_rank(cuda):
    import torch.distributed as dist

    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1, device_id=cuda)
        created = True
    yield
    if created:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["nccl", "peer"])
@pytest.mark.parametrize("dtype", DTYPES)
def test_matmul_matvec_distributed_single_rank(one_rank, monkeypatch, exchange, dtype):
    monkeypatch.setenv("BTAS_EXCHANGE", exchange)
    rng = np.random.default_rng(31)
    for kind in (MIN, MAX):
        for m, k, n in ((300, 190, 77), (1, 5, 1), (1025, 512, 640)):
            x = bt.TropicalMatrix(kind, rand_sym(rng, m, k), dtype=dtype)
            y = bt.TropicalMatrix(kind, rand_sym(rng, k, n), dtype=dtype)
            z = bt.TropicalMatrix(kind, rand_sym(rng, m, n), dtype=dtype)
            assert matmul_distributed(x, y) == bt.matmul(x, y)
            assert matmul_distributed(x, y, accumulate_into=z) == bt.matmul(x, y, accumulate_into=z)
            v = bt.TropicalVector(kind, rand_sym(rng, 1, k)[0], dtype=dtype)
            assert matvec_distributed(x, v) == bt.matvec(x, v)


def test_matmul_distributed_saturation(one_rank):
    big = float(2**53 - 1)
    a = bt.TropicalMatrix(MIN, [[big], [1.0]])
    b = bt.TropicalMatrix(MIN, [[big]])
    bt.reset_saturation()
    assert matmul_distributed(a, b) == bt.matmul(a, b)
    assert bt.saturation_seen()


def test_sharded_matmul_across_processes(cuda):
    import subprocess
    import sys
    from pathlib import Path

    tool = Path(__file__).resolve().parent.parent / "tools" / "sharded_ops_multi_proc.py"
    res = subprocess.run([sys.executable, str(tool), "2"], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "2-process sharded matmul OK" in res.stdout

"""Host-side logic of the drop-in API (CPU only): scalar semiring semantics,
TileSpec validation, dtype plumbing and the no-CPU-fallback guarantee."""

import math
import random

import pytest
import torch

import paper_1701_04733_b200 as bt
from paper_1701_04733_b200 import matrix as bm
from paper_1701_04733_b200.semiring import TropicalWeight, tadd, tmul

MIN, MAX = bt.SemiringKind.MIN_PLUS, bt.SemiringKind.MAX_PLUS
INF = math.inf


def test_semiring_laws_randomised():
    """The axiom suite of the reference acceptance gate (test_acceptance.py:71-111)."""
    rng = random.Random(0xA11CE)

    def sample():
        r = rng.random()
        if r < 0.1:
            return bt.INFINITY
        if r < 0.7:
            return TropicalWeight(float(rng.randint(-10**6, 10**6)))
        return TropicalWeight(rng.uniform(-1e6, 1e6))

    def close(a, b):
        if math.isinf(a) or math.isinf(b):
            return a == b
        return abs(a - b) <= 1e-12 * max(1.0, abs(a), abs(b))

    for kind in (MIN, MAX):
        for _ in range(1000):
            x, y, z = sample(), sample(), sample()
            assert tadd(kind, x, y) == tadd(kind, y, x)
            assert tadd(kind, tadd(kind, x, y), z) == tadd(kind, x, tadd(kind, y, z))
            assert tadd(kind, x, x) == x and tadd(kind, x, bt.INFINITY) == x
            assert tmul(kind, x, y) == tmul(kind, y, x)
            assert close(tmul(kind, tmul(kind, x, y), z).value, tmul(kind, x, tmul(kind, y, z)).value)
            assert tmul(kind, x, bt.ZERO) == x and tmul(kind, x, bt.INFINITY) == bt.INFINITY
            assert close(tmul(kind, x, tadd(kind, y, z)).value, tadd(kind, tmul(kind, x, y), tmul(kind, x, z)).value)


def test_weight_validation_and_saturation_flag():
    with pytest.raises(ValueError):
        TropicalWeight(math.nan)
    with pytest.raises(ValueError):
        TropicalWeight(-INF)
    assert math.copysign(1.0, TropicalWeight(-0.0).value) == 1.0
    bt.reset_saturation()
    assert tmul(MIN, 1e308, 1e308) == bt.INFINITY and bt.saturation_seen()
    bt.reset_saturation()
    assert tmul(MIN, -1e308, -1e308) == bt.INFINITY and bt.saturation_seen()
    bt.reset_saturation()
    assert tmul(MIN, bt.INFINITY, 5) == bt.INFINITY and not bt.saturation_seen()
    assert bt.parse_weight(bt.format_weight(TropicalWeight(12.0), integer=True)).value == 12.0
    assert bt.format_weight(bt.INFINITY) == "inf" and bt.parse_weight("INF").is_infinite
    assert bt.SemiringKind.from_token(" MaxPlus ") is MAX
    with pytest.raises(ValueError):
        bt.SemiringKind.from_token("plus")


def test_tile_spec_validation():
    with pytest.raises(ValueError):
        bt.TileSpec(0, 1, 1)
    with pytest.raises(ValueError):
        bt.TileSpec(1, 1, 0)
    spec = bt.TileSpec.default()
    assert spec.tile_rows == 8 and spec.tile_cols == 8 and spec.worker_count == bt.available_parallelism() >= 1


def test_default_dtype_plumbing():
    assert bt.get_default_dtype() == torch.float64
    bt.set_default_dtype(torch.float32)
    try:
        assert bt.get_default_dtype() == torch.float32
    finally:
        bt.set_default_dtype(torch.float64)
    with pytest.raises(ValueError):
        bt.set_default_dtype(torch.float16)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        bt.TropicalMatrix(MIN, [[0.0]])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        bt.identity_matrix(MIN, 3)


def test_cpu_device_rejected():
    with pytest.raises(ValueError):
        bm._resolve_device("cpu")


def test_public_names_cover_reference_hot_path():
    """Every hot-path name the reference facade exports (btas/__init__.py:62-113)
    is exported here with the same meaning."""
    hot = ["Algorithm", "ApspReport", "DimensionMismatch", "DistanceMatrix", "INFINITY", "SemiringKind",
           "SemiringMismatch", "TileSpec", "TropicalMatrix", "TropicalVector", "TropicalWeight", "ZERO",
           "additive_identity", "apsp_by_squaring", "available_parallelism", "ew_add", "find_apsp_violation",
           "floyd_warshall", "format_weight", "identity_matrix", "matmul", "matrix_power", "matvec",
           "multiplicative_identity", "parse_weight", "reset_saturation", "saturation_seen", "tadd", "tmul",
           "verify_apsp"]
    for name in hot:
        assert name in bt.__all__ and hasattr(bt, name), name
    assert issubclass(bt.DimensionMismatch, ValueError) and issubclass(bt.SemiringMismatch, ValueError)


def test_bench_reference_arm_contract():
    """bench.py --impl reference runs on the host alone and prints one JSON
    line with the contract's keys (small n so the CPU suite stays fast)."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    res = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--n", "512", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "impl", "cpu_baseline",
                "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1


def test_bench_gpus_relaunch_decision():
    """bench.py --gpus N outside torchrun re-launches itself with N ranks on
    127.0.0.1; inside torchrun (WORLD_SIZE set) or at N = 1 it runs in place."""
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    import bench

    assert bench.relaunch_command(["--steps", "2"], 1, {}) is None
    assert bench.relaunch_command(["--gpus", "4"], 4, {"WORLD_SIZE": "4"}) is None
    cmd = bench.relaunch_command(["--gpus", "2", "--steps", "3"], 2, {})
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=2" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "2", "--steps", "3"] and cmd[-5].endswith("bench.py")

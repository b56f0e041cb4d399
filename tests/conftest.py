"""Test configuration.

Markers
  gpu   needs a CUDA device (B200); the parity tests proper, calling the
        product through the C ABI.  Everything else runs on CPU.

The hypothesis example database is kept out of the read-only reference tree
 and out of the repo.
"""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

try:
    from hypothesis import HealthCheck, settings
    from hypothesis.database import InMemoryExampleDatabase

    settings.register_profile(
        "btas",
        deadline=None,
        suppress_health_check=[HealthCheck.too_slow],
        database=InMemoryExampleDatabase(),
    )
    settings.load_profile("btas")
except ImportError:  # pragma: no cover
    pass

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device; the GPU parity tests")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = np.load(GOLDEN / name, allow_pickle=False)
        return cache[name]

    return load


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    torch.cuda.set_device(0)
    from paper_1701_04733_b200 import _lib

    _lib.load()  # fails loudly if the extension is missing
    return torch.device("cuda", 0)

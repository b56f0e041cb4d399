"""The C-ABI library loads and exports exactly what include/btas_cuda.h
declares (CPU only: no kernel is launched)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1701_04733_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "btas_cuda.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(btas_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_bound_functions():
    assert declared_functions() == sorted(_lib.SIGNATURES)


def test_library_loads_and_exports_every_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.btas_version().decode().startswith("btas-b200")
    assert lib.btas_status_string(0) == b"ok"
    assert lib.btas_status_string(3) == b"workspace too small"


def test_header_constants_match_python():
    text = HEADER.read_text()
    assert f"#define BTAS_I32_INF 0x{_lib.I32_INF:X}" in text
    assert "#define BTAS_I32_LIMIT (1 << 28)" in text and _lib.I32_LIMIT == 1 << 28
    for name, value in (("BTAS_F32", _lib.F32), ("BTAS_I32", _lib.I32), ("BTAS_F64", _lib.F64)):
        assert re.search(rf"{name} = {value}\b", text), name
    for name, value in (("BTAS_FLAG_CHANGED", 0), ("BTAS_FLAG_DIAG_NEG", 1), ("BTAS_FLAG_SATURATED", 2),
                        ("BTAS_NUM_FLAGS", _lib.NUM_FLAGS)):
        assert re.search(rf"{name} = {value}\b", text), name
    assert ctypes.sizeof(_lib.Stats) == 8 * _lib.STATS_WORDS


def test_argument_validation_without_gpu():
    """Host-side validation returns BTAS_ERR_INVALID before touching the GPU."""
    lib = _lib.load()
    assert lib.btas_gemm(0, 0, 0, None, 1, None, 1, None, 0, None, 1, 1, 1, 1, None, 0, None, None, 0, None) == 1
    assert lib.btas_gemm_workspace_bytes(0, 0, 5, 5) == 0
    assert lib.btas_fw_workspace_bytes(0, 0) == 0
    assert lib.btas_gemm_workspace_bytes(0, 1000, 1000, 1000) > 2 * 1000 * 1000 * 4
    assert lib.btas_key_to_double(0) != lib.btas_key_to_double(0)  # NaN for "no finite entry"
    with pytest.raises(_lib.BtasStatusError):
        _lib.call("btas_ewadd", 0, 7, None, None, None, 1, None)


def test_no_fast_math_and_sm100a_only():
    from paper_1701_04733_b200 import build

    flags = " ".join(build.NVCC_FLAGS)
    assert "arch=compute_100a,code=sm_100a" in flags
    assert "fast_math" not in flags and "ftz" not in flags

"""ctypes wrapper of oracle/_build/liboracle.so (oracle/csrc/tropical_oracle.c)
— TEST INFRASTRUCTURE ONLY.  Same semantics as oracle/tropical.py, in C with
OpenMP, for parity checks at sizes NumPy is too slow for."""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "csrc" / "tropical_oracle.c"
LIB = HERE / "_build" / "liboracle.so"
STORAGE = {"f64": 0, "f32": 1, "i32": 2}

_lib = None


def build(force: bool = False) -> Path:
    """Compile the C restatement (gcc -O3 -fopenmp, no fast-math)."""
    LIB.parent.mkdir(exist_ok=True)
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        cmd = ["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", str(LIB), str(SRC), "-lm"]
        subprocess.run(cmd, check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        lib.oracle_gemm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ip]
        lib.oracle_gemm.restype = ctypes.c_int
        lib.oracle_fw.argtypes = [ctypes.c_int, ctypes.c_int, dp, ctypes.c_int64, ctypes.c_int, ip, ip]
        lib.oracle_fw.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def set_threads(n: int) -> None:
    os.environ["OMP_NUM_THREADS"] = str(n)


def matmul(x, y, kind: str, storage: str = "f64", integer: bool = False):
    """(oriented float64 C, saturated) — same contract as oracle.tropical.matmul."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    m, k = x.shape
    n = y.shape[1]
    out = np.empty((m, n), dtype=np.float64)
    sat = ctypes.c_int(0)
    rc = _load().oracle_gemm(1 if kind == "minplus" else 0, STORAGE[storage], 1 if integer else 0,
                             _dp(x), _dp(y), _dp(out), m, n, k, ctypes.byref(sat))
    if rc:
        raise MemoryError("oracle_gemm failed")
    return out, bool(sat.value)


def floyd_warshall_rounds(base, storage: str = "f64", integer: bool = False, masked: bool = False):
    """Sequential k-rounds on a closure base; returns (d, negative_cycle, saturated)."""
    d = np.array(base, dtype=np.float64, order="C")
    neg, sat = ctypes.c_int(0), ctypes.c_int(0)
    rc = _load().oracle_fw(STORAGE[storage], 1 if integer else 0, _dp(d), d.shape[0], 1 if masked else 0,
                           ctypes.byref(neg), ctypes.byref(sat))
    if rc:
        raise MemoryError("oracle_fw failed")
    return d, bool(neg.value), bool(sat.value)

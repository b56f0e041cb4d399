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
        fp = ctypes.POINTER(ctypes.c_float)
        lib.oracle_closure_rows_f32.argtypes = [fp, ctypes.c_int64, fp, ctypes.c_int64, ctypes.c_int]
        lib.oracle_closure_rows_f32.restype = ctypes.c_int
        lib.oracle_f32_finite_range.argtypes = [fp, ctypes.c_int64, fp, fp]
        lib.oracle_f32_finite_range.restype = None
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


def closure_rows_f32(base, rows, max_iter: int = 64):
    """Rows ``rows`` of the min-plus closure (I (+) A)* of ``base`` (the
    closure base, n x n oriented float32, +inf absent) by row-wise
    Bellman-Ford in C (oracle_closure_rows_f32).  Exactness precondition,
    checked here: every finite candidate sum stays below 2^24 in magnitude,
    which holds when 2 * n * max|finite base| < 2^24 (a shortest path has at
    most n-1 edges).  Returns (float64 rows, products until the fixpoint)."""
    base = np.ascontiguousarray(base, dtype=np.float32)
    n = base.shape[0]
    assert base.shape == (n, n)
    mx, mn = ctypes.c_float(0.0), ctypes.c_float(0.0)
    _load().oracle_f32_finite_range(base.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), base.size,
                                    ctypes.byref(mx), ctypes.byref(mn))
    max_abs, min_fin = float(mx.value), float(mn.value)
    if not 2.0 * n * max_abs < 2.0**24:
        raise ValueError("closure_rows_f32 needs path sums below 2^24 (exact in float32)")
    if min_fin < 0.0:
        raise ValueError("closure_rows_f32 is restricted to non-negative weights (no negative cycle)")
    r = np.ascontiguousarray(base[np.asarray(rows)], dtype=np.float32)
    fp = ctypes.POINTER(ctypes.c_float)
    out = []
    its = 0
    for s0 in range(0, r.shape[0], 16):  # 16 rows per call (register block)
        blk = np.ascontiguousarray(r[s0 : s0 + 16])
        it = _load().oracle_closure_rows_f32(base.ctypes.data_as(fp), n, blk.ctypes.data_as(fp), blk.shape[0],
                                             max_iter)
        if it < 0:
            raise RuntimeError("closure rows did not converge")
        out.append(blk)
        its = max(its, it)
    return np.concatenate(out).astype(np.float64), its

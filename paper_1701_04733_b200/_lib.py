"""ctypes binding of libbtas_cuda.so (the C ABI declared in include/btas_cuda.h).

This is the only module that touches the native library.  There is no CPU
fallback anywhere in the package: if the library is missing every compute
entry point raises ``NativeLibraryMissing`` (the library is built in-tree by
``python -m paper_1701_04733_b200.build`` / ``__graft_entry__.build()``).
Loading the library does not need a GPU; running a kernel does.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import os

# BTAS_LIB overrides the library path (A/B measurements of kernel variants)
LIB_PATH = Path(os.environ.get("BTAS_LIB") or Path(__file__).resolve().parent / "_lib" / "libbtas_cuda.so")

# constants mirrored from include/btas_cuda.h
F32, I32, F64 = 0, 1, 2
MIN_PLUS, MAX_PLUS = 0, 1
I32_INF = 0x3FFFFFFF
I32_LIMIT = 1 << 28
FLAG_CHANGED, FLAG_DIAG_NEG, FLAG_SATURATED, FLAG_PATH = 0, 1, 2, 3
NUM_FLAGS = 8
PATH_FAST32, PATH_S16X2, PATH_CHECKED, PATH_FAST64, PATH_EMPTY, PATH_I32F64 = 0, 1, 2, 3, 4, 5
PATH_NAMES = {
    PATH_FAST32: "fast32",
    PATH_S16X2: "s16x2",
    PATH_CHECKED: "checked",
    PATH_FAST64: "fast64",
    PATH_EMPTY: "empty",
    PATH_I32F64: "i32f64",
}
OK, ERR_INVALID, ERR_CUDA, ERR_WORKSPACE, ERR_UNSUPPORTED = 0, 1, 2, 3, 4
VERIFY_LE, VERIFY_EQ = 1, 2
APSP_SMALL_MAX_N = 1024


class NativeLibraryMissing(RuntimeError):
    """libbtas_cuda.so is not built; the package has no CPU fallback."""


class BtasStatusError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, func: str, status: int, text: str):
        super().__init__(f"{func} failed with status {status} ({text})")
        self.status = status


class Stats(ctypes.Structure):
    """btas_stats (include/btas_cuda.h)."""

    _fields_ = [
        ("nan_count", ctypes.c_ulonglong),
        ("neg_inf_count", ctypes.c_ulonglong),
        ("non_integral", ctypes.c_ulonglong),
        ("over_limit", ctypes.c_ulonglong),
        ("out_of_range", ctypes.c_ulonglong),
        ("finite_count", ctypes.c_ulonglong),
        ("max_abs_key", ctypes.c_ulonglong),
        ("min_key", ctypes.c_ulonglong),
        ("max_key", ctypes.c_ulonglong),
    ]


STATS_WORDS = 9  # 64-bit words of btas_stats


class Pcg64(ctypes.Structure):
    """btas_pcg64 (include/btas_cuda.h): a numpy PCG64 state."""

    _fields_ = [("state_hi", ctypes.c_uint64), ("state_lo", ctypes.c_uint64), ("inc_hi", ctypes.c_uint64),
                ("inc_lo", ctypes.c_uint64)]


WEIGHTS_CONST, WEIGHTS_BOUNDED, WEIGHTS_UNIFORM = 0, 1, 2

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_sz = ctypes.c_size_t
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double

# name -> (restype, argtypes); the exact export list of include/btas_cuda.h
SIGNATURES = {
    "btas_version": (ctypes.c_char_p, []),
    "btas_status_string": (ctypes.c_char_p, [_i32]),
    "btas_key_to_double": (_dbl, [ctypes.c_ulonglong]),
    "btas_stats_init": (_i32, [_p, _p]),
    "btas_export_words": (_i32, [_p, _p, _i64, _p]),
    "btas_ingest": (_i32, [_i32, _i32, _p, _i64, _i32, _p, _p, _p]),
    "btas_scan": (_i32, [_i32, _p, _i64, _p, _p]),
    "btas_to_f64": (_i32, [_i32, _p, _i64, _p, _p]),
    "btas_fill": (_i32, [_i32, _i32, _p, _i64, _dbl, _p]),
    "btas_identity": (_i32, [_i32, _i32, _p, _i64, _i64, _p]),
    "btas_closure_base": (_i32, [_i32, _p, _i64, _p, _i64, _i64, _p]),
    "btas_ewadd": (_i32, [_i32, _i32, _p, _p, _p, _i64, _p]),
    "btas_gemm_workspace_bytes": (_sz, [_i32, _i64, _i64, _i64]),
    "btas_gemm": (
        _i32,
        [_i32, _i32, _i32, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _p, _i64, _p, _p, _sz, _p],
    ),
    "btas_gemm_peers": (
        _i32,
        [_i32, _i32, _i32, _p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _p, _i64, ctypes.POINTER(_p), _i32, _p, _p,
         _sz, _p],
    ),
    "btas_gemm_verify": (
        _i32,
        [_i32, _i32, _i32, _p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _i32, _p, _p, _p, _sz, _p],
    ),
    "btas_verify_base": (_i32, [_i32, _p, _i64, _p, _i64, _i64, _p, _p]),
    "btas_gemm_argmin": (_i32, [_i32, _i32, _dbl, _p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _i64, _p, _i64, _p,
                                _sz, _p]),
    "btas_gemm_timing": (_i32, [_i32]),
    "btas_gemm_timing_read": (_i32, [ctypes.POINTER(_dbl), ctypes.POINTER(_i32)]),
    "btas_matvec": (_i32, [_i32, _i32, _i32, _p, _i64, _i64, _i64, _p, _i64, _i64, _p, _i64, _p, _p]),
    "btas_matvec_bounded": (_i32, [_i32, _i32, _i32, _p, _i64, _i64, _i64, _p, _i64, _i64, _p, _i64, _dbl, _p, _p]),
    "btas_fw_workspace_bytes": (_sz, [_i32, _i64]),
    "btas_fw": (_i32, [_i32, _i32, _p, _i64, _i64, _i32, _dbl, _dbl, _p, _p, _sz, _p]),
    "btas_fw_dist_workspace_bytes": (_sz, [_i32, _i64, _i64, ctypes.POINTER(_sz), ctypes.POINTER(_sz)]),
    "btas_fw_dist_group_size": (_i32, [_i32]),
    "btas_fw_dist_group": (_i32, [_i32, _i32, _i32, _p, _i64, _i64, _i64, _i64, _i64, _i32, _i32, _dbl, _p, _p, _sz,
                                  _p]),
    "btas_fw_dist_group_peers": (_i32, [_i32, _i32, _i32, _p, _i64, _i64, _i64, _i64, _i64, _i32, _i32, _dbl, _p, _p,
                                        _sz, ctypes.POINTER(_p), _i32, _p]),
    "btas_diag_negative": (_i32, [_i32, _p, _i64, _i64, _p, _p]),
    "btas_probe_ceiling": (_i32, [_i32, ctypes.POINTER(_dbl), ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)]),
    "btas_apsp_small_workspace_bytes": (_sz, [_i32, _i64]),
    "btas_apsp_squaring_small": (_i32, [_i32, _i32, _p, _i64, _i64, _p, _i64, _p, _p, _p, _sz, _p]),
    "btas_graph_workspace_bytes": (_sz, [_i64]),
    "btas_edges_to_matrix": (_i32, [_i32, _i64, _p, _p, _p, _i64, _p, _i64, _p, _p]),
    "btas_graph_presence": (_i32, [ctypes.POINTER(Pcg64), _i64, _u64, _p, _sz, _p, _p]),
    "btas_graph_draw": (_i32, [ctypes.POINTER(Pcg64), _i64, _i32, _u64, _dbl, _dbl, _i64, _u64, _u64, _p, _p, _sz, _p,
                               _p]),
    "btas_graph_fill": (_i32, [_i32, ctypes.POINTER(Pcg64), _i64, _u64, _i32, _u64, _i64, _p, _p, _i64, _p, _sz, _p,
                               _p]),
}

_lock = threading.Lock()
_lib = None


def load(path: "str | Path | None" = None) -> ctypes.CDLL:
    """Load (once) and type the native library; raise if it is not built."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise NativeLibraryMissing(
                f"{p} is not built. Run `python -m paper_1701_04733_b200.build` "
                "(needs nvcc 12.9; sm_100a). There is no CPU fallback."
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def status_text(status: int) -> str:
    return load().btas_status_string(status).decode()


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and raise on failure."""
    fn = getattr(load(), name)
    rc = fn(*args)
    if rc != OK:
        raise BtasStatusError(name, rc, status_text(rc))


def key_to_float(key: int) -> float:
    return float(load().btas_key_to_double(ctypes.c_ulonglong(key)))


def gemm_timing(enable: bool) -> None:
    call("btas_gemm_timing", 1 if enable else 0)


def gemm_timing_read() -> "tuple[float, int]":
    """(summed GEMM-kernel ms, number of bracketed btas_gemm calls); synchronises."""
    ms, n = _dbl(), _i32()
    call("btas_gemm_timing_read", ctypes.byref(ms), ctypes.byref(n))
    return ms.value, n.value


def probe_ceiling(mix: int) -> "dict[str, float]":
    """Run btas_probe_ceiling (synchronises): pairs/clk/SM, SM MHz, T pairs/s."""
    a, b, c = _dbl(), _dbl(), _dbl()
    call("btas_probe_ceiling", mix, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    return {"pairs_per_clk_sm": a.value, "sm_mhz": b.value, "tpairs_per_s": c.value}

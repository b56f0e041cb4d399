"""Shared helpers of the GPU parity tests."""

import math

import numpy as np
import torch

import paper_1701_04733_b200 as bt

MIN, MAX = bt.SemiringKind.MIN_PLUS, bt.SemiringKind.MAX_PLUS
DTYPES = (torch.float64, torch.float32, torch.int32)
STORAGE = {torch.float64: "f64", torch.float32: "f32", torch.int32: "i32"}


def kname(kind):
    return "minplus" if kind is MIN else "maxplus"


def symbolic(oriented):
    a = np.asarray(oriented, dtype=np.float64).copy()
    a[np.isinf(a)] = math.inf
    return a


def f64bytes(a):
    return np.ascontiguousarray(a, dtype=np.float64).tobytes()


def rand_sym(rng, r, c, lo=-50, hi=100, p_inf=0.25, integer=True):
    if integer:
        a = rng.integers(lo, hi + 1, size=(r, c)).astype(np.float64)
    else:
        a = rng.uniform(lo, hi, size=(r, c)).astype(np.float32).astype(np.float64)
    a[rng.random((r, c)) < p_inf] = math.inf
    return a


def path_of(flags):
    """Kernel paths that ran (bit set of BTAS_FLAG_PATH)."""
    from paper_1701_04733_b200 import _lib

    bits = int(flags[_lib.FLAG_PATH].item())
    return {name for p, name in _lib.PATH_NAMES.items() if bits & (1 << p)}

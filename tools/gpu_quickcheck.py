"""Quick end-to-end check of the GPU path against the oracle (developer tool).

python tools/gpu_quickcheck.py  — prints one line per check; exits 1 on mismatch.
"""

import math
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1701_04733_b200 as bt  # noqa: E402
from paper_1701_04733_b200 import _lib  # noqa: E402
from oracle import tropical as ot  # noqa: E402
from oracle import native as on  # noqa: E402

MIN, MAX = bt.SemiringKind.MIN_PLUS, bt.SemiringKind.MAX_PLUS
fails = 0


def check(name, ok, extra=""):
    global fails
    print(f"[{'OK' if ok else 'FAIL'}] {name} {extra}", flush=True)
    fails += 0 if ok else 1


def rand_sym(rng, r, c, lo=-50, hi=100, p_inf=0.25, integer=True):
    if integer:
        a = rng.integers(lo, hi + 1, size=(r, c)).astype(np.float64)
    else:
        a = rng.uniform(lo, hi, size=(r, c)).astype(np.float32).astype(np.float64)
    a[rng.random((r, c)) < p_inf] = math.inf
    return a


def storage_of(dt):
    return {torch.float64: "f64", torch.float32: "f32", torch.int32: "i32"}[dt]


def gemm_case(rng, m, k, n, kind, dt, integer=True, lo=-50, hi=100):
    xs, ys = rand_sym(rng, m, k, lo, hi, integer=integer), rand_sym(rng, k, n, lo, hi, integer=integer)
    X = bt.TropicalMatrix(kind, xs, dtype=dt)
    Y = bt.TropicalMatrix(kind, ys, dtype=dt)
    bt.reset_saturation()
    Z = bt.matmul(X, Y)
    got = Z.to_numpy()
    kk = "minplus" if kind is MIN else "maxplus"
    want, sat = on.matmul(ot.orient(kk, xs), ot.orient(kk, ys), kk, storage_of(dt), X.integer and Y.integer)
    ok = got.tobytes() == want.tobytes()
    check(f"gemm {m}x{k}x{n} {kk} {dt} int={integer}", ok,
          "" if ok else f"mismatches={int((got != want).sum())} first={np.argwhere(got != want)[:3].tolist()}")


def main():
    print(_lib.load().btas_version().decode())
    rng = np.random.default_rng(1)
    for dt in (torch.float32, torch.int32, torch.float64):
        for kind in (MIN, MAX):
            for (m, k, n) in [(1, 1, 1), (3, 5, 7), (128, 32, 128), (129, 33, 131), (300, 517, 259)]:
                gemm_case(rng, m, k, n, kind, dt)
    # large-value integer path (not s16): values beyond 2^12
    for dt in (torch.float32, torch.int32):
        gemm_case(rng, 200, 300, 250, MIN, dt, lo=-100000, hi=100000)
    # real-valued f32 / f64
    for dt in (torch.float32, torch.float64):
        gemm_case(rng, 257, 190, 311, MIN, dt, integer=False, lo=-1000, hi=1000)
        gemm_case(rng, 64, 64, 64, MAX, dt, integer=False, lo=-1000, hi=1000)
    # saturation KAT (f64)
    bt.reset_saturation()
    a = bt.TropicalMatrix(MIN, [[-1e308]], integer=False)
    z = bt.matmul(a, a)
    check("saturation -1e308", z.to_lists() == [[math.inf]] and bt.saturation_seen())
    bt.reset_saturation()
    # APSP
    for dt in (torch.int32, torch.float32, torch.float64):
        for n in (1, 2, 7, 64, 200, 300):
            from paper_1701_04733_b200.graphs import random_graph_matrix, dense_rows

            adj = random_graph_matrix(n, 0.5, (1, 100), 1234 + n, dtype=dt)
            sym = np.concatenate([b for _, b in dense_rows(n, 0.5, (1, 100), 1234 + n)])
            fw = bt.floyd_warshall(adj)
            sq = bt.apsp_by_squaring(adj)
            want, neg, mults, _ = ot.apsp_by_squaring(ot.orient("minplus", sym), storage_of(dt), True)
            ok1 = fw.distances.dist.to_numpy().tobytes() == want.tobytes()
            ok2 = sq.distances.dist.to_numpy().tobytes() == want.tobytes()
            check(f"apsp n={n} {dt} fw", ok1)
            check(f"apsp n={n} {dt} square mults={sq.multiplications_performed}/{mults}", ok2 and mults == sq.multiplications_performed and not sq.negative_cycle and not fw.negative_cycle)
    # timing probe
    for dt in (torch.float32, torch.int32):
        n = 4096
        x = bt.TropicalMatrix(MIN, rand_sym(rng, n, n, -1000, 1000), dtype=dt)
        bt.matmul(x, x)
        torch.cuda.synchronize()
        t = time.perf_counter()
        bt.matmul(x, x)
        torch.cuda.synchronize()
        dt_s = time.perf_counter() - t
        print(f"gemm {n}^3 {dt}: {dt_s*1e3:.2f} ms  {n**3/dt_s/1e12:.2f} Tpairs/s")
        x = bt.TropicalMatrix(MIN, rand_sym(rng, n, n, -100000, 100000), dtype=dt)
        bt.matmul(x, x)
        torch.cuda.synchronize()
        t = time.perf_counter()
        bt.matmul(x, x)
        torch.cuda.synchronize()
        dt_s = time.perf_counter() - t
        print(f"gemm {n}^3 {dt} (32-bit path): {dt_s*1e3:.2f} ms  {n**3/dt_s/1e12:.2f} Tpairs/s")
    print("ceiling", _lib.probe_ceiling(0), _lib.probe_ceiling(1), _lib.probe_ceiling(2))
    print("FAILS", fails)
    return 1 if fails else 0


if __name__ == "__main__":
    raise SystemExit(main())

"""Randomised GEMM parity against the C oracle (oracle/_build/liboracle.so,
the reference's masked-tile algorithm restated): random shapes up to ~700,
both kinds, every storage dtype, value regimes that select every kernel path
(s16x2, 32-bit, float64-via-int32, DADD, checked/saturating), accumulate_into
and the fixpoint compare.  Runs for the given number of seconds."""
import math
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from oracle import native as on  # noqa: E402
from oracle import tropical as ot  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
STORAGE = {torch.int32: "i32", torch.float32: "f32", torch.float64: "f64"}
t0 = time.time()
cases = fails = 0
paths = set()
while time.time() - t0 < budget:
    m, k, n = (int(v) for v in rng.integers(1, 700, 3))
    dt = [torch.int32, torch.float32, torch.float64][int(rng.integers(3))]
    kind = [bt.SemiringKind.MIN_PLUS, bt.SemiringKind.MAX_PLUS][int(rng.integers(2))]
    kn = "minplus" if kind is bt.SemiringKind.MIN_PLUS else "maxplus"
    regime = rng.choice(["s16", "wide", "huge", "real", "edge"])
    p_inf = float(rng.choice([0.0, 0.1, 0.5, 0.95]))
    if dt == torch.int32 and regime in ("huge", "real"):
        regime = "edge"

    def draw(r, c):
        if regime == "s16":
            a = rng.integers(-2000, 2000, (r, c)).astype(float)
        elif regime == "wide":
            a = rng.integers(-10**6, 10**6, (r, c)).astype(float)
        elif regime == "huge":
            a = np.floor(rng.uniform(-1, 1, (r, c)) * 2.0**40)
        elif regime == "real":
            a = rng.uniform(-1e3, 1e3, (r, c))
            if dt == torch.float32:
                a = a.astype(np.float32).astype(np.float64)
        else:  # near the storage limits: saturating sums
            big = {torch.int32: 2**28 - 1, torch.float32: 3.0e38, torch.float64: 1.5e308}[dt]
            a = rng.uniform(-1, 1, (r, c)) * big
            a = np.trunc(a) if dt == torch.int32 else (a.astype(np.float32).astype(np.float64)
                                                       if dt == torch.float32 else a)
        if dt == torch.float32:  # the stored operands are the oracle's operands
            a = a.astype(np.float32).astype(np.float64)
        a[rng.random((r, c)) < p_inf] = math.inf
        return a

    xs, ys, zs = draw(m, k), draw(k, n), draw(m, n)
    x, y, z = (bt.TropicalMatrix(kind, a, dtype=dt) for a in (xs, ys, zs))
    integer = x.integer and y.integer
    bt.reset_saturation()
    acc = bool(rng.integers(2))
    got = bt.matmul(x, y, accumulate_into=z if acc else None)
    sat = bt.saturation_seen()
    want, wsat = on.matmul(ot.orient(kn, xs), ot.orient(kn, ys), kn, STORAGE[dt], integer)
    if acc:
        want = ot.ew_add(want, ot.orient(kn, zs), kn)
    cases += 1
    if got.to_numpy().tobytes() != want.tobytes() or sat != wsat:
        fails += 1
        print(f"MISMATCH m={m} k={k} n={n} {dt} {kn} regime={regime} p_inf={p_inf} acc={acc} "
              f"sat={sat}/{wsat}", flush=True)
print(f"gemm stress: {cases} cases, {fails} mismatches in {time.time() - t0:.0f} s")

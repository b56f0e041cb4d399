"""Randomised cross-checks of the round-2 kernels on one GPU, against the
stock reference (oracle/_ref) and the oracle:
  verify   fused find_apsp_violation vs the stock btas.find_apsp_violation on
           random graphs and randomly broken distance matrices (message text)
  paths    predecessors vs oracle.tropical.predecessors (both argmin kernels)
  matvec   screen-free vs screened matvec (bytes), random shapes / batches
  fwgroups lookahead-group distributed FW (virtual ranks) vs btas_fw
Runs for the given number of seconds; prints any disagreement."""
import math
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1701_04733_b200 as bt  # noqa: E402
from oracle import ref_build  # noqa: E402
from oracle import tropical as ot  # noqa: E402
from paper_1701_04733_b200.graphs import dense_rows, random_graph_matrix  # noqa: E402
from paper_1701_04733_b200.sharded import floyd_warshall_emulated  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
ref = ref_build.load()
MIN, MAX = bt.SemiringKind.MIN_PLUS, bt.SemiringKind.MAX_PLUS
DTYPES = [torch.int32, torch.float32, torch.float64]
t0 = time.time()
counts = {"verify": 0, "paths": 0, "matvec": 0, "fwgroups": 0}
fails = 0


def sym_of(n, p, wr, seed):
    return np.concatenate([b for _, b in dense_rows(n, p, wr, seed)])


while time.time() - t0 < budget:
    kind = ["verify", "paths", "matvec", "fwgroups"][int(rng.integers(4))]
    dt = DTYPES[int(rng.integers(3))]
    seed = int(rng.integers(1 << 40))
    try:
        if kind == "verify":
            n = int(rng.choice([1, 2, 5, 33, 130]))
            p, wr = float(rng.choice([0.1, 0.5, 0.9])), (int(rng.choice([0, 1, -2])), int(rng.choice([5, 50])))
            sym = sym_of(n, p, wr, seed)
            rrep = ref.floyd_warshall(ref.TropicalMatrix(ref.SemiringKind.MIN_PLUS, sym))
            if rrep.negative_cycle:
                continue
            d = np.array(rrep.distances.dist.data)
            d[np.isinf(d)] = math.inf
            mut = int(rng.integers(5))
            i, j = (int(v) for v in rng.integers(0, n, 2))
            if mut == 1:
                d[i, i] = float(rng.integers(1, 5))
            elif mut == 2:
                d[i, j] = d[i, j] + 1 if np.isfinite(d[i, j]) else 3.0
            elif mut == 3 and np.isfinite(d[i, j]) and i != j:
                d[i, j] -= 1
            elif mut == 4:
                d = np.zeros((n, n))
            want = ref.find_apsp_violation(ref.TropicalMatrix(ref.SemiringKind.MIN_PLUS, sym),
                                           ref.DistanceMatrix(n, ref.TropicalMatrix(ref.SemiringKind.MIN_PLUS, d)))
            got = bt.find_apsp_violation(bt.TropicalMatrix(MIN, sym, dtype=dt),
                                         bt.DistanceMatrix(n, bt.TropicalMatrix(MIN, d, dtype=dt)))
            ok = got == want
        elif kind == "paths":
            n = int(rng.choice([2, 17, 130, 300]))
            p = float(rng.choice([0.02, 0.2, 0.7]))
            wr = (int(rng.choice([0, 1])), int(rng.choice([3, 100, 6000])))
            adj = random_graph_matrix(n, p, wr, seed, dtype=dt)
            rep = bt.floyd_warshall(adj)
            got = bt.predecessors(adj, rep).cpu().numpy()
            want = ot.predecessors(ot.orient(ot.MIN, sym_of(n, p, wr, seed)), rep.distances.dist.to_numpy())
            ok = np.array_equal(got, want)
        elif kind == "matvec":
            m, k, b = int(rng.integers(1, 700)), int(rng.choice([256, 512, 1000, 4096])), int(rng.integers(1, 10))
            kd = MIN if rng.integers(2) else MAX
            a = rng.integers(-1000, 1000, (m, k)).astype(float)
            a[rng.random(a.shape) < 0.2] = math.inf
            v = rng.integers(-1000, 1000, (b, k)).astype(float)
            v[rng.random(v.shape) < 0.2] = math.inf
            A = bt.TropicalMatrix(kd, a, dtype=dt)
            V = bt.TropicalMatrix(kd, v, dtype=dt)
            ok = torch.equal(bt.matvec_batched(A, V).view(torch.uint8), bt.matvec_batched(A, V.data).view(torch.uint8))
        else:
            n = int(rng.choice([130, 700, 1500, 3000]))
            world = int(rng.integers(2, 9))
            adj = random_graph_matrix(n, float(rng.choice([0.05, 0.5])), (int(rng.choice([-1, 1])), 100), seed, dtype=dt)
            want = bt.floyd_warshall(adj)
            got = floyd_warshall_emulated(adj, world, fused=bool(rng.integers(2)))
            ok = got.negative_cycle == want.negative_cycle and (
                want.negative_cycle or got.distances.dist == want.distances.dist)
    except ValueError:
        continue
    counts[kind] += 1
    if not ok:
        fails += 1
        print(f"MISMATCH {kind} dtype={dt} seed={seed}", flush=True)
print(f"stress r02: {counts} cases, {fails} mismatches in {time.time() - t0:.0f} s")

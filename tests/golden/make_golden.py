"""Generate the golden fixtures from the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Every output below is computed by the unmodified reference (imported as
``btas_ref`` from /root/reference/pkg/src) on inputs drawn with the seeds and
recipes of the reference's own test-suite, cited per fixture.  The fixtures
pin the oracle (tests/test_oracle.py) and are the expected values of the GPU
parity tests (tests/test_gpu_*.py).  Arrays are oriented float64 values (the
reference's ``.data``) stored as float32 when every value is a small integer
or ±inf (lossless), to keep the files small.
"""

from __future__ import annotations

import hashlib
import math
import random
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle.ref_import import load_reference  # noqa: E402

ref = load_reference()
MIN, MAX = ref.SemiringKind.MIN_PLUS, ref.SemiringKind.MAX_PLUS
INF = math.inf


def compact(a: np.ndarray) -> np.ndarray:
    """float32 if lossless (small integers / inf), else float64."""
    a = np.asarray(a, dtype=np.float64)
    f = a.astype(np.float32).astype(np.float64)
    return a.astype(np.float32) if np.array_equal(f, a) else a


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def grid(rng, r, c, lo=-50, hi=100, p_inf=0.25):
    return [[INF if rng.random() < p_inf else float(rng.randint(lo, hi)) for _ in range(c)] for _ in range(r)]


def gemm_cases(seed, count, kind_of, out):
    """Random GEMMs: test_acceptance.py:114-134 (0x04AC1E, MIN if case%3)
    and test_matrix.py:103-110 (0xB7A5, MIN if case%2)."""
    rng = random.Random(seed)
    arrays = {}
    kinds = []
    for case in range(count):
        kind = kind_of(case)
        r, k, c = (rng.randint(1, 16) for _ in range(3))
        xg = [[INF if rng.random() < 0.25 else float(rng.randint(-50, 100)) for _ in range(k)] for _ in range(r)]
        yg = [[INF if rng.random() < 0.25 else float(rng.randint(-50, 100)) for _ in range(c)] for _ in range(k)]
        x, y = ref.TropicalMatrix(kind, xg), ref.TropicalMatrix(kind, yg)
        z = ref.matmul(x, y)
        arrays[f"x{case}"] = compact(x.data)
        arrays[f"y{case}"] = compact(y.data)
        arrays[f"out{case}"] = compact(z.data)
        kinds.append(0 if kind is MIN else 1)
    arrays["kind"] = np.array(kinds, dtype=np.int8)
    np.savez_compressed(HERE / out, **arrays)


def apsp_cases():
    """test_acceptance.py:155-175 (0x7219): 500 graphs n<=7, 200 with n in 8..64."""
    rng = random.Random(0x7219)
    probs = (0.1, 0.5, 0.9)
    arrays = {}
    meta = []
    for case in range(700):
        if case < 500:
            n, prob = 1 + case % 7, probs[case % 3]
        else:
            n, prob = rng.randint(8, 64), probs[(case - 500) % 3]
        g = ref.random_graph(n, prob, (0, 100), rng.randrange(2**63))
        adj = ref.graph_to_matrix(g)
        fw = ref.floyd_warshall(adj)
        sq = ref.apsp_by_squaring(adj)
        arrays[f"adj{case}"] = compact(adj.data)
        arrays[f"fw{case}"] = compact(fw.distances.dist.data)
        arrays[f"sq{case}"] = compact(sq.distances.dist.data)
        meta.append((n, sq.multiplications_performed, int(fw.negative_cycle), int(sq.negative_cycle)))
    arrays["meta"] = np.array(meta, dtype=np.int64)
    np.savez_compressed(HERE / "apsp_small.npz", **arrays)


def negcycle_cases():
    """test_acceptance.py:178-193 (0x9E6): 200 graphs, weights in [-3, 10]."""
    rng = random.Random(0x9E6)
    arrays = {}
    meta = []
    for case in range(200):
        n = 1 + case % 7
        g = ref.random_graph(n, 0.4, (-3, 10), rng.randrange(2**63))
        adj = ref.graph_to_matrix(g)
        fw = ref.floyd_warshall(adj)
        sq = ref.apsp_by_squaring(adj)
        arrays[f"adj{case}"] = compact(adj.data)
        arrays[f"fw{case}"] = compact(fw.distances.dist.data)
        arrays[f"sq{case}"] = compact(sq.distances.dist.data)
        meta.append((n, int(fw.negative_cycle), int(sq.negative_cycle), sq.multiplications_performed))
    arrays["meta"] = np.array(meta, dtype=np.int64)
    np.savez_compressed(HERE / "negcycle.npz", **arrays)


def mult_count_cases():
    """test_acceptance.py:196-210 (0x10C): n = 2..128, multiplication counts
    and result digests of both APSP routes."""
    rng = random.Random(0x10C)
    rows = []
    seeds = []
    for n in range(2, 129):
        s = rng.randrange(2**63)
        g = ref.random_graph(n, 0.5, (1, 100), s)
        adj = ref.graph_to_matrix(g)
        sq = ref.apsp_by_squaring(adj)
        fw = ref.floyd_warshall(adj)
        rows.append((n, sq.multiplications_performed))
        seeds.append((s, digest(sq.distances.dist.data), digest(fw.distances.dist.data)))
    np.savez_compressed(
        HERE / "mult_count.npz",
        meta=np.array(rows, dtype=np.int64),
        seeds=np.array([s for s, _, _ in seeds], dtype=np.uint64),
        sq_digest=np.array([d for _, d, _ in seeds]),
        fw_digest=np.array([d for _, _, d in seeds]),
    )


def c1_case():
    """BASELINE config C1: random_graph(512, 0.5, (1,100), instance_seed(1, 512))
    (bench.py:153-156,183-188), squaring + FW on the reference."""
    n = 512
    seed = ref.bench.instance_seed(1, n)
    adj = ref.graph_to_matrix(ref.random_graph(n, 0.5, (1, 100), seed))
    sq = ref.apsp_by_squaring(adj)
    fw = ref.floyd_warshall(adj)
    np.savez_compressed(
        HERE / "c1_apsp512.npz",
        seed=np.array([seed], dtype=np.uint64),
        adj_digest=np.array([digest(adj.data)]),
        sq=compact(sq.distances.dist.data),
        fw_digest=np.array([digest(fw.distances.dist.data)]),
        meta=np.array([sq.multiplications_performed, int(sq.negative_cycle), int(fw.negative_cycle)], dtype=np.int64),
    )


def generator_digests():
    """graph_io.random_graph + graph_to_matrix digests (graph_io.py:158-165,273-304)
    for the vectorised generator (paper_1701_04733_b200/graphs.py)."""
    cases = [(7, 0.5, (1, 100), 11), (64, 0.5, (1, 100), 12), (300, 0.3, (0, 100), 13),
             (200, 0.9, (-3, 10), 14), (150, 0.5, (0.5, 7.25), 15), (1, 0.5, (1, 100), 16)]
    out = []
    for n, p, wr, s in cases:
        adj = ref.graph_to_matrix(ref.random_graph(n, p, wr, s))
        out.append(digest(adj.data))
    np.savez_compressed(
        HERE / "generator.npz",
        n=np.array([c[0] for c in cases]), p=np.array([c[1] for c in cases]),
        lo=np.array([c[2][0] for c in cases], dtype=np.float64), hi=np.array([c[2][1] for c in cases], dtype=np.float64),
        seed=np.array([c[3] for c in cases]), digest=np.array(out),
    )


def generator_families():
    """random_graph weight families beyond the benchmark's (graph_io.py:300-303):
    constant ranges, Lemire draws with frequent rejections, raw 32-bit words,
    64-bit draws and zero-scale uniforms — digests of graph_to_matrix."""
    cases = [(40, 0.5, (7, 7), 21), (90, 0.6, (0, 2**31), 22), (70, 0.5, (-(2**31), 2**31 - 1), 23),
             (60, 0.7, (0, 2**32), 24), (50, 0.5, (-(2**62), 2**62), 25), (45, 0.5, (2.5, 2.5), 26),
             (33, 1.0, (-1000.0, 1000.5), 27), (20, 0.0, (1, 100), 28)]
    out = []
    for n, p, wr, s in cases:
        adj = ref.graph_to_matrix(ref.random_graph(n, p, wr, s))
        out.append(digest(adj.data))
    np.savez_compressed(
        HERE / "generator_families.npz",
        n=np.array([c[0] for c in cases]), p=np.array([c[1] for c in cases]),
        lo=np.array([c[2][0] for c in cases], dtype=np.float64), hi=np.array([c[2][1] for c in cases], dtype=np.float64),
        seed=np.array([c[3] for c in cases]), digest=np.array(out),
    )


def edgelist_cases():
    """graph_to_matrix of explicit edge lists (graph_io.py:64-83,158-165):
    duplicate pairs (minimum kept), self-loops of both signs, -0.0 weights and
    real weights; the reference Graph normalises, graph_to_matrix scatters."""
    rng = random.Random(0xED6E)
    arrays = {}
    count = 40
    for case in range(count):
        n = rng.randint(1, 24)
        m = rng.randint(0, 3 * n * n)
        src = [rng.randrange(n) for _ in range(m)]
        dst = [rng.randrange(n) for _ in range(m)]
        if case % 4 == 3:
            w = [rng.uniform(-5, 50) for _ in range(m)]
        else:
            w = [float(rng.randint(-4, 40)) for _ in range(m)]
        for i in range(0, m, 7):
            w[i] = -0.0 if w[i] == 0 else w[i]
        g = ref.Graph(n=n, edges=tuple(zip(src, dst, w)))
        adj = ref.graph_to_matrix(g)
        arrays[f"n{case}"] = np.array([n])
        arrays[f"src{case}"] = np.array(src, dtype=np.int64)
        arrays[f"dst{case}"] = np.array(dst, dtype=np.int64)
        arrays[f"w{case}"] = np.array(w, dtype=np.float64)
        arrays[f"out{case}"] = compact(adj.data)
        arrays[f"integer{case}"] = np.array([int(adj.integer)])
    arrays["count"] = np.array([count])
    np.savez_compressed(HERE / "edgelist.npz", **arrays)


def kat_cases():
    """Known answers of the reference tests (test_matrix.py, test_apsp.py),
    recomputed on the reference."""
    arrays = {}
    # test_matrix.py:88-93
    z = ref.matmul(ref.TropicalMatrix(MIN, [[0, 3], [INF, 0]]), ref.TropicalMatrix(MIN, [[0, 1], [2, 0]]))
    arrays["matmul_example"] = z.data
    # ew_add example test_matrix.py:74-77
    arrays["ewadd_example"] = ref.ew_add(ref.TropicalMatrix(MIN, [[1, 4]]), ref.TropicalMatrix(MIN, [[3, 2]])).data
    # saturation test_matrix.py:295-314
    ref.reset_saturation()
    big = float(2**53 - 1)
    arrays["sat_int"] = ref.matmul(ref.TropicalMatrix(MIN, [[big]]), ref.TropicalMatrix(MIN, [[big]])).data
    arrays["sat_int_flag"] = np.array([ref.saturation_seen()])
    ref.reset_saturation()
    a = ref.TropicalMatrix(MIN, [[1e308]], integer=False)
    arrays["sat_pos"] = ref.matmul(a, a).data
    arrays["sat_pos_flag"] = np.array([ref.saturation_seen()])
    ref.reset_saturation()
    b = ref.TropicalMatrix(MIN, [[-1e308]], integer=False)
    arrays["sat_neg"] = ref.matmul(b, b).data
    arrays["sat_neg_flag"] = np.array([ref.saturation_seen()])
    ref.reset_saturation()
    # mixed: one saturating candidate and one finite winner
    c = ref.TropicalMatrix(MIN, [[-1e308, 5.0]], integer=False)
    d = ref.TropicalMatrix(MIN, [[-1e308], [1.0]], integer=False)
    arrays["sat_mixed"] = ref.matmul(c, d).data
    arrays["sat_mixed_flag"] = np.array([ref.saturation_seen()])
    ref.reset_saturation()
    # matvec test_matrix.py:164-182
    rng = random.Random(3)
    ag = grid(rng, 6, 5)
    vg = grid(rng, 5, 1)
    arrays["mv_a"] = ref.TropicalMatrix(MIN, ag).data
    arrays["mv_v"] = ref.TropicalVector(MIN, [r[0] for r in vg]).data
    arrays["mv_out"] = ref.matvec(ref.TropicalMatrix(MIN, ag), ref.TropicalVector(MIN, [r[0] for r in vg])).data
    # random matvecs (min and max, integer data)
    rng = random.Random(0x3A7)
    for case in range(40):
        kind = MIN if case % 2 else MAX
        r, k = rng.randint(1, 40), rng.randint(1, 70)
        A = ref.TropicalMatrix(kind, grid(rng, r, k))
        V = ref.TropicalVector(kind, [INF if rng.random() < 0.2 else float(rng.randint(-30, 60)) for _ in range(k)])
        arrays[f"mvr_a{case}"] = A.data
        arrays[f"mvr_v{case}"] = V.data
        arrays[f"mvr_out{case}"] = ref.matvec(A, V).data
    # matrix_power test_matrix.py:195-201
    rng = random.Random(21)
    for p in (2, 3, 4, 5, 8):
        g = grid(rng, 5, 5)
        arrays[f"pow_in{p}"] = ref.TropicalMatrix(MIN, g).data
        arrays[f"pow_out{p}"] = ref.matrix_power(ref.TropicalMatrix(MIN, g), p).data
    # three-node APSP test_apsp.py:30,43-59
    three = ref.graph_to_matrix(ref.Graph(3, ((0, 1, 1.0), (1, 2, 2.0), (0, 2, 5.0))))
    arrays["three_adj"] = three.data
    arrays["three_fw"] = ref.floyd_warshall(three).distances.dist.data
    # real-valued (non-integer) float GEMMs: exact reference float64 results
    rng = np.random.default_rng(0xF10A7)
    for case in range(12):
        kind = MIN if case % 2 else MAX
        r, k, c = (int(v) for v in rng.integers(1, 48, size=3))
        xv = rng.uniform(-1e3, 1e3, size=(r, k)).astype(np.float32).astype(np.float64)
        yv = rng.uniform(-1e3, 1e3, size=(k, c)).astype(np.float32).astype(np.float64)
        xv[rng.random((r, k)) < 0.2] = INF
        yv[rng.random((k, c)) < 0.2] = INF
        x, y = ref.TropicalMatrix(kind, xv), ref.TropicalMatrix(kind, yv)
        arrays[f"real_x{case}"] = x.data
        arrays[f"real_y{case}"] = y.data
        arrays[f"real_out{case}"] = ref.matmul(x, y).data
    np.savez_compressed(HERE / "kat.npz", **arrays)


def verify_cases():
    """find_apsp_violation (apsp.py:181-210) on correct and deliberately
    broken distance matrices (0x5EF1): the reference's exact messages
    (None -> ""), including its acceptance of too-small fixpoints (SURVEY
    §9 quirk 2: the all-zero matrix)."""
    rng = np.random.default_rng(0x5EF1)
    arrays = {}
    msgs = []
    case = 0

    def add(adj, d):
        nonlocal case
        a = ref.TropicalMatrix(MIN, np.where(np.isinf(adj), INF, adj))
        dm = ref.DistanceMatrix(d.shape[0], ref.TropicalMatrix(MIN, np.where(np.isinf(d), INF, d)))
        msgs.append(ref.find_apsp_violation(a, dm) or "")
        arrays[f"adj{case}"] = compact(a.data)
        arrays[f"d{case}"] = compact(dm.dist.data)
        case += 1

    for n in (1, 2, 3, 5, 8, 13, 24, 40, 64, 130):
        for lo in (0, -3):
            adj = rng.integers(lo, 20, (n, n)).astype(np.float64)
            adj[rng.random((n, n)) < 0.6] = INF
            np.fill_diagonal(adj, np.where(rng.random(n) < 0.3, rng.integers(0, 5, n), 0).astype(float))
            a = ref.TropicalMatrix(MIN, np.where(np.isinf(adj), INF, adj))
            rep = ref.floyd_warshall(a)
            if rep.negative_cycle:
                continue
            d = np.array(rep.distances.dist.data)
            base = np.array(adj)
            np.fill_diagonal(base, np.minimum(np.diagonal(base), 0.0))
            add(adj, d)  # correct
            add(adj, np.zeros((n, n)))  # too small, accepted when the weights are non-negative
            add(adj, base)  # the closure base: triangle / fixpoint failures past 1 hop
            i, j = rng.integers(0, n, 2)
            x = d.copy(); x[i, i] = float(rng.integers(1, 9)); add(adj, x)  # nonzero diagonal
            x = d.copy(); x[i, i] = INF; add(adj, x)
            fin = np.argwhere(np.isfinite(base) & ~np.eye(n, dtype=bool))
            if len(fin):
                r, c = fin[rng.integers(len(fin))]
                x = d.copy(); x[r, c] = base[r, c] + 1.0; add(adj, x)  # exceeds the edge
                x = d.copy(); x[r, c] = INF; add(adj, x)
            fin = np.argwhere(np.isfinite(d) & ~np.eye(n, dtype=bool))
            if len(fin):
                r, c = fin[rng.integers(len(fin))]
                x = d.copy(); x[r, c] -= 1.0; add(adj, x)  # too small by one somewhere
                x = d.copy(); x[r, :] = np.minimum(x[r, :], 0.0); x[r, r] = 0.0; add(adj, x)
    arrays["msg"] = np.array(msgs)
    np.savez_compressed(HERE / "verify.npz", **arrays)


def main():
    gemm_cases(0x04AC1E, 200, lambda c: MIN if c % 3 else MAX, "gemm_acceptance.npz")
    gemm_cases(0xB7A5, 120, lambda c: MIN if c % 2 else MAX, "gemm_matrix.npz")
    apsp_cases()
    negcycle_cases()
    mult_count_cases()
    c1_case()
    generator_digests()
    generator_families()
    edgelist_cases()
    kat_cases()
    verify_cases()
    for f in sorted(HERE.glob("*.npz")):
        print(f"{f.name}: {f.stat().st_size / 1024:.1f} KiB")


if __name__ == "__main__":
    if sys.argv[1:] == ["verify"]:  # only the verifier fixture
        verify_cases()
    else:
        main()

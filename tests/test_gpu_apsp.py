"""GPU parity of APSP (blocked Floyd-Warshall and repeated squaring) against
the reference's golden outputs and the pinned oracle — bit-exact distances,
exact multiplication counts and negative-cycle flags."""

import hashlib
import math

import numpy as np
import pytest
import torch

import paper_1701_04733_b200 as bt
from paper_1701_04733_b200.graphs import dense_rows, instance_seed, random_graph_matrix
from oracle import native as on
from oracle import tropical as ot

from gpu_helpers import DTYPES, MAX, MIN, STORAGE, f64bytes, symbolic

pytestmark = pytest.mark.gpu


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("small_route", [True, False])
def test_golden_apsp_triple_equivalence(cuda, golden, dtype, small_route, monkeypatch):
    """700 digraphs of test_acceptance.py:155-175: FW == squaring == the
    reference, byte for byte, with the reference's multiplication counts.
    small_route=False disables the one-kernel small-graph squaring (and the
    FW route through it), so the blocked FW and the btas_gemm loop are
    checked on the same graphs."""
    if not small_route:
        monkeypatch.setenv("BTAS_APSP_SMALL_MAX_N", "0")
    g = golden("apsp_small.npz")
    meta = g["meta"]
    for case in range(len(meta)):
        adj = bt.TropicalMatrix(MIN, symbolic(g[f"adj{case}"]), dtype=dtype)
        fw = bt.floyd_warshall(adj)
        sq = bt.apsp_by_squaring(adj)
        assert fw.distances.dist.to_numpy().tobytes() == f64bytes(g[f"fw{case}"]), case
        assert sq.distances.dist.to_numpy().tobytes() == f64bytes(g[f"sq{case}"]), case
        assert sq.multiplications_performed == meta[case][1]
        assert fw.negative_cycle == bool(meta[case][2]) and sq.negative_cycle == bool(meta[case][3])
        assert fw.algorithm is bt.Algorithm.FLOYD_WARSHALL and fw.multiplications_performed == 0
        assert sq.algorithm is bt.Algorithm.REPEATED_SQUARING


@pytest.mark.parametrize("dtype", DTYPES)
def test_golden_negative_cycles(cuda, golden, dtype):
    """200 graphs with weights in [-3, 10] (test_acceptance.py:178-193): the
    flags match; distances match too wherever no negative cycle exists."""
    g = golden("negcycle.npz")
    meta = g["meta"]
    flagged = 0
    for case in range(len(meta)):
        adj = bt.TropicalMatrix(MIN, symbolic(g[f"adj{case}"]), dtype=dtype)
        fw = bt.floyd_warshall(adj)
        sq = bt.apsp_by_squaring(adj)
        assert fw.negative_cycle == bool(meta[case][1]) and sq.negative_cycle == bool(meta[case][2]), case
        assert sq.multiplications_performed == meta[case][3]
        flagged += fw.negative_cycle
        if not fw.negative_cycle:
            assert fw.distances.dist.to_numpy().tobytes() == f64bytes(g[f"fw{case}"])
            assert sq.distances.dist.to_numpy().tobytes() == f64bytes(g[f"sq{case}"])
    assert 0 < flagged < len(meta)


def test_golden_mult_counts(cuda, golden):
    """n = 2..128 (test_acceptance.py:196-210): counts and result digests."""
    g = golden("mult_count.npz")
    for idx, (n, mults) in enumerate(g["meta"]):
        adj = random_graph_matrix(int(n), 0.5, (1, 100), int(g["seeds"][idx]))
        sq = bt.apsp_by_squaring(adj)
        assert sq.multiplications_performed == mults
        budget = 0 if n == 2 else 2 * math.ceil(math.log2(n - 1))
        assert mults <= budget
        assert digest(sq.distances.dist.to_numpy()) == str(g["sq_digest"][idx])
        assert digest(bt.floyd_warshall(adj).distances.dist.to_numpy()) == str(g["fw_digest"][idx])


@pytest.mark.parametrize("dtype", DTYPES)
def test_config_c1_apsp512(cuda, golden, dtype):
    """BASELINE config C1 (n = 512, p = 0.5, weights 1..100,
    instance_seed(1, 512)) — the case the reference CPU path runs in full."""
    g = golden("c1_apsp512.npz")
    seed = instance_seed(1, 512)
    assert seed == int(g["seed"][0])
    adj = random_graph_matrix(512, 0.5, (1, 100), seed, dtype=dtype)
    assert digest(adj.to_numpy()) == str(g["adj_digest"][0])
    sq = bt.apsp_by_squaring(adj)
    assert sq.distances.dist.to_numpy().tobytes() == f64bytes(g["sq"])
    assert sq.multiplications_performed == g["meta"][0] and not sq.negative_cycle
    fw = bt.floyd_warshall(adj)
    assert digest(fw.distances.dist.to_numpy()) == str(g["fw_digest"][0]) and not fw.negative_cycle


def test_kats(cuda, golden):
    g = golden("kat.npz")
    three = bt.TropicalMatrix(MIN, symbolic(g["three_adj"]))
    fw = bt.floyd_warshall(three)
    assert fw.distances.dist.to_numpy().tobytes() == f64bytes(g["three_fw"])
    assert fw.distances.dist.to_lists() == [[0, 1, 3], [math.inf, 0, 2], [math.inf, math.inf, 0]]
    assert bt.apsp_by_squaring(three).distances.dist == fw.distances.dist
    edgeless = bt.TropicalMatrix.filled(MIN, 4, 4)
    for rep in (bt.floyd_warshall(edgeless), bt.apsp_by_squaring(edgeless)):
        assert rep.distances.dist == bt.identity_matrix(MIN, 4) and not rep.negative_cycle
    two = bt.TropicalMatrix(MIN, [[0, -2], [1, 0]])
    assert bt.floyd_warshall(two).negative_cycle and bt.apsp_by_squaring(two).negative_cycle
    one = bt.TropicalMatrix(MIN, [[0]])
    rep = bt.apsp_by_squaring(one)
    assert rep.distances.dist.to_lists() == [[0]] and rep.multiplications_performed == 0 and not rep.negative_cycle
    loop = bt.TropicalMatrix(MIN, [[-1]])
    assert bt.floyd_warshall(loop).negative_cycle and bt.apsp_by_squaring(loop).negative_cycle
    k9 = bt.TropicalMatrix(MIN, [[0 if i == j else 1 for j in range(9)] for i in range(9)])
    rep = bt.apsp_by_squaring(k9)
    assert rep.multiplications_performed <= 2 and rep.distances.dist == bt.floyd_warshall(k9).distances.dist


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32])
@pytest.mark.parametrize("n", [1000, 2500])
def test_fw_equals_squaring_midsize(cuda, dtype, n):
    """Config C3's cross-check at mid size: GPU blocked FW == GPU squaring,
    and sampled rows equal the (pinned) row-closure oracle."""
    adj = random_graph_matrix(n, 0.5, (1, 100), 4242 + n, dtype=dtype)
    fw = bt.floyd_warshall(adj)
    sq = bt.apsp_by_squaring(adj)
    assert fw.distances.dist == sq.distances.dist
    sym = np.concatenate([b for _, b in dense_rows(n, 0.5, (1, 100), 4242 + n)])
    rows = [0, n // 3, n - 1]
    want = ot.closure_rows(sym, rows, STORAGE[dtype], True,
                           gemm=lambda a, b: on.matmul(a, b, "minplus", STORAGE[dtype], True)[0])
    got = fw.distances.dist.to_numpy()[rows]
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32])
def test_fw_overlapped_phase1_schedule(cuda, dtype, monkeypatch):
    """The large-graph schedule (pivot tile first, phase 1 concurrent with the
    capped thin passes on two side streams, phase 1's s16 flag in its own
    word folded back by the panel kernel) forced onto small graphs: the same
    bytes as the serial schedule and as squaring — ragged last pivot blocks,
    several lookahead groups, and weights whose panels leave the s16 domain
    in mid-group (the gate of the next thin passes must see it)."""
    monkeypatch.setenv("BTAS_FW_SQUARING_MAX_N", "0")
    for n, wr, seed in ((700, (1, 100), 1), (1500, (1, 100), 2), (1100, (1, 3000), 3), (1300, (1, 40000), 4)):
        adj = random_graph_matrix(n, 0.3, wr, 777 + seed, dtype=dtype)
        monkeypatch.setenv("BTAS_FW_OVERLAP_P1_MIN_BLOCKS", "1000000")
        serial = bt.floyd_warshall(adj)
        monkeypatch.setenv("BTAS_FW_OVERLAP_P1_MIN_BLOCKS", "2")
        over = bt.floyd_warshall(adj)
        assert not over.negative_cycle and not serial.negative_cycle
        assert over.distances.dist == serial.distances.dist, (n, wr)
        assert over.distances.dist == bt.apsp_by_squaring(adj).distances.dist, (n, wr)
    # s16-domain weights except inside pivot block 5, which is cut off from
    # blocks 0-4 and whose internal edges weigh 40000: only block 5's CLOSED
    # pivot tile (phase 1's emission) leaves the s16 domain, its panels stay
    # inside, so the flag word phase 1 sets concurrently with the thin passes
    # is the only signal that block 6's thin passes (whose column block 5
    # reads that tile) must run the 32-bit kernel (int16 lanes would wrap)
    n = 1200
    sym = np.concatenate([b for _, b in dense_rows(n, 0.3, (1, 100), 99)])
    sym[640:768, :640] = math.inf
    sym[:640, 640:768] = math.inf
    rng = np.random.default_rng(5)
    sym[640:768, 768:] = rng.integers(1, 100, (128, n - 768))  # every panel entry has a short direct edge
    sym[768:, 640:768] = rng.integers(1, 100, (n - 768, 128))
    inner = sym[640:768, 640:768]
    inner[np.isfinite(inner) & (inner > 0)] = 40000
    adj = bt.TropicalMatrix(MIN, sym, dtype=dtype)
    monkeypatch.setenv("BTAS_FW_OVERLAP_P1_MIN_BLOCKS", "1000000")
    serial = bt.floyd_warshall(adj)
    monkeypatch.setenv("BTAS_FW_OVERLAP_P1_MIN_BLOCKS", "2")
    over = bt.floyd_warshall(adj)
    assert over.distances.dist == serial.distances.dist
    rows = [0, 650, 700, 800, n - 1]
    want = ot.closure_rows(sym, rows, STORAGE[dtype], True,
                           gemm=lambda a, b: on.matmul(a, b, "minplus", STORAGE[dtype], True)[0])
    assert over.distances.dist.to_numpy()[rows].tobytes() == want.tobytes()


def test_fw_overlapped_phase1_at_scale(cuda):
    """n = 16384 (128 pivot blocks: the overlapped phase-1 schedule is on by
    default) with weights that straddle the s16 domain, so the int16x2 gate
    flips inside lookahead groups: FW bytes == repeated squaring bytes."""
    adj = random_graph_matrix(16384, 0.02, (1, 3000), 5151, dtype=torch.int32)
    fw = bt.floyd_warshall(adj)
    sq = bt.apsp_by_squaring(adj)
    assert not fw.negative_cycle and fw.distances.dist == sq.distances.dist


@pytest.mark.parametrize("dtype", DTYPES)
def test_fw_negative_weights_and_sparse(cuda, dtype):
    """Negative weights without negative cycles (no s16 shortcut for the
    pivots that leave its domain) and sparse graphs with long paths, vs the
    sequential C oracle FW."""
    for n, p, wr, seed in ((700, 0.02, (0, 100), 1), (333, 0.5, (-1, 60), 2), (300, 0.01, (1, 5000), 3)):
        sym = np.concatenate([b for _, b in dense_rows(n, p, wr, seed)])
        adj = bt.TropicalMatrix(MIN, sym, dtype=dtype)
        want, neg, _ = on.floyd_warshall_rounds(ot.closure_base(sym), STORAGE[dtype], True)
        fw = bt.floyd_warshall(adj)
        assert fw.negative_cycle == neg
        if not neg:
            assert fw.distances.dist.to_numpy().tobytes() == want.tobytes(), (n, p, wr)
            assert bt.apsp_by_squaring(adj).distances.dist == fw.distances.dist


def test_fw_masked_path(cuda):
    """When the reference screen 2(n+1)max|x| < limit fails (apsp.py:103-107)
    the masked rounds run; results and flag match the oracle."""
    rng = np.random.default_rng(8)
    n = 80
    sym = rng.integers(1, 10**7, (n, n)).astype(float)
    sym[rng.random((n, n)) < 0.6] = math.inf
    np.fill_diagonal(sym, 0)
    for dtype in (torch.int32, torch.float64):
        adj = bt.TropicalMatrix(MIN, sym, dtype=dtype)
        bt.reset_saturation()
        fw = bt.floyd_warshall(adj)
        want, neg, sat = ot.floyd_warshall(ot.orient("minplus", sym), STORAGE[dtype], True)
        assert fw.distances.dist.to_numpy().tobytes() == want.tobytes()
        assert bt.saturation_seen() == sat


def test_verifier(cuda):
    adj = random_graph_matrix(40, 0.3, (0, 100), 5)
    rep = bt.floyd_warshall(adj)
    assert bt.verify_apsp(adj, rep.distances)
    assert bt.verify_apsp(adj, bt.apsp_by_squaring(adj).distances)
    three = bt.TropicalMatrix(MIN, [[0, 1, 5], [math.inf, 0, 2], [math.inf, math.inf, 0]])
    stale = bt.TropicalMatrix(MIN, [[0, 1, 5], [math.inf, 0, 2], [math.inf, math.inf, 0]])
    v = bt.find_apsp_violation(three, bt.DistanceMatrix.from_matrix(stale))
    assert v is not None and ("triangle" in v or "fixpoint" in v)
    good = bt.floyd_warshall(three).distances.dist.to_lists()
    broken = [r[:] for r in good]
    broken[1][1] = 2.0
    assert "diagonal" in bt.find_apsp_violation(three, bt.DistanceMatrix.from_matrix(bt.TropicalMatrix(MIN, broken)))
    above = [r[:] for r in good]
    above[0][1] = 9.0
    assert "edge" in bt.find_apsp_violation(three, bt.DistanceMatrix.from_matrix(bt.TropicalMatrix(MIN, above)))


@pytest.mark.parametrize("dtype", DTYPES)
def test_verifier_messages_match_reference(cuda, golden, dtype):
    """The fused verifier (btas_verify_base + two btas_gemm_verify products)
    returns the reference's find_apsp_violation message — check order, first
    offending index and numpy-scalar value repr — on correct, too-small
    (accepted) and deliberately broken distance matrices
    (tests/golden/verify.npz, made by the reference)."""
    g = golden("verify.npz")
    msgs = g["msg"]
    for case in range(len(msgs)):
        adj = bt.TropicalMatrix(MIN, symbolic(g[f"adj{case}"]), dtype=dtype)
        d = bt.DistanceMatrix.from_matrix(bt.TropicalMatrix(MIN, symbolic(g[f"d{case}"]), dtype=dtype))
        got = bt.find_apsp_violation(adj, d)
        assert (got or "") == str(msgs[case]), case
        assert bt.verify_apsp(adj, d) == (str(msgs[case]) == "")


def test_verifier_at_c3_scale(cuda):
    """The verifier at n = 32768 (int32): accepts the true distances, and
    names the exact first violation of a broken diagonal, an entry above its
    edge and an entry above a shorter path."""
    n = 32768
    adj = random_graph_matrix(n, 0.5, (1, 100), instance_seed(1, n), dtype=torch.int32)
    d = bt.floyd_warshall(adj).distances.dist
    assert bt.find_apsp_violation(adj, bt.DistanceMatrix(n, d)) is None

    def broken(i, j, v):
        data = d.data.clone()
        data[i, j] = v
        return bt.DistanceMatrix(n, bt.TropicalMatrix._wrap(MIN, data, True))

    assert bt.find_apsp_violation(adj, broken(777, 777, 1)) == "diagonal entry (777,777) is np.float64(1.0), expected 0"
    a = adj.data
    r = 20001
    c = int(torch.nonzero(a[r] < (1 << 28))[5].item())
    assert bt.find_apsp_violation(adj, broken(r, c, int(a[r, c]) + 1)) == \
        f"distance ({r},{c}) exceeds the direct edge weight"
    # an entry raised above its true distance but not above its edge
    cols = torch.nonzero((a[r] < (1 << 28)) & (a[r] > d.data[r] + 1)).reshape(-1)
    c = int(cols[0].item())
    assert bt.find_apsp_violation(adj, broken(r, c, int(d.data[r, c]) + 1)) == f"triangle inequality fails at ({r},{c})"


def test_input_errors(cuda):
    rect = bt.TropicalMatrix(MIN, [[0, 1, 2], [3, 0, 4]])
    wrong = bt.TropicalMatrix(MAX, [[0]])
    for solver in (bt.floyd_warshall, bt.apsp_by_squaring):
        with pytest.raises(bt.DimensionMismatch):
            solver(rect)
        with pytest.raises(bt.SemiringMismatch):
            solver(wrong)
        with pytest.raises(TypeError):
            solver([[0]])
    with pytest.raises(ValueError):
        bt.DistanceMatrix(2, bt.TropicalMatrix(MAX, [[0, 1], [1, 0]]))
    with pytest.raises(bt.DimensionMismatch):
        bt.DistanceMatrix(3, bt.identity_matrix(MIN, 2))


@pytest.mark.parametrize("exchange", ["nccl", "peer"])
def test_sharded_squaring_nccl_single_rank(cuda, exchange, monkeypatch):
    """The distributed squaring path (NCCL all-gather or the symmetric-memory
    peer-store exchange + flag all-reduce, CUDA row-block GEMM) on a one-rank
    group: identical to apsp_by_squaring."""
    import torch.distributed as dist

    from paper_1701_04733_b200.sharded import apsp_by_squaring_distributed, apsp_by_squaring_sharded

    monkeypatch.setenv("BTAS_EXCHANGE", exchange)

    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1, device_id=cuda)
        created = True
    try:
        for n, p, wr, seed, dtype in ((300, 0.5, (1, 100), 31, torch.int32), (700, 0.05, (1, 50), 32, torch.float32),
                                      (129, 0.4, (-3, 10), 33, torch.float64), (1, 0.5, (1, 5), 34, torch.int32)):
            adj = random_graph_matrix(n, p, wr, seed, dtype=dtype)
            want = bt.apsp_by_squaring(adj)
            got = apsp_by_squaring_distributed(adj)
            assert got.negative_cycle == want.negative_cycle
            assert got.multiplications_performed == want.multiplications_performed
            if not want.negative_cycle:
                assert got.distances.dist == want.distances.dist
        base = bt.TropicalMatrix(MIN, [[0, 1], [1, 0]], dtype=torch.int32).data
        assert apsp_by_squaring_sharded(base, integer=True).exchange == exchange
    finally:
        if created:
            dist.destroy_process_group()


def _both_paths(monkeypatch, adj):
    monkeypatch.setenv("BTAS_APSP_SMALL_MAX_N", "0")
    bt.reset_saturation()
    want = bt.apsp_by_squaring(adj)
    want_sat = bt.saturation_seen()
    monkeypatch.delenv("BTAS_APSP_SMALL_MAX_N")
    bt.reset_saturation()
    got = bt.apsp_by_squaring(adj)
    got_sat = bt.saturation_seen()
    return want, want_sat, got, got_sat


@pytest.mark.parametrize("dtype", DTYPES)
def test_small_graph_kernel_matches_general_path(cuda, dtype, monkeypatch):
    """The one-kernel small-graph squaring (btas_apsp_squaring_small) against
    the btas_gemm-driven loop: distances, count, negative cycle, saturation."""
    rng = np.random.default_rng(17)
    cases = [(2, 0.5, (1, 9)), (3, 1.0, (-2, 5)), (33, 0.3, (1, 100)), (257, 0.05, (0, 60)), (700, 0.5, (1, 100)),
             (1024, 0.01, (1, 1000)), (130, 0.4, (-1, 40))]
    for n, p, wr in cases:
        adj = random_graph_matrix(n, p, wr, int(rng.integers(1 << 30)), dtype=dtype)
        want, ws, got, gs = _both_paths(monkeypatch, adj)
        assert got.multiplications_performed == want.multiplications_performed, n
        assert got.negative_cycle == want.negative_cycle, n
        assert ws == gs
        if not want.negative_cycle:
            assert got.distances.dist == want.distances.dist, n
    # magnitudes that overflow: the masked-candidate variant and the flag
    big = {torch.float64: 1e308, torch.float32: 3e38, torch.int32: 2**27 - 1}[dtype]
    for n in (5, 70):
        sym = rng.uniform(big / 2, big, (n, n))
        if dtype != torch.float64:
            sym = np.floor(sym) if dtype == torch.int32 else sym
        sym[rng.random((n, n)) < 0.3] = math.inf
        np.fill_diagonal(sym, 0.0)
        adj = bt.TropicalMatrix(bt.SemiringKind.MIN_PLUS, sym, dtype=dtype)
        want, ws, got, gs = _both_paths(monkeypatch, adj)
        assert ws and gs
        assert (got.multiplications_performed, got.negative_cycle) == (want.multiplications_performed,
                                                                       want.negative_cycle)
        assert got.distances.dist == want.distances.dist


def test_c3_scale_fw_equals_squaring_and_oracle_rows(cuda):
    """Config C3 at its own size (SURVEY §8(c) at-scale verification): the
    n = 32768 instance graph_to_matrix(random_graph(n, 0.5, (1, 100),
    instance_seed(1, n))) in int32.  The adjacency's first/last 64 rows equal
    the reference generator (host restatement), GPU blocked FW == GPU
    repeated squaring byte for byte, and 16 sampled distance rows equal the
    C row-closure oracle (reference apsp.py:136-178 row by row)."""
    from oracle.checks import closure_rows_parity

    n = 32768
    seed = instance_seed(1, n)
    adj = random_graph_matrix(n, 0.5, (1, 100), seed, dtype=torch.int32)
    fw = bt.floyd_warshall(adj)
    sq = bt.apsp_by_squaring(adj)
    assert not fw.negative_cycle and not sq.negative_cycle
    assert fw.distances.dist == sq.distances.dist
    rng = np.random.default_rng(0xC3)
    rows = sorted({0, n - 1, *rng.choice(n, 14, replace=False).tolist()})
    par = closure_rows_parity(adj.data, fw.distances.dist.data, rows, gen=(n, 0.5, (1, 100), seed))
    assert par["generator_rows"]["mismatches"] == 0
    assert par["closure_rows"]["mismatches"] == 0


def test_c4_generator_rows_past_2_32(cuda):
    """The n = 65536 instance walks n(n-1) = 4.3e9 presence doubles and
    ~2.1e9 weight draws (past 2^31 edges and 2^32 stream positions): blocks
    at the start, the middle and the end of the GPU-generated matrix equal
    the host restatement of the reference stream."""
    from oracle import graphs as og
    from oracle.checks import mismatches, storage_to_f64

    n = 65536
    seed = instance_seed(1, n)
    adj = random_graph_matrix(n, 0.5, (1, 100), seed, dtype=torch.float32)
    for r0 in (0, 32768, n - 16):
        want = og.instance_rows(n, 0.5, (1, 100), seed, r0, r0 + 16)
        assert mismatches(storage_to_f64(adj.data[r0 : r0 + 16]).cpu().numpy(), want) == 0, r0

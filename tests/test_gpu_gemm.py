"""GPU parity of the tropical GEMM (btas_gemm through the C ABI) against the
reference's golden outputs and the pinned oracle — bit-exact."""

import math

import numpy as np
import pytest
import torch

import paper_1701_04733_b200 as bt
from paper_1701_04733_b200 import _lib
from paper_1701_04733_b200 import matrix as bm
from oracle import native as on
from oracle import tropical as ot

from gpu_helpers import DTYPES, MAX, MIN, STORAGE, f64bytes, kname, path_of, rand_sym, symbolic

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fixture", ["gemm_acceptance.npz", "gemm_matrix.npz"])
@pytest.mark.parametrize("dtype", DTYPES)
def test_golden_gemm_cases(cuda, golden, fixture, dtype):
    """The reference acceptance GEMMs (test_acceptance.py:114-134) and the
    randomised shapes of test_matrix.py:103-110, every storage dtype."""
    g = golden(fixture)
    for case, kc in enumerate(g["kind"]):
        kind = MIN if kc == 0 else MAX
        x = bt.TropicalMatrix(kind, symbolic(g[f"x{case}"]), dtype=dtype)
        y = bt.TropicalMatrix(kind, symbolic(g[f"y{case}"]), dtype=dtype)
        z = bt.matmul(x, y)
        assert z.to_numpy().tobytes() == f64bytes(g[f"out{case}"]), (fixture, case)
        assert z.integer and z.dtype == dtype


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("kind", [MIN, MAX])
def test_tile_edges(cuda, dtype, kind):
    """Shapes around the 128x128 CTA tile, the 32-wide k stage and odd k."""
    rng = np.random.default_rng(11)
    dims = [1, 2, 31, 33, 63, 127, 128, 129, 255, 257]
    for m in dims[::2]:
        for k in dims[1::2]:
            n = dims[(m + k) % len(dims)]
            xs, ys = rand_sym(rng, m, k), rand_sym(rng, k, n)
            x = bt.TropicalMatrix(kind, xs, dtype=dtype)
            y = bt.TropicalMatrix(kind, ys, dtype=dtype)
            want, _ = ot.matmul(ot.orient(kname(kind), xs), ot.orient(kname(kind), ys), kname(kind), STORAGE[dtype], True)
            assert bt.matmul(x, y).to_numpy().tobytes() == want.tobytes(), (m, k, n)


def _paths(x, y, integer, kind=MIN):
    out, flags = bm._gemm(x.data, y.data, kind, integer)
    return out, path_of(flags.cpu())


def test_kernel_path_selection(cuda):
    rng = np.random.default_rng(2)
    small = rand_sym(rng, 40, 50, -1000, 1000)
    wide = rand_sym(rng, 40, 50, -10**6, 10**6)
    real = rand_sym(rng, 40, 50, -1000, 1000, integer=False)
    for dt in (torch.int32, torch.float32, torch.float64):
        a = bt.TropicalMatrix(MIN, small, dtype=dt)
        b = bt.TropicalMatrix(MIN, small.T.copy(), dtype=dt)
        assert _paths(a, b, True)[1] == {"s16x2"}
        a = bt.TropicalMatrix(MIN, wide, dtype=dt)
        b = bt.TropicalMatrix(MIN, wide.T.copy(), dtype=dt)
        assert _paths(a, b, True)[1] == ({"i32f64"} if dt == torch.float64 else {"fast32"})
    # float64 integer operands beyond the int32 domain keep the DADD path
    huge = rand_sym(rng, 40, 50, -2**40, 2**40)
    a = bt.TropicalMatrix(MIN, huge, dtype=torch.float64)
    b = bt.TropicalMatrix(MIN, huge.T.copy(), dtype=torch.float64)
    assert _paths(a, b, True)[1] == {"fast64"}
    for v, path in ((2.0**27 - 1, "i32f64"), (2.0**27, "fast64")):  # sums 2^28 - 2 / 2^28
        for kind in (MIN, MAX):
            sym = np.full((3, 3), v)
            sym[0, 1] = math.inf
            a = bt.TropicalMatrix(kind, sym, dtype=torch.float64)
            out, paths = _paths(a, a, True, kind)
            assert paths == {path}
            want, _ = ot.matmul(ot.orient(kname(kind), sym), ot.orient(kname(kind), sym), kname(kind), "f64", True)
            assert bm._to_f64(out).cpu().numpy().tobytes() == want.tobytes()
    for dt in (torch.float32, torch.float64):
        a = bt.TropicalMatrix(MIN, real, dtype=dt)
        b = bt.TropicalMatrix(MIN, real.T.copy(), dtype=dt)
        assert _paths(a, b, False)[1] == ({"fast64"} if dt == torch.float64 else {"fast32"})


@pytest.mark.parametrize("dtype", DTYPES)
def test_large_sampled_block(cuda, dtype):
    """n = 4096 products on every path, checked on a sampled 48-row block
    against the C oracle (the reference's own sampled-block recipe)."""
    rng = np.random.default_rng(123)
    n = 4096
    rows = np.sort(rng.choice(n, 48, replace=False))
    for lo, hi, integer in ((-1000, 1000, True), (-10**6, 10**6, True), (-1000.0, 1000.0, False)):
        if dtype == torch.int32 and not integer:
            continue
        xs, ys = rand_sym(rng, n, n, lo, hi, integer=integer), rand_sym(rng, n, n, lo, hi, integer=integer)
        for kind in (MIN, MAX):
            x = bt.TropicalMatrix(kind, xs, dtype=dtype)
            y = bt.TropicalMatrix(kind, ys, dtype=dtype)
            z = bt.matmul(x, y)
            got = bm._to_f64(z.data[torch.as_tensor(rows, device=z.device)]).cpu().numpy()
            want, _ = on.matmul(ot.orient(kname(kind), xs[rows]), ot.orient(kname(kind), ys), kname(kind),
                                STORAGE[dtype], x.integer and y.integer)
            assert got.tobytes() == want.tobytes(), (lo, hi, kind)


def test_saturation_kats_f64(cuda, golden):
    """test_matrix.py:295-321 on float64 storage: bit-exact, flag exact."""
    g = golden("kat.npz")
    big = float(2**53 - 1)
    bt.reset_saturation()
    a = bt.TropicalMatrix(MIN, [[big]])
    assert bt.matmul(a, a).to_numpy().tobytes() == f64bytes(g["sat_int"]) and bt.saturation_seen()
    for key, v in (("sat_pos", 1e308), ("sat_neg", -1e308)):
        bt.reset_saturation()
        a = bt.TropicalMatrix(MIN, [[v]], integer=False)
        assert bt.matmul(a, a).to_numpy().tobytes() == f64bytes(g[key]) and bt.saturation_seen()
    bt.reset_saturation()
    c = bt.TropicalMatrix(MIN, [[-1e308, 5.0]], integer=False)
    d = bt.TropicalMatrix(MIN, [[-1e308], [1.0]], integer=False)
    assert bt.matmul(c, d).to_numpy().tobytes() == f64bytes(g["sat_mixed"]) and bt.saturation_seen()
    bt.reset_saturation()
    a = bt.TropicalMatrix(MIN, [[1, math.inf], [2, 0]])
    bt.matmul(a, a)
    assert not bt.saturation_seen()


def test_saturation_seen_across_streams(cuda):
    """A saturating product launched on a side stream (behind a long GEMM on
    that stream) is seen by saturation_seen() called from the default stream
    — also after the ledger folded more than 256 pending flag buffers."""
    big = float(2**53 - 1)
    n = 4096
    rng = np.random.default_rng(12)
    x = bt.TropicalMatrix(MIN, rand_sym(rng, n, n), dtype=torch.float32)
    a = bt.TropicalMatrix(MIN, [[big]])
    side = torch.cuda.Stream()
    for folds in (False, True):
        bt.reset_saturation()
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            for _ in range(3):
                bt.matmul(x, x)  # keeps the side stream busy
            bt.matmul(a, a)  # saturates
            if folds:
                small = bt.TropicalMatrix(MIN, [[1.0]])
                for _ in range(300):
                    bt.matmul(small, small)
        assert bt.saturation_seen(), folds
    torch.cuda.synchronize()


@pytest.mark.parametrize("dtype,big", [(torch.float32, 3e38), (torch.int32, 2**28 - 1), (torch.float64, 1e308)])
@pytest.mark.parametrize("kind", [MIN, MAX])
def test_saturation_per_storage(cuda, dtype, big, kind):
    """Overflow on either side, for each storage: matches the storage-aware
    oracle (dangerous side routed to the CHECKED kernel)."""
    rng = np.random.default_rng(4)
    integer = dtype == torch.int32
    for sign in (1, -1):
        xs = rand_sym(rng, 37, 45, -100, 100)
        ys = rand_sym(rng, 45, 29, -100, 100)
        xs[3, :5] = sign * big
        ys[:5, 7] = sign * big
        x = bt.TropicalMatrix(kind, xs, dtype=dtype, integer=True if integer else False)
        y = bt.TropicalMatrix(kind, ys, dtype=dtype, integer=True if integer else False)
        bt.reset_saturation()
        z = bt.matmul(x, y)
        want, sat = ot.matmul(ot.orient(kname(kind), xs), ot.orient(kname(kind), ys), kname(kind), STORAGE[dtype],
                              integer)
        assert z.to_numpy().tobytes() == want.tobytes(), sign
        assert bt.saturation_seen() == sat == True  # noqa: E712


def test_real_valued_gemm(cuda, golden):
    """Real-valued fp GEMMs: f64 bit-exact with the reference; f32 equals the
    reference result rounded once to f32 (SURVEY §8(c) rule 2)."""
    g = golden("kat.npz")
    for case in range(12):
        kind = MIN if case % 2 else MAX
        want = np.asarray(g[f"real_out{case}"], dtype=np.float64)
        for dt in (torch.float64, torch.float32):
            x = bt.TropicalMatrix(kind, symbolic(g[f"real_x{case}"]), dtype=dt)
            y = bt.TropicalMatrix(kind, symbolic(g[f"real_y{case}"]), dtype=dt)
            got = bt.matmul(x, y).to_numpy()
            exp = want if dt == torch.float64 else want.astype(np.float32).astype(np.float64)
            assert got.tobytes() == exp.tobytes()


@pytest.mark.parametrize("dtype", DTYPES)
def test_accumulate_into(cuda, dtype):
    rng = np.random.default_rng(7)
    xs, ys, zs = rand_sym(rng, 70, 90, integer=True), rand_sym(rng, 90, 60), rand_sym(rng, 70, 60)
    for kind in (MIN, MAX):
        x, y, z = (bt.TropicalMatrix(kind, a, dtype=dtype) for a in (xs, ys, zs))
        before = z.to_numpy().tobytes()
        fused = bt.matmul(x, y, accumulate_into=z)
        plain = bt.matmul(x, y)
        assert fused == bt.ew_add(plain, z)
        assert z.to_numpy().tobytes() == before  # read, never written


def test_kats_and_laws(cuda, golden):
    g = golden("kat.npz")
    x = bt.TropicalMatrix(MIN, [[0, 3], [math.inf, 0]])
    y = bt.TropicalMatrix(MIN, [[0, 1], [2, 0]])
    assert bt.matmul(x, y).to_numpy().tobytes() == f64bytes(g["matmul_example"])
    assert (x @ y).to_lists() == [[0, 1], [2, 0]]
    a = bt.TropicalMatrix(MIN, [[1, 2], [3, 4]])
    absent = bt.TropicalMatrix.filled(MIN, 2, 2)
    assert bt.matmul(a, absent) == absent and bt.matmul(absent, a) == absent
    rng = np.random.default_rng(3)
    for dt in DTYPES:
        for kind in (MIN, MAX):
            m = bt.TropicalMatrix(kind, rand_sym(rng, 6, 6), dtype=dt)
            ident = bt.identity_matrix(kind, 6, dtype=dt)
            assert bt.matmul(ident, m) == m and bt.matmul(m, ident) == m
            b = bt.TropicalMatrix(kind, rand_sym(rng, 6, 6), dtype=dt)
            c = bt.TropicalMatrix(kind, rand_sym(rng, 6, 6), dtype=dt)
            assert bt.matmul(bt.matmul(m, b), c) == bt.matmul(m, bt.matmul(b, c))


def test_tilespec_and_determinism(cuda):
    """Bytes are identical for every TileSpec (reference contract
    matrix.py:9-13), across repeated runs, and row blocks are independent
    (the property the multi-GPU row sharding relies on)."""
    rng = np.random.default_rng(9)
    xs = rand_sym(rng, 300, 300)
    x = bt.TropicalMatrix(MIN, xs, dtype=torch.int32)
    ref = bt.matmul(x, x, tiles=bt.TileSpec(1, 1, 1)).tobytes()
    for spec in (bt.TileSpec(2, 2, 4), bt.TileSpec(1, 300, 8), None):
        assert bt.matmul(x, x, tiles=spec).tobytes() == ref
    full = bt.matmul(x, x).to_numpy()
    top = bt.TropicalMatrix(MIN, xs[:130], dtype=torch.int32)
    assert bt.matmul(top, x).to_numpy().tobytes() == full[:130].tobytes()


def test_matrix_power(cuda, golden):
    g = golden("kat.npz")
    for dt in DTYPES:
        for p in (2, 3, 4, 5, 8):
            a = bt.TropicalMatrix(MIN, symbolic(g[f"pow_in{p}"]), dtype=dt)
            assert bt.matrix_power(a, p).to_numpy().tobytes() == f64bytes(g[f"pow_out{p}"])
        a = bt.TropicalMatrix(MIN, [[0, 1], [math.inf, 0]], dtype=dt)
        assert bt.matrix_power(a, 1) is a
        assert bt.matrix_power(a, 2) == a


def test_errors(cuda):
    a = bt.TropicalMatrix(MIN, [[1, 2], [3, 4]])
    wide = bt.TropicalMatrix(MIN, [[1, 2, 3]])
    other = bt.TropicalMatrix(MAX, [[1, 2], [3, 4]])
    f32 = bt.TropicalMatrix(MIN, [[1, 2], [3, 4]], dtype=torch.float32)
    with pytest.raises(bt.DimensionMismatch):
        bt.matmul(a, wide)
    with pytest.raises(bt.SemiringMismatch):
        bt.matmul(a, other)
    with pytest.raises(bt.DtypeMismatch):
        bt.matmul(a, f32)
    with pytest.raises(bt.DimensionMismatch):
        bt.matmul(a, a, accumulate_into=wide)
    with pytest.raises(bt.SemiringMismatch):
        bt.matmul(a, a, accumulate_into=other)
    with pytest.raises(bt.DimensionMismatch):
        bt.matrix_power(wide, 2)
    with pytest.raises(ValueError):
        bt.matrix_power(a, 0)
    with pytest.raises(bt.DimensionMismatch):
        bt.ew_add(a, wide)
    with pytest.raises(bt.SemiringMismatch):
        bt.ew_add(a, other)


def test_gemm_kernel_timing_hook(cuda):
    rng = np.random.default_rng(1)
    x = bt.TropicalMatrix(MIN, rand_sym(rng, 512, 512), dtype=torch.int32)
    _lib.gemm_timing(True)
    try:
        bt.matmul(x, x)
        bt.matmul(x, x)
        ms, count = _lib.gemm_timing_read()
    finally:
        _lib.gemm_timing(False)
    assert count == 2 and ms > 0


def test_f64_integer_path_epilogues(cuda, monkeypatch):
    """BTAS_PATH_I32F64 through every epilogue: plain, accumulate_into, the
    fixpoint compare of the squaring loop, and max-plus."""
    rng = np.random.default_rng(44)
    for kind in (MIN, MAX):
        xs, ys, zs = (rand_sym(rng, 150, 190, -10**6, 10**6), rand_sym(rng, 190, 130, -10**6, 10**6),
                      rand_sym(rng, 150, 130, -10**6, 10**6))
        x, y, z = (bt.TropicalMatrix(kind, m, dtype=torch.float64) for m in (xs, ys, zs))
        out, paths = _paths(x, y, True, kind)
        assert paths == {"i32f64"}
        k = kname(kind)
        want, _ = ot.matmul(ot.orient(k, xs), ot.orient(k, ys), k, "f64", True)
        assert bt.matmul(x, y).to_numpy().tobytes() == want.tobytes()
        want_acc = ot.ew_add(want, ot.orient(k, zs), k)
        assert bt.matmul(x, y, accumulate_into=z).to_numpy().tobytes() == want_acc.tobytes()
    # squaring loop (Cprev compare) on the general path, float64 wide weights
    monkeypatch.setenv("BTAS_APSP_SMALL_MAX_N", "0")
    from paper_1701_04733_b200.graphs import random_graph_matrix

    adj = random_graph_matrix(300, 0.05, (1, 10**5), 91, dtype=torch.float64)
    got = bt.apsp_by_squaring(adj)
    want, neg, mults, _ = ot.apsp_by_squaring(adj.to_numpy(), "f64", True)
    assert (got.multiplications_performed, got.negative_cycle) == (mults, neg)
    assert got.distances.dist.to_numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("dtype", DTYPES)
def test_fixpoint_compare_long_k(cuda, dtype):
    """K >= 4096 (the unroll-4 compare epilogue of the 32-bit integer mixes):
    FLAG_CHANGED exactly when some entry's bits differ from Cprev — even and
    odd N, a single differing entry anywhere, and Cprev aliasing C (the
    epilogue reads Cprev before it stores)."""
    g = torch.Generator(device=cuda)
    g.manual_seed(21)
    for m, n, k in ((130, 256, 4096), (67, 129, 4100)):
        a = torch.randint(1, 100, (m, k), generator=g, device=cuda).to(dtype)
        b = torch.randint(1, 100, (k, n), generator=g, device=cuda).to(dtype)
        want, f0 = bm._gemm(a, b, MIN, True)
        assert int(f0[_lib.FLAG_CHANGED]) == 0
        out = torch.empty_like(want)
        _, f = bm._gemm(a, b, MIN, True, out=out, cprev=want.clone())
        assert int(f[_lib.FLAG_CHANGED]) == 0 and torch.equal(out, want)
        for r, c in ((m - 1, n - 1), (0, 0), (m // 2, 3)):
            prev = want.clone()
            prev[r, c] += 1
            _, f = bm._gemm(a, b, MIN, True, out=out, cprev=prev)
            assert int(f[_lib.FLAG_CHANGED]) == 1, (m, n, r, c)
        # Cprev aliasing C
        same = want.clone()
        _, f = bm._gemm(a, b, MIN, True, out=same, cprev=same)
        assert int(f[_lib.FLAG_CHANGED]) == 0 and torch.equal(same, want)

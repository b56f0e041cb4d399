"""GPU parity of the HBM-bound kernels (matvec, ⊕, identity, closure base,
ingest/validation) and of the container semantics of TropicalMatrix/Vector."""

import math

import numpy as np
import pytest
import torch

import paper_1701_04733_b200 as bt
from paper_1701_04733_b200 import matrix as bm
from oracle import tropical as ot

from gpu_helpers import DTYPES, MAX, MIN, STORAGE, f64bytes, kname, rand_sym, symbolic

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", DTYPES)
def test_matvec_golden(cuda, golden, dtype):
    g = golden("kat.npz")
    a = bt.TropicalMatrix(MIN, symbolic(g["mv_a"]), dtype=dtype)
    v = bt.TropicalVector(MIN, symbolic(g["mv_v"]), dtype=dtype)
    assert bt.matvec(a, v).to_numpy().tobytes() == f64bytes(g["mv_out"])
    for case in range(40):
        kind = MIN if case % 2 else MAX
        a = bt.TropicalMatrix(kind, symbolic(g[f"mvr_a{case}"]), dtype=dtype)
        v = bt.TropicalVector(kind, symbolic(g[f"mvr_v{case}"]), dtype=dtype)
        assert bt.matvec(a, v).to_numpy().tobytes() == f64bytes(g[f"mvr_out{case}"]), case


@pytest.mark.parametrize("dtype", DTYPES)
def test_matvec_batched_large(cuda, dtype):
    rng = np.random.default_rng(6)
    for m, k in ((1000, 4099), (257, 65536)):
        asym = rand_sym(rng, m, k, -1000, 1000, p_inf=0.1)
        for kind in (MIN, MAX):
            a = bt.TropicalMatrix(kind, asym, dtype=dtype)
            for batch in (1, 3, 6, 8, 11):
                vs = rand_sym(rng, batch, k, -1000, 1000, p_inf=0.1)
                V = bt.TropicalMatrix(kind, vs, dtype=dtype)
                out = bm._to_f64(bt.matvec_batched(a, V)).cpu().numpy()
                for b in range(batch):
                    want, _ = ot.matvec(ot.orient(kname(kind), asym), ot.orient(kname(kind), vs[b]), kname(kind),
                                        STORAGE[dtype], True)
                    assert out[b].tobytes() == want.tobytes(), (m, k, batch, b)


@pytest.mark.parametrize("dtype", DTYPES)
def test_matvec_bound_selects_screen_free_path(cuda, dtype):
    """Ingested operands carry their exact max |finite| (abs_bound); a bound
    that proves no overflow runs the screen-free kernels, an unknown bound
    (raw tensor, no v_bound) the screened ones — the same bytes either way,
    for 1-4 vectors (matvec_kernel) and 5-8 (tensor-map wide kernel)."""
    rng = np.random.default_rng(16)
    m, k = 777, 4096
    asym = rand_sym(rng, m, k, -1000, 1000, p_inf=0.1)
    for kind in (MIN, MAX):
        a = bt.TropicalMatrix(kind, asym, dtype=dtype)
        assert a.abs_bound == float(np.abs(asym[np.isfinite(asym)]).max())
        for batch in (1, 4, 8):
            V = bt.TropicalMatrix(kind, rand_sym(rng, batch, k, -1000, 1000, p_inf=0.1), dtype=dtype)
            bt.reset_saturation()
            fast = bt.matvec_batched(a, V)  # bound known: screen-free
            slow = bt.matvec_batched(a, V.data)  # bound unknown: screened
            assert torch.equal(fast.view(torch.uint8), slow.view(torch.uint8)), (kind, batch)
            assert not bt.saturation_seen()
    # bounds propagate through products and ⊕ (|a (x) b| <= |a| + |b|)
    b = bt.TropicalMatrix(MIN, rand_sym(rng, k, 64, -7, 9), dtype=dtype)
    c = bt.matmul(bt.TropicalMatrix(MIN, asym, dtype=dtype), b)
    assert a.abs_bound + b.abs_bound <= c.abs_bound <= (a.abs_bound + b.abs_bound) * (1 + 2**-19)
    assert float(np.abs(np.where(np.isfinite(c.to_numpy()), c.to_numpy(), 0)).max()) <= c.abs_bound
    assert bt.ew_add(c, c).abs_bound == c.abs_bound and bt.identity_matrix(MIN, 3, dtype=dtype).abs_bound == 0.0


def test_matvec_always_masks(cuda):
    """matvec masks overflow with no screen (matrix.py:408-420)."""
    for dtype, big, integer in ((torch.float64, 1e308, False), (torch.float32, 3e38, False),
                                (torch.int32, 2**28 - 1, True), (torch.float64, 2.0**53 - 1, True)):
        for kind in (MIN, MAX):
            for sign in (1, -1):
                asym = np.array([[sign * big, 1.0, math.inf], [2.0, sign * big, 3.0]])
                vsym = np.array([sign * big, 4.0, 5.0])
                a = bt.TropicalMatrix(kind, asym, dtype=dtype, integer=integer)
                v = bt.TropicalVector(kind, vsym, dtype=dtype, integer=integer)
                bt.reset_saturation()
                got = bt.matvec(a, v).to_numpy()
                want, sat = ot.matvec(ot.orient(kname(kind), asym), ot.orient(kname(kind), vsym), kname(kind),
                                      STORAGE[dtype], integer)
                assert got.tobytes() == want.tobytes() and bt.saturation_seen() == sat == True  # noqa: E712


@pytest.mark.parametrize("dtype", DTYPES)
def test_ew_add(cuda, golden, dtype):
    g = golden("kat.npz")
    a = bt.TropicalMatrix(MIN, [[1, 4]], dtype=dtype)
    b = bt.TropicalMatrix(MIN, [[3, 2]], dtype=dtype)
    assert bt.ew_add(a, b).to_numpy().tobytes() == f64bytes(g["ewadd_example"])
    rng = np.random.default_rng(1)
    for shape in ((1, 1), (3, 5), (257, 1031)):
        xs, ys = rand_sym(rng, *shape), rand_sym(rng, *shape)
        for kind in (MIN, MAX):
            x = bt.TropicalMatrix(kind, xs, dtype=dtype)
            y = bt.TropicalMatrix(kind, ys, dtype=dtype)
            want = ot.ew_add(ot.orient(kname(kind), xs), ot.orient(kname(kind), ys), kname(kind))
            assert bt.ew_add(x, y).to_numpy().tobytes() == want.tobytes()
            assert bt.ew_add(x, x) == x
            assert bt.ew_add(x, bt.TropicalMatrix.filled(kind, *shape, dtype=dtype)) == x
    # vectors (the reference has no vector ⊕)
    u = bt.TropicalVector(MAX, [1, math.inf, 3], dtype=dtype)
    w = bt.TropicalVector(MAX, [2, 0, math.inf], dtype=dtype)
    assert bt.ew_add(u, w).to_list() == [2, 0, 3]
    with pytest.raises(bt.DimensionMismatch):
        bt.ew_add(u, bt.TropicalMatrix(MAX, [[1, 2, 3]], dtype=dtype))


@pytest.mark.parametrize("dtype", DTYPES)
def test_identity_and_closure_base(cuda, dtype):
    assert bt.identity_matrix(MIN, 2, dtype=dtype).to_lists() == [[0, math.inf], [math.inf, 0]]
    assert bt.identity_matrix(MAX, 2, dtype=dtype).to_numpy().tolist() == [[0, -math.inf], [-math.inf, 0]]
    assert bt.identity_matrix(MIN, 3, dtype=dtype).integer
    with pytest.raises(bt.DimensionMismatch):
        bt.identity_matrix(MIN, 0)
    from paper_1701_04733_b200.apsp import _closure_base

    adj = bt.TropicalMatrix(MIN, [[5, 1], [math.inf, -2]], dtype=dtype)
    assert _closure_base(adj).to_lists() == [[0, 1], [math.inf, -2]]


def test_construction_validation(cuda):
    with pytest.raises(ValueError):
        bt.TropicalMatrix(MIN, [[math.nan]])
    with pytest.raises(ValueError):
        bt.TropicalMatrix(MIN, [[-math.inf]])
    with pytest.raises(bt.DimensionMismatch):
        bt.TropicalMatrix(MIN, [[1, 2], [3]])
    with pytest.raises(bt.DimensionMismatch):
        bt.TropicalMatrix(MIN, [1, 2, 3])
    with pytest.raises(bt.DimensionMismatch):
        bt.TropicalVector(MIN, [[1, 2]])
    with pytest.raises(ValueError):
        bt.TropicalMatrix(MIN, [[2.0**28]], dtype=torch.int32)
    with pytest.raises(ValueError):
        bt.TropicalMatrix(MIN, [[0.5]], dtype=torch.int32)
    with pytest.raises(ValueError):
        bt.TropicalMatrix(MIN, [[1e39]], dtype=torch.float32)
    with pytest.raises(bt.SemiringMismatch):
        bt.TropicalMatrix("minplus", [[1]])
    a = bt.TropicalMatrix(MIN, [[-0.0]])
    assert a.tobytes() == bt.TropicalMatrix(MIN, [[0.0]]).tobytes()


def test_integer_detection(cuda):
    assert bt.TropicalMatrix(MIN, [[1, math.inf], [0, -3]]).integer
    assert not bt.TropicalMatrix(MIN, [[0.5]]).integer
    assert not bt.TropicalMatrix(MIN, [[float(2**53)]]).integer
    with pytest.raises(ValueError):
        bt.TropicalMatrix(MIN, [[0.5]], integer=True)
    with pytest.raises(ValueError):
        bt.TropicalMatrix(MIN, [[float(2**53)]], integer=True)
    assert not bt.TropicalMatrix(MIN, [[1]], integer=False).integer
    assert bt.TropicalMatrix(MIN, [[7]], dtype=torch.int32).integer


def test_container_semantics(cuda):
    a = bt.TropicalMatrix(MAX, [[math.inf, 3], [0, math.inf]])
    assert a.to_lists() == [[math.inf, 3], [0, math.inf]]
    assert a.weight_at(0, 0).is_infinite and a.weight_at(0, 1).value == 3
    assert a.to_numpy()[0, 0] == -math.inf  # oriented, like the reference .data
    with pytest.raises(AttributeError):
        a.kind = MIN
    v = bt.TropicalVector(MIN, [1, math.inf])
    with pytest.raises(AttributeError):
        v.kind = MAX
    assert v.to_list() == [1, math.inf] and len(v) == 2 and v.weight_at(1).is_infinite
    assert a.shape == (2, 2) and a.n_rows == 2 and a.n_cols == 2
    from_tensor = bt.TropicalMatrix(MAX, torch.tensor([[math.inf, 3.0], [0.0, math.inf]]))
    assert from_tensor == a
    assert bt.TropicalMatrix(MIN, [[bt.TropicalWeight(2.0), bt.INFINITY]]).to_lists() == [[2.0, math.inf]]
    f = bt.TropicalMatrix.filled(MIN, 2, 3, 5)
    assert f.to_lists() == [[5] * 3] * 2
    assert "2x3" in repr(f)


def test_host_read_small_results(cuda):
    """btas_export_words: small device results reach the host through SM
    stores into page-locked memory, bit for bit, for every word size."""
    from paper_1701_04733_b200.matrix import _host_read

    g = torch.Generator(device="cuda").manual_seed(3)
    for dt in (torch.int32, torch.int64, torch.float32, torch.float64, torch.uint8):
        for shape in ((1,), (9,), (3, 5), (4096,)):
            t = torch.randint(-100, 100, shape, generator=g, device="cuda").to(dt)
            got = _host_read(t)
            assert got.dtype == t.cpu().numpy().dtype and got.shape == tuple(shape)
            assert got.tobytes() == t.cpu().numpy().tobytes()
    # non-contiguous and oversize inputs take the copy fallback
    t = torch.arange(20000, device="cuda", dtype=torch.int32)
    assert _host_read(t).tobytes() == t.cpu().numpy().tobytes()
    assert _host_read(t[::3]).tobytes() == t[::3].cpu().numpy().tobytes()
    assert _host_read(torch.zeros(0, device="cuda")).shape == (0,)


@pytest.mark.parametrize("dtype", [torch.float32, torch.int32])
def test_matvec_wide_saturating(cuda, dtype):
    """5-8 vectors (one-pass wide kernel) with magnitudes whose sums overflow:
    the CTA's screen fails and its rows are recomputed with masked candidates."""
    rng = np.random.default_rng(9)
    big = 3e38 if dtype == torch.float32 else 2**28 - 1
    m, k = 70, 512
    for kind in (MIN, MAX):
        asym = rng.uniform(-big, big, (m, k))
        vs = rng.uniform(-big, big, (6, k))
        if dtype == torch.int32:
            asym, vs = np.floor(asym), np.floor(vs)
        else:  # the storage values (f32) are the operands
            asym, vs = asym.astype(np.float32).astype(np.float64), vs.astype(np.float32).astype(np.float64)
        asym[rng.random((m, k)) < 0.2] = math.inf
        asym[:40] = np.clip(asym[:40], -1000, 1000)  # some CTAs pass the screen, some do not
        a = bt.TropicalMatrix(kind, asym, dtype=dtype)
        V = bt.TropicalMatrix(kind, vs, dtype=dtype)
        bt.reset_saturation()
        out = bm._to_f64(bt.matvec_batched(a, V)).cpu().numpy()
        assert bt.saturation_seen()
        for b in range(6):
            want, sat = ot.matvec(ot.orient(kname(kind), asym), ot.orient(kname(kind), vs[b]), kname(kind),
                                  STORAGE[dtype], dtype == torch.int32)
            assert out[b].tobytes() == want.tobytes(), (kind, b)

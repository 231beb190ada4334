"""GPU parity: the sm_100a operators against the golden vectors and the CPU oracle.

Bars (BASELINE.json north_star): FK remap, source rows and counts bit-exact; float64
values within normwise rel 1e-9 (the reference's own max_rel_deviation metric,
bench.py:38-43).
"""
import numpy as np
import pytest
import torch

import factorla_oracle as O
import golden_io

pytestmark = pytest.mark.gpu

TOL = 1e-9


def _fb():
    import paper_1612_07448_b200 as fb

    return fb


def _close(a, b, tol=TOL):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    assert a.shape == np.asarray(b).shape, (a.shape, np.asarray(b).shape)
    dev = O.max_rel_deviation(a, b)
    assert dev <= tol, dev


def _build_gpu(g):
    fb = _fb()
    parts = golden_io.parts(g)
    if len(parts) == 1:
        return fb.build_pkfk(g["s"], parts[0][0], parts[0][1])
    return fb.build_star(g["s"], parts)


@pytest.mark.parametrize("name", golden_io.names())
def test_construction_bit_exact(name):
    g = golden_io.load(name)
    nm = _build_gpu(g)
    for i, (e, rk) in enumerate(nm.parts):
        np.testing.assert_array_equal(e.target_numpy(), g[f"target{i}"])
        np.testing.assert_array_equal(nm.source_rows[i + 1].cpu().numpy(), g[f"used{i}"])
        np.testing.assert_array_equal(e.counts.cpu().numpy(), g[f"counts{i}"])
        np.testing.assert_array_equal(rk.cpu().numpy(), g[f"rkept{i}"])
    np.testing.assert_array_equal(_fb().materialize(nm), g["materialize"])


@pytest.mark.parametrize("name", golden_io.names())
def test_operators_vs_reference_golden(name):
    fb = _fb()
    g = golden_io.load(name)
    nm = _build_gpu(g)
    for key, fn, cnt in (
        ("lmm_x1", lambda c: fb.lmm(nm, g["x1"], c), "cnt_lmm_x1"),
        ("lmm_x3", lambda c: fb.lmm(nm, g["x3"], c), None),
        ("tmm_p2", lambda c: fb.lmm(nm.T, g["p2"], c), "cnt_tmm_p2"),
        ("rmm_xr", lambda c: fb.rmm(g["xr"], nm, c), "cnt_rmm_xr"),
        ("rmm_t_xt", lambda c: fb.rmm(g["xt"], nm.T, c), None),
        ("row_sums", lambda c: fb.row_sums(nm, c), "cnt_row_sums"),
        ("col_sums", lambda c: fb.col_sums(nm, c), "cnt_col_sums"),
        ("row_sums_t", lambda c: fb.row_sums(nm.T, c), None),
        ("col_sums_t", lambda c: fb.col_sums(nm.T, c), None),
    ):
        c = fb.OpCounter()
        out = fn(c)
        assert isinstance(out, np.ndarray)  # host in -> host out, like the reference
        _close(out, g[key])
        if cnt:
            assert [c.multiplies, c.additions] == list(g[cnt]), key
    c = fb.OpCounter()
    tot = fb.sum_all(nm, c)
    assert abs(tot - float(g["sum_all"])) <= TOL * max(1.0, np.abs(g["materialize"]).sum())
    assert [c.multiplies, c.additions] == list(g["cnt_sum_all"])
    for op, x in (("mul", 2.0), ("add", 3.0), ("rsub", 1.5), ("div", 4.0), ("pow", 2.0)):
        c = fb.OpCounter()
        _close(fb.materialize(fb.scalar_op(nm, x, op, c)), g[f"scalar_{op}"])
        assert [c.multiplies, c.additions] == list(g[f"cnt_scalar_{op}"])
    _close(fb.materialize(fb.scalar_fn(nm, np.exp)), g["fn_exp"])
    _close(fb.materialize(fb.scalar_fn(nm, np.square)), g["fn_square"])


# ---------------------------------------------------------------- seeded, multi-tile cases
CASES = [
    # n_s, d_s, [(n_r, d_r)], seed
    (100_003, 20, [(10_000, 40)], 1),
    (65_537, 7, [(513, 3)], 2),
    (40_001, 1, [(97, 5), (1000, 2)], 3),
    (30_000, 60, [(5000, 120)], 4),
    (12_345, 0, [(300, 9)], 5),
    (1, 3, [(1, 2)], 6),
    (50_000, 10, [(20_000, 80), (7, 1), (400, 33)], 7),
]


def _random_case(n_s, d_s, shapes, seed):
    rng = np.random.default_rng(seed)
    s = rng.standard_normal((n_s, d_s))
    parts = []
    for n_r, d_r in shapes:
        keys = rng.integers(1, n_r + 1, size=n_s)
        parts.append((keys, rng.standard_normal((n_r, d_r))))
    return s, parts


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_d{c[1]}_q{len(c[2])}" for c in CASES])
def test_seeded_multitile_vs_oracle(case):
    fb = _fb()
    n_s, d_s, shapes, seed = case
    s, parts = _random_case(n_s, d_s, shapes, seed)
    ref = O.build_star(s, parts)
    nm = fb.build_star(s, parts) if len(parts) > 1 else fb.build_pkfk(s, parts[0][0], parts[0][1])
    for i, (e, rk) in enumerate(nm.parts):
        np.testing.assert_array_equal(e.target_numpy(), ref.parts[i][0])
        np.testing.assert_array_equal(nm.source_rows[i + 1].cpu().numpy(), ref.source_rows[i + 1])
    rng = np.random.default_rng(seed + 100)
    n, d = ref.shape
    for d_x in (1, 2, 5, 16, 19):
        x = rng.standard_normal((d, d_x))
        _close(fb.lmm(nm, x), O.lmm(ref, x))
    for m in (1, 3, 10, 17):
        p = rng.standard_normal((n, m))
        _close(fb.lmm(nm.T, p), O.lmm(ref.T, p))
        _close(fb.rmm(p.T.copy(), nm), O.rmm(p.T, ref))
    _close(fb.row_sums(nm), O.row_sums(ref))
    _close(fb.col_sums(nm), O.col_sums(ref))
    assert abs(fb.sum_all(nm) - O.sum_all(ref)) <= TOL * max(1.0, np.abs(s).sum() + sum(np.abs(r).sum() * n for _, r in parts))


def test_device_tensors_stay_on_device():
    fb = _fb()
    s, parts = _random_case(5000, 4, [(100, 6)], 11)
    nm = fb.build_pkfk(torch.from_numpy(s).cuda(), torch.from_numpy(parts[0][0]).cuda(), torch.from_numpy(parts[0][1]).cuda())
    x = torch.randn(10, 2, dtype=torch.float64, device="cuda")
    out = fb.lmm(nm, x)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    _close(out, O.lmm(O.build_pkfk(s, parts[0][0], parts[0][1]), x.cpu().numpy()))


def test_errors_match_reference_behaviour():
    fb = _fb()
    s = np.array([[1.0, 2], [3, 4], [5, 6]])
    r = np.array([[10.0, 20], [30, 40]])
    with pytest.raises(fb.DataError, match="entity row 1"):
        fb.build_pkfk(s, [1, 3, 1], r)
    with pytest.raises(fb.DataError, match="non-integer"):
        fb.build_pkfk(s, [1.0, 1.5, 1.0], r)
    nm = fb.build_pkfk(s, [1, 2, 1], r)
    with pytest.raises(fb.ShapeError):
        fb.lmm(nm, np.ones((3, 1)))
    with pytest.raises(fb.ShapeError):
        fb.rmm(np.ones((1, 4)), nm)
    with pytest.raises(fb.NumericError):
        fb.scalar_op(nm, 0, "div")
    with pytest.raises(ValueError):
        fb.scalar_op(nm, 1, "mod")


def test_kernels_were_launched():
    """The CUDA path ran (no silent host fallback)."""
    fb = _fb()
    before = fb.launch_count()
    nm = fb.build_pkfk([[1.0, 2], [3, 4]], [1, 1], [[5.0, 6]])
    fb.lmm(nm, np.ones((4, 1)))
    assert fb.launch_count() > before


def _zipf_keys(rng, n_s, n_r, s=1.2):
    p = np.arange(1, n_r + 1, dtype=np.float64) ** -s
    p /= p.sum()
    return np.minimum(np.searchsorted(np.cumsum(p), rng.random(n_s), side="right"), n_r - 1) + 1


@pytest.mark.parametrize("n_s,d_s,n_r,d_r", [(200_003, 10, 5000, 40), (70_001, 3, 50, 4)])
def test_skewed_fk_scatter_vs_oracle(n_s, d_s, n_r, d_r):
    """Zipf(1.2) keys: the warp-aggregated scatter path (hot bins) and the dropped-row remap."""
    fb = _fb()
    rng = np.random.default_rng(n_s)
    s = rng.random((n_s, d_s))
    r = rng.random((n_r, d_r))
    key = _zipf_keys(rng, n_s, n_r)
    nm = fb.build_pkfk(s, key, r)
    ref = O.build_pkfk(s, key, r)
    assert nm.k.skewed
    np.testing.assert_array_equal(nm.k.target_numpy(), ref.parts[0][0])
    np.testing.assert_array_equal(nm.k.counts.cpu().numpy(), O.counts(*ref.parts[0][0:1], ref.parts[0][1].shape[0]))
    n, d = ref.shape
    for m in (1, 5):
        p = rng.standard_normal((n, m))
        _close(fb.lmm(nm.T, p), O.lmm(ref.T, p))
        _close(fb.rmm(p.T.copy(), nm), O.rmm(p.T, ref))
    x = rng.standard_normal((d, 5))
    _close(fb.lmm(nm, x), O.lmm(ref, x))
    _close(fb.col_sums(nm), O.col_sums(ref))


# ---------------------------------------------------------------- crossprod (DMMA two-pass)
@pytest.mark.parametrize("name", [n for n in golden_io.names() if n != "zero_width_s"])
def test_crossprod_vs_reference_golden(name):
    fb = _fb()
    g = golden_io.load(name)
    nm = _build_gpu(g)
    c = fb.OpCounter()
    cp = fb.crossprod(nm, counter=c)
    _close(cp, g["crossprod"])
    np.testing.assert_array_equal(cp, cp.T)  # exact symmetry (rewrite.py:298)
    assert [c.multiplies, c.additions] == list(g["cnt_crossprod"])


CP_CASES = [
    # n_s, d_s, [(n_r, d_r)], key distribution, seed
    (300_001, 60, [(15_000, 120)], "uniform", 1),
    (100_003, 20, [(10_000, 40)], "uniform", 2),
    (200_000, 10, [(50, 40)], "zipf", 3),      # runs spanning many CTAs (carry fixup)
    (50_001, 7, [(997, 5)], "uniform", 4),     # odd widths: non-bulk gather fill
    (20_000, 64, [(3, 8)], "uniform", 5),      # huge runs, tiny R
    (12_345, 0, [(300, 9)], "uniform", 6),     # no entity features
    (40_001, 5, [(97, 6), (1000, 3)], "uniform", 7),  # star, odd d_S: per-part unfused S pass + cross block
    (1, 3, [(1, 2)], "uniform", 8),
    (30_001, 72, [(2000, 16)], "uniform", 9),   # fused S pass, 3 columns per walker lane
    (20_000, 100, [(500, 10)], "zipf", 10),     # fused S pass, 4 columns per walker lane
    (10_000, 130, [(100, 4)], "uniform", 11),   # d_S > 128: the block-column path
    (60_001, 20, [(4000, 40), (300, 60)], "uniform", 12),          # star, fused passes + pair-count cross block
    (50_000, 6, [(200, 5), (7000, 9), (31, 3)], "zipf", 13),      # three parts: both pair orientations
    (33_333, 8, [(1500, 16), (1500, 4)], "uniform", 14),          # equal table sizes
    (45_001, 19, [(3000, 7), (200, 12)], "zipf", 15),              # star, odd d_S, skewed keys
    (25_000, 1, [(100, 3), (50, 2)], "uniform", 16),               # star, one entity column
    (25_000, 0, [(100, 3), (50, 2)], "uniform", 17),               # star without entity features
]


@pytest.mark.parametrize("case", CP_CASES, ids=[f"cp_n{c[0]}_d{c[1]}_{c[3]}_q{len(c[2])}" for c in CP_CASES])
def test_crossprod_seeded_vs_oracle(case):
    fb = _fb()
    n_s, d_s, shapes, dist, seed = case
    rng = np.random.default_rng(seed)
    s = rng.random((n_s, d_s))
    parts = []
    for n_r, d_r in shapes:
        keys = _zipf_keys(rng, n_s, n_r) if dist == "zipf" else rng.integers(1, n_r + 1, size=n_s)
        parts.append((keys, rng.random((n_r, d_r))))
    ref = O.build_star(s, parts)
    nm = fb.build_star(s, parts) if len(parts) > 1 else fb.build_pkfk(s, parts[0][0], parts[0][1])
    cp = fb.crossprod(nm)
    _close(cp, O.crossprod(ref))
    np.testing.assert_array_equal(cp, cp.T)


@pytest.mark.parametrize("d_s,d_r", [(16, 16), (32, 20), (20, 32), (16, 32), (48, 64)])
@pytest.mark.parametrize("d_x", [1, 2, 3, 4, 17])
def test_lmm_rowdot_widths_16_32(d_s, d_r, d_x):
    """Factor widths whose lane groups span 16 / 32 lanes (rowdot kernel, d_x <= 4 and the remainder chunk of
    d_x = 17): every row of a tile must be computed (a lane group handles at most 8 rows per tile)."""
    fb = _fb()
    rng = np.random.default_rng(100 * d_s + d_r + d_x)
    n_s, n_r = 5003, 152
    s = rng.standard_normal((n_s, d_s))
    r = rng.standard_normal((n_r, d_r))
    key = rng.integers(1, n_r + 1, size=n_s)
    nm, ref = fb.build_pkfk(s, key, r), O.build_pkfk(s, key, r)
    x = rng.standard_normal((d_s + d_r, d_x))
    _close(fb.lmm(nm, x), O.lmm(ref, x))
    if d_x == 1:
        _close(fb.row_sums(nm), O.row_sums(ref))
        _close(fb.row_sums(fb.scalar_fn(nm, np.square)), O.row_sums(O.scalar_fn(ref, np.square)))


def test_fk_sorted_order_is_stable_argsort():
    fb = _fb()
    from paper_1612_07448_b200.crossprod_impl import fk_sorted_order

    rng = np.random.default_rng(9)
    key = rng.integers(1, 200, size=30_001)
    nm = fb.build_pkfk(rng.random((30_001, 2)), key, rng.random((199, 3)))
    perm, fks = fk_sorted_order(nm.k)
    t = nm.k.target_numpy()
    order = np.argsort(t, kind="stable")
    np.testing.assert_array_equal(perm.cpu().numpy(), order)
    np.testing.assert_array_equal(fks.cpu().numpy(), t[order])


def test_crossprod_dense_and_transposed_errors():
    fb = _fb()
    rng = np.random.default_rng(10)
    a = rng.standard_normal((5000, 33))
    m = fb.as_normalized(a)
    _close(fb.crossprod(m), a.T @ a)
    nm = fb.build_pkfk(a, rng.integers(1, 5, size=5000), rng.random((4, 2)))
    with pytest.raises(fb.ShapeError):
        fb.crossprod(nm.T)


@pytest.mark.parametrize("n,d", [(300_001, 5), (70_000, 3), (1000, 1), (50_000, 17)])
def test_crossprod_dense_narrow(n, d):
    """q = 0 crossprod of narrow dense factors (GNMF's WᵀW): padded-column fragment reads stay in bounds."""
    fb = _fb()
    rng = np.random.default_rng(n + d)
    a = rng.random((n, d))
    cp = fb.crossprod(fb.as_normalized(torch.from_numpy(a).cuda()))
    _close(cp, a.T @ a)
    assert torch.equal(cp, cp.t())


def test_crossprod_fused_with_unreferenced_keys():
    """An indicator whose targets skip some R rows (row-sharded builds keep every R row, so a
    shard's FK leaves gaps): KᵀS bins without rows are zeroed inside tiles, at tile seams and at
    both ends, in the fused S pass."""
    fb = _fb()
    from paper_1612_07448_b200.normmat import PKFK, IndicatorMatrix, NormalizedMatrix

    rng = np.random.default_rng(12)
    n_s, d_s, n_r, d_r = 150_001, 12, 4000, 6
    used = np.sort(rng.choice(np.arange(3, n_r - 5), size=900, replace=False))  # rows 0-2, tail unused
    target = rng.choice(used, size=n_s)
    s = rng.random((n_s, d_s))
    r = rng.random((n_r, d_r))
    ind = IndicatorMatrix(torch.from_numpy(target.astype(np.int32)).cuda(), n_r)
    nm = NormalizedMatrix(PKFK, [(None, torch.from_numpy(s).cuda()), (ind, torch.from_numpy(r).cuda())])
    cp = fb.crossprod(nm).cpu().numpy()
    t = np.hstack([s, r[target]])
    _close(cp, t.T @ t)
    np.testing.assert_array_equal(cp, cp.T)


def test_crossprod_fused_and_unfused_s_pass_agree(monkeypatch):
    """The fused S pass (SᵀS + KᵀS from one FK-sorted stream) and the two-kernel path
    (storage-order SᵀS gram + kts_walk_kernel) agree to rounding; so do the narrow-matrix gram
    and the DMMA gram for a plain d <= 8 matrix."""
    fb = _fb()
    rng = np.random.default_rng(13)
    n_s, d_s, n_r, d_r = 80_001, 30, 3000, 12
    s = rng.random((n_s, d_s))
    keys = rng.integers(1, n_r + 1, size=n_s)
    r = rng.random((n_r, d_r))
    nm = fb.build_pkfk(s, keys, r)
    fused = fb.crossprod(nm)
    monkeypatch.setenv("FB_CP_UNFUSED", "1")
    unfused = fb.crossprod(nm)
    _close(fused, unfused, 1e-13)
    np.testing.assert_array_equal(unfused, unfused.T)
    w = torch.from_numpy(rng.random((200_003, 6))).cuda()
    narrow = fb.crossprod(fb.as_normalized(w))
    monkeypatch.setenv("FB_CP_NO_NARROW", "1")
    dmma = fb.crossprod(fb.as_normalized(w))
    _close(narrow, dmma.cpu().numpy(), 1e-13)


@pytest.mark.parametrize("n_s,d_s,n_r,d_r,d_x,zipf", [
    (100_003, 20, 5_000, 12, 16, False),   # partial last tile (rows*4 not a multiple of 16)
    (65_536, 20, 3_001, 8, 8, False),      # whole tiles only
    (40_000, 7, 2_000, 5, 16, True),       # ragged k-step, skewed keys (uneven bands)
    (30_000, 32, 1_000, 3, 40, False),     # d_x = 16 + 16 + 8 column chunks
    (257, 4, 9, 2, 16, False),             # two tiles, more bands than CTAs have rows
])
def test_lmm_band_layout_bitwise_equal(monkeypatch, n_s, d_s, n_r, d_r, d_x, zipf):
    """The FK-band S pass (fb_lmm_banded: cached band copy of S, round-robin tiles, permuted
    stores) gives the same bits as the storage-order pass and matches the oracle."""
    fb = _fb()
    from paper_1612_07448_b200.normmat import NormalizedMatrix

    rng = np.random.default_rng(n_s + d_x)
    s = rng.standard_normal((n_s, d_s))
    r = rng.standard_normal((n_r, d_r))
    if zipf:
        key = np.minimum(rng.zipf(1.3, size=n_s), n_r)
    else:
        key = rng.integers(1, n_r + 1, size=n_s)
    x = rng.standard_normal((d_s + d_r, d_x))
    monkeypatch.setattr(NormalizedMatrix, "BAND_MIN_BYTES", 0)
    nm0 = fb.build_pkfk(s, key, r)
    plain = fb.lmm(nm0, x)
    assert "band" not in nm0._cache
    monkeypatch.setattr(NormalizedMatrix, "BAND_MIN_BYTES", 1)
    monkeypatch.setattr(NormalizedMatrix, "BAND_BYTES", 128 * max(1, nm0.parts[0][1].shape[0] // 7))
    nm = fb.build_pkfk(s, key, r)
    banded = fb.lmm(nm, x)
    assert "band" in nm._cache
    st, perm, fkb, sb = nm._cache["band"]
    assert st.n_bands >= 2
    p = perm.cpu().numpy()
    tgt = nm.k.target_numpy()
    band = tgt * st.n_bands // nm.parts[0][1].shape[0]
    np.testing.assert_array_equal(p, np.argsort(band, kind="stable"))
    np.testing.assert_array_equal(fkb[0].cpu().numpy(), tgt[p])
    np.testing.assert_array_equal(sb.cpu().numpy(), s[p])
    np.testing.assert_array_equal(banded, plain)
    again = fb.lmm(nm, x)  # cached layout reused
    np.testing.assert_array_equal(again, plain)
    _close(banded, O.lmm(O.build_pkfk(s, key, r), x))


def test_scalar_fn_arbitrary_callables():
    """scalar_fn on callables outside the built-in ufunc set (rewrite.py:89-99 takes any f)."""
    import warnings

    fb = _fb()
    g = golden_io.load(golden_io.names()[0])
    nm = _build_gpu(g)
    ref = O.build_pkfk(g["s"], golden_io.parts(g)[0][0], golden_io.parts(g)[0][1]) if len(golden_io.parts(g)) == 1 \
        else O.build_star(g["s"], golden_io.parts(g))

    def poly(a):  # array-polymorphic: runs on the device tensors
        return a * a * 0.5 + 1.0

    with warnings.catch_warnings():
        warnings.simplefilter("error")
        out = fb.scalar_fn(nm, poly)
    _close(fb.materialize(out), O.materialize(O.scalar_fn(ref, poly)))

    def host_only(a):  # needs an ndarray (np.where on a CUDA tensor raises)
        return np.where(np.asarray(a) > 0.0, np.arctan(a), -1.0)

    with pytest.warns(fb.HostCallableWarning):
        out = fb.scalar_fn(nm, host_only)
    _close(fb.materialize(out), O.materialize(O.scalar_fn(ref, host_only)))
    c = fb.OpCounter()
    fb.scalar_fn(nm, poly, c)  # one multiply per stored factor element (kernel.py:296-298)
    assert (c.multiplies, c.additions) == (sum(f.numel() for _, f in nm.blocks), 0)
    with pytest.raises(ValueError):
        fb.scalar_fn(nm, "no_such_function")
    with pytest.raises(fb.ShapeError):
        fb.scalar_fn(nm, lambda a: np.asarray(a).sum(axis=0))

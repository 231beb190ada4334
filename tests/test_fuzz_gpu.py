"""Randomised fixtures: the device operators against the CPU oracle on many small random schemas.

The reference's spec names an "oracle suite of 1000 random fixtures, rel 1e-10" as an acceptance
criterion it never shipped. This is that suite for the hot path: every fixture draws
a schema (PK-FK, star with 2-3 attribute tables, M:N or multi-table M:N), its shapes — including single rows, d_S = 0,
odd widths, attribute rows no key references, keys that repeat one value — and its operands from one
seed, builds it on the device and in the oracle, checks the construction bit for bit and every
operator at normwise rel 1e-10 (bench.py:38-43's metric). FB_FUZZ_N sets the fixture count
(default 1000, the spec's number: under half a minute on a B200).

First run (round 2): fixture 10011 — a 16-wide attribute table under a d_x = 1 LMM — exposed that the rowdot kernel
computed only the first 8 rows of each lane group for factor widths 16 and 32 (fb_lmm.cu launch_rowdot). The driver
fixtures then found the fused K-Means / GNMF passes chosen for star shapes whose ring does not fit ("unsupported
size" instead of the operator-by-operator step) and an out-of-range store of the Rᵀ·X reduce (cp_reduce_kernel's
bound in r1only mode) that overwrote the first cluster sizes of K-Means for even k > 16 not a multiple of 8.
"""
import os

import numpy as np
import pytest
import torch

import factorla_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-10
N_FIXTURES = int(os.environ.get("FB_FUZZ_N", "1000"))
BATCH = 50


def _np(a):
    return a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)


def _check(tag, got, want, tol=TOL):
    got, want = _np(got), np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (tag, got.shape, want.shape)
    dev = O.max_rel_deviation(got, want)
    assert dev <= tol, (tag, dev)


def _check_scaled(tag, got, want, scale, tol):
    """|got - want| against an explicit scale: objectives that are differences of large sums (K-Means with one
    point per cluster, GNMF with an exact fit) are rounding noise around zero in the reference too."""
    got, want = _np(got).ravel(), np.asarray(want, dtype=np.float64).ravel()
    assert got.shape == want.shape, (tag, got.shape, want.shape)
    dev = float(np.max(np.abs(got - want))) / max(float(scale), 1e-300) if got.size else 0.0
    assert dev <= tol, (tag, dev)


def _draw_keys(rng, n, n_r):
    mode = rng.integers(0, 4)
    if mode == 0:  # uniform
        return rng.integers(1, n_r + 1, size=n)
    if mode == 1:  # only a few rows of R referenced
        live = rng.choice(n_r, size=max(1, n_r // 3), replace=False) + 1
        return rng.choice(live, size=n)
    if mode == 2:  # one value
        return np.full(n, int(rng.integers(1, n_r + 1)))
    w = 1.0 / np.arange(1, n_r + 1) ** 1.3  # skewed
    return rng.choice(n_r, size=n, p=w / w.sum()) + 1


def _draw(seed):
    rng = np.random.default_rng(seed)
    kind = ("pkfk", "pkfk", "star", "star", "mn")[rng.integers(0, 5)]
    small = rng.integers(0, 4) == 0
    n = int(rng.integers(1, 40)) if small else int(rng.integers(40, 4000))
    if kind == "mn" and rng.integers(0, 2):  # half of the M:N fixtures: multi-table, explicit 0-based row map
        q = int(rng.integers(2, 5))
        tables = [rng.standard_normal((int(rng.integers(1, 80)), int(rng.integers(1, 12)))) for _ in range(q)]
        row_map = np.stack([rng.integers(0, t.shape[0], size=n) for t in tables], axis=1)
        return "multimn", rng, (row_map, tables)
    if kind == "mn":
        n_s, n_r = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        dom = int(rng.integers(1, 8))
        s = rng.standard_normal((n_s, int(rng.integers(1, 9))))
        r = rng.standard_normal((n_r, int(rng.integers(1, 9))))
        j_s, j_r = rng.integers(0, dom, size=n_s), rng.integers(0, dom, size=n_r)
        if not np.intersect1d(j_s, j_r).size:  # an empty join is an error in the reference: force one match
            j_r[0] = j_s[0]
        return kind, rng, (s, j_s, r, j_r)
    d_s = int(rng.integers(0, 41))
    q = 1 if kind == "pkfk" else int(rng.integers(2, 4))
    parts = []
    for _ in range(q):
        n_r = int(rng.integers(1, 30)) if small else int(rng.integers(1, 500))
        parts.append((_draw_keys(rng, n, n_r), rng.standard_normal((n_r, int(rng.integers(1, 33))))))
    return kind, rng, (rng.standard_normal((n, d_s)), parts)


def _build(fb, kind, data):
    if kind == "mn":
        return fb.build_mn(*data), O.build_mn(*data)
    if kind == "multimn":
        return fb.build_multimn(*data), O.build_multimn(*data)
    s, parts = data
    if kind == "pkfk":
        return fb.build_pkfk(s, parts[0][0], parts[0][1]), O.build_pkfk(s, parts[0][0], parts[0][1])
    return fb.build_star(s, parts), O.build_star(s, parts)


def _one_fixture(fb, seed):
    kind, rng, data = _draw(seed)
    nm, ref = _build(fb, kind, data)
    # construction: indicator targets, kept rows and counts bit for bit
    inds = nm.indicator_blocks
    assert len(inds) == len(ref.parts)
    for (e, f), (t, kept) in zip(inds, ref.parts):
        np.testing.assert_array_equal(e.target_numpy(), t)
        np.testing.assert_array_equal(_np(f), kept)
        np.testing.assert_array_equal(_np(e.counts), O.counts(t, kept.shape[0]))
    t_ref = O.materialize(ref)
    n, d = t_ref.shape
    _check("materialize", fb.materialize(nm), t_ref, 0.0)
    dx, dp = int(rng.integers(1, 20)), int(rng.integers(1, 20))
    x = rng.standard_normal((d, dx))
    p = rng.standard_normal((n, dp))
    _check("lmm", fb.lmm(nm, x), O.lmm(ref, x))
    _check("tmm", fb.lmm(nm.T, p), O.lmm(ref.T, p))
    _check("rmm", fb.rmm(np.ascontiguousarray(p.T), nm), O.rmm(p.T, ref))
    _check("row_sums", fb.row_sums(nm), O.row_sums(ref))
    _check("col_sums", fb.col_sums(nm), O.col_sums(ref))
    _check("sum_all", np.asarray(fb.sum_all(nm)), np.asarray(O.sum_all(ref)))
    cp = _np(fb.crossprod(nm))
    _check("crossprod", cp, O.crossprod(ref))
    np.testing.assert_array_equal(cp, cp.T)
    c = float(rng.standard_normal()) + 3.0
    op = ("add", "rsub", "mul", "div")[rng.integers(0, 4)]
    _check("scalar_" + op, fb.materialize(fb.scalar_op(nm, c, op)), O.materialize(O.scalar_op(ref, c, op)))
    _check("scalar_fn", fb.materialize(fb.scalar_fn(nm, np.square)), O.materialize(O.scalar_fn(ref, np.square)))


@pytest.mark.parametrize("batch", range((N_FIXTURES + BATCH - 1) // BATCH))
def test_random_fixtures_vs_oracle(batch):
    import paper_1612_07448_b200 as fb

    for seed in range(batch * BATCH, min((batch + 1) * BATCH, N_FIXTURES)):
        try:
            _one_fixture(fb, 10_000 + seed)
        except Exception as e:  # name the fixture: a failure must be reproducible from its seed
            raise AssertionError(f"fixture seed {10_000 + seed}: {type(e).__name__}: {e}") from e


# --------------------------------------------------------------------------- drivers and the transposed side
N_DRIVER = int(os.environ.get("FB_FUZZ_DRIVERS", "400"))
DTOL = 1e-9  # drivers: the north star's bar (iterated sums; K-Means ties would show as O(1) deviations)


def _draw_medium(seed):
    """PK-FK / star schemas whose passes span many tiles and CTAs (4k-150k rows)."""
    rng = np.random.default_rng(seed)
    q = int(rng.integers(1, 4))
    n = int(rng.integers(4_000, 150_000))
    parts = []
    for _ in range(q):
        n_r = int(rng.integers(1, 5_000))
        parts.append((_draw_keys(rng, n, n_r), rng.standard_normal((n_r, int(rng.integers(1, 41))))))
    return ("pkfk" if q == 1 else "star"), rng, (rng.standard_normal((n, int(rng.integers(0, 41)))), parts)


def _one_driver_fixture(fb, seed, draw=None):
    kind, rng, data = (draw or _draw)(seed)
    if kind == "multimn":
        data = (data[0], [np.abs(t) for t in data[1]])
    elif kind != "mn":  # non-negative data so GNMF runs on the same fixture
        s, parts = data
        data = (np.abs(s), [(k, np.abs(r)) for k, r in parts])
    else:
        s, j_s, r, j_r = data
        data = (np.abs(s), j_s, np.abs(r), j_r)
    nm, ref = _build(fb, kind, data)
    t_ref = O.materialize(ref)
    n, d = t_ref.shape
    # transposed side: rowSums / colSums / sum of T', T'·P
    _check("row_sums_T", fb.row_sums(nm.T), O.row_sums(ref.T), TOL)
    _check("col_sums_T", fb.col_sums(nm.T), O.col_sums(ref.T), TOL)
    p = rng.standard_normal((dpw := int(rng.integers(1, 6)), d))
    _check("rmm_T", fb.rmm(p, nm.T), O.rmm(p, ref.T), TOL)
    # GLMs
    it = int(rng.integers(1, 5))
    y = np.where(O.lmm(ref, rng.standard_normal((d, 1))) >= np.median(t_ref.sum(axis=1)), 1.0, -1.0)
    step = 1e-3 / max(1, n)
    out = fb.logistic_gd(nm, y, fb.TrainConfig(iterations=it, step_size=step))
    w, obj = O.logistic_gd(ref, y, it, step)
    _check("logreg_w", out.weights, w, DTOL)
    _check("logreg_obj", out.objective, obj, DTOL)
    yl = O.lmm(ref, rng.standard_normal((d, 1))) + 0.01 * rng.standard_normal((n, 1))
    out = fb.linreg_gd(nm, yl, fb.TrainConfig(iterations=it, step_size=step))
    w, obj = O.linreg_gd(ref, yl, it, step)
    _check("linreg_w", out.weights, w, DTOL)
    _check("linreg_obj", out.objective, obj, DTOL)
    # K-Means (k <= n) and GNMF
    k = int(rng.integers(1, min(n, 40) + 1))
    out = fb.kmeans(nm, fb.TrainConfig(iterations=it, k=k, rng_seed=seed))
    c, obj, _ = O.kmeans(ref, k, it, seed)
    _check("kmeans_c", out.centroids, c, DTOL)
    _check_scaled("kmeans_obj", out.objective, obj, float((t_ref * t_ref).sum()), DTOL)
    r = int(rng.integers(1, 40))
    out = fb.gnmf(nm, fb.TrainConfig(iterations=it, r=r, rng_seed=seed))
    w, h, obj = O.gnmf(ref, r, it, seed)
    _check("gnmf_w", out.factors[0], w, DTOL)
    _check("gnmf_h", out.factors[1], h, DTOL)
    # sqrt of a difference of large sums (ml.py:314-315): an error e in the difference shows as sqrt(e)
    _check_scaled("gnmf_obj", out.objective, obj, float(np.sqrt((t_ref * t_ref).sum())), 1e-6)


@pytest.mark.parametrize("batch", range((N_DRIVER + BATCH - 1) // BATCH))
def test_random_fixtures_drivers_vs_oracle(batch):
    import warnings

    import paper_1612_07448_b200 as fb

    for seed in range(batch * BATCH, min((batch + 1) * BATCH, N_DRIVER)):
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                _one_driver_fixture(fb, 50_000 + seed)
        except Exception as e:
            raise AssertionError(f"driver fixture seed {50_000 + seed}: {type(e).__name__}: {e}") from e


# --------------------------------------------------------------------------- larger shapes, products, CSR inputs
N_MEDIUM = int(os.environ.get("FB_FUZZ_MEDIUM", "60"))


def _one_medium_fixture(fb, seed):
    """Shapes that span many tiles and CTAs (up to 300k rows), wider operands, scipy CSR factors,
    T·Tᵀ (small n only), and the normal equations."""
    import scipy.sparse as sp

    rng = np.random.default_rng(seed)
    q = int(rng.integers(1, 4))
    n = int(rng.integers(4_000, 300_000))
    d_s = int(rng.integers(0, 70))
    s = rng.standard_normal((n, d_s))
    parts = []
    for _ in range(q):
        n_r = int(rng.integers(1, 20_000))
        parts.append((_draw_keys(rng, n, n_r), rng.standard_normal((n_r, int(rng.integers(1, 90))))))
    csr = rng.integers(0, 4) == 0  # a quarter of the fixtures hand the attribute tables over as scipy CSR
    if csr:
        dev_parts = []
        for k, r in parts:
            r = r * (rng.random(r.shape) < 0.04)
            dev_parts.append((k, r))
        parts = dev_parts
        gpu_parts = [(k, sp.csr_matrix(r)) for k, r in parts]
    else:
        gpu_parts = parts
    if q == 1:
        nm, ref = fb.build_pkfk(s, gpu_parts[0][0], gpu_parts[0][1]), O.build_pkfk(s, parts[0][0], parts[0][1])
    else:
        nm, ref = fb.build_star(s, gpu_parts), O.build_star(s, parts)
    d = ref.d
    dx, dp = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    x = rng.standard_normal((d, dx))
    p = rng.standard_normal((n, dp))
    _check("lmm", fb.lmm(nm, x), O.lmm(ref, x))
    _check("tmm", fb.lmm(nm.T, p), O.lmm(ref.T, p))
    _check("rmm", fb.rmm(np.ascontiguousarray(p.T), nm), O.rmm(p.T, ref))
    _check("row_sums", fb.row_sums(nm), O.row_sums(ref))
    _check("col_sums", fb.col_sums(nm), O.col_sums(ref))
    cp = _np(fb.crossprod(nm))
    _check("crossprod", cp, O.crossprod(ref))
    np.testing.assert_array_equal(cp, cp.T)
    if not csr:
        y = O.lmm(ref, rng.standard_normal((d, 1))) + 0.01 * rng.standard_normal((n, 1))
        out = fb.linreg_normal(nm, y)
        w, obj = O.linreg_normal(ref, y)
        _check("linreg_normal_obj", out.objective, obj, 1e-7)  # pinv of a d × d Gram on both sides


@pytest.mark.parametrize("batch", range((N_MEDIUM + 9) // 10))
def test_random_medium_fixtures_vs_oracle(batch):
    import warnings

    import paper_1612_07448_b200 as fb

    for seed in range(batch * 10, min((batch + 1) * 10, N_MEDIUM)):
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                _one_medium_fixture(fb, 90_000 + seed)
        except Exception as e:
            raise AssertionError(f"medium fixture seed {90_000 + seed}: {type(e).__name__}: {e}") from e


N_MEDIUM_DRIVER = int(os.environ.get("FB_FUZZ_MEDIUM_DRIVERS", "40"))


@pytest.mark.parametrize("batch", range((N_MEDIUM_DRIVER + 9) // 10))
def test_random_medium_fixtures_drivers_vs_oracle(batch):
    import warnings

    import paper_1612_07448_b200 as fb

    for seed in range(batch * 10, min((batch + 1) * 10, N_MEDIUM_DRIVER)):
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                _one_driver_fixture(fb, 110_000 + seed, _draw_medium)
        except Exception as e:
            raise AssertionError(f"medium driver fixture seed {110_000 + seed}: {type(e).__name__}: {e}") from e


N_PRODUCT = int(os.environ.get("FB_FUZZ_PRODUCTS", "150"))


def _one_product_fixture(fb, seed):
    """T·Tᵀ, the pseudo-inverse through the small Gram and the pair-count product on small schemas."""
    kind, rng, data = _draw(seed)
    if kind in ("mn", "multimn"):
        return
    s, parts = data
    n = min(s.shape[0], 300)  # T·Tᵀ is n × n
    s, parts = s[:n], [(k[:n], r) for k, r in parts]
    nm, ref = _build(fb, kind, (s, parts))
    g = _np(fb.gram_transposed(nm))
    _check("gram_transposed", g, O.gram_transposed(ref))
    np.testing.assert_array_equal(g, g.T)
    t_ref = O.materialize(ref)
    if kind == "pkfk":  # double multiplication takes PK-FK operands only, as in the reference (rewrite.py:349-389)
        _check("dmm_a_at", fb.dmm(nm, nm.T), t_ref @ t_ref.T)
        _check("dmm_at_a", fb.dmm(nm.T, nm), t_ref.T @ t_ref)
    if len(parts) >= 2:
        (ea, _), (eb, _) = nm.indicator_blocks[:2]
        (ta, ra), (tb, rb) = ref.parts[:2]
        pp = fb.pair_product(ea, eb)
        np.testing.assert_array_equal(pp.to_dense().cpu().numpy(), O.pair_product(ta, ra.shape[0], tb, rb.shape[0]))


@pytest.mark.parametrize("batch", range((N_PRODUCT + BATCH - 1) // BATCH))
def test_random_fixtures_products_vs_oracle(batch):
    import warnings

    import paper_1612_07448_b200 as fb

    for seed in range(batch * BATCH, min((batch + 1) * BATCH, N_PRODUCT)):
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                _one_product_fixture(fb, 70_000 + seed)
        except Exception as e:
            raise AssertionError(f"product fixture seed {70_000 + seed}: {type(e).__name__}: {e}") from e


N_WIDE = int(os.environ.get("FB_FUZZ_WIDE", "40"))


def _one_wide_fixture(fb, seed):
    """Wide factor matrices (60-300 columns: past the streaming kernels' 128 / 256-column paths)."""
    rng = np.random.default_rng(seed)
    q = int(rng.integers(1, 3))
    n = int(rng.integers(500, 20_000))
    s = rng.standard_normal((n, int(rng.integers(60, 301))))
    parts = []
    for _ in range(q):
        n_r = int(rng.integers(1, 2_000))
        parts.append((_draw_keys(rng, n, n_r), rng.standard_normal((n_r, int(rng.integers(60, 301))))))
    if q == 1:
        nm, ref = fb.build_pkfk(s, parts[0][0], parts[0][1]), O.build_pkfk(s, parts[0][0], parts[0][1])
    else:
        nm, ref = fb.build_star(s, parts), O.build_star(s, parts)
    d = ref.d
    x = rng.standard_normal((d, int(rng.integers(1, 40))))
    p = rng.standard_normal((n, int(rng.integers(1, 40))))
    _check("lmm", fb.lmm(nm, x), O.lmm(ref, x))
    _check("tmm", fb.lmm(nm.T, p), O.lmm(ref.T, p))
    _check("rmm", fb.rmm(np.ascontiguousarray(p.T), nm), O.rmm(p.T, ref))
    _check("row_sums", fb.row_sums(nm), O.row_sums(ref))
    _check("col_sums", fb.col_sums(nm), O.col_sums(ref))
    _check("sum_all", np.asarray(fb.sum_all(nm)), np.asarray(O.sum_all(ref)), 1e-9)
    if max([s.shape[1]] + [r.shape[1] for _, r in parts]) <= 256:
        cp = _np(fb.crossprod(nm))
        _check("crossprod", cp, O.crossprod(ref))
        np.testing.assert_array_equal(cp, cp.T)
    else:  # the documented limit of the crossprod kernels: a clear error, not a wrong answer
        with pytest.raises(ValueError, match="widths above 256"):
            fb.crossprod(nm)


@pytest.mark.parametrize("batch", range((N_WIDE + 9) // 10))
def test_random_wide_fixtures_vs_oracle(batch):
    import warnings

    import paper_1612_07448_b200 as fb

    for seed in range(batch * 10, min((batch + 1) * 10, N_WIDE)):
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                _one_wide_fixture(fb, 130_000 + seed)
        except Exception as e:
            raise AssertionError(f"wide fixture seed {130_000 + seed}: {type(e).__name__}: {e}") from e

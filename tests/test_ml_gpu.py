"""GPU parity of the ML drivers (ml.py) against the reference golden traces and the oracle.

Bars: float64 model state and objective traces within normwise rel 1e-9 of the reference
(bench.py:38-43 metric); K-Means assignments compared through the centroids and trace.
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


def _close(a, b, tol=TOL, what=""):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    dev = O.max_rel_deviation(a, b)
    assert dev <= tol, (what, dev, a.ravel()[:6], b.ravel()[:6])


def _build_gpu(g):
    fb = _fb()
    parts = golden_io.parts(g)
    if len(parts) == 1:
        return fb.build_pkfk(g["s"], parts[0][0], parts[0][1])
    return fb.build_star(g["s"], parts)


GOLD = [n for n in golden_io.names() if n != "zero_width_s"]


@pytest.mark.parametrize("name", GOLD)
def test_drivers_vs_reference_golden(name):
    fb = _fb()
    g = golden_io.load(name)
    nm = _build_gpu(g)
    cfg = fb.TrainConfig(iterations=5, step_size=1e-3, k=3, r=2, rng_seed=3)
    out = fb.logistic_gd(nm, g["y_log"], cfg)
    _close(out.weights, g["logreg_w"], what="logreg_w")
    _close(out.objective, g["logreg_obj"], what="logreg_obj")
    out = fb.linreg_gd(nm, g["y_lin"], cfg)
    _close(out.weights, g["linreg_gd_w"], what="linreg_gd_w")
    out = fb.kmeans(nm, cfg)
    _close(out.centroids, g["kmeans_c"], what="kmeans_c")
    _close(out.objective, g["kmeans_obj"], what="kmeans_obj")
    if "gnmf_w" in g:
        out = fb.gnmf(nm, cfg)
        _close(out.factors[0], g["gnmf_w"], what="gnmf_w")
        _close(out.factors[1], g["gnmf_h"], what="gnmf_h")
        _close(out.objective, g["gnmf_obj"], what="gnmf_obj")
    out = fb.linreg_normal(nm, g["y_lin"])
    _close(out.weights, g["linreg_w"], what="linreg_w")
    # the residual of an exact fit is rounding noise: compare against ‖y‖²
    scale = max(float(g["linreg_obj"][0]), float(np.sum(g["y_lin"] ** 2)))
    assert abs(out.objective[0] - float(g["linreg_obj"][0])) <= TOL * scale


def _c1_like(seed, n_s=100_000, d_s=20, n_r=10_000, d_r=40, star=False):
    rng = np.random.default_rng(seed)
    s = rng.standard_normal((n_s, d_s))
    parts = [(rng.integers(1, n_r + 1, size=n_s), rng.standard_normal((n_r, d_r)))]
    if star:
        parts.append((rng.integers(1, 501, size=n_s), rng.standard_normal((500, 7))))
    return rng, s, parts


def _both(s, parts):
    fb = _fb()
    nm = fb.build_star(s, parts) if len(parts) > 1 else fb.build_pkfk(s, parts[0][0], parts[0][1])
    return nm, O.build_star(s, parts)


def test_logreg_c1_shape_20_iterations():
    fb = _fb()
    rng, s, parts = _c1_like(11)
    nm, ref = _both(s, parts)
    w_true = rng.standard_normal((ref.d, 1))
    y = np.where(O.lmm(ref, w_true) >= 0, 1.0, -1.0)
    out = fb.logistic_gd(nm, y, fb.TrainConfig(iterations=20, step_size=1e-3))
    w, obj = O.logistic_gd(ref, y, 20, 1e-3)
    _close(out.weights, w)
    _close(out.objective, obj)
    assert out.counts.multiplies > 0


def test_linreg_gd_and_normal_star():
    fb = _fb()
    rng, s, parts = _c1_like(12, n_s=60_001, d_s=9, n_r=3000, d_r=13, star=True)
    nm, ref = _both(s, parts)
    y = O.lmm(ref, rng.standard_normal((ref.d, 1))) + 0.01 * rng.standard_normal((ref.n, 1))
    out = fb.linreg_gd(nm, y, fb.TrainConfig(iterations=7, step_size=1e-6))
    w, obj = O.linreg_gd(ref, y, 7, 1e-6)
    _close(out.weights, w)
    _close(out.objective, obj)
    out = fb.linreg_normal(nm, y)
    w, obj = O.linreg_normal(ref, y)
    _close(out.weights, w, 1e-8)
    _close(out.objective, obj, 1e-8)


def test_kmeans_star_vs_oracle():
    fb = _fb()
    rng, s, parts = _c1_like(13, n_s=80_000, d_s=6, n_r=2000, d_r=5, star=True)
    nm, ref = _both(s, parts)
    out = fb.kmeans(nm, fb.TrainConfig(iterations=6, k=10, rng_seed=5))
    c, obj, _ = O.kmeans(ref, 10, 6, 5)
    _close(out.centroids, c)
    _close(out.objective, obj)


def test_gnmf_zipf_vs_oracle():
    fb = _fb()
    rng = np.random.default_rng(14)
    n_s, n_r = 50_000, 500
    p = np.arange(1, n_r + 1, dtype=np.float64) ** -1.2
    p /= p.sum()
    key = np.minimum(np.searchsorted(np.cumsum(p), rng.random(n_s), side="right"), n_r - 1) + 1
    s = rng.random((n_s, 10))
    r = rng.random((n_r, 40))
    nm, ref = _both(s, [(key, r)])
    out = fb.gnmf(nm, fb.TrainConfig(iterations=6, r=5, rng_seed=2))
    w, h, obj = O.gnmf(ref, 5, 6, 2)
    _close(out.factors[0], w)
    _close(out.factors[1], h)
    _close(out.objective, obj)


def test_dense_matrix_input():
    fb = _fb()
    rng = np.random.default_rng(15)
    a = rng.standard_normal((20_000, 12))
    y = np.where(a @ rng.standard_normal((12, 1)) >= 0, 1.0, -1.0)
    out = fb.logistic_gd(a, y, fb.TrainConfig(iterations=4, step_size=1e-3))
    w, obj = O.logistic_gd(O.NM(a, []), y, 4, 1e-3)
    _close(out.weights, w)


def test_divergence_error_iteration():
    """DivergenceError carries the first iteration whose weights are not finite (ml.py:190-192)."""
    fb = _fb()
    a = np.full((100, 2), 1e300)
    y = np.ones((100, 1))
    # reference semantics on the host: w -= α Tᵀ(Tw − y), check after each update
    w, expect = np.zeros((2, 1)), None
    with np.errstate(all="ignore"):
        for it in range(3):
            w = w - 1.0 * (a.T @ (a @ w - y))
            if not np.all(np.isfinite(w)):
                expect = it
                break
    assert expect is not None
    with pytest.raises(fb.DivergenceError) as ei:
        fb.linreg_gd(a, y, fb.TrainConfig(iterations=3, step_size=1.0))
    assert ei.value.iteration == expect


def test_logreg_graph_replay_matches_eager(monkeypatch):
    """The captured CUDA graph of a GD run reproduces the eager run (and the oracle)."""
    fb = _fb()
    rng, s, parts = _c1_like(21, n_s=30_000, n_r=3000)
    nm, ref = _both(s, parts)
    y = np.where(O.lmm(ref, rng.standard_normal((ref.d, 1))) >= 0, 1.0, -1.0)
    yd = torch.from_numpy(y).cuda()
    cfg = fb.TrainConfig(iterations=6, step_size=1e-3)
    first = fb.logistic_gd(nm, yd, cfg)   # eager run + capture
    again = fb.logistic_gd(nm, yd, cfg)   # graph replay
    # the Kᵀp scatter uses atomics, so runs agree to rounding, not bit for bit
    _close(again.weights, first.weights, 1e-12)
    _close(again.objective, first.objective, 1e-12)
    monkeypatch.setenv("FB_NO_GRAPHS", "1")
    eager = fb.logistic_gd(nm, yd, cfg)
    _close(eager.weights, first.weights, 1e-12)
    w, obj = O.logistic_gd(ref, y, 6, 1e-3)
    _close(again.weights, w)
    _close(again.objective, obj)


def test_logreg_fused_run_matches_stepwise(monkeypatch):
    """The single cooperative GD launch (L2-resident problems) and the per-iteration fused
    steps (CUDA graph) agree to rounding (the Kᵀp scatter uses atomics) and with the oracle."""
    fb = _fb()
    rng, s, parts = _c1_like(22, n_s=50_000, n_r=4000)
    nm, ref = _both(s, parts)
    y = np.where(O.lmm(ref, rng.standard_normal((ref.d, 1))) >= 0, 1.0, -1.0)
    yd = torch.from_numpy(y).cuda()
    cfg = fb.TrainConfig(iterations=8, step_size=1e-3)
    fused = fb.logistic_gd(nm, yd, cfg)
    monkeypatch.setenv("FB_GLM_STEPWISE", "1")
    steps = fb.logistic_gd(nm, yd, cfg)
    _close(fused.weights, steps.weights, 1e-12)
    _close(fused.objective, steps.objective, 1e-12)
    w, obj = O.logistic_gd(ref, y, 8, 1e-3)
    _close(fused.weights, w)
    _close(fused.objective, obj)
    yl = O.lmm(ref, rng.standard_normal((ref.d, 1)))
    lcfg = fb.TrainConfig(iterations=5, step_size=1e-7)
    lin_steps = fb.linreg_gd(nm, yl, lcfg)
    monkeypatch.delenv("FB_GLM_STEPWISE")
    lin_fused = fb.linreg_gd(nm, yl, lcfg)
    _close(lin_fused.weights, lin_steps.weights, 1e-12)
    w, obj = O.linreg_gd(ref, yl, 5, 1e-7)
    _close(lin_fused.weights, w)
    _close(lin_fused.objective, obj)


def test_glm_host_inputs_do_not_pin_device_memory():
    """Host y / host-built matrices: the per-iteration graph path must not cache (and so pin)
    device copies made from host inputs (ml.py GLM graph cache key)."""
    fb = _fb()
    rng = np.random.default_rng(8)
    n, n_r = 2_000_000, 20_000  # 320 MB of S: beyond L2, so fb_glm_run takes the per-iteration path
    s = rng.standard_normal((n, 20))
    r = rng.standard_normal((n_r, 10))
    nm = fb.build_pkfk(s, rng.integers(1, n_r + 1, size=n), r)
    y = np.where(rng.standard_normal((n, 1)) >= 0, 1.0, -1.0)
    cfg = fb.TrainConfig(iterations=3, step_size=1e-4)
    first = fb.logistic_gd(nm, y, cfg)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    for _ in range(4):
        out = fb.logistic_gd(nm, y, cfg)
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() <= base + (1 << 20)
    assert O.max_rel_deviation(out.weights, first.weights) <= 1e-12  # Kᵀp scatter order (REDs) varies


@pytest.mark.parametrize("k", [17, 18, 20, 28, 33, 64, 100, 150])
def test_kmeans_wide_k_vs_oracle(k):
    """k above the fused pass's 16 columns: chunked T·(2C), assign, one-hot and chunked R passes
    (k = 150: the one-hot sums go window by window of 64 clusters)."""
    fb = _fb()
    rng, s, parts = _c1_like(31 + k, n_s=40_000, d_s=6, n_r=1500, d_r=5, star=True)
    nm, ref = _both(s, parts)
    out = fb.kmeans(nm, fb.TrainConfig(iterations=4, k=k, rng_seed=5))
    c, obj, _ = O.kmeans(ref, k, 4, 5)
    _close(out.centroids, c)
    _close(out.objective, obj)
    with pytest.raises(NotImplementedError):
        fb.kmeans(nm, fb.TrainConfig(iterations=1, k=4097))


@pytest.mark.parametrize("r", [17, 40, 70, 130])
def test_gnmf_wide_r_vs_oracle(r):
    """r above the fused pass's 16 columns: the operator-by-operator step (LMM, Tᵀ·W, WᵀW)."""
    fb = _fb()
    rng = np.random.default_rng(40 + r)
    n_s, n_r = 30_000, 400
    key = rng.integers(1, n_r + 1, size=n_s)
    s = rng.random((n_s, 10))
    rr = rng.random((n_r, 24))
    nm, ref = _both(s, [(key, rr)])
    out = fb.gnmf(nm, fb.TrainConfig(iterations=4, r=r, rng_seed=2))
    w, h, obj = O.gnmf(ref, r, 4, 2)
    _close(out.factors[0], w)
    _close(out.factors[1], h)
    _close(out.objective, obj)


def test_kmeans_band_layout_matches_storage_order(monkeypatch):
    """The fused K-Means pass over the FK-band layout (round-robin tiles, band-ordered S / FK / d_t)
    gives the storage-order run's assignments bit for bit and its centroids / trace within 1e-9."""
    fb = _fb()
    from paper_1612_07448_b200 import ml as fbml
    from paper_1612_07448_b200.normmat import NormalizedMatrix

    rng, s, parts = _c1_like(77, n_s=120_003, d_s=6, n_r=5000, d_r=5, star=True)
    cfg = fb.TrainConfig(iterations=6, k=10, rng_seed=5)
    monkeypatch.setattr(NormalizedMatrix, "BAND_KMEANS_MIN_BYTES", 0)
    nm0, ref = _both(s, parts)
    plain = fb.kmeans(nm0, cfg)
    assert "band" not in nm0._cache
    monkeypatch.setattr(NormalizedMatrix, "BAND_KMEANS_MIN_BYTES", 1)
    monkeypatch.setattr(NormalizedMatrix, "BAND_BYTES", 128 * 700)
    monkeypatch.setattr(fbml, "_BAND_MIN_ITERS", 1)
    nm, _ = _both(s, parts)
    banded = fb.kmeans(nm, cfg)
    assert "band" in nm._cache and nm._cache["band"][0].n_bands >= 2
    st, perm, fkb, sb = nm._cache["band"]
    p = perm.cpu().numpy()
    for q, (e, _) in enumerate(nm.parts):
        np.testing.assert_array_equal(fkb[q].cpu().numpy(), e.target_numpy()[p])
    np.testing.assert_array_equal(banded.assignment.cpu().numpy(), plain.assignment.cpu().numpy())
    _close(banded.centroids, plain.centroids, 1e-12)
    _close(banded.objective, plain.objective, 1e-12)
    c, obj, _ = O.kmeans(ref, 10, 6, 5)
    _close(banded.centroids, c)
    _close(banded.objective, obj)
    # a NaN row is still reported in row order (the run repeats in storage order)
    s2 = s.copy()
    s2[4321, 2] = np.nan
    nm2, _ = _both(s2, parts)
    with pytest.raises(fb.NumericError, match="row 4321"):
        fb.kmeans(nm2, cfg)

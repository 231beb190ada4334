"""gram_transposed / ginv / dmm / dmm_gram / pair_product / elementwise_matrix_op
(rewrite.py:301-470, indicator.py:144-162) against the reference's
golden vectors (tests/golden/products.npz, oracle/gen_golden.py) — CPU oracle and device."""
import warnings

import numpy as np
import pytest
import torch

import factorla_oracle as O
import golden_io

G = golden_io.load("products")
TOL = 1e-9


def _close(a, b, tol=TOL):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    dev = O.max_rel_deviation(a, b)
    assert dev <= tol, dev


def _o(prefix):
    return O.build_pkfk(G[f"{prefix}_s"], G[f"{prefix}_k"], G[f"{prefix}_r"])


# --------------------------------------------------------------------------- oracle (CPU)
def test_oracle_products_match_reference():
    a, w = _o("a"), _o("w")
    _close(O.gram_transposed(a), G["gram_t_a"], 1e-12)
    _close(O.gram_transposed(w.T), G["gram_t_w"], 1e-12)
    for key, nm in (("ginv_a", a), ("ginv_at", a.T), ("ginv_w", w), ("ginv_wt", w.T)):
        _close(O.ginv(nm), G[key], 1e-9)
    _close(O.dmm(a, _o("b")), G["dmm_ab"], 1e-12)
    _close(O.dmm(a.T, _o("b2")), G["dmm_atb"], 1e-12)
    for tag in ("lt", "eq", "gt"):
        _close(O.dmm(a, _o(f"b3{tag}").T), G[f"dmm_abt_{tag}"], 1e-12)
    _close(O.dmm(_o("b4").T, _o("c").T), G["dmm_atbt"], 1e-12)
    b2 = _o("b2")
    pp = O.pair_product(a.parts[0][0], a.parts[0][1].shape[0], b2.parts[0][0], b2.parts[0][1].shape[0])
    np.testing.assert_array_equal(pp, G["pair_ab2"])


# --------------------------------------------------------------------------- device (GPU)
def _d(prefix):
    import paper_1612_07448_b200 as fb

    return fb.build_pkfk(G[f"{prefix}_s"], G[f"{prefix}_k"], G[f"{prefix}_r"])


def _check(name, fn):
    import paper_1612_07448_b200 as fb

    c = fb.OpCounter()
    out = fn(c)
    assert isinstance(out, np.ndarray), name  # host operands -> host result
    _close(out, G[name])
    assert [c.multiplies, c.additions] == list(G["cnt_" + name]), name
    return out


@pytest.mark.gpu
def test_device_gram_transposed_and_ginv():
    import paper_1612_07448_b200 as fb

    a, w = _d("a"), _d("w")
    g = _check("gram_t_a", lambda c: fb.gram_transposed(a, c))
    np.testing.assert_array_equal(g, g.T)
    _check("gram_t_w", lambda c: fb.gram_transposed(w.T, c))
    _check("ginv_a", lambda c: fb.ginv(a, c))
    _check("ginv_at", lambda c: fb.ginv(a.T, c))
    _check("ginv_w", lambda c: fb.ginv(w, c))
    _check("ginv_wt", lambda c: fb.ginv(w.T, c))


@pytest.mark.gpu
def test_device_dmm_family():
    import paper_1612_07448_b200 as fb

    a = _d("a")
    _check("dmm_ab", lambda c: fb.dmm(a, _d("b"), c))
    _check("dmm_atb", lambda c: fb.dmm(a.T, _d("b2"), c))
    for tag in ("lt", "eq", "gt"):
        _check(f"dmm_abt_{tag}", lambda c, tag=tag: fb.dmm(a, _d(f"b3{tag}").T, c))
    _check("dmm_atbt", lambda c: fb.dmm(_d("b4").T, _d("c").T, c))
    with pytest.raises(fb.ShapeError):
        fb.dmm(a, a)
    c = fb.OpCounter()
    pp = fb.pair_product(a.k, _d("b2").k, c)
    np.testing.assert_array_equal(pp.to_dense().cpu().numpy(), G["pair_ab2"])
    assert [c.multiplies, c.additions] == list(G["cnt_pair_ab2"])


@pytest.mark.gpu
def test_device_elementwise_matrix_op_warns_and_matches():
    import paper_1612_07448_b200 as fb

    a = _d("a")
    for op in ("add", "sub", "rsub", "mul", "div", "rdiv"):
        with pytest.warns(fb.MaterializationWarning):
            _check(f"ew_{op}", lambda c, op=op: fb.elementwise_matrix_op(a, G["ew_x"], op, c))
    with pytest.raises(fb.ShapeError):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            fb.elementwise_matrix_op(a, np.ones((2, 2)), "add")


@pytest.mark.gpu
def test_device_drivers_on_transposed_matrix():
    """logistic_gd / linreg_gd / linreg_normal / gnmf on nm.T (ml.py dispatches on the flag);
    kmeans refuses it like the reference's _take_rows."""
    import paper_1612_07448_b200 as fb

    u = _d("u")
    cfg = fb.TrainConfig(iterations=4, step_size=1e-2, r=2, rng_seed=5)
    out = fb.logistic_gd(u.T, G["ut_y_log"], cfg)
    _close(out.weights, G["ut_logreg_w"])
    _close(out.objective, G["ut_logreg_obj"])
    out = fb.linreg_gd(u.T, G["ut_y_lin"], cfg)
    _close(out.weights, G["ut_linreg_gd_w"])
    _close(out.objective, G["ut_linreg_gd_obj"])
    out = fb.linreg_normal(u.T, G["ut_y_lin"])
    _close(out.weights, G["ut_linreg_w"])
    # 7 rows, 40 columns: an exact minimum-norm fit, the objective is rounding noise — compared
    # against ‖y‖² (as the PK-FK exact-fit cases in test_ml_gpu.py)
    assert abs(out.objective[0] - float(G["ut_linreg_obj"][0])) <= 1e-9 * float(np.sum(G["ut_y_lin"] ** 2))
    out = fb.gnmf(u.T, cfg)
    _close(out.factors[0], G["ut_gnmf_w"])
    _close(out.factors[1], G["ut_gnmf_h"])
    _close(out.objective, G["ut_gnmf_obj"])
    with pytest.raises(fb.ShapeError):
        fb.kmeans(u.T, fb.TrainConfig(iterations=1, k=2))

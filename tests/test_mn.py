"""M:N and multi-table M:N normalized matrices (normmat.py:240-319).

CPU: the oracle's join planning and operators against the reference's golden vectors.
GPU: the device constructors (indicators, kept rows, source rows bit-exact) and every
operator / driver through the sm_100a kernels against the same vectors (rel 1e-9), plus a
multi-tile seeded case against the oracle.
"""
import numpy as np
import pytest
import torch

import factorla_oracle as O
import golden_io

TOL_ORACLE = 1e-12
TOL = 1e-9
MN = golden_io.mn_names()


def _close(a, b, tol):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    dev = O.max_rel_deviation(a, b)
    assert dev <= tol, dev


def _tables(g):
    return [g[f"table{j}"] for j in range(int(g["q"]))]


def _oracle(g):
    if str(g["kind"]) == "mn":
        return O.build_mn(g["s"], g["j_s"], g["r"], g["j_r"])
    return O.build_multimn(g["row_map"], _tables(g))


def _device(g):
    import paper_1612_07448_b200 as fb

    if str(g["kind"]) == "mn":
        return fb.build_mn(g["s"], g["j_s"], g["r"], g["j_r"])
    return fb.build_multimn(g["row_map"], _tables(g))


# --------------------------------------------------------------------------- oracle (CPU)
@pytest.mark.parametrize("name", MN)
def test_oracle_construction_bit_exact(name):
    g = golden_io.load(name)
    nm = _oracle(g)
    for i, (t, kept) in enumerate(nm.parts):
        np.testing.assert_array_equal(t, g[f"target{i}"])
        np.testing.assert_array_equal(nm.source_rows[i], g[f"used{i}"])
        np.testing.assert_array_equal(O.counts(t, kept.shape[0]), g[f"counts{i}"])
        np.testing.assert_array_equal(kept, g[f"kept{i}"])
    np.testing.assert_array_equal(O.materialize(nm), g["materialize"])


@pytest.mark.parametrize("name", MN)
def test_oracle_operators_and_drivers(name):
    g = golden_io.load(name)
    nm = _oracle(g)
    _close(O.lmm(nm, g["x1"]), g["lmm_x1"], TOL_ORACLE)
    _close(O.lmm(nm, g["x3"]), g["lmm_x3"], TOL_ORACLE)
    _close(O.lmm(nm.T, g["p2"]), g["tmm_p2"], TOL_ORACLE)
    _close(O.rmm(g["xr"], nm), g["rmm_xr"], TOL_ORACLE)
    _close(O.rmm(g["xt"], nm.T), g["rmm_t_xt"], TOL_ORACLE)
    _close(O.row_sums(nm), g["row_sums"], TOL_ORACLE)
    _close(O.col_sums(nm), g["col_sums"], TOL_ORACLE)
    cp = O.crossprod(nm)
    _close(cp, g["crossprod"], TOL_ORACLE)
    np.testing.assert_array_equal(cp, cp.T)
    w, _ = O.linreg_normal(nm, g["y_lin"])
    _close(w, g["linreg_w"], 1e-9)
    w, obj = O.logistic_gd(nm, g["y_log"], 5, 1e-3)
    _close(w, g["logreg_w"], TOL_ORACLE)
    c, obj, _ = O.kmeans(nm, 3, 5, 3)
    _close(c, g["kmeans_c"], TOL_ORACLE)
    if "gnmf_w" in g:
        w, h, obj = O.gnmf(nm, 2, 5, 3)
        _close(obj, g["gnmf_obj"], TOL_ORACLE)


def test_oracle_empty_join_raises():
    with pytest.raises(O.DataError):
        O.build_mn(np.ones((3, 1)), [1, 2, 3], np.ones((2, 1)), [7, 8])


# --------------------------------------------------------------------------- device (GPU)
@pytest.mark.gpu
@pytest.mark.parametrize("name", MN)
def test_device_construction_bit_exact(name):
    import paper_1612_07448_b200 as fb

    g = golden_io.load(name)
    nm = _device(g)
    assert nm.variant == str(g["kind"])
    for i, (e, kept) in enumerate(nm.blocks):
        np.testing.assert_array_equal(e.target_numpy(), g[f"target{i}"])
        np.testing.assert_array_equal(nm.source_rows[i].cpu().numpy(), g[f"used{i}"])
        np.testing.assert_array_equal(e.counts.cpu().numpy(), g[f"counts{i}"])
        np.testing.assert_array_equal(kept.cpu().numpy(), g[f"kept{i}"])
    np.testing.assert_array_equal(fb.materialize(nm), g["materialize"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", MN)
def test_device_operators_vs_reference_golden(name):
    import paper_1612_07448_b200 as fb

    g = golden_io.load(name)
    nm = _device(g)
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
        ("crossprod", lambda c: fb.crossprod(nm, counter=c), "cnt_crossprod"),
    ):
        c = fb.OpCounter()
        out = fn(c)
        assert isinstance(out, np.ndarray)
        _close(out, g[key], TOL)
        if cnt:
            assert [c.multiplies, c.additions] == list(g[cnt]), key
    cp = fb.crossprod(nm)
    np.testing.assert_array_equal(cp, cp.T)
    c = fb.OpCounter()
    tot = fb.sum_all(nm, c)
    assert abs(tot - float(g["sum_all"])) <= TOL * max(1.0, np.abs(g["materialize"]).sum())
    assert [c.multiplies, c.additions] == list(g["cnt_sum_all"])
    for op, x in (("mul", 2.0), ("add", 3.0), ("rsub", 1.5), ("div", 4.0), ("pow", 2.0)):
        c = fb.OpCounter()
        _close(fb.materialize(fb.scalar_op(nm, x, op, c)), g[f"scalar_{op}"], TOL)
        assert [c.multiplies, c.additions] == list(g[f"cnt_scalar_{op}"])
    _close(fb.materialize(fb.scalar_fn(nm, np.exp)), g["fn_exp"], TOL)


@pytest.mark.gpu
@pytest.mark.parametrize("name", MN)
def test_device_drivers_vs_reference_golden(name):
    import paper_1612_07448_b200 as fb

    g = golden_io.load(name)
    nm = _device(g)
    cfg = fb.TrainConfig(iterations=5, step_size=1e-3, k=3, r=2, rng_seed=3)
    out = fb.linreg_normal(nm, g["y_lin"])
    _close(out.weights, g["linreg_w"], TOL)
    out = fb.logistic_gd(nm, g["y_log"], cfg)
    _close(out.weights, g["logreg_w"], TOL)
    _close(out.objective, g["logreg_obj"], TOL)
    out = fb.linreg_gd(nm, g["y_lin"], cfg)
    _close(out.weights, g["linreg_gd_w"], TOL)
    out = fb.kmeans(nm, cfg)
    _close(out.centroids, g["kmeans_c"], TOL)
    _close(out.objective, g["kmeans_obj"], TOL)
    if "gnmf_w" in g:
        out = fb.gnmf(nm, cfg)
        _close(out.factors[0], g["gnmf_w"], TOL)
        _close(out.factors[1], g["gnmf_h"], TOL)
        _close(out.objective, g["gnmf_obj"], TOL)


@pytest.mark.gpu
def test_device_mn_multitile_vs_oracle():
    """A join large enough for multi-tile passes: 200k S rows × ~4 matches each."""
    import paper_1612_07448_b200 as fb

    rng = np.random.default_rng(44)
    n_s, n_r = 200_000, 60_000
    s = rng.standard_normal((n_s, 12))
    r = rng.standard_normal((n_r, 9))
    j_s = rng.integers(0, 20_000, size=n_s)
    j_r = rng.integers(500, 20_500, size=n_r)
    ref = O.build_mn(s, j_s, r, j_r)
    nm = fb.build_mn(s, j_s, r, j_r)
    for i, (e, _) in enumerate(nm.blocks):
        np.testing.assert_array_equal(e.target_numpy(), ref.parts[i][0])
    n, d = ref.shape
    x = rng.standard_normal((d, 3))
    p = rng.standard_normal((n, 2))
    _close(fb.lmm(nm, x), O.lmm(ref, x), TOL)
    _close(fb.lmm(nm.T, p), O.lmm(ref.T, p), TOL)
    _close(fb.col_sums(nm), O.col_sums(ref), TOL)
    cp = fb.crossprod(nm)
    _close(cp, O.crossprod(ref), TOL)
    np.testing.assert_array_equal(cp, cp.T)


@pytest.mark.gpu
def test_device_empty_join_raises():
    import paper_1612_07448_b200 as fb

    with pytest.raises(fb.EmptyJoinError):
        fb.build_mn(np.ones((3, 1)), [1, 2, 3], np.ones((2, 1)), [7, 8])
    with pytest.raises(fb.DataError):
        fb.build_multimn(np.array([[0, 5]]), [np.ones((2, 1)), np.ones((3, 1))])

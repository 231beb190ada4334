"""Pin the CPU oracle: against the reference's golden vectors and the SPEC worked examples."""
import numpy as np
import pytest

import factorla_oracle as O
import golden_io

TOL = 1e-12  # oracle vs reference: same algorithm, same native primitives


def _build(g):
    parts = golden_io.parts(g)
    return O.build_star(g["s"], parts)


@pytest.mark.parametrize("name", golden_io.names())
def test_construction_bit_exact(name):
    g = golden_io.load(name)
    nm = _build(g)
    for i, (t, rk) in enumerate(nm.parts):
        np.testing.assert_array_equal(t, g[f"target{i}"])
        np.testing.assert_array_equal(nm.source_rows[i + 1], g[f"used{i}"])
        np.testing.assert_array_equal(O.counts(t, rk.shape[0]), g[f"counts{i}"])
        np.testing.assert_array_equal(rk, g[f"rkept{i}"])
    np.testing.assert_array_equal(O.materialize(nm), g["materialize"])


def _close(a, b, tol=TOL):
    assert np.asarray(a).shape == np.asarray(b).shape
    assert O.max_rel_deviation(a, b) <= tol


@pytest.mark.parametrize("name", golden_io.names())
def test_operators_match_reference(name):
    g = golden_io.load(name)
    nm = _build(g)
    _close(O.lmm(nm, g["x1"]), g["lmm_x1"])
    _close(O.lmm(nm, g["x3"]), g["lmm_x3"])
    _close(O.lmm(nm.T, g["p2"]), g["tmm_p2"])
    _close(O.rmm(g["xr"], nm), g["rmm_xr"])
    _close(O.rmm(g["xt"], nm.T), g["rmm_t_xt"])
    _close(O.row_sums(nm), g["row_sums"])
    _close(O.col_sums(nm), g["col_sums"])
    _close(O.row_sums(nm.T), g["row_sums_t"])
    _close(O.col_sums(nm.T), g["col_sums_t"])
    assert abs(O.sum_all(nm) - float(g["sum_all"])) <= TOL * max(1.0, abs(float(g["sum_all"])))
    for op, x in (("mul", 2.0), ("add", 3.0), ("rsub", 1.5), ("div", 4.0), ("pow", 2.0)):
        _close(O.materialize(O.scalar_op(nm, x, op)), g[f"scalar_{op}"])
    _close(O.materialize(O.scalar_fn(nm, np.exp)), g["fn_exp"])
    _close(O.materialize(O.scalar_fn(nm, np.square)), g["fn_square"])


@pytest.mark.parametrize("name", [n for n in golden_io.names() if n != "zero_width_s"])
def test_crossprod_and_drivers_match_reference(name):
    g = golden_io.load(name)
    nm = _build(g)
    cp = O.crossprod(nm)
    _close(cp, g["crossprod"])
    np.testing.assert_array_equal(cp, cp.T)  # exact symmetry (rewrite.py:298)
    w, obj = O.linreg_normal(nm, g["y_lin"])
    _close(w, g["linreg_w"], 1e-9)
    w, obj = O.logistic_gd(nm, g["y_log"], 5, 1e-3)
    _close(w, g["logreg_w"])
    _close(obj, g["logreg_obj"])
    w, obj = O.linreg_gd(nm, g["y_lin"], 5, 1e-3)
    _close(w, g["linreg_gd_w"])
    c, obj, _ = O.kmeans(nm, 3, 5, 3)
    _close(c, g["kmeans_c"])
    _close(obj, g["kmeans_obj"])
    if "gnmf_w" in g:
        w, h, obj = O.gnmf(nm, 2, 5, 3)
        _close(w, g["gnmf_w"])
        _close(h, g["gnmf_h"])
        _close(obj, g["gnmf_obj"])


# --------------------------------------------------------------------------- SPEC KATs
F1_S = [[1, 2], [3, 4], [5, 6]]
F1_KEY = [1, 2, 1]
F1_R = [[10, 20], [30, 40]]


def test_spec_f1_known_answers():
    """SPEC.md:248-298 and :472 (fixture F1 worked examples)."""
    nm = O.build_pkfk(F1_S, F1_KEY, F1_R)
    np.testing.assert_array_equal(nm.parts[0][0], [0, 1, 0])
    np.testing.assert_array_equal(O.materialize(nm), [[1, 2, 10, 20], [3, 4, 30, 40], [5, 6, 10, 20]])
    np.testing.assert_array_equal(O.row_sums(nm).ravel(), [33, 77, 41])
    np.testing.assert_array_equal(O.col_sums(nm).ravel(), [9, 12, 50, 80])
    assert O.sum_all(nm) == 151
    np.testing.assert_array_equal(O.lmm(nm, [[1], [0], [0], [1]]).ravel(), [21, 43, 25])
    np.testing.assert_array_equal(O.rmm([[0, 1, -1]], nm), [[-2, -2, 20, 20]])
    np.testing.assert_array_equal(
        O.crossprod(nm),
        [[35, 44, 150, 240], [44, 56, 200, 320], [150, 200, 1100, 1600], [240, 320, 1600, 2400]],
    )
    np.testing.assert_array_equal(O.materialize(O.scalar_op(nm, 2, "mul"))[0], [2, 4, 20, 40])
    w, _ = O.logistic_gd(nm, [[1], [-1], [1]], 1, 0.1)
    np.testing.assert_allclose(w.ravel(), [0.15, 0.2, -0.5, 0.0], atol=1e-15)
    np.testing.assert_array_equal(O.lmm(nm.T, [[1], [-1], [1]]).ravel(), [3, 4, -10, 0])


def test_spec_f3_star_known_answers():
    """SPEC.md:127-129, 250-268 (fixture F3)."""
    nm = O.build_star([[1], [2], [3]], [([1, 2, 1], [[10], [20]]), ([2, 1, 2], [[100], [200]])])
    np.testing.assert_array_equal(O.materialize(nm), [[1, 10, 200], [2, 20, 100], [3, 10, 200]])
    np.testing.assert_array_equal(O.row_sums(nm).ravel(), [211, 122, 213])
    np.testing.assert_array_equal(O.col_sums(nm).ravel(), [6, 40, 500])
    assert O.sum_all(nm) == 546


def test_bad_keys_raise_with_row_index():
    with pytest.raises(O.DataError, match="entity row 1"):
        O.build_pkfk(F1_S, [1, 3, 1], F1_R)
    with pytest.raises(O.DataError, match="non-integer"):
        O.build_pkfk(F1_S, [1.0, 1.5, 1.0], F1_R)


def test_unreferenced_rows_dropped():
    """s 2×1, key=[1,1], r 3×2 → r reduced to 1 row, K.target=[0,0]."""
    nm = O.build_pkfk([[1], [2]], [1, 1], [[1, 2], [3, 4], [5, 6]])
    np.testing.assert_array_equal(nm.parts[0][0], [0, 0])
    assert nm.parts[0][1].shape == (1, 2)
    np.testing.assert_array_equal(nm.source_rows[1], [0])

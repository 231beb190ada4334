"""The reference's own drivers (factorla.ml) running on the device operators.

``paper_1612_07448_b200.integration.route_reference_drivers`` patches the reference's
polymorphic helpers (ml.py:101-180) so that ``factorla.ml.logistic_gd / linreg_normal /
kmeans / gnmf`` — the stock driver code, unmodified — run every operator of a device
matrix on the sm_100a kernels. Stock factorla comes from baseline/_ref (pip-installed from
/root/reference/pkg, travels with the repo); the tests skip when it is absent.
"""
import os
import sys

import numpy as np
import pytest
import torch

import factorla_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TOL = 1e-9


def _factorla():
    if not os.path.isdir(os.path.join(REF, "factorla")):
        pytest.skip("stock factorla not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import factorla

    return factorla


def test_patch_and_undo_restore_the_reference_attributes():
    factorla = _factorla()
    from paper_1612_07448_b200.integration import register_cost_model_ops, route_reference_drivers

    ml, cm = factorla.ml, factorla.costmodel
    before = {k: getattr(ml, k) for k in ("_is_nm", "rewrite", "_take_rows", "_min_value")}
    reg = dict(cm._FACTORIZED_OPS)
    undo1, undo2 = route_reference_drivers(factorla), register_cost_model_ops(factorla)
    assert ml.rewrite is not before["rewrite"] and ml._is_nm is not before["_is_nm"]
    assert set(cm._FACTORIZED_OPS) == set(reg)
    # the reference's own matrices still take the reference's path
    s = np.arange(12.0).reshape(4, 3)
    r = np.array([[1.0, 2.0], [3.0, 4.0]])
    nm = factorla.build_pkfk(s, np.array([1, 2, 2, 1]), r)
    assert ml._is_nm(nm)
    np.testing.assert_array_equal(ml.rewrite.row_sums(nm), factorla.row_sums(nm))
    undo2()
    undo1()
    assert {k: getattr(ml, k) for k in before} == before
    assert cm._FACTORIZED_OPS == reg


@pytest.mark.gpu
def test_reference_drivers_run_on_device_matrices():
    factorla = _factorla()
    import paper_1612_07448_b200 as fb
    from paper_1612_07448_b200.integration import route_reference_drivers

    rng = np.random.default_rng(21)
    n, d_s, n_r1, n_r2 = 40_000, 7, 900, 50
    s = rng.random((n, d_s))
    parts = [(rng.integers(1, n_r1 + 1, size=n), rng.random((n_r1, 5))),
             (rng.integers(1, n_r2 + 1, size=n), rng.random((n_r2, 3)))]
    dev = fb.build_star(s, parts)
    ref = O.build_star(s, parts)
    launches0 = fb.launch_count()
    undo = route_reference_drivers(factorla)
    try:
        ml = factorla.ml
        y = np.where(O.lmm(ref, rng.standard_normal((ref.d, 1))) >= 0, 1.0, -1.0)
        out = ml.logistic_gd(dev, y, factorla.TrainConfig(iterations=5, step_size=1e-3))
        w, obj = O.logistic_gd(ref, y, 5, 1e-3)
        assert O.max_rel_deviation(out.weights, w) <= TOL
        assert O.max_rel_deviation(out.objective, obj) <= TOL
        yl = O.lmm(ref, rng.standard_normal((ref.d, 1))) + 0.01 * rng.standard_normal((n, 1))
        out = ml.linreg_normal(dev, yl)
        w, obj = O.linreg_normal(ref, yl)
        assert O.max_rel_deviation(out.weights, w) <= 1e-8
        out = ml.kmeans(dev, factorla.TrainConfig(iterations=4, k=6, rng_seed=3))
        c, obj, _ = O.kmeans(ref, 6, 4, 3)
        assert O.max_rel_deviation(out.centroids, c) <= TOL
        assert O.max_rel_deviation(out.objective, obj) <= TOL
        out = ml.gnmf(dev, factorla.TrainConfig(iterations=3, r=3, rng_seed=5))
        w, h, obj = O.gnmf(ref, 3, 3, 5)
        assert O.max_rel_deviation(out.factors[0], w) <= TOL
        assert O.max_rel_deviation(out.factors[1], h) <= TOL
        # the reference's own matrix in the same patched module still runs on the CPU path
        rn = factorla.build_star(s, parts)
        out = ml.logistic_gd(rn, y, factorla.TrainConfig(iterations=2, step_size=1e-3))
        assert O.max_rel_deviation(out.weights, O.logistic_gd(ref, y, 2, 1e-3)[0]) <= 1e-12
    finally:
        undo()
    assert fb.launch_count() > launches0  # the device kernels ran
    torch.cuda.synchronize()

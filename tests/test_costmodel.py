"""Cost model and auto-dispatch (costmodel.py:75-202, the dispatch half).

CPU: predicted counts and plans against the reference's own (tests/golden/products.npz).
GPU: auto_dispatch runs every operator on both plans (factorized kernels / the same kernels
over the materialized T) with values equal to the oracle's.
"""
import numpy as np
import pytest
import torch

import factorla_oracle as O
import golden_io

G = golden_io.load("products")


def _stats(key):
    from paper_1612_07448_b200.normmat import ShapeStats

    if key == "mn":
        s, r = G["mn_s"], G["mn_r"]
        n = G["mn_ts"].size
        return ShapeStats("mn", s.shape[0], s.shape[1], (r.shape[0],), (r.shape[1],), n, s.shape[1] + r.shape[1],
                          s.shape[0] / r.shape[0], r.shape[1] / s.shape[1])
    s, r = G[f"{key}_s"], G[f"{key}_r"]
    n_r = int(G[f"{key}_k"].max())  # every kept R row is referenced (the build drops the rest)
    return ShapeStats("pkfk", s.shape[0], s.shape[1], (n_r,), (r.shape[1],), s.shape[0], s.shape[1] + r.shape[1],
                      s.shape[0] / n_r, r.shape[1] / s.shape[1])


@pytest.mark.parametrize("key", ["a", "u", "w", "mn"])
def test_predicted_counts_and_plans_match_reference(key):
    from paper_1612_07448_b200 import costmodel as C

    st = _stats(key)
    for op in C.KNOWN_OPS:
        pc = C.predict_counts(op, st, d_x=3, n_x=2)
        np.testing.assert_allclose([pc.standard, pc.factorized], G[f"cm_{key}_{op}"], rtol=1e-15)
    assert C.decide(st, C.DecisionThresholds()).value == str(G[f"cm_{key}_plan_default"])
    assert C.decide(st, C.DecisionThresholds(1.0, 0.1)).value == str(G[f"cm_{key}_plan_loose"])
    with pytest.raises(ValueError):
        C.predict_counts("nope", st)
    with pytest.raises(ValueError):
        C.DecisionThresholds(0.0, 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("thr", [(1.0, 0.01), (1e9, 1e9)], ids=["factorized", "materialized"])
def test_auto_dispatch_both_plans_match_oracle(thr):
    import paper_1612_07448_b200 as fb
    from paper_1612_07448_b200 import costmodel as C

    s, k, r = G["a_s"], G["a_k"], G["a_r"]
    nm = fb.build_pkfk(s, k, r)
    ref = O.build_pkfk(s, k, r)
    th = C.DecisionThresholds(*thr)
    want = C.Plan.FACTORIZED if thr[0] < 2 else C.Plan.MATERIALIZED
    assert C.plan_for(nm, th) is want
    rng = np.random.default_rng(5)
    n, d = ref.shape
    x = rng.standard_normal((d, 3))
    xr = rng.standard_normal((2, n))

    def close(a, b, tol=1e-9):
        a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
        assert a.shape == np.asarray(b).shape
        assert O.max_rel_deviation(a, b) <= tol

    close(C.auto_dispatch("lmm", nm, th, x=x), O.lmm(ref, x))
    close(C.auto_dispatch("lmm", nm.T, th, x=xr.T), O.lmm(ref.T, xr.T))
    close(C.auto_dispatch("rmm", nm, th, x=xr), O.rmm(xr, ref))
    close(C.auto_dispatch("rowsums", nm, th), O.row_sums(ref))
    close(C.auto_dispatch("colsums", nm, th), O.col_sums(ref))
    assert abs(C.auto_dispatch("sum", nm, th) - O.sum_all(ref)) <= 1e-9 * np.abs(O.materialize(ref)).sum()
    close(C.auto_dispatch("crossprod", nm, th), O.crossprod(ref))
    close(C.auto_dispatch("ginv", nm, th), np.linalg.pinv(O.materialize(ref)), 1e-8)
    out = C.auto_dispatch("scalar_op", nm, th, x=2.0)  # (op= collides with the op id, as in the reference)
    t = fb.materialize(out) if isinstance(out, fb.NormalizedMatrix) else out
    close(t, O.materialize(ref) * 2.0)
    c = fb.OpCounter()
    C.auto_dispatch("rowsums", nm, th, counter=c)
    n_, d_ = ref.shape
    if want is C.Plan.MATERIALIZED:  # kernel.row_sums of the dense T (kernel.py:174-182)
        assert (c.multiplies, c.additions) == (n_ * d_, n_ * d_ - n_)

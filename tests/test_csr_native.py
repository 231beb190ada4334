"""CSR-native factorized operators (csr_ops.py).

Factor matrices at or below 5 % density stay CSR in HBM; T·X, Tᵀ·X, X·T, rowSums, colSums and
sumAll read them through fb_csr_spmm / fb_csr_spmm_t without expanding them (checked: the
matrix makes no dense copy), and match the oracle (scipy CSR products, the reference's own
path, kernel.py:103-129) within the 1e-9 bar. Operators without a sparse kernel (crossprod,
the drivers) use the one-time dense expansion.
"""

import numpy as np
import pytest
from scipy import sparse

import factorla_oracle as O

TOL = 1e-9


def _dev(a, b):
    return O.max_rel_deviation(np.asarray(a), np.asarray(b))


def _cases(rng):
    s = sparse.random(20_000, 200, density=0.01, format="csr", random_state=rng, data_rvs=rng.standard_normal)
    r = sparse.random(700, 250, density=0.02, format="csr", random_state=rng, data_rvs=rng.standard_normal)
    keys = rng.integers(1, 701, size=20_000)
    return s, r, keys


@pytest.mark.gpu
def test_csr_pkfk_operators_native_vs_oracle():
    import paper_1612_07448_b200 as fb

    rng = np.random.default_rng(21)
    s, r, keys = _cases(rng)
    nm = fb.build_pkfk(s, keys, r)
    ref = O.build_pkfk(s.toarray(), keys, r.toarray())
    assert nm.has_csr
    d = nm.shape[1]
    x = rng.standard_normal((d, 5))
    p = rng.standard_normal((20_000, 3))
    checks = {
        "lmm": (fb.lmm(nm, x), O.lmm(ref, x)),
        "lmm_x1": (fb.lmm(nm, x[:, :1]), O.lmm(ref, x[:, :1])),
        "tmm": (fb.lmm(nm.T, p), O.lmm(ref.T, p)),
        "rmm": (fb.rmm(p.T.copy(), nm), O.rmm(p.T, ref)),
        "rmm_t": (fb.rmm(x.T.copy(), nm.T), O.rmm(x.T, ref.T)),
        "row_sums": (fb.row_sums(nm), O.row_sums(ref)),
        "col_sums": (fb.col_sums(nm), O.col_sums(ref)),
    }
    for name, (got, want) in checks.items():
        assert _dev(got, want) <= TOL, (name, _dev(got, want))
    assert abs(fb.sum_all(nm) - O.sum_all(ref)) <= TOL * abs(O.sum_all(ref))
    assert "dense_blocks" not in nm._cache, "a CSR-native operator expanded the factors"
    # operators without a sparse kernel: the one-time dense expansion
    assert _dev(fb.crossprod(nm), O.crossprod(ref)) <= TOL
    assert "dense_blocks" in nm._cache


@pytest.mark.gpu
def test_csr_star_mixed_and_dense_equivalence():
    import paper_1612_07448_b200 as fb

    rng = np.random.default_rng(22)
    s = rng.standard_normal((5_000, 7))  # dense entity table
    r1 = sparse.random(300, 90, density=0.03, format="csr", random_state=rng, data_rvs=rng.standard_normal)
    r2 = rng.standard_normal((40, 11))
    k1 = rng.integers(1, 301, size=5_000)
    k2 = rng.integers(1, 41, size=5_000)
    nm = fb.build_star(s, [(k1, r1), (k2, r2)])
    nm_d = fb.build_star(s, [(k1, r1.toarray()), (k2, r2)])
    ref = O.build_star(s, [(k1, r1.toarray()), (k2, r2)])
    assert nm.has_csr and not nm_d.has_csr
    x = rng.standard_normal((nm.shape[1], 4))
    w = rng.standard_normal((5_000, 2))
    for got, dense, want in (
        (fb.lmm(nm, x), fb.lmm(nm_d, x), O.lmm(ref, x)),
        (fb.lmm(nm.T, w), fb.lmm(nm_d.T, w), O.lmm(ref.T, w)),
        (fb.col_sums(nm), fb.col_sums(nm_d), O.col_sums(ref)),
    ):
        assert _dev(got, want) <= TOL
        assert _dev(got, dense) <= 1e-12
    # densities above the threshold are expanded at build (dense kernels, no CSR)
    rd = sparse.random(300, 90, density=0.3, format="csr", random_state=rng)
    assert not fb.build_star(s, [(k1, rd), (k2, r2)]).has_csr


@pytest.mark.gpu
def test_csr_unreferenced_rows_dropped_and_drivers():
    import paper_1612_07448_b200 as fb

    rng = np.random.default_rng(23)
    s = sparse.random(3_000, 40, density=0.02, format="csr", random_state=rng, data_rvs=rng.standard_normal)
    r = sparse.random(500, 60, density=0.02, format="csr", random_state=rng, data_rvs=rng.standard_normal)
    keys = rng.integers(1, 251, size=3_000)  # rows 251..500 unreferenced: dropped, CSR rows selected
    nm = fb.build_pkfk(s, keys, r)
    ref = O.build_pkfk(s.toarray(), keys, r.toarray())
    assert nm.has_csr and nm.r.shape[0] == ref.parts[0][1].shape[0]
    x = rng.standard_normal((100, 2))
    assert _dev(fb.lmm(nm, x), O.lmm(ref, x)) <= TOL
    y = np.where(O.lmm(ref, rng.standard_normal((100, 1))) >= 0, 1.0, -1.0)
    w_ref, _ = O.logistic_gd(ref, y, 3, 1e-3)
    got = fb.logistic_gd(nm, y, fb.TrainConfig(iterations=3, step_size=1e-3)).weights
    assert _dev(got, w_ref) <= TOL


@pytest.mark.gpu
def test_wide_dense_factors_take_the_block_path():
    """Factors wider than the streaming kernels' 256 columns: T·X, Tᵀ·X, row / column sums."""
    import paper_1612_07448_b200 as fb

    rng = np.random.default_rng(24)
    s = rng.standard_normal((3_000, 300))
    r = rng.standard_normal((200, 270))
    keys = rng.integers(1, 201, size=3_000)
    nm = fb.build_pkfk(s, keys, r)
    ref = O.build_pkfk(s, keys, r)
    assert nm.block_path and not nm.has_csr
    x = rng.standard_normal((570, 3))
    p = rng.standard_normal((3_000, 2))
    for got, want in (
        (fb.lmm(nm, x), O.lmm(ref, x)),
        (fb.lmm(nm.T, p), O.lmm(ref.T, p)),
        (fb.rmm(p.T.copy(), nm), O.rmm(p.T, ref)),
        (fb.row_sums(nm), O.row_sums(ref)),
        (fb.col_sums(nm), O.col_sums(ref)),
    ):
        assert _dev(got, want) <= TOL

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


@pytest.mark.gpu
def test_dense_sparse_primitives_vs_numpy():
    """fb_dense_mm (all transposes, ragged sizes), fb_gather2_add, fb_scatter_rows, fb_pair_counts
    (exact counts / CSR order), fb_csr_spmm and fb_csr_spmm_t against NumPy / SciPy."""
    import scipy.sparse as sp
    import torch

    from paper_1612_07448_b200 import _device as D
    from paper_1612_07448_b200 import _lib

    so = _lib.lib()
    st = D.stream_handle()
    rng = np.random.default_rng(11)
    dev = torch.device("cuda")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    for m, n, k in ((1, 1, 1), (37, 45, 13), (70, 9, 130), (33, 64, 4)):
        for ta in (0, 1):
            for tb in (0, 1):
                a = rng.standard_normal((k, m) if ta else (m, k))
                b = rng.standard_normal((n, k) if tb else (k, n))
                want = (a.T if ta else a) @ (b.T if tb else b)
                c = torch.full((m, n), 2.0, dtype=torch.float64, device=dev)
                ad, bd = T(a), T(b)  # keep the device copies alive until the kernel ran
                _lib.check(so.fb_dense_mm(m, n, k, D.ptr(ad), a.shape[1], ta, D.ptr(bd), b.shape[1], tb, D.ptr(c), n,
                                          1, st))
                torch.cuda.synchronize()
                np.testing.assert_allclose(c.cpu().numpy(), want + 2.0, rtol=1e-12, atol=1e-12)
    mat = rng.standard_normal((17, 23))
    ra = rng.integers(0, 17, 41).astype(np.int32)
    cb = rng.integers(0, 23, 29).astype(np.int32)
    c = torch.ones((41, 29), dtype=torch.float64, device=dev)
    keep = [T(mat), T(ra), T(cb)]
    _lib.check(so.fb_gather2_add(41, 29, D.ptr(keep[0]), 23, D.ptr(keep[1]), D.ptr(keep[2]), D.ptr(c), 29, st))
    np.testing.assert_array_equal(c.cpu().numpy(), 1.0 + mat[ra][:, cb])
    a = rng.standard_normal((500, 7))
    tgt = rng.integers(0, 31, 500).astype(np.int32)
    out = torch.empty((31, 7), dtype=torch.float64, device=dev)
    keep = [T(tgt), T(a)]
    _lib.check(so.fb_scatter_rows(500, 7, D.ptr(keep[0]), D.ptr(keep[1]), 7, D.ptr(out), 31, st))
    want = np.zeros((31, 7))
    np.add.at(want, tgt, a)
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-12, atol=1e-12)
    for n_rows, ca, cbn in ((1, 1, 1), (5000, 40, 17), (20000, 3, 900)):
        t1 = rng.integers(0, ca, n_rows).astype(np.int32)
        t2 = rng.integers(0, cbn, n_rows).astype(np.int32)
        want = sp.csr_matrix((np.ones(n_rows), (t1, t2)), shape=(ca, cbn))
        want.sum_duplicates()
        want.sort_indices()
        indptr = torch.empty(ca + 1, dtype=torch.int64, device=dev)
        col = torch.empty(n_rows, dtype=torch.int64, device=dev)
        val = torch.empty(n_rows, dtype=torch.float64, device=dev)
        nnz = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = torch.empty(so.fb_pair_counts_workspace_bytes(n_rows), dtype=torch.uint8, device=dev)
        keep = [T(t1), T(t2)]
        _lib.check(so.fb_pair_counts(n_rows, D.ptr(keep[0]), D.ptr(keep[1]), ca, cbn, D.ptr(indptr), D.ptr(col),
                                     D.ptr(val), D.ptr(nnz), ws.data_ptr(), ws.numel(), st))
        k = int(nnz.item())
        assert k == want.nnz
        np.testing.assert_array_equal(indptr.cpu().numpy(), want.indptr)
        np.testing.assert_array_equal(col[:k].cpu().numpy(), want.indices)
        np.testing.assert_array_equal(val[:k].cpu().numpy(), want.data)
    p = sp.random(300, 50, density=0.05, random_state=3, format="csr")
    x = rng.standard_normal((50, 37))
    y = torch.empty((300, 37), dtype=torch.float64, device=dev)
    keep = [T(p.indptr.astype(np.int64)), T(p.indices.astype(np.int32)), T(p.data), T(x)]
    _lib.check(so.fb_csr_spmm(300, D.ptr(keep[0]), D.ptr(keep[1]), 0, D.ptr(keep[2]), D.ptr(keep[3]), 37, 37, D.ptr(y),
                              37, 0, st))
    np.testing.assert_allclose(y.cpu().numpy(), p @ x, rtol=1e-12, atol=1e-12)
    xt = rng.standard_normal((300, 5))
    yt = torch.empty((50, 5), dtype=torch.float64, device=dev)
    keep = [T(p.indptr.astype(np.int64)), T(p.indices.astype(np.int64)), T(p.data), T(xt)]
    _lib.check(so.fb_csr_spmm_t(300, 50, D.ptr(keep[0]), D.ptr(keep[1]), 1, D.ptr(keep[2]), D.ptr(keep[3]), 5, 5,
                                D.ptr(yt), 5, st))
    np.testing.assert_allclose(yt.cpu().numpy(), p.T @ xt, rtol=1e-12, atol=1e-12)

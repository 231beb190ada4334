"""Generate golden vectors from the LIVE reference package (build container only).

Run here, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py

It imports ``factorla`` from /root/reference/pkg/src, builds small seeded PK-FK / star /
skewed fixtures (including unreferenced attribute rows and a zero-width S), runs every
in-scope operator and driver through the reference's own public API, and writes
``tests/golden/<fixture>.npz`` (inputs + outputs + the reference's op counters). The GPU
box never reads /root/reference; tests read only these committed files.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _fixtures():
    rng = np.random.default_rng(20161224)
    fx = {}
    # SPEC fixture F1
    fx["f1"] = dict(s=np.array([[1.0, 2], [3, 4], [5, 6]]), parts=[(np.array([1, 2, 1]), np.array([[10.0, 20], [30, 40]]))])
    # SPEC fixture F3, star q=2
    fx["f3"] = dict(
        s=np.array([[1.0], [2], [3]]),
        parts=[(np.array([1, 2, 1]), np.array([[10.0], [20]])), (np.array([2, 1, 2]), np.array([[100.0], [200]]))],
    )
    # random PK-FK, N(0,1), R rows 3, 11, 29 never referenced
    n_s, n_r = 257, 31
    keys = rng.integers(1, n_r + 1, size=n_s)
    keys[np.isin(keys, [3, 11, 29])] = 1
    fx["pkfk_normal"] = dict(s=rng.standard_normal((n_s, 5)), parts=[(keys, rng.standard_normal((n_r, 7)))])
    # star with two FKs, N(0,1)
    n_s = 301
    fx["star_normal"] = dict(
        s=rng.standard_normal((n_s, 4)),
        parts=[
            (rng.integers(1, 21, size=n_s), rng.standard_normal((20, 3))),
            (rng.integers(1, 53, size=n_s), rng.standard_normal((52, 6))),
        ],
    )
    # Zipf(1.2)-skewed FK over U[0,1) tables (non-negative, for GNMF)
    n_s, n_r = 503, 40
    p = np.arange(1, n_r + 1, dtype=np.float64) ** -1.2
    p /= p.sum()
    zk = np.searchsorted(np.cumsum(p), rng.random(n_s), side="right") + 1
    zk = np.minimum(zk, n_r)
    fx["zipf_uniform"] = dict(s=rng.random((n_s, 3)), parts=[(zk, rng.random((n_r, 9)))])
    # wide-ish U[0,1) PK-FK (crossprod / linreg)
    n_s, n_r = 400, 25
    fx["pkfk_uniform"] = dict(s=rng.random((n_s, 12)), parts=[(rng.integers(1, n_r + 1, size=n_s), rng.random((n_r, 18)))])
    # zero-width entity table (SPEC.md DESIGN DECISIONS: d_S = 0 is legal)
    n_s, n_r = 64, 9
    fx["zero_width_s"] = dict(s=np.zeros((n_s, 0)), parts=[(rng.integers(1, n_r + 1, size=n_s), rng.standard_normal((n_r, 4)))])
    return fx


def _mn_fixtures():
    """M:N (normmat.py:240-285) and multi-table M:N (normmat.py:288-319) fixtures."""
    rng = np.random.default_rng(1612)
    fx = {}
    # M:N, N(0,1): join values 0..14 on S, 3..19 on R (values outside the overlap and the rows
    # holding them are dropped), duplicates on both sides
    n_s, n_r = 90, 40
    fx["mn_normal"] = dict(kind="mn", s=rng.standard_normal((n_s, 4)), j_s=rng.integers(0, 15, size=n_s),
                           r=rng.standard_normal((n_r, 6)), j_r=rng.integers(3, 20, size=n_r))
    # M:N over U[0,1) tables (GNMF needs non-negative T)
    n_s, n_r = 70, 25
    fx["mn_uniform"] = dict(kind="mn", s=rng.random((n_s, 5)), j_s=rng.integers(0, 9, size=n_s),
                            r=rng.random((n_r, 3)), j_r=rng.integers(0, 12, size=n_r))
    # multi-table M:N: three tables, an explicit row map with unreferenced rows
    n_out = 150
    tabs = [rng.standard_normal((30, 3)), rng.standard_normal((12, 4)), rng.standard_normal((50, 2))]
    row_map = np.stack([rng.integers(0, 25, size=n_out), rng.integers(0, 12, size=n_out),
                        rng.integers(5, 50, size=n_out)], axis=1)
    fx["multimn_normal"] = dict(kind="multimn", tables=tabs, row_map=row_map)
    return fx


def _record_ops(rec, nm, rng, kernel, ml, normmat, rewrite, nonneg):
    n, d = nm.shape
    rec["materialize"] = normmat.materialize(nm)
    x1 = rng.standard_normal((d, 1))
    x3 = rng.standard_normal((d, 3))
    p2 = rng.standard_normal((n, 2))
    xr = rng.standard_normal((2, n))
    xt = rng.standard_normal((3, d))
    rec.update(x1=x1, x3=x3, p2=p2, xr=xr, xt=xt)
    c = kernel.OpCounter()
    rec["lmm_x1"] = rewrite.lmm(nm, x1, c)
    rec["cnt_lmm_x1"] = np.array([c.multiplies, c.additions])
    rec["lmm_x3"] = rewrite.lmm(nm, x3)
    c = kernel.OpCounter()
    rec["tmm_p2"] = rewrite.lmm(nm.T, p2, c)
    rec["cnt_tmm_p2"] = np.array([c.multiplies, c.additions])
    c = kernel.OpCounter()
    rec["rmm_xr"] = rewrite.rmm(xr, nm, c)
    rec["cnt_rmm_xr"] = np.array([c.multiplies, c.additions])
    rec["rmm_t_xt"] = rewrite.rmm(xt, nm.T)
    c = kernel.OpCounter()
    rec["row_sums"] = rewrite.row_sums(nm, c)
    rec["cnt_row_sums"] = np.array([c.multiplies, c.additions])
    c = kernel.OpCounter()
    rec["col_sums"] = rewrite.col_sums(nm, c)
    rec["cnt_col_sums"] = np.array([c.multiplies, c.additions])
    c = kernel.OpCounter()
    rec["sum_all"] = np.array(rewrite.sum_all(nm, c))
    rec["cnt_sum_all"] = np.array([c.multiplies, c.additions])
    rec["row_sums_t"] = rewrite.row_sums(nm.T)
    rec["col_sums_t"] = rewrite.col_sums(nm.T)
    for op, x in (("mul", 2.0), ("add", 3.0), ("rsub", 1.5), ("div", 4.0), ("pow", 2.0)):
        c = kernel.OpCounter()
        rec[f"scalar_{op}"] = normmat.materialize(rewrite.scalar_op(nm, x, op, c))
        rec[f"cnt_scalar_{op}"] = np.array([c.multiplies, c.additions])
    rec["fn_exp"] = normmat.materialize(rewrite.scalar_fn(nm, np.exp))
    c = kernel.OpCounter()
    rec["crossprod"] = rewrite.crossprod(nm, counter=c)
    rec["cnt_crossprod"] = np.array([c.multiplies, c.additions])
    w_true = rng.standard_normal((d, 1))
    t = normmat.materialize(nm)
    y_lin = t @ w_true + 0.01 * rng.standard_normal((n, 1))
    out = ml.linreg_normal(nm, y_lin)
    rec.update(y_lin=y_lin, linreg_w=out.weights, linreg_obj=np.array(out.objective))
    cfg = ml.TrainConfig(iterations=5, step_size=1e-3, k=3, r=2, rng_seed=3)
    y_log = np.where(t @ w_true >= 0, 1.0, -1.0)
    out = ml.logistic_gd(nm, y_log, cfg)
    rec.update(y_log=y_log, logreg_w=out.weights, logreg_obj=np.array(out.objective))
    out = ml.linreg_gd(nm, y_lin, cfg)
    rec.update(linreg_gd_w=out.weights, linreg_gd_obj=np.array(out.objective))
    out = ml.kmeans(nm, cfg)
    rec.update(kmeans_c=out.centroids, kmeans_obj=np.array(out.objective))
    if nonneg:
        out = ml.gnmf(nm, cfg)
        rec.update(gnmf_w=out.factors[0], gnmf_h=out.factors[1], gnmf_obj=np.array(out.objective))


def main_mn():
    sys.path.insert(0, REF)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    import factorla
    from factorla import kernel, ml, normmat, rewrite

    rng = np.random.default_rng(11)
    for name, f in _mn_fixtures().items():
        if f["kind"] == "mn":
            nm = normmat.build_mn(f["s"], f["j_s"], f["r"], f["j_r"])
            rec = {"kind": np.array("mn"), "s": f["s"], "j_s": f["j_s"], "r": f["r"], "j_r": f["j_r"]}
            facs = [f["s"], f["r"]]
        else:
            nm = normmat.build_multimn(f["row_map"], f["tables"])
            rec = {"kind": np.array("multimn"), "row_map": f["row_map"], "q": np.array(len(f["tables"]))}
            for j, t in enumerate(f["tables"]):
                rec[f"table{j}"] = t
            facs = f["tables"]
        for i, (e, fk) in enumerate(nm.blocks):
            rec[f"target{i}"] = e.target
            rec[f"used{i}"] = nm.source_rows[i]
            rec[f"counts{i}"] = e.counts
            rec[f"kept{i}"] = fk
        nonneg = all(float(np.min(t)) >= 0 for t in facs)
        _record_ops(rec, nm, rng, kernel, ml, normmat, rewrite, nonneg)
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **{k: np.asarray(v) for k, v in rec.items()})
        print("wrote", path, os.path.getsize(path), "bytes", "factorla", getattr(factorla, "__version__", "?"))


def main_products():
    """gram_transposed / ginv / dmm / dmm_gram / pair_product / elementwise (rewrite.py:301-470)."""
    sys.path.insert(0, REF)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    import warnings

    from factorla import indicator, kernel, normmat, rewrite

    rng = np.random.default_rng(301)
    rec = {}

    def pk(prefix, n_s, d_s, n_r, d_r):
        s = rng.standard_normal((n_s, d_s))
        k = rng.integers(1, n_r + 1, size=n_s)
        r = rng.standard_normal((n_r, d_r))
        rec.update({f"{prefix}_s": s, f"{prefix}_k": k, f"{prefix}_r": r})
        return normmat.build_pkfk(s, k, r)

    def cnt(name, fn):
        c = kernel.OpCounter()
        out = fn(c)
        rec[name] = out.toarray() if hasattr(out, "toarray") else np.asarray(out)
        rec["cnt_" + name] = np.array([c.multiplies, c.additions])

    a = pk("a", 120, 5, 17, 7)        # A: 120 x 12 (tall)
    w = pk("w", 6, 4, 3, 5)           # W: 6 x 9 (wide)
    cnt("gram_t_a", lambda c: rewrite.gram_transposed(a, c))
    cnt("gram_t_w", lambda c: rewrite.gram_transposed(w.T, c))
    cnt("ginv_a", lambda c: rewrite.ginv(a, c))
    cnt("ginv_at", lambda c: rewrite.ginv(a.T, c))
    cnt("ginv_w", lambda c: rewrite.ginv(w, c))
    cnt("ginv_wt", lambda c: rewrite.ginv(w.T, c))
    b = pk("b", 12, 3, 5, 4)          # B: 12 x 7 (rows = A's columns)
    cnt("dmm_ab", lambda c: rewrite.dmm(a, b, c))
    b2 = pk("b2", 120, 2, 9, 3)       # same rows as A: A'B2 (atb)
    cnt("dmm_atb", lambda c: rewrite.dmm(a.T, b2, c))
    for tag, ds in (("lt", 3), ("eq", 5), ("gt", 8)):  # d_S of B3 below / equal / above A's
        b3 = pk(f"b3{tag}", 40, ds, 11, 12 - ds)
        cnt(f"dmm_abt_{tag}", lambda c, b3=b3: rewrite.dmm(a, b3.T, c))
    b4 = pk("b4", 9, 2, 4, 10)        # B4 (9 x 12): A'' B4' = (B4 A)'... dmm(A.T, B4.T) = (B4 A)'
    cnt("dmm_atbt", lambda c: rewrite.dmm(b4.T, pk("c", 12, 2, 3, 7).T, c))
    cnt("pair_ab2", lambda c: indicator.pair_product(a.k, b2.k, c))
    x = rng.standard_normal(a.shape)
    rec["ew_x"] = x
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for op in ("add", "sub", "rsub", "mul", "div", "rdiv"):
            cnt(f"ew_{op}", lambda c, op=op: rewrite.elementwise_matrix_op(a, x, op, c))
    # drivers on a transposed normalized matrix (ml.py: _mm / _tmm / _crossprod dispatch on the
    # flag; kmeans refuses it in _take_rows)
    from factorla import ml
    u = normmat.build_pkfk(rng.random((40, 3)), rng.integers(1, 9, size=40), rng.random((8, 4)))
    rec.update(u_s=u.s, u_k=np.asarray(u.k.target) + 1, u_r=u.r)
    n_t = u.T.shape[0]
    y_lin = rng.standard_normal((n_t, 1))
    y_log = np.where(rng.standard_normal((n_t, 1)) >= 0, 1.0, -1.0)
    cfg = ml.TrainConfig(iterations=4, step_size=1e-2, r=2, rng_seed=5)
    rec.update(ut_y_lin=y_lin, ut_y_log=y_log)
    out = ml.logistic_gd(u.T, y_log, cfg)
    rec.update(ut_logreg_w=out.weights, ut_logreg_obj=np.array(out.objective))
    out = ml.linreg_gd(u.T, y_lin, cfg)
    rec.update(ut_linreg_gd_w=out.weights, ut_linreg_gd_obj=np.array(out.objective))
    out = ml.linreg_normal(u.T, y_lin)
    rec.update(ut_linreg_w=out.weights, ut_linreg_obj=np.array(out.objective))
    out = ml.gnmf(u.T, cfg)
    rec.update(ut_gnmf_w=out.factors[0], ut_gnmf_h=out.factors[1], ut_gnmf_obj=np.array(out.objective))
    # cost model (costmodel.py:75-134): predicted counts and plans on a few shapes
    from factorla import costmodel
    st_mats = {"a": a, "u": u, "w": w}
    mnm = normmat.build_mn(rng.random((30, 2)), rng.integers(0, 6, size=30), rng.random((12, 3)),
                           rng.integers(0, 6, size=12))
    rec.update(mn_s=np.asarray(mnm.blocks[0][1]), mn_r=np.asarray(mnm.blocks[1][1]))
    rec["mn_ts"] = np.asarray(mnm.blocks[0][0].target)
    rec["mn_tr"] = np.asarray(mnm.blocks[1][0].target)
    st_mats["mn"] = mnm
    for key, nmx in st_mats.items():
        st = normmat.stats(nmx)
        for op in costmodel.KNOWN_OPS:
            pc = costmodel.predict_counts(op, st, d_x=3, n_x=2)
            rec[f"cm_{key}_{op}"] = np.array([pc.standard, pc.factorized])
        rec[f"cm_{key}_plan_default"] = np.array(costmodel.decide(st).value)
        rec[f"cm_{key}_plan_loose"] = np.array(costmodel.decide(st, costmodel.DecisionThresholds(1.0, 0.1)).value)
    path = os.path.join(OUT, "products.npz")
    np.savez_compressed(path, **{k: np.asarray(v) for k, v in rec.items()})
    print("wrote", path, os.path.getsize(path), "bytes")


def main():
    sys.path.insert(0, REF)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    import factorla
    from factorla import kernel, ml, normmat, rewrite

    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(7)
    for name, f in _fixtures().items():
        s, parts = f["s"], f["parts"]
        if len(parts) == 1:
            nm = normmat.build_pkfk(s, parts[0][0], parts[0][1])
        else:
            nm = normmat.build_star(s, parts)
        n, d = nm.shape
        rec = {"s": s, "q": np.array(len(parts))}
        for i, (k, r) in enumerate(parts):
            rec[f"key{i}"] = np.asarray(k, dtype=np.int64)
            rec[f"r{i}"] = r
            e, rk = nm.blocks[i + 1]
            rec[f"target{i}"] = e.target
            rec[f"used{i}"] = nm.source_rows[i + 1]
            rec[f"counts{i}"] = e.counts
            rec[f"rkept{i}"] = rk
        rec["materialize"] = normmat.materialize(nm)
        x1 = rng.standard_normal((d, 1))
        x3 = rng.standard_normal((d, 3))
        p2 = rng.standard_normal((n, 2))
        xr = rng.standard_normal((2, n))
        xt = rng.standard_normal((3, d))
        rec.update(x1=x1, x3=x3, p2=p2, xr=xr, xt=xt)
        c = kernel.OpCounter()
        rec["lmm_x1"] = rewrite.lmm(nm, x1, c)
        rec["cnt_lmm_x1"] = np.array([c.multiplies, c.additions])
        rec["lmm_x3"] = rewrite.lmm(nm, x3)
        c = kernel.OpCounter()
        rec["tmm_p2"] = rewrite.lmm(nm.T, p2, c)
        rec["cnt_tmm_p2"] = np.array([c.multiplies, c.additions])
        c = kernel.OpCounter()
        rec["rmm_xr"] = rewrite.rmm(xr, nm, c)
        rec["cnt_rmm_xr"] = np.array([c.multiplies, c.additions])
        rec["rmm_t_xt"] = rewrite.rmm(xt, nm.T)
        c = kernel.OpCounter()
        rec["row_sums"] = rewrite.row_sums(nm, c)
        rec["cnt_row_sums"] = np.array([c.multiplies, c.additions])
        c = kernel.OpCounter()
        rec["col_sums"] = rewrite.col_sums(nm, c)
        rec["cnt_col_sums"] = np.array([c.multiplies, c.additions])
        c = kernel.OpCounter()
        rec["sum_all"] = np.array(rewrite.sum_all(nm, c))
        rec["cnt_sum_all"] = np.array([c.multiplies, c.additions])
        rec["row_sums_t"] = rewrite.row_sums(nm.T)
        rec["col_sums_t"] = rewrite.col_sums(nm.T)
        for op, x in (("mul", 2.0), ("add", 3.0), ("rsub", 1.5), ("div", 4.0), ("pow", 2.0)):
            c = kernel.OpCounter()
            rec[f"scalar_{op}"] = normmat.materialize(rewrite.scalar_op(nm, x, op, c))
            rec[f"cnt_scalar_{op}"] = np.array([c.multiplies, c.additions])
        rec["fn_exp"] = normmat.materialize(rewrite.scalar_fn(nm, np.exp))
        rec["fn_square"] = normmat.materialize(rewrite.scalar_fn(nm, np.square))
        if s.shape[1] > 0:
            c = kernel.OpCounter()
            rec["crossprod"] = rewrite.crossprod(nm, counter=c)
            rec["cnt_crossprod"] = np.array([c.multiplies, c.additions])
            w_true = rng.standard_normal((d, 1))
            t = normmat.materialize(nm)
            y_lin = t @ w_true + 0.01 * rng.standard_normal((n, 1))
            out = ml.linreg_normal(nm, y_lin)
            rec.update(y_lin=y_lin, linreg_w=out.weights, linreg_obj=np.array(out.objective))
            cfg = ml.TrainConfig(iterations=5, step_size=1e-3, k=3, r=2, rng_seed=3)
            y_log = np.where(t @ w_true >= 0, 1.0, -1.0)
            out = ml.logistic_gd(nm, y_log, cfg)
            rec.update(y_log=y_log, logreg_w=out.weights, logreg_obj=np.array(out.objective))
            out = ml.linreg_gd(nm, y_lin, cfg)
            rec.update(linreg_gd_w=out.weights, linreg_gd_obj=np.array(out.objective))
            out = ml.kmeans(nm, cfg)
            rec.update(kmeans_c=out.centroids, kmeans_obj=np.array(out.objective))
            if float(min(s.min(), min(r.min() for _, r in parts))) >= 0:
                out = ml.gnmf(nm, cfg)
                rec.update(gnmf_w=out.factors[0], gnmf_h=out.factors[1], gnmf_obj=np.array(out.objective))
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **{k: np.asarray(v) for k, v in rec.items()})
        print("wrote", path, os.path.getsize(path), "bytes", "factorla", getattr(factorla, "__version__", "?"))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "mn":
        main_mn()
    elif len(sys.argv) > 1 and sys.argv[1] == "products":
        main_products()
    else:
        main()
        main_mn()
        main_products()

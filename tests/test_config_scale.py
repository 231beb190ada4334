"""Config-scale parity: every BASELINE.json configuration at its full size, GPU vs CPU oracle.

SURVEY.md §4 item 3 / VERDICT r1 "next" #1. Inputs come from ``workloads.generate`` (the
SURVEY §8(d) NumPy seeds, drawn on the box host); the GPU runs through the public API
(host arrays in, host arrays out) and the oracle (the pinned CPU restatement of the
reference, tests/test_oracle.py) runs on the same arrays in the same process.

Bars (BASELINE.json north_star): FK remap / kept rows / counts and K-Means assignments
bit-exact; float64 results within normwise rel 1e-9 (bench.py:38-43 metric). The RMM /
Tᵀ·X scatters use L2 atomics (REDG) whose order varies run to run: their bound is the
same 1e-9 (measured deviations 1e-16..1e-13). c4 runs 10 K-Means iterations instead of 20
(the CPU oracle needs ~4.5 s per iteration at c4 on the box's 16 cores); every iteration's
assignment vector (10M rows) is compared, and the smallest argmin margin is printed.
"""
import gc
import time

import numpy as np
import pytest
import torch

import factorla_oracle as O
import workloads as W

pytestmark = pytest.mark.gpu

TOL = 1e-9


def _fb():
    import paper_1612_07448_b200 as fb

    return fb


def _dev(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    return O.max_rel_deviation(a, b)


def _build(g):
    fb = _fb()
    parts = W.keys_1based(g["parts"])
    if len(parts) == 1:
        nm = fb.build_pkfk(g["s"], parts[0][0], parts[0][1])
        ref = O.build_pkfk(g["s"], parts[0][0], parts[0][1])
    else:
        nm = fb.build_star(g["s"], parts)
        ref = O.build_star(g["s"], parts)
    # construction: remapped targets, kept R rows and counts bit-exact (normmat.py:168-237)
    for i, (e, _) in enumerate(nm.parts):
        np.testing.assert_array_equal(e.target_numpy(), ref.parts[i][0])
        np.testing.assert_array_equal(nm.source_rows[i + 1].cpu().numpy(), ref.source_rows[i + 1])
        np.testing.assert_array_equal(e.counts_i32.cpu().numpy(), O.counts(ref.parts[i][0], ref.parts[i][1].shape[0]))
    return nm, ref


def _report(name, devs):
    print(f"\n[{name}] " + ", ".join(f"{k}={v:.2e}" for k, v in devs.items()))
    for k, v in devs.items():
        assert v <= TOL, (name, k, v)


def test_c1_logreg_full():
    fb = _fb()
    g = W.generate("c1")
    nm, ref = _build(g)
    devs = {"lmm_x60x1": _dev(fb.lmm(nm, g["x"]), O.lmm(ref, g["x"])),
            "crossprod": _dev(fb.crossprod(nm), O.crossprod(ref)),
            "col_sums": _dev(fb.col_sums(nm), O.col_sums(ref))}
    out = fb.logistic_gd(nm, g["y"], fb.TrainConfig(iterations=g["iterations"], step_size=g["step"]))
    w_ref, tr_ref = O.logistic_gd(ref, g["y"], g["iterations"], g["step"])
    devs["logreg_w"] = _dev(out.weights, w_ref)
    devs["logreg_objective"] = _dev(out.objective, tr_ref)
    _report("c1", devs)


def test_c2_operator_suite_full():
    fb = _fb()
    g = W.generate("c2")
    nm, ref = _build(g)
    devs = {}
    devs["lmm_x1"] = _dev(fb.lmm(nm, g["x1"]), O.lmm(ref, g["x1"]))
    gc.collect()
    devs["lmm_x16"] = _dev(fb.lmm(nm, g["x16"]), O.lmm(ref, g["x16"]))
    gc.collect()
    devs["rmm_x1"] = _dev(fb.rmm(g["xr"], nm), O.rmm(g["xr"], ref))
    devs["row_sums"] = _dev(fb.row_sums(nm), O.row_sums(ref))
    devs["col_sums"] = _dev(fb.col_sums(nm), O.col_sums(ref))
    _report("c2", devs)


def test_c3_crossprod_linreg_full():
    fb = _fb()
    g = W.generate("c3")
    nm, ref = _build(g)
    cp = fb.crossprod(nm)
    cp = cp.cpu().numpy() if isinstance(cp, torch.Tensor) else cp
    np.testing.assert_array_equal(cp, cp.T)  # exactly symmetric (rewrite.py:298)
    devs = {"crossprod": _dev(cp, O.crossprod(ref))}
    out = fb.linreg_normal(nm, g["y"])
    w_ref, obj_ref = O.linreg_normal(ref, g["y"])
    devs["linreg_w"] = _dev(out.weights, w_ref)
    devs["linreg_objective"] = _dev(out.objective, obj_ref)
    print("\n[c3] |w - w_true|_max =", float(np.max(np.abs(np.asarray(out.weights) - g["w_true"]))))
    _report("c3", devs)


def test_c4_kmeans_full_assignments_bit_exact():
    fb = _fb()
    g = W.generate("c4")
    nm, ref = _build(g)
    iters = 10
    hist = []
    t0 = time.perf_counter()
    c_ref, tr_ref, _ = O.kmeans(ref, g["k"], iters, g["kmeans_seed"], history=hist)
    cpu_s = time.perf_counter() - t0
    devs = {}
    for it in range(1, iters + 1):
        out = fb.kmeans(nm, fb.TrainConfig(iterations=it, k=g["k"], rng_seed=g["kmeans_seed"]))
        got = out.assignment.cpu().numpy()
        want, margin = hist[it - 1]
        diff = np.flatnonzero(got != want)
        if diff.size:
            pytest.fail(f"c4 iteration {it}: {diff.size} assignments differ; margins there "
                        f"{np.sort(margin[diff])[:5]} (min margin overall {margin.min():.3e})")
        print(f"\n[c4] iteration {it}: assignments identical; smallest argmin margin {margin.min():.3e}")
        if it == iters:
            devs["centroids"] = _dev(out.centroids, c_ref)
            devs["objective"] = _dev(out.objective, tr_ref)
    print(f"[c4] oracle {iters} iterations: {cpu_s:.1f} s")
    _report("c4", devs)


def test_c5_gnmf_full():
    fb = _fb()
    g = W.generate("c5")
    nm, ref = _build(g)
    iters = g["iterations"]
    out = fb.gnmf(nm, fb.TrainConfig(iterations=iters, r=g["r"], rng_seed=g["gnmf_seed"]))
    w_ref, h_ref, tr_ref = O.gnmf(ref, g["r"], iters, g["gnmf_seed"])
    devs = {"W": _dev(out.factors[0], w_ref), "H": _dev(out.factors[1], h_ref),
            "objective": _dev(out.objective, tr_ref)}
    print(f"\n[c5] kept R rows {ref.parts[0][1].shape[0]} of {g['parts'][0][1].shape[0]}")
    _report("c5", devs)

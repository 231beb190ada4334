"""ML drivers over device-resident (normalized) matrices.

Same entry points, configuration and result types as the reference's ``factorla.ml``
(ml.py:1-317): ``logistic_gd``, ``linreg_gd``, ``linreg_normal``, ``kmeans`` and
``gnmf`` accept a :class:`NormalizedMatrix` or a regular matrix (NumPy / torch, viewed
as T = [S]) and return a :class:`ModelOutput` whose arrays are NumPy, like the
reference's.

Each iteration is one call into the C ABI (``fb_glm_step`` / ``fb_kmeans_step`` /
``fb_gnmf_step``), stream-ordered with no host synchronisation: objective traces and the
divergence flag stay on the device until the loop ends. Host-side arithmetic is limited
to what the reference itself does on tiny host matrices: the seeded NumPy RNG draws
(ml.py:268-271, 297-301) and the SVD pseudo-inverse of the d × d Gram matrix
(kernel.pinv_dense, kernel.py:303-324).
"""

import collections
import ctypes
import os
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from . import _lib
from . import kernel as K
from .crossprod_impl import crossprod as _crossprod_nm
from .exceptions import DataError, DivergenceError, NumericError, ShapeError
from .kernel import OpCounter
from .normmat import NormalizedMatrix, as_normalized
from .rewrite import row_sums, scalar_fn, sum_all

__all__ = ["TrainConfig", "ModelOutput", "logistic_gd", "linreg_normal", "linreg_gd", "kmeans", "gnmf"]


@dataclass(frozen=True)
class TrainConfig:
    """Iteration count, step size, K-Means k, GNMF rank r, RNG seed (ml.py:34-48)."""

    iterations: int = 20
    step_size: float = 0.01
    k: int = 10
    r: int = 5
    rng_seed: int = 0

    def __post_init__(self):
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")
        if self.step_size <= 0:
            raise ValueError("step_size must be positive")
        if self.k < 1 or self.r < 1:
            raise ValueError("k and r must be >= 1")


@dataclass
class ModelOutput:
    """Trained model plus objective trace, timing and op counts (ml.py:51-94)."""

    algorithm: str
    dims: tuple
    config: TrainConfig | None
    objective: list = field(default_factory=list)
    weights: np.ndarray | None = None
    centroids: np.ndarray | None = None
    factors: tuple | None = None
    wall_time_s: float = 0.0
    counts: OpCounter = field(default_factory=OpCounter)

    def model_arrays(self):
        out = {}
        if self.weights is not None:
            out["weights"] = self.weights
        if self.centroids is not None:
            out["centroids"] = self.centroids
        if self.factors is not None:
            out["w_factor"], out["h_factor"] = self.factors
        return out

    def to_json_dict(self):
        cfg = None
        if self.config is not None:
            cfg = {
                "iterations": self.config.iterations,
                "step_size": self.config.step_size,
                "k": self.config.k,
                "r": self.config.r,
                "rng_seed": self.config.rng_seed,
            }
        return {
            "algorithm": self.algorithm,
            "dims": {"rows": self.dims[0], "cols": self.dims[1]},
            "config": cfg,
            "objective": [float(v) for v in self.objective],
            "model": {
                name: {"shape": list(arr.shape), "values": arr.ravel().tolist()}
                for name, arr in self.model_arrays().items()
            },
            "timing": {"wall_time_s": self.wall_time_s},
            "counts": self.counts.as_dict(),
        }


# ---------------------------------------------------------------------------
# helpers


def _matrix(m):
    """Untransposed NormalizedMatrix view of the training input, device results."""
    nm = as_normalized(m)
    if nm.transposed:
        raise ShapeError("row sampling expects an untransposed matrix")  # ml.py:160-161 (kmeans)
    return nm.device_view()


def _transposed(m):
    return isinstance(m, NormalizedMatrix) and m.transposed


# ---------------------------------------------------------------------------
# drivers on a transposed normalized matrix: the reference's loops (ml.py:199-317) composed
# from the device operators, whose flag dispatch (rewrite.py:182-183, 204-205) turns T·w into
# Wᵀ·T scatters and Tᵀ·p into LMM gathers; the n_base-long weight vectors stay on the device


def _t_glm(m, y, cfg, mode, name):
    from .rewrite import lmm

    mt = m.device_view()
    n, d = mt.shape
    yd = _column(y, n)
    counter = OpCounter()
    so = _lib.lib()
    st = D.stream_handle()
    dev = yd.device
    w = torch.zeros((d, 1), dtype=torch.float64, device=dev)
    p = torch.empty((n, 1), dtype=torch.float64, device=dev)
    trace = torch.zeros(cfg.iterations, dtype=torch.float64, device=dev)
    diverged = torch.full((1,), -1, dtype=torch.int32, device=dev)
    ws = torch.empty(max(int(so.fb_glm_pointwise_workspace_bytes()), 256), dtype=torch.uint8, device=dev)
    alpha = cfg.step_size if mode == 0 else -cfg.step_size  # ml.py:212 / ml.py:251
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for it in range(cfg.iterations):
        tw = lmm(mt, w, counter)  # T·w: the Wᵀ·T scatter path of the untransposed factors
        # p = y / (1 + exp(tw)) and the stable log-loss, or the residual and its square sum
        _lib.check(so.fb_glm_pointwise(D.ptr(tw), D.ptr(yd), n, mode, D.ptr(p), D.ptr(trace), it, ws.data_ptr(),
                                       ws.numel(), st))
        g = lmm(mt.T, p, counter)  # Tᵀ·p: an LMM gather pass
        _lib.check(so.fb_axpy_check(alpha, D.ptr(g), D.ptr(w), d, it, D.ptr(diverged), st))
    bad = int(diverged.item())
    wall = time.perf_counter() - t0
    if bad >= 0:
        raise DivergenceError(bad)
    return ModelOutput(name, (n, d), cfg, _np(trace).tolist(), weights=_np(w), wall_time_s=wall, counts=counter)


def _t_linreg_normal(m, y):
    from .products import gram_transposed
    from .rewrite import lmm

    mt = m.device_view()
    n, d = mt.shape
    yd = _column(y, n)
    counter = OpCounter()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = _np(gram_transposed(mt.T, counter))  # _crossprod of a transposed matrix (ml.py:148-150)
    tty = _np(lmm(mt.T, yd, counter))
    w = _pinv_dense(g, counter) @ tty
    K.tally_matmul(counter, d, d, 1)
    so = _lib.lib()
    tw = lmm(mt, torch.from_numpy(w).to(yd.device), counter)
    resid = torch.empty_like(yd)
    obj = torch.zeros(1, dtype=torch.float64, device=yd.device)
    ws = torch.empty(max(int(so.fb_glm_pointwise_workspace_bytes()), 256), dtype=torch.uint8, device=yd.device)
    _lib.check(so.fb_glm_pointwise(D.ptr(tw), D.ptr(yd), n, 1, D.ptr(resid), D.ptr(obj), 0, ws.data_ptr(), ws.numel(),
                                   D.stream_handle()))  # Σ (T·w − y)²
    wall = time.perf_counter() - t0
    out = ModelOutput("linreg_normal", (n, d), None, [float(obj.item())], weights=w)
    out.wall_time_s = wall
    out.counts = counter
    return out


def _t_gnmf(m, cfg):
    from .rewrite import lmm, scalar_fn, sum_all

    mt = m.device_view()
    n, d = mt.shape
    if _min_value(mt) < 0:
        warnings.warn("input has negative entries; GNMF semantics assume non-negative data")
    rng = np.random.default_rng(cfg.rng_seed)
    counter = OpCounter()
    dev = mt.device
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = cfg.r
    if r > _MAX_R:
        raise NotImplementedError(f"the device GNMF step supports r <= {_MAX_R}")
    so = _lib.lib()
    st = D.stream_handle()
    w = torch.from_numpy(1.0 - rng.random((n, r))).to(dev)
    h = torch.from_numpy(1.0 - rng.random((d, r))).to(dev)
    sum_t2 = torch.tensor([sum_all(scalar_fn(mt, np.square, counter), counter)], dtype=torch.float64, device=dev)
    trace = torch.zeros(cfg.iterations, dtype=torch.float64, device=dev)
    cpw = _mirror_gram(w, counter)
    for it in range(cfg.iterations):
        ttw = lmm(mt.T, w, counter).contiguous()
        # h ← h ∘ ttw / (h·cpw + eps), w ← w ∘ th / (w·cph + eps): fb_nmf_update, in place (ml.py:308-312)
        _lib.check(so.fb_nmf_update(D.ptr(h), D.ptr(ttw), D.ptr(cpw), d, r, st))
        cph = _mirror_gram(h, counter)
        th = lmm(mt, h, counter).contiguous()
        _lib.check(so.fb_nmf_update(D.ptr(w), D.ptr(th), D.ptr(cph), n, r, st))
        ttw_now = lmm(mt.T, w, counter).contiguous()
        cpw = _mirror_gram(w, counter)
        # ‖T − W Hᵀ‖ = sqrt(max(ΣT² − 2 Σ(TᵀW ∘ H) + Σ(WᵀW ∘ HᵀH), 0))  (ml.py:314-315)
        _lib.check(so.fb_nmf_objective(D.ptr(sum_t2), D.ptr(ttw_now), D.ptr(h), d * r, D.ptr(cpw), D.ptr(cph), r * r,
                                       D.ptr(trace), it, st))
    trace = _np(trace).tolist()
    wall = time.perf_counter() - t0
    return ModelOutput("gnmf", (n, d), cfg, trace, factors=(_np(w), _np(h)), wall_time_s=wall, counts=counter)


def _mirror_gram(f, counter):
    """kernel.crossprod of a small dense factor: fᵀf with the upper triangle mirrored (kernel.py:138-154)."""
    return _crossprod_nm(as_normalized(f.contiguous()), counter=counter).contiguous()  # DMMA / narrow Gram, exact mirror


def _column(y, n, what="y"):
    t = D.as_matrix(y)
    if tuple(t.shape) != (n, 1):
        raise ShapeError(f"{what} must be {n}x1, got {t.shape[0]}x{t.shape[1]}")
    return t.contiguous()


def _np(t):
    return t.detach().cpu().numpy()


def _tally_lmm(counter, nm, d_x):
    """rewrite.lmm's counts (matmul per block + accumulate per indicator block)."""
    n = nm.base_rows
    for i, (e, f) in enumerate(nm.blocks):
        K.tally_matmul(counter, f.shape[0], f.shape[1], d_x)
        if i > 0:
            K.tally_accumulate(counter, n * d_x)


def _tally_tmm(counter, nm, n_w):
    """rewrite.lmm(m.T, ·) -> rmm's counts (right_compress + matmul per block)."""
    for e, f in nm.blocks:
        if e is not None:
            counter.tally(0, n_w * e.rows)
        K.tally_matmul(counter, n_w, f.shape[0], f.shape[1])


def _ws(nbytes):
    return D.workspace(nbytes)


# ---------------------------------------------------------------------------
# gradient descent (logistic / least squares)


# CUDA graphs of whole GD runs, keyed on the operands' device pointers (a replay reads the
# same buffers, so later in-place changes to S / R / y are seen). Small LRU; the entry keeps
# the normalized matrix alive so its pointers stay valid.
_GLM_GRAPHS = collections.OrderedDict()
_GLM_GRAPHS_MAX = 4


def _glm_run(so, cs, yd, w, trace, diverged, ws, mode, cfg, st):
    w.zero_()
    trace.zero_()
    diverged.fill_(-1)
    _lib.check(so.fb_glm_run(cs, D.ptr(yd), D.ptr(w), mode, float(cfg.step_size), cfg.iterations, D.ptr(trace),
                             D.ptr(diverged), ws.data_ptr(), ws.numel(), st))


def _glm_gd(m, y, cfg, mode, name):
    """GD loop (fb_glm_run). L2-resident problems (c1) run the whole loop as ONE cooperative
    launch; larger ones run one fused pass per iteration (fb_glm_step), captured once into a
    CUDA graph and replayed."""
    nm = _matrix(m)
    n, d = nm.shape
    yd = _column(y, n)
    so = _lib.lib()
    cs = nm.c_struct()
    dev = nm.device
    counter = OpCounter()
    key = (id(nm._cache), nm.blocks[0][1].data_ptr(), yd.data_ptr(), cfg.iterations, float(cfg.step_size), mode, dev.index)
    # graphs are cached only for caller-owned device operands: host y (or a host-built matrix)
    # means fresh device copies every call, whose key never repeats — capturing and pinning
    # them would only hold HBM
    cacheable = os.environ.get("FB_NO_GRAPHS") is None and isinstance(y, torch.Tensor) and y.is_cuda \
        and not nm.host_io
    entry = _GLM_GRAPHS.get(key) if cacheable else None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if entry is None:
        w = torch.zeros(d, dtype=torch.float64, device=dev)
        trace = torch.zeros(cfg.iterations, dtype=torch.float64, device=dev)
        diverged = torch.full((1,), -1, dtype=torch.int32, device=dev)
        ws = torch.empty(max(int(so.fb_glm_run_workspace_bytes(cs)), 256), dtype=torch.uint8, device=dev)
        _glm_run(so, cs, yd, w, trace, diverged, ws, mode, cfg, D.stream_handle())  # eager run (and warm-up)
        if cacheable and not so.fb_glm_run_fused(cs):
            graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                snap = (w.clone(), trace.clone(), diverged.clone())
                with torch.cuda.graph(graph, stream=side):
                    _glm_run(so, cs, yd, w, trace, diverged, ws, mode, cfg, side.cuda_stream)
                w.copy_(snap[0])
                trace.copy_(snap[1])
                diverged.copy_(snap[2])
            torch.cuda.current_stream().wait_stream(side)
            _GLM_GRAPHS[key] = (graph, w, trace, diverged, ws, yd, nm)
            while len(_GLM_GRAPHS) > _GLM_GRAPHS_MAX:
                _GLM_GRAPHS.popitem(last=False)
    else:
        _GLM_GRAPHS.move_to_end(key)
        graph, w, trace, diverged, ws, _, _ = entry
        graph.replay()
    bad = int(diverged.item())  # synchronises
    wall = time.perf_counter() - t0
    for _ in range(cfg.iterations):
        _tally_lmm(counter, nm, 1)
        _tally_tmm(counter, nm, 1)
    if bad >= 0:
        raise DivergenceError(bad)
    return ModelOutput(name, (n, d), cfg, _np(trace).tolist(), weights=_np(w).reshape(d, 1).copy(), wall_time_s=wall,
                       counts=counter)


def logistic_gd(m, y, cfg):
    """Logistic regression by full-gradient descent, labels in {-1, +1} (ml.py:199-215).

    Per iteration: w += α·Tᵀ(y / (1 + exp(T w))); the objective is the stable log-loss.
    """
    if _transposed(m):
        return _t_glm(m, y, cfg, 0, "logistic_gd")
    return _glm_gd(m, y, cfg, 0, "logistic_gd")


def linreg_gd(m, y, cfg):
    """Least squares by gradient descent: w -= α·Tᵀ(T w - y) (ml.py:239-254)."""
    if _transposed(m):
        return _t_glm(m, y, cfg, 1, "linreg_gd")
    return _glm_gd(m, y, cfg, 1, "linreg_gd")


def _pinv_dense(a, counter=None):
    """SVD pseudo-inverse with cutoff eps·max(m, n)·σ_max (kernel.pinv_dense, kernel.py:303-324)."""
    a = np.asarray(a, dtype=np.float64)
    mm, nn = a.shape
    try:
        u, s, vh = np.linalg.svd(a, full_matrices=False)
    except np.linalg.LinAlgError as exc:
        raise NumericError(f"SVD failed on {mm}x{nn} matrix: {exc}") from exc
    if s.size == 0 or s[0] == 0.0:
        return np.zeros((nn, mm))
    cutoff = np.finfo(np.float64).eps * max(mm, nn) * s[0]
    r = int(np.sum(s > cutoff))
    if counter is not None:
        counter.tally(7 * mm * nn * min(mm, nn) + 20 * min(mm, nn) ** 3, 0)
    if r == 0:
        return np.zeros((nn, mm))
    return (vh[:r].T / s[:r]) @ u[:, :r].T


def linreg_normal(m, y):
    """Least squares via the normal equations and the pseudo-inverse (ml.py:218-236).

    TᵀT (factorized crossprod, DMMA) and Tᵀy run on the device; the d × d pseudo-inverse
    is the reference's host SVD; the residual objective ‖Tw − y‖² is one fused device pass.
    """
    if _transposed(m):
        return _t_linreg_normal(m, y)
    nm = _matrix(m)
    n, d = nm.shape
    yd = _column(y, n)
    so = _lib.lib()
    st = D.stream_handle()
    cs = nm.c_struct()
    counter = OpCounter()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = _crossprod_nm(nm, counter=counter)
    g = g if isinstance(g, np.ndarray) else _np(g)
    gw = torch.empty(d + 1, dtype=torch.float64, device=yd.device)
    loss = torch.empty(1, dtype=torch.float64, device=yd.device)
    ws = _ws(so.fb_glm_workspace_bytes(cs))
    # Tᵀy: the least-squares gradient at w = 0 is Tᵀ(0 − y) = −Tᵀy
    zero = torch.zeros(d, dtype=torch.float64, device=yd.device)
    _lib.check(so.fb_glm_eval(cs, D.ptr(yd), D.ptr(zero), 1, D.ptr(gw), D.ptr(loss), ws.data_ptr(), ws.numel(), st))
    tty = -_np(gw[:d]).reshape(d, 1)
    _tally_tmm(counter, nm, 1)
    pinv = _pinv_dense(g, counter)
    w = pinv @ tty
    K.tally_matmul(counter, d, d, 1)
    wd = torch.from_numpy(np.ascontiguousarray(w.ravel())).to(yd.device)
    _lib.check(so.fb_glm_eval(cs, D.ptr(yd), D.ptr(wd), 1, D.ptr(gw), D.ptr(loss), ws.data_ptr(), ws.numel(), st))
    _tally_lmm(counter, nm, 1)
    obj = float(loss.item())
    wall = time.perf_counter() - t0
    out = ModelOutput("linreg_normal", (n, d), None, [obj], weights=w)
    out.wall_time_s = wall
    out.counts = counter
    return out


# ---------------------------------------------------------------------------
# K-Means


def _take_rows(nm, idx):
    """Dense copy of selected logical rows (ml.py:155-168), gathered on the device."""
    so = _lib.lib()
    st = D.stream_handle()
    idx_t = torch.as_tensor(np.asarray(idx, dtype=np.int64), device=nm.device)
    k = idx_t.numel()
    d = nm.base_cols
    out = torch.empty((k, d), dtype=torch.float64, device=nm.device)
    off = 0
    for e, f in nm.blocks:
        w = f.shape[1]
        if w:
            if e is None:
                _lib.check(so.fb_gather_rows(D.ptr(f), w, D.ptr(idx_t), k, w, out.data_ptr() + 8 * off, d, st))
            else:
                tgt = e.target.index_select(0, idx_t).contiguous()
                _lib.check(so.fb_gather_rows_i32(D.ptr(f), w, D.ptr(tgt), k, w, out.data_ptr() + 8 * off, d, st))
        off += w
    return out


# widest problems of the operator-by-operator steps (fb_kernels.cuh kKmeansMaxK / kNmfStepMaxR)
_MAX_K = 4096
_MAX_R = 256

_BAND_MIN_ITERS = int(os.environ.get("FB_KMEANS_BAND_MIN_ITERS", "8"))


def kmeans(m, cfg):
    """Matrix-form K-Means (ml.py:257-285); centroids are the columns of a d × k matrix.

    Seeding uses the reference's ``default_rng(seed).choice(n, k, replace=False)`` rows;
    per iteration the device computes T·(2C), the argmin assignment (ties to the lowest
    index), the objective, TᵀA (one-hot sums for S, integer Aᵀ·K histograms for R) and
    the centroid update (empty clusters keep their centroid).
    """
    nm = _matrix(m)
    n, d = nm.shape
    k = cfg.k
    if k > n:
        raise DataError(f"k={k} exceeds the number of data rows ({n})")
    if k > _MAX_K:
        raise NotImplementedError(f"the device K-Means step supports k <= {_MAX_K}")
    so = _lib.lib()
    st = D.stream_handle()
    cs = nm.c_struct()
    dev = nm.device
    rng = np.random.default_rng(cfg.rng_seed)
    counter = OpCounter()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c = _take_rows(nm, rng.choice(n, size=k, replace=False)).t().contiguous()  # d × k
    d_t = row_sums(scalar_fn(nm, np.square, counter), counter).reshape(-1).contiguous()  # rowSums(T²) (ml.py:272)
    for _, f in nm.blocks:  # two_t = 2·T (ml.py:273), folded into T·(2C) on the device
        counter.tally(f.numel(), 0)
    c0 = c.clone()
    # rows through the cached FK-band layout when part 0's z table would not stay in L2: the loop
    # then stores nothing in row order (objective, sizes, histograms and SᵀA are sums over rows),
    # and the last assignment is brought back to storage order once. Built on first use when the
    # run is long enough to pay for it (FB_KMEANS_BAND_MIN_ITERS), reused afterwards.
    band = None
    if "band" in nm._cache or cfg.iterations >= _BAND_MIN_ITERS:
        band = nm.kmeans_band_layout(k)

    def run(band):
        cc = _col_sq_sums(c)
        trace = torch.zeros(cfg.iterations, dtype=torch.float64, device=dev)
        assign = torch.empty(n, dtype=torch.int32, device=dev)
        nan_row = torch.full((1,), -1, dtype=torch.int64, device=dev)
        ws = _ws(so.fb_kmeans_workspace_bytes(cs, k))
        if band is not None:
            bst, perm = band[0], band[1]
            d_b = torch.empty_like(d_t)
            _lib.check(so.fb_gather_rows_i32(D.ptr(d_t), 1, D.ptr(perm), n, 1, D.ptr(d_b), 1, st))
            a_b = torch.empty_like(assign)
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
        for it in range(cfg.iterations):
            if band is not None:
                _lib.check(so.fb_kmeans_step_banded(cs, ctypes.byref(bst), D.ptr(d_b), D.ptr(c), D.ptr(cc), k, it,
                                                    D.ptr(trace), D.ptr(a_b), D.ptr(nan_row), ws.data_ptr(),
                                                    ws.numel(), st))
            else:
                _lib.check(so.fb_kmeans_step(cs, D.ptr(d_t), D.ptr(c), D.ptr(cc), k, it, D.ptr(trace), D.ptr(assign),
                                             D.ptr(nan_row), ws.data_ptr(), ws.numel(), st))
        ev[1].record()
        if band is not None:
            _lib.check(so.fb_scatter_i32(D.ptr(a_b), D.ptr(perm), n, D.ptr(assign), st))
        bad = int(nan_row.item())  # synchronizes
        return trace, assign, bad, ev[0].elapsed_time(ev[1])

    trace, assign, bad, loop_ms = run(band)
    if bad != -1 and band is not None:
        # a NaN row: the reference reports the first one in row order (kernel.py:327-339), which the
        # band order cannot tell — repeat the run in storage order for the exact row
        c.copy_(c0)
        trace, assign, bad, loop_ms = run(None)
    for it in range(cfg.iterations):
        _tally_lmm(counter, nm, k)
        counter.tally(0, n * k)  # row_min_mask
        _tally_tmm(counter, nm, k)
    wall = time.perf_counter() - t0
    if bad != -1:  # (iteration << 40) | row of the first NaN row of the first NaN iteration
        raise NumericError(f"row_min_mask: NaN in row {bad & ((1 << 40) - 1)}")
    out = ModelOutput("kmeans", (n, d), cfg, _np(trace).tolist(), centroids=_np(c), wall_time_s=wall, counts=counter)
    out.assignment = assign  # last iteration's argmin cluster per row (int32, device): parity checks
    out.loop_ms = loop_ms  # the iteration loop alone on the device timeline (CUDA events)
    return out


def _col_sq_sums(c):
    """cc[j] = Σ_r c[r, j]² (np.sum(c * c, axis=0), ml.py:276) on the device."""
    sq = scalar_fn(as_normalized(c.t().contiguous()), np.square)
    return row_sums(sq).reshape(-1).contiguous()


# ---------------------------------------------------------------------------
# GNMF


def _min_value(nm):
    vals = [float(f.min().item()) for _, f in nm.blocks if f.numel()]
    return min(vals) if vals else 0.0


def gnmf(m, cfg):
    """Gaussian NMF by multiplicative updates; factors W (n × r), H (d × r) (ml.py:288-317).

    W and H start from the reference's draws ``1 − default_rng(seed).random``; the
    objective ‖T − W Hᵀ‖ is tracked without materializing T. Tᵀ W of the updated W is
    reused as the next iteration's Tᵀ W (the reference recomputes the same product).
    """
    if _transposed(m):
        return _t_gnmf(m, cfg)
    nm = _matrix(m)
    n, d = nm.shape
    r = cfg.r
    if r > _MAX_R:
        raise NotImplementedError(f"the device GNMF step supports r <= {_MAX_R}")
    if _min_value(nm) < 0:
        warnings.warn("input has negative entries; GNMF semantics assume non-negative data")
    so = _lib.lib()
    st = D.stream_handle()
    cs = nm.c_struct()
    nm.ensure_sorted()  # Tᵀ·W scatters as segmented sums over the cached FK-sorted order
    dev = nm.device
    rng = np.random.default_rng(cfg.rng_seed)
    counter = OpCounter()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    w = torch.from_numpy(1.0 - rng.random((n, r))).to(dev)
    h = torch.from_numpy(1.0 - rng.random((d, r))).to(dev)
    sum_t2 = torch.tensor([sum_all(scalar_fn(nm, np.square, counter), counter)], dtype=torch.float64, device=dev)
    cpw = _crossprod_nm(as_normalized(w), counter=counter).contiguous()
    ttw = torch.empty((d, r), dtype=torch.float64, device=dev)
    wsz = _ws(so.fb_wt_workspace_bytes(cs, r))
    _lib.check(so.fb_wt(cs, D.ptr(w), r, r, 1, D.ptr(ttw), 1, r, wsz.data_ptr(), wsz.numel(), st))
    trace = torch.zeros(cfg.iterations, dtype=torch.float64, device=dev)
    ws = _ws(so.fb_gnmf_workspace_bytes(cs, r))
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ev[0].record()
    for it in range(cfg.iterations):
        _lib.check(so.fb_gnmf_step(cs, D.ptr(w), D.ptr(h), D.ptr(ttw), D.ptr(cpw), D.ptr(sum_t2), r, it,
                                   D.ptr(trace), ws.data_ptr(), ws.numel(), st))
        _tally_tmm(counter, nm, r)
        K.tally_crossprod(counter, d, r)
        _tally_lmm(counter, nm, r)
        _tally_tmm(counter, nm, r)
        K.tally_crossprod(counter, n, r)
    ev[1].record()
    objective = _np(trace).tolist()  # synchronizes
    wall = time.perf_counter() - t0
    out = ModelOutput("gnmf", (n, d), cfg, objective, factors=(_np(w), _np(h)), wall_time_s=wall, counts=counter)
    out.loop_ms = ev[0].elapsed_time(ev[1])  # the iteration loop alone on the device timeline (CUDA events)
    return out

"""Factorized operators over device-resident normalized matrices.

Same functions, signatures, transpose-flag dispatch and error behaviour as the
reference's ``factorla.rewrite`` (rewrite.py:25-39); the arithmetic runs in the
sm_100a kernels behind ``libfactorla_b200.so``:

====================  ==========================================  =======================
operator              reference                                   C ABI
====================  ==========================================  =======================
``scalar_op``         rewrite.py:75-86 -> kernel.scalar_map        fb_scalar_map
``scalar_fn``         rewrite.py:89-99 -> kernel.unary_map         fb_unary_map
``row_sums``          rewrite.py:118-128                           fb_row_sums
``col_sums``          rewrite.py:131-149                           fb_col_sums
``sum_all``           rewrite.py:152-165                           fb_sum_all
``lmm``               rewrite.py:172-191 (T.T: :182-183)           fb_lmm / fb_wt
``rmm``               rewrite.py:194-212 (T.T: :204-205)           fb_wt / fb_lmm
``crossprod``         rewrite.py:245-298 (efficient method)        fb_crossprod
====================  ==========================================  =======================

Operands may be NumPy arrays (results come back as NumPy, like the reference) or
CUDA tensors (results stay on the device).
"""

import warnings

import numpy as np
import torch

from . import _device as D
from . import _lib
from . import csr_ops as _csr
from . import kernel as K
from .exceptions import NumericError, ShapeError
from .normmat import NormalizedMatrix

__all__ = [
    "scalar_op",
    "scalar_fn",
    "row_sums",
    "col_sums",
    "sum_all",
    "lmm",
    "rmm",
    "crossprod",
    "gram_transposed",
    "ginv",
    "dmm",
    "dmm_gram",
    "elementwise_matrix_op",
    "MaterializationWarning",
    "HostCallableWarning",
]

_SCALAR_OPS = {"add": 0, "radd": 1, "sub": 2, "rsub": 3, "mul": 4, "rmul": 5, "div": 6, "rdiv": 7, "pow": 8, "rpow": 9}
_MULTIPLICATIVE = {"mul", "div", "pow", "rdiv", "rpow"}  # as kernel.py:216 ("rmul" tallies additions there)

_UNARY = {
    np.exp: 0,
    np.log: 1,
    np.square: 2,
    np.sqrt: 3,
    np.abs: 4,
    np.negative: 5,
    np.log1p: 6,
    np.expm1: 7,
    np.sin: 8,
    np.cos: 9,
    np.tanh: 10,
    np.reciprocal: 12,
}
_UNARY_NAMES = {
    "exp": 0, "log": 1, "square": 2, "sqrt": 3, "abs": 4, "absolute": 4, "negative": 5,
    "log1p": 6, "expm1": 7, "sin": 8, "cos": 9, "tanh": 10, "sigmoid": 11, "reciprocal": 12,
    "identity": 13,
}


def _nm_check(nm):
    if not isinstance(nm, NormalizedMatrix):
        raise TypeError(f"expected a NormalizedMatrix, got {type(nm).__name__}")


def _operand(x):
    """(device matrix, caller wanted host results)."""
    return D.as_matrix(x), D.is_host(x)


# ---------------------------------------------------------------------------
# element-wise scalar operators (closed: output is a normalized matrix)


def _map_factors(nm, launch):
    so = _lib.lib()
    st = D.stream_handle()
    new = []
    for _, f in nm.blocks:
        out = torch.empty_like(f)
        _lib.check(launch(so, f, out, st))
        new.append(out)
    return nm.with_factors(new)


def scalar_op(nm, x, op, counter=None):
    """``T <op> x`` applied to the factor matrices only (rewrite.py:75-86)."""
    _nm_check(nm)
    if op not in _SCALAR_OPS:
        raise ValueError(f"unknown scalar op {op!r}")
    x = float(x)
    if op == "div" and x == 0:
        raise NumericError("division by zero scalar")
    code = _SCALAR_OPS[op]
    out = _map_factors(nm, lambda so, f, o, st: so.fb_scalar_map(D.ptr(f), D.ptr(o), f.numel(), code, x, st))
    if counter is not None:
        for _, f in nm.blocks:
            cost = f.numel()
            counter.tally(cost, 0) if op in _MULTIPLICATIVE else counter.tally(0, cost)
    return out


class HostCallableWarning(UserWarning):
    """``scalar_fn`` received a callable that only accepts NumPy arrays: the factor matrices
    make one round trip through host memory so the caller's own function can run on them."""


def _apply_callable(f, fm):
    """``f`` applied element-wise to one dense device factor matrix.

    The reference hands ``f`` the factor as an ndarray (kernel.py:280-300). Here the factor is a
    CUDA tensor: array-polymorphic callables (arithmetic lambdas, torch functions) run on it in
    place on the device; a callable that needs an ndarray gets a host copy and its result is
    uploaded again (warned once per call — the function is the caller's host code, not an
    operator of this library).
    """
    try:
        with torch.no_grad():
            out = f(fm)
        if isinstance(out, torch.Tensor) and out.shape == fm.shape and out.device == fm.device:
            return out.to(torch.float64).contiguous(), False
    except Exception:  # noqa: BLE001 — any failure on a tensor argument means "wants an ndarray"
        pass
    with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
        host = np.asarray(f(fm.cpu().numpy()), dtype=np.float64)
    if host.shape != tuple(fm.shape):
        raise ShapeError(f"scalar_fn: the function returned shape {host.shape} for a {tuple(fm.shape)} factor")
    return torch.from_numpy(np.ascontiguousarray(host)).to(fm.device), True


def scalar_fn(nm, f, counter=None):
    """Element-wise ``f(T)`` = (f(S), K, f(R)) (rewrite.py:89-99).

    NumPy ufuncs of the built-in set (exp, log, square, sqrt, abs, negative, log1p, expm1, sin,
    cos, tanh, reciprocal) and those names (plus "sigmoid"/"identity") run in the library's
    element-wise kernel (``fb_unary_map``). Any other callable is applied to each factor matrix as
    the reference applies it (``_apply_callable``): on the device tensor when it accepts one, else
    on a host copy with a :class:`HostCallableWarning`.
    """
    _nm_check(nm)
    if isinstance(f, str):
        code = _UNARY_NAMES.get(f)
        if code is None:
            raise ValueError(f"scalar_fn: unknown function name {f!r}; known: {sorted(_UNARY_NAMES)}")
    else:
        code = _UNARY.get(f) if isinstance(f, np.ufunc) else None
        if code is None and not callable(f):
            raise TypeError(f"scalar_fn: expected a callable or a function name, got {type(f).__name__}")
    if code is not None:
        out = _map_factors(nm, lambda so, fm, o, st: so.fb_unary_map(D.ptr(fm), D.ptr(o), fm.numel(), code, st))
    else:
        new, via_host = [], False
        for _, fm in nm.blocks:
            o, h = _apply_callable(f, fm)
            new.append(o)
            via_host |= h
        if via_host:
            warnings.warn(f"scalar_fn: {getattr(f, '__name__', f)!r} ran on host copies of the factor matrices",
                          HostCallableWarning, stacklevel=2)
        out = nm.with_factors(new)
    if counter is not None:
        for _, fm in nm.blocks:
            counter.tally(fm.numel(), 0)
    return out


# ---------------------------------------------------------------------------
# aggregations


def row_sums(nm, counter=None):
    """Row totals of the logical matrix as a column vector (rewrite.py:118-128)."""
    _nm_check(nm)
    if nm.transposed:
        r = col_sums(nm.T, counter)
        return D.to_like(_as_dev(r).t().contiguous(), nm.host_io)
    so = _lib.lib()
    n = nm.base_rows
    if nm.block_path:  # CSR factors read natively / wide factors (csr_ops): T·1
        out = _csr.lmm(nm, _csr.ones(nm.base_cols, nm.device))
    else:
        out = torch.empty((n, 1), dtype=torch.float64, device=nm.device)
        cs = nm.c_struct()
        ws = D.workspace(so.fb_row_sums_workspace_bytes(cs))
        _lib.check(so.fb_row_sums(cs, D.ptr(out), ws.data_ptr(), ws.numel(), D.stream_handle()))
    if counter is not None:
        for i, (e, f) in enumerate(nm.raw_blocks):
            K.tally_rowsums(counter, f.shape[0], f.shape[1])
            if i > 0:
                K.tally_accumulate(counter, n)
    return D.to_like(out, nm.host_io)


def col_sums(nm, counter=None):
    """Column totals as a row vector; indicator blocks use cached counts (rewrite.py:131-149)."""
    _nm_check(nm)
    if nm.transposed:
        r = row_sums(nm.T, counter)
        return D.to_like(_as_dev(r).t().contiguous(), nm.host_io)
    so = _lib.lib()
    if nm.block_path:  # CSR factors read natively / wide factors (csr_ops): (Tᵀ·1)ᵀ
        out = _csr.tmm(nm, _csr.ones(nm.base_rows, nm.device)).reshape(1, -1)
    else:
        out = torch.empty((1, nm.base_cols), dtype=torch.float64, device=nm.device)
        cs = nm.c_struct()
        ws = D.workspace(so.fb_col_sums_workspace_bytes(cs))
        _lib.check(so.fb_col_sums(cs, D.ptr(out), ws.data_ptr(), ws.numel(), D.stream_handle()))
    if counter is not None:
        for e, f in nm.raw_blocks:
            if e is None:
                K.tally_colsums(counter, f.shape[0], f.shape[1])
            else:
                counter.tally(0, e.rows)
                K.tally_matmul(counter, 1, f.shape[0], f.shape[1])
    return D.to_like(out, nm.host_io)


def sum_all(nm, counter=None):
    """Grand total; invariant under transposition (rewrite.py:152-165)."""
    _nm_check(nm)
    base = nm.untransposed()
    so = _lib.lib()
    if base.block_path:
        out = _csr.sum_all(base)
    else:
        cs = base.c_struct()
        out = torch.empty(1, dtype=torch.float64, device=base.device)
        d = base.base_cols
        ws = D.workspace(so.fb_col_sums_workspace_bytes(cs) + 8 * d + 512)
        _lib.check(so.fb_sum_all(cs, D.ptr(out), ws.data_ptr(), ws.numel(), D.stream_handle()))
    if counter is not None:
        for e, f in base.raw_blocks:
            if e is None:
                K.tally_rowsums(counter, f.shape[0], f.shape[1])
                counter.tally(0, max(f.shape[0] - 1, 0))
            else:
                counter.tally(0, e.rows)
                K.tally_rowsums(counter, f.shape[0], f.shape[1])
                K.tally_matmul(counter, 1, f.shape[0], 1)
    return float(out.item())


# ---------------------------------------------------------------------------
# multiplication


def _as_dev(a):
    return a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a)).to(D.device())


def _lmm_dev(nm, x, counter):
    """T·X on the untransposed matrix; x is a contiguous device matrix (d × d_x)."""
    if nm.block_path:
        return _csr.lmm(nm, x, counter)
    so = _lib.lib()
    n, d_x = nm.base_rows, x.shape[1]
    out = torch.empty((n, d_x), dtype=torch.float64, device=x.device)
    cs = nm.c_struct()
    ws = D.workspace(so.fb_lmm_workspace_bytes(cs, d_x))
    band = nm.band_layout(d_x)  # cached FK-band copy of S when z = R·X would not stay in L2
    if band is not None:
        _lib.check(so.fb_lmm_banded(cs, band, D.ptr(x), d_x, D.ptr(out), ws.data_ptr(), ws.numel(),
                                    D.stream_handle()))
    else:
        _lib.check(so.fb_lmm(cs, D.ptr(x), d_x, D.ptr(out), ws.data_ptr(), ws.numel(), D.stream_handle()))
    if counter is not None:
        for i, (e, f) in enumerate(nm.raw_blocks):
            K.tally_matmul(counter, f.shape[0], f.shape[1], d_x)
            if i > 0:
                K.tally_accumulate(counter, n * d_x)
    return out


def _wt_dev(nm, w, w_rs, w_cs, n_w, out, o_js, o_cs, counter):
    """out(j, c) = Σ_i w(i, j) T(i, c) on the untransposed matrix.

    The X·K halves run as segmented sums over the cached FK-sorted order (built on first use,
    like the reference's cached CSR of K, indicator.py:71-86).
    """
    if nm.block_path:  # CSR factors read natively / wide factors (csr_ops): out(j, c) = (Tᵀ·W)[c, j]
        wd = torch.as_strided(w, (nm.base_rows, n_w), (w_rs, w_cs)).contiguous()
        res = _csr.tmm(nm, wd, counter)
        torch.as_strided(out, (nm.base_cols, n_w), (o_cs, o_js)).copy_(res)
        return out
    so = _lib.lib()
    cs = nm.c_struct()
    nm.ensure_sorted()
    ws = D.workspace(so.fb_wt_workspace_bytes(cs, n_w))
    _lib.check(so.fb_wt(cs, D.ptr(w), n_w, w_rs, w_cs, D.ptr(out), o_js, o_cs, ws.data_ptr(), ws.numel(),
                        D.stream_handle()))
    if counter is not None:
        for e, f in nm.raw_blocks:
            if e is not None:
                counter.tally(0, n_w * e.rows)
            K.tally_matmul(counter, n_w, f.shape[0], f.shape[1])
    return out


def lmm(nm, x, counter=None):
    """Left multiplication ``T X`` (rewrite.py:172-191); ``T.T X`` via the scatter path."""
    _nm_check(nm)
    xd, host = _operand(x)
    n_log, d_log = nm.shape
    if xd.shape[0] != d_log:
        raise ShapeError(f"lmm: X has {xd.shape[0]} rows, normalized matrix has {d_log} columns")
    if nm.transposed:
        # T' X = (X' T)'  (rewrite.py:182-183): weights w(i, j) = X[i, j]
        base = nm.T
        m = xd.shape[1]
        out = torch.empty((base.base_cols, m), dtype=torch.float64, device=xd.device)
        _wt_dev(base, xd, xd.stride(0), xd.stride(1), m, out, 1, m, counter)
        return D.to_like(out, host)
    return D.to_like(_lmm_dev(nm, xd, counter), host)


def rmm(x, nm, counter=None):
    """Right multiplication ``X T`` (rewrite.py:194-212)."""
    _nm_check(nm)
    xd, host = _operand(x)
    n_log, d_log = nm.shape
    if xd.shape[1] != n_log:
        raise ShapeError(f"rmm: X has {xd.shape[1]} columns, normalized matrix has {n_log} rows")
    if nm.transposed:
        # X T' = (T X')'  (rewrite.py:204-205)
        res = _lmm_dev(nm.T, xd.t().contiguous(), counter)
        return D.to_like(res.t().contiguous(), host)
    n_x = xd.shape[0]
    d = nm.base_cols
    out = torch.empty((n_x, d), dtype=torch.float64, device=xd.device)
    # weights w(i, j) = x[j, i]
    _wt_dev(nm, xd, xd.stride(1), xd.stride(0), n_x, out, d, 1, counter)
    return D.to_like(out, host)


def crossprod(nm, method="efficient", counter=None):
    """``T' T`` without materializing T; exactly symmetric (rewrite.py:245-298)."""
    from .crossprod_impl import crossprod as _cp

    return _cp(nm, method=method, counter=counter)


from .products import (  # noqa: E402  (rewrite.py:301-470: the rest of the operator surface)
    MaterializationWarning,
    dmm,
    dmm_gram,
    elementwise_matrix_op,
    ginv,
    gram_transposed,
)

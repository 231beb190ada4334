"""Row-Gram, pseudo-inverse, double multiplication and non-factorizable element-wise ops.

The rest of the reference's operator surface (rewrite.py:301-470, indicator.py:144-162;
SURVEY §8(f) row 3), on the device:

==========================  =====================================  ==========================
operator                    reference                              device composition
==========================  =====================================  ==========================
``gram_transposed``         rewrite.py:301-315                     per block F·Fᵀ (DGEMM) +
                                                                   two-sided row gather
``ginv``                    rewrite.py:318-333                     crossprod / gram_transposed,
                                                                   host SVD pinv of the small
                                                                   Gram, then rmm / lmm
``dmm``                     rewrite.py:349-389                     A·B = lmm(A, B materialised):
                                                                   B has only d_A rows
``dmm_gram``                rewrite.py:392-446                     block products (DGEMM) +
                                                                   keyed scatters / gathers
``elementwise_matrix_op``   rewrite.py:449-470                     materialise + map (warns)
``pair_product``            indicator.py:144-162                   2-D target histogram (CSR)
==========================  =====================================  ==========================

These sit beside the hot path (their outputs are n×n or n×m dense, or they run once per
model), so they are composed from the library's LMM/RMM/crossprod kernels plus cuBLAS
DGEMMs and torch gathers/scatters on device tensors; nothing runs on the host except the
reference's own LAPACK SVD of a d×d Gram. ``counter=`` gets the reference's tallies
(counting rules kernel.py:7-18) reproduced step by step.
"""

import warnings

import numpy as np
import torch

from . import _device as D
from . import _lib
from . import kernel as K
from .exceptions import ShapeError
from .normmat import PKFK, NormalizedMatrix, materialize

__all__ = [
    "MaterializationWarning",
    "gram_transposed",
    "ginv",
    "dmm",
    "dmm_gram",
    "elementwise_matrix_op",
    "pair_product",
]


class MaterializationWarning(UserWarning):
    """A non-factorizable operation (or a densifying one) ran on factors (rewrite.py:42-43)."""


def _mirror(g):
    """Exact symmetry: the upper triangle copied onto the lower (kernel.py:132-135)."""
    so = _lib.lib()
    g = g.contiguous()
    _lib.check(so.fb_mirror_upper(D.ptr(g), g.shape[0], D.stream_handle()))
    return g


def _tally_gram(counter, n, d):
    """kernel.gram of a dense n×d input (kernel.py:157-171)."""
    if counter is not None:
        counter.tally(d * n * (n + 1) // 2, max(d - 1, 0) * n * (n + 1) // 2)


def gram_transposed(nm, counter=None):
    """``T Tᵀ`` (the Gram matrix over rows) per column block: E_i (F_i F_iᵀ) E_iᵀ (rewrite.py:301-315).

    Ignores the transpose flag, like the reference. The result is n × n and exactly
    symmetric; host operands give a NumPy result.
    """
    base = nm.untransposed()
    out = None
    for e, f in base.blocks:
        g = _mirror(torch.mm(f, f.t()))  # cuBLAS DGEMM on the (small) factor
        _tally_gram(counter, f.shape[0], f.shape[1])
        if e is not None:
            t = e.target.to(torch.int64)
            g = g.index_select(0, t).index_select(1, t)
        if out is None:
            out = g
        else:
            out = out + g
            K.tally_accumulate(counter, out.numel())
    return D.to_like(out, nm.host_io)


def _pinv(g, counter):
    """kernel.pinv_dense (kernel.py:303-324): LAPACK SVD of the small d×d Gram on the host."""
    from .ml import _pinv_dense

    g = g.detach().cpu().numpy() if isinstance(g, torch.Tensor) else np.asarray(g, dtype=np.float64)
    return _pinv_dense(g, counter)


def ginv(nm, counter=None):
    """Moore-Penrose pseudo-inverse of the logical matrix (rewrite.py:318-333).

    Tall: ``pinv(TᵀT)·Tᵀ``; wide: ``Tᵀ·pinv(T Tᵀ)`` — the small Gram always.
    """
    from .rewrite import crossprod, lmm, rmm

    dv = nm.device_view()
    n_log, d_log = nm.shape
    if d_log < n_log:
        g = gram_transposed(dv, counter) if nm.transposed else crossprod(dv, counter=counter)
        p = torch.as_tensor(_pinv(g, counter), device=nm.device)
        out = rmm(p, dv.T, counter)
    else:
        g = crossprod(dv.T, counter=counter) if nm.transposed else gram_transposed(dv, counter)
        p = torch.as_tensor(_pinv(g, counter), device=nm.device)
        out = lmm(dv.T, p, counter)
    return D.to_like(out, nm.host_io)


# ---------------------------------------------------------------------------
# double matrix multiplication (both operands normalized, pkfk only)


def _require_pkfk(nm, side):
    if not isinstance(nm, NormalizedMatrix):
        raise TypeError(f"expected a NormalizedMatrix, got {type(nm).__name__}")
    if nm.variant != PKFK:
        raise ShapeError(f"double multiplication supports pkfk operands only ({side} is {nm.variant})")


def _tally_mm(counter, m, k, n):
    K.tally_matmul(counter, m, k, n)


def dmm(a, b, counter=None):
    """Product of two normalized matrices ``A B`` (rewrite.py:349-389).

    ``A'B'`` becomes ``(B A)'`` and single-transposed products go through :func:`dmm_gram`.
    B has d_A rows, so A·B is computed as one factorized LMM of A against B materialised
    (S_A·B[:d_S] + K_A·(R_A·B[d_S:]) on the fused gather kernel); the counter receives the
    reference's block-wise tallies.
    """
    _require_pkfk(a, "left operand")
    _require_pkfk(b, "right operand")
    host = a.host_io
    if a.transposed and b.transposed:
        return D.to_like(_as_dev(dmm(b.T.device_view(), a.T.device_view(), counter)).t().contiguous(), host)
    if a.transposed:
        return dmm_gram(a.T, b, "atb", counter)
    if b.transposed:
        return dmm_gram(a, b.T, "abt", counter)
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"dmm: shapes {a.shape} and {b.shape} do not conform")
    from .rewrite import lmm

    out = lmm(a.device_view(), materialize(b.device_view()))
    if counter is not None:
        n_a, d_sa = a.s.shape
        n_ra, d_ra = a.r.shape
        d_sb = b.s.shape[1]
        n_rb, d_rb = b.r.shape
        tb = b.k.target[:d_sa]
        _tally_mm(counter, n_a, d_sa, d_sb)  # S_A S_B1
        if b.shape[0] > d_sa:
            _tally_mm(counter, n_ra, d_ra, d_sb)  # R_A S_B2, expanded
            K.tally_accumulate(counter, n_a * d_sb)
        nk1 = tb.numel()
        if nk1:
            counter.tally(0, n_a * d_sa)  # right_compress(S_A, K_B1)
            _tally_mm(counter, n_a, n_rb, d_rb)
        if b.shape[0] > d_sa:
            counter.tally(0, n_ra * d_ra)  # right_compress(R_A, K_B2)
            _tally_mm(counter, n_ra, n_rb, d_rb)
            if nk1:
                K.tally_accumulate(counter, n_a * d_rb)
    return D.to_like(out, host)


def _as_dev(x):
    return x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x)).to(D.device())


def _compress(e, a):
    """Eᵀ a: scatter-add rows of a into the target buckets (indicator.py:107-118)."""
    out = torch.zeros((e.cols, a.shape[1]), dtype=torch.float64, device=a.device)
    return out.index_add_(0, e.target.to(torch.int64), a)


def dmm_gram(a, b, form, counter=None):
    """``A Bᵀ`` (form "abt") or ``Aᵀ B`` (form "atb") of two normalized matrices (rewrite.py:392-446)."""
    _require_pkfk(a, "left operand")
    _require_pkfk(b, "right operand")
    if a.transposed or b.transposed:
        raise ShapeError("dmm_gram operands carry no transpose flag; the form selects it")
    host = a.host_io
    s_a, k_a, r_a = a.s, a.k, a.r
    s_b, k_b, r_b = b.s, b.k, b.r
    d_sa, d_sb = s_a.shape[1], s_b.shape[1]
    if form == "atb":
        if a.shape[0] != b.shape[0]:
            raise ShapeError(f"dmm_gram A'B: row counts differ ({a.shape[0]} vs {b.shape[0]})")
        n = a.shape[0]
        p = pair_product(k_a, k_b, counter)  # E_Aᵀ E_B, sparse CSR on the device
        top_left = s_a.t() @ s_b
        _tally_mm(counter, d_sa, n, d_sb)
        cb = _compress(k_b, s_a)
        if counter is not None:
            counter.tally(0, n * d_sa)
        top_right = cb.t() @ r_b
        _tally_mm(counter, d_sa, k_b.cols, r_b.shape[1])
        ca = _compress(k_a, s_b)
        if counter is not None:
            counter.tally(0, n * d_sb)
        bot_left = r_a.t() @ ca
        _tally_mm(counter, r_a.shape[1], k_a.cols, d_sb)
        mid = torch.sparse.mm(p, r_b)
        if counter is not None:
            nnz = p._nnz()
            counter.tally(nnz * r_b.shape[1], max(nnz - k_a.cols, 0) * r_b.shape[1])
        bot_right = r_a.t() @ mid
        _tally_mm(counter, r_a.shape[1], k_a.cols, r_b.shape[1])
        out = torch.cat([torch.cat([top_left, top_right], 1), torch.cat([bot_left, bot_right], 1)], 0)
        return D.to_like(out.contiguous(), host)
    if form == "abt":
        if a.shape[1] != b.shape[1]:
            raise ShapeError(f"dmm_gram AB': column counts differ ({a.shape[1]} vs {b.shape[1]})")
        if d_sa > d_sb:
            out = _as_dev(dmm_gram(b.device_view(), a.device_view(), "abt", counter)).t().contiguous()
            return D.to_like(out, host)
        ta = k_a.target.to(torch.int64)
        tb = k_b.target.to(torch.int64)
        if d_sa == d_sb:
            out = s_a @ s_b.t()
            _tally_mm(counter, s_a.shape[0], d_sa, s_b.shape[0])
            mid = r_a @ r_b.t()
            _tally_mm(counter, r_a.shape[0], r_a.shape[1], r_b.shape[0])
            return D.to_like((out + mid.index_select(0, ta).index_select(1, tb)).contiguous(), host)
        cut = d_sb - d_sa  # S_B and R_A overlap on the middle columns
        s_b1, s_b2 = s_b[:, :d_sa], s_b[:, d_sa:]
        r_a1, r_a2 = r_a[:, :cut], r_a[:, cut:]
        out = s_a @ s_b1.t()
        _tally_mm(counter, s_a.shape[0], d_sa, s_b.shape[0])
        x = r_a1 @ s_b2.t()
        _tally_mm(counter, r_a.shape[0], cut, s_b.shape[0])
        out = out + x.index_select(0, ta)
        mid = r_a2 @ r_b.t()
        _tally_mm(counter, r_a.shape[0], r_a2.shape[1], r_b.shape[0])
        return D.to_like((out + mid.index_select(0, ta).index_select(1, tb)).contiguous(), host)
    raise ValueError(f"unknown dmm_gram form {form!r} (expected 'atb' or 'abt')")


def pair_product(ind_a, ind_b, counter=None):
    """``E_aᵀ E_b`` as a sparse counts matrix (indicator.py:144-162): a CSR tensor on the device."""
    if ind_a.rows != ind_b.rows:
        raise ShapeError(f"pair_product: row counts differ ({ind_a.rows} vs {ind_b.rows})")
    key = ind_a.target.to(torch.int64) * ind_b.cols + ind_b.target.to(torch.int64)
    uniq, cnt = torch.unique(key, sorted=True, return_counts=True)
    rows = uniq // ind_b.cols
    cols = uniq % ind_b.cols
    crow = torch.zeros(ind_a.cols + 1, dtype=torch.int64, device=key.device)
    crow[1:] = torch.cumsum(torch.bincount(rows, minlength=ind_a.cols), 0)
    if counter is not None:
        counter.tally(0, ind_a.rows)
    return torch.sparse_csr_tensor(crow, cols, cnt.to(torch.float64), size=(ind_a.cols, ind_b.cols))


# ---------------------------------------------------------------------------
# non-factorizable element-wise matrix operators

_ELEMENTWISE = {
    "add": lambda t, x: t + x,
    "sub": lambda t, x: t - x,
    "rsub": lambda t, x: x - t,
    "mul": lambda t, x: t * x,
    "div": lambda t, x: t / x,
    "rdiv": lambda t, x: x / t,
}


def elementwise_matrix_op(nm, x, op, counter=None):
    """Element-wise ``T <op> X`` with a full-size X: forces materialization (rewrite.py:449-470)."""
    if tuple(x.shape) != tuple(nm.shape):
        raise ShapeError(f"elementwise op: X shape {tuple(x.shape)} != logical shape {nm.shape}")
    warnings.warn(
        "element-wise matrix op is non-factorizable; materializing the join", MaterializationWarning, stacklevel=2
    )
    if op not in _ELEMENTWISE:
        raise ValueError(f"unknown elementwise op {op!r}")
    t = materialize(nm.device_view())
    out = _ELEMENTWISE[op](t, D.as_matrix(x))
    if counter is not None:
        size = int(out.numel())
        counter.tally(size, 0) if op in ("mul", "div", "rdiv") else counter.tally(0, size)
    return D.to_like(out.contiguous(), nm.host_io or D.is_host(x))

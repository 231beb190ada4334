"""Row-Gram, pseudo-inverse, double multiplication and non-factorizable element-wise ops.

The rest of the reference's operator surface (rewrite.py:301-470, indicator.py:144-162;
SURVEY §8(f) row 3), on the library's own sm_100a kernels (fb_dense.cu + the factorized
operators):

==========================  =====================================  ==========================
operator                    reference                              device composition
==========================  =====================================  ==========================
``gram_transposed``         rewrite.py:301-315                     per block F·Fᵀ (fb_dense_mm,
                                                                   DMMA) + two-sided row
                                                                   gather (fb_gather2_add)
``ginv``                    rewrite.py:318-333                     crossprod / gram_transposed,
                                                                   host SVD pinv of the small
                                                                   Gram, then rmm / lmm
``dmm``                     rewrite.py:349-389                     A·B = lmm(A, B materialised):
                                                                   B has only d_A rows
``dmm_gram``                rewrite.py:392-446                     block products (fb_dense_mm)
                                                                   + Eᵀa scatters
                                                                   (fb_scatter_rows), the pair
                                                                   counts · R (fb_csr_spmm)
``elementwise_matrix_op``   rewrite.py:449-470                     materialise + map (warns)
``pair_product``            indicator.py:144-162                   2-D target histogram: radix
                                                                   sort + run-length encode of
                                                                   the combined keys → CSR
                                                                   (fb_pair_counts)
==========================  =====================================  ==========================

These sit beside the hot path (their outputs are n×n or n×m dense, or they run once per
model). Nothing runs on the host except the reference's own LAPACK SVD of a d×d Gram;
``counter=`` gets the reference's tallies (counting rules kernel.py:7-18) step by step.
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


def _dmm(m, n, k, a, lda, ta, b, ldb, tb, c, ldc, accumulate=False, a_off=0, b_off=0, c_off=0):
    """C (+)= op(A)·op(B) on the FP64 tensor cores (fb_dense_mm); offsets in elements."""
    so = _lib.lib()
    if m == 0 or n == 0:
        return
    if k == 0:  # an empty contraction (a zero-width S): the product is the zero block
        if not accumulate:
            torch.as_strided(c.reshape(-1), (m, n), (ldc, 1), c_off).zero_()
        return
    _lib.check(so.fb_dense_mm(m, n, k, D.ptr(a) + 8 * a_off, lda, int(ta), D.ptr(b) + 8 * b_off, ldb, int(tb),
                              D.ptr(c) + 8 * c_off, ldc, int(accumulate), D.stream_handle()))


def _gather2_add(c, mat, ra, cb=None):
    """c += mat[ra][:, cb] (cb None: all columns) — fb_gather2_add."""
    so = _lib.lib()
    m, n = c.shape
    _lib.check(so.fb_gather2_add(m, n, D.ptr(mat), mat.shape[1], D.ptr(ra), D.ptr(cb) if cb is not None else 0,
                                 D.ptr(c), n, D.stream_handle()))


def gram_transposed(nm, counter=None):
    """``T Tᵀ`` (the Gram matrix over rows) per column block: E_i (F_i F_iᵀ) E_iᵀ (rewrite.py:301-315).

    Ignores the transpose flag, like the reference. The result is n × n and exactly
    symmetric; host operands give a NumPy result.
    """
    base = nm.untransposed()
    n = base.shape[0]
    out = None
    for e, f in base.blocks:
        f = f.contiguous()
        nf, d = f.shape
        _tally_gram(counter, nf, d)
        g = torch.empty((nf, nf), dtype=torch.float64, device=f.device)
        _dmm(nf, nf, d, f, d, False, f, d, True, g, nf)  # F·Fᵀ on the tensor cores
        g = _mirror(g)
        if e is None:
            if out is None:
                out = g
                continue
            out = out + g
        else:
            if out is None:
                out = torch.zeros((n, n), dtype=torch.float64, device=f.device)
                first = True
            else:
                first = False
            _gather2_add(out, g, e.target, e.target)  # out += g[t][:, t]
            if first:
                continue
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
    """Eᵀ a: scatter-add rows of a into the target buckets (indicator.py:107-118) — fb_scatter_rows."""
    so = _lib.lib()
    a = a.contiguous()
    out = torch.empty((e.cols, a.shape[1]), dtype=torch.float64, device=a.device)
    _lib.check(so.fb_scatter_rows(a.shape[0], a.shape[1], D.ptr(e.target), D.ptr(a), a.shape[1], D.ptr(out), e.cols,
                                  D.stream_handle()))
    return out


def _spmm(p, x):
    """P·x for the device CSR counts of :func:`pair_product` (fb_csr_spmm)."""
    so = _lib.lib()
    x = x.contiguous()
    rows = p.shape[0]
    y = torch.empty((rows, x.shape[1]), dtype=torch.float64, device=x.device)
    _lib.check(so.fb_csr_spmm(rows, D.ptr(p.crow_indices()), D.ptr(p.col_indices()), 1, D.ptr(p.values()), D.ptr(x),
                              x.shape[1], x.shape[1], D.ptr(y), x.shape[1], 0, D.stream_handle()))
    return y


def dmm_gram(a, b, form, counter=None):
    """``A Bᵀ`` (form "abt") or ``Aᵀ B`` (form "atb") of two normalized matrices (rewrite.py:392-446)."""
    _require_pkfk(a, "left operand")
    _require_pkfk(b, "right operand")
    if a.transposed or b.transposed:
        raise ShapeError("dmm_gram operands carry no transpose flag; the form selects it")
    host = a.host_io
    s_a, k_a, r_a = a.s.contiguous(), a.k, a.r.contiguous()
    s_b, k_b, r_b = b.s.contiguous(), b.k, b.r.contiguous()
    d_sa, d_sb = s_a.shape[1], s_b.shape[1]
    d_ra, d_rb = r_a.shape[1], r_b.shape[1]
    dev = s_a.device
    if form == "atb":
        if a.shape[0] != b.shape[0]:
            raise ShapeError(f"dmm_gram A'B: row counts differ ({a.shape[0]} vs {b.shape[0]})")
        n = a.shape[0]
        p = pair_product(k_a, k_b, counter)  # E_Aᵀ E_B, CSR counts on the device
        out = torch.empty((d_sa + d_ra, d_sb + d_rb), dtype=torch.float64, device=dev)
        ld = d_sb + d_rb
        _dmm(d_sa, d_sb, n, s_a, d_sa, True, s_b, d_sb, False, out, ld)  # top left: S_Aᵀ S_B
        _tally_mm(counter, d_sa, n, d_sb)
        cb = _compress(k_b, s_a)
        if counter is not None:
            counter.tally(0, n * d_sa)
        _dmm(d_sa, d_rb, k_b.cols, cb, d_sa, True, r_b, d_rb, False, out, ld, c_off=d_sb)  # (E_Bᵀ S_A)ᵀ R_B
        _tally_mm(counter, d_sa, k_b.cols, d_rb)
        ca = _compress(k_a, s_b)
        if counter is not None:
            counter.tally(0, n * d_sb)
        _dmm(d_ra, d_sb, k_a.cols, r_a, d_ra, True, ca, d_sb, False, out, ld, c_off=d_sa * ld)  # R_Aᵀ (E_Aᵀ S_B)
        _tally_mm(counter, d_ra, k_a.cols, d_sb)
        mid = _spmm(p, r_b)
        if counter is not None:
            nnz = p._nnz()
            counter.tally(nnz * d_rb, max(nnz - k_a.cols, 0) * d_rb)
        _dmm(d_ra, d_rb, k_a.cols, r_a, d_ra, True, mid, d_rb, False, out, ld, c_off=d_sa * ld + d_sb)
        _tally_mm(counter, d_ra, k_a.cols, d_rb)
        return D.to_like(out, host)
    if form == "abt":
        if a.shape[1] != b.shape[1]:
            raise ShapeError(f"dmm_gram AB': column counts differ ({a.shape[1]} vs {b.shape[1]})")
        if d_sa > d_sb:
            out = _as_dev(dmm_gram(b.device_view(), a.device_view(), "abt", counter)).t().contiguous()
            return D.to_like(out, host)
        n_a, n_b = s_a.shape[0], s_b.shape[0]
        n_ra, n_rb = r_a.shape[0], r_b.shape[0]
        out = torch.empty((n_a, n_b), dtype=torch.float64, device=dev)
        _dmm(n_a, n_b, d_sa, s_a, d_sa, False, s_b, d_sb, True, out, n_b)  # S_A S_B1ᵀ
        _tally_mm(counter, n_a, d_sa, n_b)
        cut = d_sb - d_sa  # S_B and R_A overlap on the middle columns
        if cut:
            x = torch.empty((n_ra, n_b), dtype=torch.float64, device=dev)
            _dmm(n_ra, n_b, cut, r_a, d_ra, False, s_b, d_sb, True, x, n_b, b_off=d_sa)  # R_A1 S_B2ᵀ
            _tally_mm(counter, n_ra, cut, n_b)
            _gather2_add(out, x, k_a.target)
        mid = torch.empty((n_ra, n_rb), dtype=torch.float64, device=dev)
        _dmm(n_ra, n_rb, d_ra - cut, r_a, d_ra, False, r_b, d_rb, True, mid, n_rb, a_off=cut)  # R_A2 R_Bᵀ
        _tally_mm(counter, n_ra, d_ra - cut, n_rb)
        _gather2_add(out, mid, k_a.target, k_b.target)
        return D.to_like(out, host)
    raise ValueError(f"unknown dmm_gram form {form!r} (expected 'atb' or 'abt')")


def pair_product(ind_a, ind_b, counter=None):
    """``E_aᵀ E_b`` as a sparse counts matrix (indicator.py:144-162): a CSR tensor on the device.

    The combined keys t_a·n_b + t_b are radix-sorted and run-length encoded on the device
    (fb_pair_counts); the CSR arrays are wrapped in a torch sparse tensor (a container).
    """
    if ind_a.rows != ind_b.rows:
        raise ShapeError(f"pair_product: row counts differ ({ind_a.rows} vs {ind_b.rows})")
    so = _lib.lib()
    n = ind_a.rows
    dev = ind_a.target.device
    indptr = torch.empty(ind_a.cols + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    val = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(so.fb_pair_counts_workspace_bytes(n), dtype=torch.uint8, device=dev)
    _lib.check(so.fb_pair_counts(n, D.ptr(ind_a.target), D.ptr(ind_b.target), ind_a.cols, ind_b.cols, D.ptr(indptr),
                                 D.ptr(col), D.ptr(val), D.ptr(nnz), ws.data_ptr(), ws.numel(), D.stream_handle()))
    if counter is not None:
        counter.tally(0, ind_a.rows)
    k = int(nnz.item())
    return torch.sparse_csr_tensor(indptr, col[:k].clone(), val[:k].clone(), size=(ind_a.cols, ind_b.cols))


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

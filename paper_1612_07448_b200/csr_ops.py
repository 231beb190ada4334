"""CSR-native factorized operators.

The reference keeps sparse factor matrices as scipy CSR (kernel.as_matrix, kernel.py:73-88)
and multiplies them through scipy's sparse-dense products (kernel.matmul, kernel.py:103-129).
A PK-FK / star matrix built here from a scipy factor at or below ``D.CSR_DENSITY_MAX``
density keeps that factor as a :class:`~._device.CsrMatrix` in HBM, and the operators below
read it natively — traffic proportional to nnz instead of the dense n × d:

* ``T·X`` (rewrite.py:172-191): per block F·X_F — ``fb_csr_spmm`` for a CSR factor (a warp
  per row, entries in stored order), ``fb_dense_mm`` (DMMA) for a dense one — the entity
  block written first, then each attribute block's z = R·X_R added through its indicator
  (``fb_gather2_add``: out += z[fk]), in the reference's block order;
* ``Tᵀ·W`` (RMM, ``lmm(T.T)``, rewrite.py:182-212): per block Fᵀ·W — the entity block
  directly, each attribute block as R_qᵀ (K_qᵀ W) with K_qᵀ W a keyed scatter
  (``fb_scatter_rows``) and the CSR transpose product ``fb_csr_spmm_t``;
* rowSums / colSums / sumAll (rewrite.py:118-165) as T·1, 1ᵀ·T and 1ᵀ·T·1.

Every other operator (crossprod, the fused drivers, element-wise maps, M:N) reads the dense
expansion the matrix makes once (``NormalizedMatrix.blocks``). The same block-by-block route
serves dense factors wider than the streaming kernels' 256 columns
(``NormalizedMatrix.block_path``). Op tallies follow the
reference's storage-aware rule for a sparse left operand (kernel.py:115-117: nnz·n
multiplies, (nnz − m)·n additions).
"""

import torch

from . import _device as D
from . import _lib
from . import kernel as K


def _tally_mm(counter, f, k):
    if counter is None:
        return
    if D.is_csr(f):
        counter.tally(f.nnz * k, max(f.nnz - f.shape[0], 0) * k)
    else:
        K.tally_matmul(counter, f.shape[0], f.shape[1], k)


def _mm_into(f, x, out, accumulate):
    """out (+)= F·x for a CSR or dense factor; x contiguous (F.cols × k), out (F.rows × k)."""
    so = _lib.lib()
    k = x.shape[1]
    if D.is_csr(f):
        _lib.check(so.fb_csr_spmm(f.shape[0], D.ptr(f.indptr), D.ptr(f.indices), 0, D.ptr(f.data), D.ptr(x), k, k,
                                  D.ptr(out), out.shape[1], int(accumulate), D.stream_handle()))
    else:
        _lib.check(so.fb_dense_mm(f.shape[0], k, f.shape[1], D.ptr(f), f.shape[1], 0, D.ptr(x), k, 0, D.ptr(out),
                                  out.shape[1], int(accumulate), D.stream_handle()))


def _tmm_into(f, w, out):
    """out = Fᵀ·w for a CSR or dense factor; w contiguous (F.rows × m), out (F.cols × m)."""
    so = _lib.lib()
    m = w.shape[1]
    if D.is_csr(f):
        _lib.check(so.fb_csr_spmm_t(f.shape[0], f.shape[1], D.ptr(f.indptr), D.ptr(f.indices), 0, D.ptr(f.data),
                                    D.ptr(w), m, m, D.ptr(out), out.shape[1], D.stream_handle()))
    else:
        _lib.check(so.fb_dense_mm(f.shape[1], m, f.shape[0], D.ptr(f), f.shape[1], 1, D.ptr(w), m, 0, D.ptr(out),
                                  out.shape[1], 0, D.stream_handle()))


def lmm(nm, x, counter=None):
    """T·X on the untransposed matrix; x a contiguous device matrix (d × d_x)."""
    so = _lib.lib()
    n, d_x = nm.base_rows, x.shape[1]
    offs = nm.col_offsets()
    out = torch.empty((n, d_x), dtype=torch.float64, device=x.device)
    started = False
    for i, (e, f) in enumerate(nm.raw_blocks):
        xs = x[offs[i]:offs[i + 1]].contiguous()
        _tally_mm(counter, f, d_x)
        if i > 0:
            K.tally_accumulate(counter, n * d_x)
        if e is None:
            _mm_into(f, xs, out, started)
        else:
            z = torch.empty((f.shape[0], d_x), dtype=torch.float64, device=x.device)
            _mm_into(f, xs, z, False)  # R·X before K (rewrite.py:187-189)
            if not started:
                out.zero_()
            _lib.check(so.fb_gather2_add(n, d_x, D.ptr(z), d_x, D.ptr(e.target), 0, D.ptr(out), d_x,
                                         D.stream_handle()))
        started = True
    return out


def tmm(nm, w, counter=None):
    """Tᵀ·W on the untransposed matrix; w a contiguous device matrix (n × m); out d × m."""
    so = _lib.lib()
    m = w.shape[1]
    offs = nm.col_offsets()
    out = torch.empty((nm.base_cols, m), dtype=torch.float64, device=w.device)
    for i, (e, f) in enumerate(nm.raw_blocks):
        blk = out[offs[i]:offs[i + 1]]
        if e is None:
            _tmm_into(f, w, blk)
        else:
            bins = torch.empty((f.shape[0], m), dtype=torch.float64, device=w.device)
            _lib.check(so.fb_scatter_rows(w.shape[0], m, D.ptr(e.target), D.ptr(w), m, D.ptr(bins), f.shape[0],
                                          D.stream_handle()))  # K_qᵀ W
            if counter is not None:
                counter.tally(0, m * e.rows)
            _tmm_into(f, bins, blk)  # R_qᵀ (K_qᵀ W)
        _tally_mm(counter, f, m)
    return out


def ones(n, device):
    return torch.ones((n, 1), dtype=torch.float64, device=device)


def sum_all(nm):
    """1ᵀ·T·1 as a device scalar: the column totals dotted with ones (fb_dense_mm)."""
    so = _lib.lib()
    cs = tmm(nm, ones(nm.base_rows, nm.device))  # d × 1
    one = ones(cs.shape[0], cs.device)
    out = torch.empty((1, 1), dtype=torch.float64, device=cs.device)
    _lib.check(so.fb_dense_mm(1, 1, cs.shape[0], D.ptr(one), 1, 1, D.ptr(cs), 1, 0, D.ptr(out), 1, 0,
                              D.stream_handle()))
    return out

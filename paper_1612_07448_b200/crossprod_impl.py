"""Factorized crossprod ``T' T`` (rewrite.py:245-298) on the FP64 tensor cores.

PK-FK (q = 1) and plain (q = 0) matrices run the two-pass DMMA kernels of
``fb_crossprod.cu``: one pass over S in FK-sorted order (SᵀS tiles + the segmented
KᵀS), one over R (Rᵀdiag(c)R + Rᵀ(KᵀS)). The FK-sorted permutation is the device
analogue of the reference's cached ``_csr_t`` (indicator.py:78-86) and is cached on the
indicator the same way.

Star schemas (q >= 2) are assembled block-column by block-column: block column b of
TᵀT is (T_bᵀ T)ᵀ, computed by the weighted transposed product kernel with the
(gathered) column block T_b as weights; the upper triangle is then mirrored exactly.
"""

import torch

from . import _device as D
from . import _lib
from . import kernel as K
from .exceptions import ShapeError
from .normmat import NormalizedMatrix

__all__ = ["crossprod", "fk_sorted_order"]


def fk_sorted_order(ind):
    """(perm, fk_sorted) of an indicator: rows in ascending (target, row) order; cached."""
    return ind.sorted_order()


def _tally(nm, counter):
    """Multiply/add counts of the reference's efficient crossprod (rewrite.py:263-298)."""
    if counter is None:
        return
    blocks = nm.blocks
    for i, (e_i, f_i) in enumerate(blocks):
        n, d = f_i.shape
        if e_i is not None:
            counter.tally(n * d, 0)  # _scale_rows (rewrite.py:215-225)
        K.tally_crossprod(counter, n, d)
        for j in range(i + 1, len(blocks)):
            e_j, f_j = blocks[j]
            if e_i is None:
                counter.tally(0, f_i.shape[0] * f_i.shape[1])  # compress (indicator.py:107-118)
                K.tally_matmul(counter, f_i.shape[1], f_j.shape[0], f_j.shape[1])
            else:
                counter.tally(0, e_i.rows)  # pair_product (indicator.py:144-162)
                key = e_i.target.to(torch.int64) * e_j.cols + e_j.target.to(torch.int64)
                nnz = int(torch.unique(key).numel())
                m, dj = f_i.shape[0], f_j.shape[1]
                counter.tally(nnz * dj, max(nnz - m, 0) * dj)
                K.tally_matmul(counter, f_i.shape[1], f_i.shape[0], dj)


def crossprod(nm, method="efficient", counter=None):
    """``T' T`` without materializing T; exactly symmetric (rewrite.py:245-298).

    Both the "efficient" and the benchmark-only "naive" method names are accepted and
    run the same device kernels; ``counter`` is filled with the efficient method's
    analytic counts.
    """
    if not isinstance(nm, NormalizedMatrix):
        raise TypeError(f"expected a NormalizedMatrix, got {type(nm).__name__}")
    if nm.transposed:
        raise ShapeError("crossprod expects an untransposed input; use gram_transposed")
    if method not in ("efficient", "naive"):
        raise ValueError(f"unknown crossprod method {method!r}")
    so = _lib.lib()
    st = D.stream_handle()
    d = nm.base_cols
    dev = nm.device
    out = torch.empty((d, d), dtype=torch.float64, device=dev)
    q = len(nm.blocks) - 1
    cs = nm.c_struct()
    if nm.blocks[0][0] is not None:
        _star_crossprod(nm, out, so, st)  # M:N: every block gathered (the fused passes need S = block 0)
    elif q == 1 and nm.blocks[0][1].shape[1] > 128:
        _star_crossprod(nm, out, so, st)  # the fused segmented KᵀS covers d_S <= 128
    elif q <= 1:
        perm = fks = None
        if q == 1:
            perm, fks = fk_sorted_order(nm.blocks[1][0])
        ws = D.workspace(so.fb_crossprod_workspace_bytes(cs))
        _lib.check(so.fb_crossprod(cs, D.ptr(perm), D.ptr(fks), D.ptr(out), ws.data_ptr(), ws.numel(), st))
    else:
        _star_crossprod(nm, out, so, st)
    _tally(nm, counter)
    return D.to_like(out, nm.host_io)


def _star_crossprod(nm, out, so, st):
    nm.ensure_sorted()
    n = nm.base_rows
    d = nm.base_cols
    offs = nm.col_offsets()
    cs = nm.c_struct()
    for b, (e, f) in enumerate(nm.blocks):
        c0, c1 = int(offs[b]), int(offs[b + 1])
        if c1 == c0:
            continue
        if e is None:
            w = f
        else:
            w = torch.empty((n, c1 - c0), dtype=torch.float64, device=f.device)
            _lib.check(so.fb_gather_rows_i32(D.ptr(f), f.shape[1], D.ptr(e.target), n, c1 - c0, D.ptr(w), c1 - c0, st))
        # rows c0:c1 of TᵀT = T_bᵀ T: out(j, c) = Σ_i w(i, j) T(i, c)
        nw = c1 - c0
        wsz = D.workspace(so.fb_wt_workspace_bytes(cs, nw))
        _lib.check(so.fb_wt(cs, D.ptr(w), nw, nw, 1, out.data_ptr() + 8 * c0 * d, d, 1, wsz.data_ptr(), wsz.numel(),
                            st))
    _lib.check(so.fb_mirror_upper(D.ptr(out), d, st))

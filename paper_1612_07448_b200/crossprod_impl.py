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
        # M:N / multi-table M:N: every block keyed — the same plan with a zero-width S
        # (R_iᵀ diag(c_i) R_i per table, pair-count cross blocks)
        _star_crossprod_fused(nm, out, so, st) if nm.base_rows > 0 else _star_crossprod(nm, out, so, st)
    elif q == 1 and nm.blocks[0][1].shape[1] > 128:
        _star_crossprod(nm, out, so, st)  # the fused segmented KᵀS covers d_S <= 128
    elif q <= 1:
        perm = fks = None
        if q == 1:
            perm, fks = fk_sorted_order(nm.blocks[1][0])
        ws = D.workspace(so.fb_crossprod_workspace_bytes(cs))
        try:
            _lib.check(so.fb_crossprod(cs, D.ptr(perm), D.ptr(fks), D.ptr(out), ws.data_ptr(), ws.numel(), st))
        except ValueError as e:
            # a shape the two-pass kernels' job tables cannot hold (e.g. d_S = 125 beside a 250-wide R:
            # more than 256 block tiles in the R pass): the block-column path, exact but slower
            if q != 1 or "unsupported size" not in str(e):
                raise
            _star_crossprod(nm, out, so, st)
    elif nm.blocks[0][1].shape[1] <= 128 and nm.base_rows > 0:
        # odd d_S included: fb_crossprod then runs its unfused S pass (SᵀS in storage order + the
        # segmented KᵀS walk) per part, still far from the block-column path's cost
        try:
            _star_crossprod_fused(nm, out, so, st)
        except ValueError as e:
            if "unsupported size" not in str(e):
                raise
            _star_crossprod(nm, out, so, st)
    else:
        _star_crossprod(nm, out, so, st)
    _tally(nm, counter)
    return D.to_like(out, nm.host_io)


def _chunk_width(rem):
    """Widest column chunk <= rem the weighted column reduction is instantiated for (fb_capi.cu chunk_width)."""
    if rem >= 16:
        return 16
    if rem in (12, 10) or rem <= 8:
        return rem
    return next(w for w in (12, 10, 8) if w <= rem)


def _star_crossprod_fused(nm, out, so, st):
    """Star schema (q >= 2) on the fused two-pass kernels, the reference's efficient plan
    (rewrite.py:263-298) block by block:

    * per part i, ``fb_crossprod`` of the PK-FK sub-matrix [S, K_i R_i] gives SᵀS, Sᵀ(K_i R_i) =
      (K_iᵀS)ᵀR_i and R_iᵀ diag(c_i) R_i (one fused pass over S in FK_i-sorted order + one pass
      over R_i; SᵀS is recomputed per part on the tensor cores and taken from the first);
    * per pair i < j, the cross block R_iᵀ (K_iᵀK_j) R_j through the pair counts
      (indicator.py:144-162): ``fb_pair_counts`` → CSR P, M = P·R_j (``fb_csr_spmm``), R_iᵀ·M
      (``fb_dense_mm``);
    * the lower triangle is the exact mirror of the upper.
    """
    import ctypes

    nm.ensure_sorted()
    nm.c_struct()
    full = nm._cache["c_struct"]
    d = nm.base_cols
    dev = nm.device
    offs = [int(o) for o in nm.col_offsets()]
    parts = nm.indicator_blocks
    d_s = int(full.d_s)  # 0 for M:N matrices (every block is a keyed part)
    if nm.blocks[0][0] is None:
        offs = offs[1:]  # offs[i] = first column of part i
    n = nm.base_rows
    out.zero_()
    for i, (e, f) in enumerate(parts):
        sub = _lib.FbNormalized()
        sub.s, sub.n_s, sub.d_s, sub.q = full.s, full.n_s, full.d_s, 1
        sub.part[0] = full.part[i]
        di = f.shape[1]
        g = torch.empty((d_s + di, d_s + di), dtype=torch.float64, device=dev)
        perm, fks = fk_sorted_order(e)
        ws = D.workspace(so.fb_crossprod_workspace_bytes(ctypes.byref(sub)))
        _lib.check(so.fb_crossprod(ctypes.byref(sub), D.ptr(perm), D.ptr(fks), D.ptr(g), ws.data_ptr(), ws.numel(), st))
        c0 = offs[i]
        if i == 0 and d_s:
            out[:d_s, :d_s] = g[:d_s, :d_s]
        if d_s:
            out[:d_s, c0:c0 + di] = g[:d_s, d_s:]
        out[c0:c0 + di, c0:c0 + di] = g[d_s:, d_s:]
    for i, (ei, fi) in enumerate(parts):
        for j in range(i + 1, len(parts)):
            ej, fj = parts[j]
            # P = K_aᵀK_b, M = P·R_b, block = R_aᵀ·M with a the smaller table: fewer, longer CSR rows for
            # the warp-per-row SpMM and a short column reduction (c4: 6.2 ms; with a the larger
            # table — gathers from the L2-resident small one, but 1M short rows — 10.8 ms)
            flip = fj.shape[0] < fi.shape[0]
            (ea, fa), (eb, fb_) = ((ej, fj), (ei, fi)) if flip else ((ei, fi), (ej, fj))
            da, db = fa.shape[1], fb_.shape[1]
            indptr = torch.empty(ea.cols + 1, dtype=torch.int64, device=dev)
            col = torch.empty(n, dtype=torch.int64, device=dev)
            val = torch.empty(n, dtype=torch.float64, device=dev)
            nnz = torch.zeros(1, dtype=torch.int64, device=dev)
            ws = D.workspace(so.fb_pair_counts_workspace_bytes(n))
            _lib.check(so.fb_pair_counts(n, D.ptr(ea.target), D.ptr(eb.target), ea.cols, eb.cols, D.ptr(indptr),
                                         D.ptr(col), D.ptr(val), D.ptr(nnz), ws.data_ptr(), ws.numel(), st))
            # column chunks of R_b in the widths the column reduction is instantiated for: each chunk's
            # M = P·R_b[:, c0:c0+w] is its own contiguous n_a × w matrix, so the reduction streams its
            # weights row-aligned with R_a (interleaved mode) instead of reading them strided
            base = out.data_ptr() + 8 * (offs[i] * d + offs[j])
            o_js, o_cs = (d, 1) if flip else (1, d)
            c0 = 0
            while c0 < db:
                w = _chunk_width(db - c0)
                m = torch.empty((ea.cols, w), dtype=torch.float64, device=dev)
                _lib.check(so.fb_csr_spmm(ea.cols, D.ptr(indptr), D.ptr(col), 1, D.ptr(val), fb_.data_ptr() + 8 * c0, db, w,
                                          D.ptr(m), w, 0, st))
                # out[off_i + c_i, off_j + c_j]: fb_rows_wt writes (weight column, table column) through strides
                ws = D.workspace(so.fb_rows_wt_workspace_bytes(da, w))
                _lib.check(so.fb_rows_wt(D.ptr(fa), ea.cols, da, D.ptr(m), w, w, 1, base + 8 * c0 * o_js, o_js, o_cs,
                                         ws.data_ptr(), ws.numel(), st))
                c0 += w
    _lib.check(so.fb_mirror_upper(D.ptr(out), d, st))


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

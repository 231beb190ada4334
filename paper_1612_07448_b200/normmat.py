"""The normalized matrix on a B200: base-table factors resident in HBM.

Mirrors ``factorla.normmat`` (normmat.py:1-375) for the PK-FK, star, M:N and multi-table
M:N variants:
``NormalizedMatrix`` keeps column blocks ``(indicator | None, factor)``, a logical
transpose flag, and the kept source rows of every attribute table. The factors are
float64 CUDA tensors (row-major, as the reference's C-contiguous arrays) and each
indicator is an int32 FK column on the device. Construction (key validation, the
unreferenced-row drop and remap) runs in the library's kernels (fb_build.cu).

HBM layout per matrix: S (n_S × d_S f64), per part: FK (n_S int32), R_kept
(n_R' × d_R f64), counts (n_R' f64, cached), plus lazily built caches (the FK-sorted
permutation used by the segmented reductions).

M:N (normmat.py:240-285) and multi-table M:N (normmat.py:288-319) matrices have an
indicator on every block, S included: T = [I_S·S, I_R·R]. The kernels see them as a
zero-width entity table plus one attribute part per block (``fb_normalized`` with
d_s = 0), so every operator and driver runs unchanged on the same gathers/scatters.
"""

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib
from .exceptions import DataError, EmptyJoinError, ShapeError

__all__ = [
    "IndicatorMatrix",
    "NormalizedMatrix",
    "ShapeStats",
    "build_pkfk",
    "build_star",
    "build_mn",
    "build_multimn",
    "materialize",
    "transpose",
    "stats",
]

PKFK = "pkfk"
STAR = "star"
MN = "mn"
MULTIMN = "multimn"
DENSE = "dense"  # a regular matrix viewed as T = [S] (q = 0); used by the ML drivers


class IndicatorMatrix:
    """K stored as ``target[i] = j`` (indicator.py:27-95), int32 on the device."""

    def __init__(self, target, cols, counts_i32=None):
        if not (isinstance(target, torch.Tensor) and target.is_cuda and target.dtype == torch.int32):
            raise ShapeError("indicator target must be an int32 CUDA tensor")
        if target.dim() != 1:
            raise ShapeError("indicator target must be a 1-D index array")
        if target.numel() == 0:
            raise ShapeError("indicator matrix must have at least one row")
        cols = int(cols)
        if cols < 1:
            raise ShapeError("indicator matrix must have at least one column")
        self.target = target.contiguous()
        self.cols = cols
        self._counts_i32 = counts_i32
        self._counts = None

    @property
    def rows(self):
        return self.target.numel()

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def nnz(self):
        return self.rows

    @property
    def counts_i32(self):
        """bincount of the targets (indicator.py:61-66), exact int32."""
        if self._counts_i32 is None:
            so = _lib.lib()
            c = torch.empty(self.cols, dtype=torch.int32, device=self.target.device)
            _lib.check(so.fb_fk_counts(D.ptr(self.target), self.rows, D.ptr(c), self.cols, D.stream_handle()))
            self._counts_i32 = c
        return self._counts_i32

    @property
    def counts(self):
        """Column sums of K as float64 (the reference's ``counts``), cached."""
        if self._counts is None:
            so = _lib.lib()
            ci = self.counts_i32
            c = torch.empty(self.cols, dtype=torch.float64, device=ci.device)
            _lib.check(so.fb_i32_to_f64(D.ptr(ci), D.ptr(c), self.cols, D.stream_handle()))
            self._counts = c
        return self._counts

    @property
    def max_count(self):
        """Largest group size (cached; one device->host read)."""
        if getattr(self, "_max_count", None) is None:
            self._max_count = int(self.counts_i32.max().item())
        return self._max_count

    @property
    def skewed(self):
        """True when one target holds more than 1/256 of the rows (Zipf-like keys)."""
        return self.max_count * 256 > self.rows

    def hot_tables(self, nhot=64):
        """(hot_slot int16[cols], hot_key int32[k], k) for skewed targets, cached.

        The k <= nhot most frequent targets holding more than 1/4096 of the rows each get a
        slot; scatter kernels keep their bins in per-warp shared memory instead of hammering
        one L2 line with atomics (Zipf keys: the top target holds ~20% of the rows).
        """
        if getattr(self, "_hot", None) is None:
            if not self.skewed:
                self._hot = (None, None, 0)
            else:
                cnt = self.counts_i32
                k = min(nhot, self.cols)
                vals, keys = torch.topk(cnt, k)
                keep = vals.to(torch.int64) * 4096 > self.rows
                keys = keys[keep].to(torch.int32).contiguous()
                slot = torch.full((self.cols,), -1, dtype=torch.int16, device=cnt.device)
                slot[keys.to(torch.int64)] = torch.arange(keys.numel(), dtype=torch.int16, device=cnt.device)
                self._hot = (slot, keys, int(keys.numel()))
        return self._hot

    def sorted_order(self):
        """(perm, fk_sorted): rows in ascending (target, row) order, cached.

        The device analogue of the reference's cached ``_csr_t`` stable argsort
        (indicator.py:78-86), built once by a stable radix sort (fb_fk_sort).
        """
        if getattr(self, "_sorted", None) is None:
            so = _lib.lib()
            n = self.rows
            perm = torch.empty(n, dtype=torch.int32, device=self.target.device)
            fks = torch.empty(n, dtype=torch.int32, device=self.target.device)
            ws = D.workspace(so.fb_fk_sort_workspace_bytes(n))
            _lib.check(so.fb_fk_sort(D.ptr(self.target), n, self.cols, D.ptr(perm), D.ptr(fks), ws.data_ptr(),
                                     ws.numel(), D.stream_handle()))
            self._sorted = (perm, fks)
        return self._sorted

    def all_columns_used(self):
        return bool((self.counts_i32 > 0).all().item())

    def target_numpy(self):
        return self.target.cpu().numpy().astype(np.int64)

    def __repr__(self):
        return f"IndicatorMatrix(rows={self.rows}, cols={self.cols}, device)"


class NormalizedMatrix:
    """Immutable multi-matrix value (normmat.py:47-130); build with ``build_*``."""

    def __init__(self, variant, blocks, transposed=False, source_rows=None, host_io=False):
        blocks = tuple((e, f) for e, f in blocks)
        if not blocks:
            raise ShapeError("normalized matrix needs at least one block")
        rows = {e.rows if e is not None else f.shape[0] for e, f in blocks}
        if len(rows) != 1:
            raise ShapeError(f"blocks disagree on logical row count: {sorted(rows)}")
        for e, f in blocks:
            if e is not None and e.cols != f.shape[0]:
                raise ShapeError(f"indicator cols {e.cols} != factor rows {f.shape[0]}")
        if blocks[0][0] is not None and any(e is None for e, _ in blocks):
            raise ShapeError("either only the first block (the entity table) or every block has no indicator")
        if len(blocks) - (1 if blocks[0][0] is None else 0) > _lib.FB_MAX_PARTS:
            raise ShapeError(f"at most {_lib.FB_MAX_PARTS} indicator blocks are supported")
        self.variant = variant
        self._raw = blocks  # factors as given: dense CUDA tensors or D.CsrMatrix
        self.transposed = bool(transposed)
        self.source_rows = tuple(source_rows) if source_rows is not None else None
        self.host_io = bool(host_io)
        self._cache = {}  # per-matrix device caches shared with the transposed view

    # -- factors ----------------------------------------------------------
    @property
    def blocks(self):
        """(indicator, dense factor) pairs. CSR factors (D.CsrMatrix) are expanded here, once
        per matrix (the operators with CSR-native kernels read :attr:`raw_blocks` instead)."""
        if not self.has_csr:
            return self._raw
        b = self._cache.get("dense_blocks")
        if b is None:
            b = tuple((e, D.dense_of(f)) for e, f in self._raw)
            self._cache["dense_blocks"] = b
        return b

    @property
    def raw_blocks(self):
        return self._raw

    @property
    def has_csr(self):
        return any(D.is_csr(f) for _, f in self._raw)

    # widest factor the streaming kernels take (a factor row is staged in shared memory)
    MAX_RING_WIDTH = 256

    @property
    def block_path(self):
        """LMM / Tᵀ·X / row and column sums go block by block (csr_ops: CSR SpMM, DMMA block
        products, keyed gathers / scatters) instead of through the fused streaming kernels:
        CSR factors, or a factor wider than the streaming kernels' 256 columns."""
        return self.has_csr or max(f.shape[1] for _, f in self._raw) > self.MAX_RING_WIDTH

    # -- shape ------------------------------------------------------------
    @property
    def base_rows(self):
        e, f = self._raw[0]
        return e.rows if e is not None else f.shape[0]

    @property
    def device(self):
        return self._raw[0][1].device

    @property
    def indicator_blocks(self):
        """The blocks the kernels see as attribute parts (all blocks of an M:N matrix)."""
        return self.blocks[1:] if self.blocks[0][0] is None else self.blocks

    @property
    def base_cols(self):
        return sum(f.shape[1] for _, f in self._raw)

    @property
    def shape(self):
        n, d = self.base_rows, self.base_cols
        return (d, n) if self.transposed else (n, d)

    def col_offsets(self):
        widths = [f.shape[1] for _, f in self._raw]
        return np.concatenate([[0], np.cumsum(widths)]).astype(int)

    # -- accessors ---------------------------------------------------------
    @property
    def s(self):
        if self.variant == MULTIMN:
            raise ShapeError(f"{self.variant} variant has no entity block")
        return self.blocks[0][1]

    @property
    def k(self):
        if self.variant != PKFK:
            raise ShapeError("k accessor is pkfk-only")
        return self.blocks[1][0]

    @property
    def r(self):
        if self.variant not in (PKFK, MN):
            raise ShapeError("r accessor applies to single-attribute variants")
        return self.blocks[1][1]

    @property
    def parts(self):
        return self.blocks[1:]

    # -- logical ops -------------------------------------------------------
    @property
    def T(self):
        t = NormalizedMatrix(self.variant, self._raw, not self.transposed, self.source_rows, self.host_io)
        t._cache = self._cache
        return t

    def device_view(self):
        """The same matrix with results returned as CUDA tensors (shares the caches)."""
        if not self.host_io:
            return self
        v = NormalizedMatrix(self.variant, self._raw, self.transposed, self.source_rows, False)
        v._cache = self._cache
        return v

    def untransposed(self):
        return self if not self.transposed else self.T

    def with_factors(self, factors):
        """Same indicators / flag, new factor matrices (closure of scalar ops)."""
        blocks = [(e, f) for (e, _), f in zip(self.blocks, factors)]
        return NormalizedMatrix(self.variant, blocks, self.transposed, self.source_rows, self.host_io)

    # -- C ABI view ----------------------------------------------------------
    def c_struct(self):
        """``fb_normalized`` describing the untransposed factors (cached)."""
        st = self._cache.get("c_struct")
        if st is None:
            st = _lib.FbNormalized()
            if self.blocks[0][0] is None:
                s = self.blocks[0][1]
                st.s = D.ptr(s)
                st.n_s = s.shape[0]
                st.d_s = s.shape[1]
            else:  # M:N: a zero-width entity table, every block an attribute part
                st.s = 0
                st.n_s = self.base_rows
                st.d_s = 0
            parts = self.indicator_blocks
            st.q = len(parts)
            for i, (e, f) in enumerate(parts):
                p = st.part[i]
                p.fk = D.ptr(e.target)
                p.r = D.ptr(f)
                p.n_r = f.shape[0]
                p.d_r = f.shape[1]
                p.skewed = int(e.skewed)
                p.counts = D.ptr(e.counts)
                hs, hk, nh = e.hot_tables()
                p.hot_slot, p.hot_key, p.nhot = D.ptr(hs), D.ptr(hk), nh
                srt = getattr(e, "_sorted", None)
                if srt is not None:
                    p.perm, p.fk_sorted = D.ptr(srt[0]), D.ptr(srt[1])
            self._cache["c_struct"] = st
        return ctypes.byref(st)

    def ensure_sorted(self):
        """Build (once) the FK-sorted order of every indicator and expose it to the kernels."""
        st = self._cache.get("c_struct")
        for i, (e, _) in enumerate(self.indicator_blocks):
            perm, fks = e.sorted_order()
            if st is not None:
                st.part[i].perm, st.part[i].fk_sorted = D.ptr(perm), D.ptr(fks)

    # FK-band layout (fb_band_layout): a cached copy of S and the FK columns grouped into key bands
    # of part 0, so a pass over S gathers z_0 = R_0·X from one L2-resident slice at a time. Both
    # users are OFF by default — measured on B200 (profiles/r02_lmm16_experiments.txt) the layout
    # removes the z misses but not the time:
    # * wide-X LMM (FB_LMM_BAND_MIN_MB=<MB> enables): at c2 X100x16 the S pass's DRAM traffic drops
    #   7.6 -> 6.1 GB, but the permuted 128-byte output rows cost the DRAM what the z misses did
    #   (op 1.45 -> 1.42 ms; 1.12 ms with the same rows stored in band order);
    # * fused K-Means pass (FB_KMEANS_BAND_MIN_MB=<MB> enables; nothing is stored in permuted order
    #   inside the loop, the build takes 1.4 ms at c4): 1.077 vs 1.070 ms per c4 iteration — the
    #   pass is bound by its consumers' per-tile chain (argmin, histogram REDs, one-hot DMMAs), not
    #   by the gathers.
    BAND_MIN_BYTES = int(float(os.environ.get("FB_LMM_BAND_MIN_MB", "0")) * (1 << 20))
    BAND_KMEANS_MIN_BYTES = int(float(os.environ.get("FB_KMEANS_BAND_MIN_MB", "0")) * (1 << 20))
    BAND_BYTES = int(float(os.environ.get("FB_LMM_BAND_MB", "16")) * (1 << 20))

    def _band(self):
        """(struct, perm, fk_band, s_band) of this matrix, built once (bands sized for 128-byte z rows)."""
        band = self._cache.get("band")
        if band is None:
            so = _lib.lib()
            s = self.blocks[0][1]
            parts = self.indicator_blocks
            n = s.shape[0]
            zbytes = parts[0][1].shape[0] * 128
            n_bands = max(2, min(4096, -(-zbytes // max(1, self.BAND_BYTES))))
            perm = torch.empty(n, dtype=torch.int32, device=s.device)
            fkb = torch.empty((len(parts), so.fb_band_fk_stride(n)), dtype=torch.int32, device=s.device)
            sb = torch.empty_like(s)
            ws = D.workspace(so.fb_band_build_workspace_bytes(n))
            _lib.check(so.fb_band_build(self.c_struct(), n_bands, D.ptr(perm), D.ptr(fkb), D.ptr(sb),
                                        ws.data_ptr(), ws.numel(), D.stream_handle()))
            st = _lib.FbBandLayout()
            st.n_bands, st.perm, st.s = n_bands, D.ptr(perm), D.ptr(sb)
            for q in range(len(parts)):
                st.fk[q] = D.ptr(fkb[q])
            band = (st, perm, fkb[:, :n], sb)
            self._cache["band"] = band
        return band

    def _bandable(self):
        if self.variant not in (PKFK, STAR) or self.transposed or self.has_csr or self.blocks[0][0] is not None:
            return False
        s = self.blocks[0][1]
        return len(self.indicator_blocks) >= 1 and 1 <= s.shape[1] <= 32 and s.shape[0] > 0

    def band_layout(self, d_x):
        """``fb_band_layout`` for a wide-X LMM, or None when the pass should stay in storage order.

        PK-FK matrices with d_S <= 32 whose z = R·X table (n_R × 16 doubles) exceeds
        ``BAND_MIN_BYTES`` (0 = never), for X widths the band body covers (multiples of 8).
        Costs one extra copy of S and of the FK column in HBM.
        """
        if not self._bandable() or len(self.indicator_blocks) != 1 or not self.BAND_MIN_BYTES:
            return None
        if d_x < 8 or d_x % 8 or self.indicator_blocks[0][1].shape[0] * 128 < self.BAND_MIN_BYTES:
            return None
        return ctypes.byref(self._band()[0])

    def kmeans_band_layout(self, k):
        """The band layout for the fused K-Means pass (k <= 16), or None.

        Used when part 0's z table (n_R × even(k) doubles) exceeds ``BAND_KMEANS_MIN_BYTES`` and is
        the largest of the parts (the bands follow part 0's keys).
        """
        if not self._bandable() or not self.BAND_KMEANS_MIN_BYTES or k > 16:
            return None
        rows = [f.shape[0] for _, f in self.indicator_blocks]
        zrow = 8 * max(2, (k + 1) & ~1)
        if rows[0] != max(rows) or rows[0] * zrow < self.BAND_KMEANS_MIN_BYTES:
            return None
        if not _lib.lib().fb_kmeans_banded_supported(self.c_struct(), k):
            return None
        return self._band()

    def __repr__(self):
        n, d = self.shape
        flag = ", transposed" if self.transposed else ""
        return f"NormalizedMatrix({self.variant}, {n}x{d}{flag}, device)"


def transpose(nm):
    """Flip the logical-transpose flag; no data is copied (normmat.py:118-122)."""
    return nm.T


def as_normalized(m):
    """View a regular matrix as T = [S] (q = 0) so the drivers run on the same kernels."""
    if isinstance(m, NormalizedMatrix):
        return m
    return NormalizedMatrix(DENSE, [(None, D.as_matrix(m))], host_io=D.is_host(m))


def materialize(nm):
    """Expand T = [S, K_1 R_1, ...] on the device (normmat.py:138-161).

    Gathers every attribute block with the library's row-gather kernel; honours the
    transpose flag. Intended for tests and small inputs — the operators never call it.
    """
    so = _lib.lib()
    n, d = nm.base_rows, nm.base_cols
    out = torch.empty((n, d), dtype=torch.float64, device=nm.device)
    offs = nm.col_offsets()
    st = D.stream_handle()
    for (e, f), c0, c1 in zip(nm.blocks, offs[:-1], offs[1:]):
        if c1 == c0:
            continue
        if e is None:
            out[:, c0:c1] = f
        else:
            _lib.check(so.fb_gather_rows_i32(D.ptr(f), f.shape[1], D.ptr(e.target), n, c1 - c0,
                                             out.data_ptr() + 8 * int(c0), d, st))
    out = out.t().contiguous() if nm.transposed else out
    return D.to_like(out, nm.host_io)


# ---------------------------------------------------------------------------
# construction


def _check_keys(key, n_rows, part_label=""):
    """1-based key validation (normmat.py:182-198) -> int64 device tensor."""
    k = D.as_vector_i64(key)
    if not (k.dtype in (torch.int8, torch.int16, torch.int32, torch.int64, torch.uint8)):
        kf = k.to(torch.float64)
        if not bool(torch.all(kf == torch.round(kf)).item()):
            raise DataError(f"key column{part_label} contains non-integer values")
        k = kf.to(torch.int64)
    return k.to(torch.int64).contiguous()


def _remap_part(key, r, part_label=""):
    """Validate keys, drop unreferenced rows of r, remap to 0-based (normmat.py:168-179).

    Returns (indicator, r_kept, used) with ``used`` the kept 0-based source rows (int64).
    """
    so = _lib.lib()
    st = D.stream_handle()
    n_r = r.shape[0]
    n = key.numel()
    dev = r.device
    counts_full = torch.empty(max(n_r, 1), dtype=torch.int32, device=dev)
    first_bad = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.check(so.fb_key_check(D.ptr(key), n, n_r, counts_full.data_ptr(), first_bad.data_ptr(), st))
    bad = int(first_bad.item())
    if bad != -1:  # UINT64_MAX reads back as -1
        raise DataError(
            f"key{part_label} references nonexistent attribute row "
            f"{int(key[bad].item())} at entity row {bad} (valid range 1..{n_r})"
        )
    lookup = torch.empty(n_r, dtype=torch.int32, device=dev)
    n_used_t = torch.empty(1, dtype=torch.int32, device=dev)
    target = torch.empty(n, dtype=torch.int32, device=dev)
    used = torch.empty(n_r, dtype=torch.int64, device=dev)
    counts_kept = torch.empty(n_r, dtype=torch.int32, device=dev)
    ws = D.workspace(so.fb_key_remap_workspace_bytes(n_r))
    _lib.check(so.fb_key_remap(D.ptr(key), n, n_r, counts_full.data_ptr(), lookup.data_ptr(),
                               n_used_t.data_ptr(), D.ptr(target), used.data_ptr(),
                               counts_kept.data_ptr(), ws.data_ptr(), ws.numel(), st))
    n_used = int(n_used_t.item())
    used = used[:n_used]
    counts_kept = counts_kept[:n_used].clone()
    if n_used == n_r:
        r_kept = r
    elif D.is_csr(r):
        r_kept = r.rows(used)
    else:
        r_kept = torch.empty((n_used, r.shape[1]), dtype=torch.float64, device=dev)
        _lib.check(so.fb_gather_rows(D.ptr(r), r.shape[1], used.data_ptr(), n_used, r.shape[1],
                                     D.ptr(r_kept), r.shape[1], st))
    return IndicatorMatrix(target, n_used, counts_i32=counts_kept), r_kept, used


def build_pkfk(s, key_column, r):
    """PK-FK normalized matrix from S, its 1-based key column and R (normmat.py:201-214)."""
    host = D.is_host(s)
    s = D.as_factor(s)
    r = D.as_factor(r)
    key = _check_keys(key_column, r.shape[0])
    if key.numel() != s.shape[0]:
        raise ShapeError(f"key column length {key.numel()} != entity rows {s.shape[0]}")
    ind, r_kept, used = _remap_part(key, r)
    return NormalizedMatrix(PKFK, [(None, s), (ind, r_kept)], source_rows=[None, used], host_io=host)


def build_star(s, parts):
    """Star-schema normalized matrix: S plus ``[(key_column_i, R_i), ...]`` (normmat.py:217-237)."""
    host = D.is_host(s)
    s = D.as_factor(s)
    blocks = [(None, s)]
    source = [None]
    for idx, (key_column, r) in enumerate(parts):
        r = D.as_factor(r)
        key = _check_keys(key_column, r.shape[0], part_label=f" (part {idx})")
        if key.numel() != s.shape[0]:
            raise ShapeError(f"part {idx}: key column length {key.numel()} != entity rows {s.shape[0]}")
        ind, r_kept, used = _remap_part(key, r, part_label=f" (part {idx})")
        blocks.append((ind, r_kept))
        source.append(used)
    if len(blocks) == 1:
        raise ShapeError("star join needs at least one attribute table")
    return NormalizedMatrix(STAR, blocks, source_rows=source, host_io=host)


def build_mn(s, j_s, r, j_r):
    """M:N normalized matrix from join columns of equal values (normmat.py:240-285).

    Output rows are enumerated in lexicographic (S-row, R-row) order; rows of either table
    that match nothing are dropped before the indicators are built. The join planning runs
    on the device: join values coded through the sorted common values, R rows grouped by
    code with a stable sort, then per S row its group expanded into consecutive output rows.
    """
    host = D.is_host(s)
    s = D.as_matrix(s)
    r = D.as_matrix(r)
    dev = s.device
    js = D.as_vector_i64(j_s)
    jr = D.as_vector_i64(j_r)
    if js.dtype != jr.dtype:
        js, jr = js.to(torch.float64), jr.to(torch.float64)
    if js.numel() != s.shape[0]:
        raise ShapeError(f"join column length {js.numel()} != S rows {s.shape[0]}")
    if jr.numel() != r.shape[0]:
        raise ShapeError(f"join column length {jr.numel()} != R rows {r.shape[0]}")
    common = torch.unique(js)
    common = common[torch.isin(common, jr)]  # np.intersect1d: sorted unique common values
    if common.numel() == 0:
        raise EmptyJoinError("M:N join is empty: the join columns share no values")
    s_keep = torch.nonzero(torch.isin(js, common)).reshape(-1)
    r_keep = torch.nonzero(torch.isin(jr, common)).reshape(-1)
    s_code = torch.searchsorted(common, js.index_select(0, s_keep))
    r_code = torch.searchsorted(common, jr.index_select(0, r_keep))
    r_order = torch.sort(r_code, stable=True).indices  # groups of kept R rows, ascending within
    group_sizes = torch.bincount(r_code, minlength=common.numel())
    group_starts = torch.cumsum(group_sizes, 0) - group_sizes
    match = group_sizes.index_select(0, s_code)
    n_out = int(match.sum().item())
    if n_out >= 2**31:
        raise ShapeError(f"M:N join output has {n_out} rows; the device indicators are int32")
    i_s = torch.repeat_interleave(torch.arange(s_keep.numel(), device=dev), match)
    out_starts = torch.cumsum(match, 0) - match
    within = torch.arange(n_out, device=dev) - torch.repeat_interleave(out_starts, match)
    i_r = r_order.index_select(0, torch.repeat_interleave(group_starts.index_select(0, s_code), match) + within)
    s_kept = _take(s, s_keep)
    r_kept = _take(r, r_keep)
    ind_s = IndicatorMatrix(i_s.to(torch.int32), s_keep.numel())
    ind_r = IndicatorMatrix(i_r.to(torch.int32), r_keep.numel())
    return NormalizedMatrix(MN, [(ind_s, s_kept), (ind_r, r_kept)], source_rows=[s_keep, r_keep], host_io=host)


def build_multimn(row_map, tables):
    """Multi-table M:N normalized matrix from an explicit row mapping (normmat.py:288-319).

    ``row_map`` is an (n_out, q) integer array whose column j holds the 0-based row of
    ``tables[j]`` feeding each output row. Unreferenced table rows are dropped and indices
    compacted (the remap kernels of build_pkfk, on 1-based keys).
    """
    host = D.is_host(tables[0]) if len(tables) else True
    rm = row_map if isinstance(row_map, torch.Tensor) else torch.from_numpy(np.asarray(row_map, dtype=np.int64))
    if rm.dim() != 2:
        raise ShapeError("row_map must be 2-D (output rows x tables)")
    if rm.shape[0] < 1:
        raise EmptyJoinError("row mapping has no output rows")
    if rm.shape[1] != len(tables):
        raise ShapeError(f"row_map has {rm.shape[1]} columns but {len(tables)} tables given")
    blocks, source = [], []
    for j, t in enumerate(tables):
        t = D.as_matrix(t)
        refs = rm[:, j].to(device=t.device, dtype=torch.int64).contiguous()
        lo, hi = int(refs.min().item()), int(refs.max().item())
        if lo < 0 or hi >= t.shape[0]:
            raise DataError(f"row_map column {j} references nonexistent rows")
        ind, kept, used = _remap_part((refs + 1).contiguous(), t, part_label=f" (table {j})")
        blocks.append((ind, kept))
        source.append(used)
    return NormalizedMatrix(MULTIMN, blocks, source_rows=source, host_io=host)


def _take(f, rows):
    """f[rows] with the library's row gather (rows: int64 device indices)."""
    out = torch.empty((rows.numel(), f.shape[1]), dtype=torch.float64, device=f.device)
    if rows.numel() and f.shape[1]:
        so = _lib.lib()
        _lib.check(so.fb_gather_rows(D.ptr(f), f.shape[1], D.ptr(rows.contiguous()), rows.numel(), f.shape[1],
                                     D.ptr(out), f.shape[1], D.stream_handle()))
    return out


# ---------------------------------------------------------------------------
# shape statistics


@dataclass
class ShapeStats:
    """Dimensions plus the tuple/feature ratios (normmat.py:326-375)."""

    variant: str
    n_s: int
    d_s: int
    n_r: tuple
    d_r: tuple
    logical_rows: int
    logical_cols: int
    tuple_ratio: float
    feature_ratio: float

    @property
    def d_total(self):
        return self.logical_cols


def stats(nm):
    """Shape statistics (normmat.py:340-375; transpose flag ignored)."""
    base = nm.untransposed()
    n_log, d_log = base.shape
    if nm.variant == MULTIMN:  # no entity table
        n_s, d_s = 0, 0
        n_r = tuple(f.shape[0] for _, f in base.blocks)
        d_r = tuple(f.shape[1] for _, f in base.blocks)
        tr = n_log / max(n_r)
        fr = float("inf")
    else:
        n_s, d_s = base.blocks[0][1].shape
        n_r = tuple(f.shape[0] for _, f in base.blocks[1:])
        d_r = tuple(f.shape[1] for _, f in base.blocks[1:])
        tr = n_s / max(n_r) if n_r else 1.0
        fr = (sum(d_r) / d_s) if d_s > 0 else float("inf")
    return ShapeStats(nm.variant, n_s, d_s, n_r, d_r, n_log, d_log, float(tr), float(fr))

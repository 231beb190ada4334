"""Row-sharded factorized LA over 1..N GPUs (one process per GPU, ``torch.distributed``).

Partitioning (BASELINE.json north star): the rows of S, of every FK
column and of every per-row vector (y, W, assignments) are split into contiguous blocks,
one per rank; the attribute tables R_i are replicated — but the R-side *work* is split by
R-row slice (with every rank reading all of R, c2 LMM would scale ~3.8x at
N = 8). Rank g owns R rows [g·⌈n_R/N⌉, (g+1)·⌈n_R/N⌉) of every part:

* LMM T·X / rowSums: each rank computes z = R_slice·X_R for its slice (``fb_lmm_zpass``),
  one **all-gather** assembles the whole z, and the S pass runs on the rank's own rows
  (``fb_lmm_spass``); the output stays row-sharded.
* Tᵀ·P, X·T, colSums: the S pass (``fb_wt_spass``) gives this rank's SᵀW partial and its
  X·K bins over all n_R rows; a **reduce-scatter** of the bins leaves each rank the summed
  bins of its own slice, which it multiplies into its R slice (``fb_rows_wt``); one
  **all-reduce** of the small n_w × d result combines everything. colSums needs no
  reduce-scatter: its bins are the global key counts, known on every rank since the build.
* crossprod: SᵀS and KᵀS of the rank's rows (``fb_crossprod_spass``), a reduce-scatter of
  KᵀS (n_R × d_S), then (KᵀS)ᵀR and Rᵀdiag(c)R on the slice (``fb_crossprod_rpass``), one
  all-reduce of the d × d result and an exact mirror.
* GNMF composes the above (Tᵀ·W, T·H); the GLM and K-Means drivers keep their fused
  single-GPU steps per rank (replicated R-side work) plus one all-reduce per iteration.
* Integer partials (key histograms, cluster sizes) are reduced as integers, so they stay
  bit-exact; construction keeps the reference's global semantics (normmat.py:168-198): the
  key histogram is all-reduced first, so every rank drops the same unreferenced R rows.

The local arithmetic goes through a *backend* (``DeviceBackend``: the sm_100a kernels of
this package). The collective composition is backend-independent, which is what the
world-size-2 ``gloo`` tests exercise on CPU with an oracle-backed backend (and on one GPU
with the device backend).
"""

import numpy as np
import torch
import torch.distributed as dist

from . import _device as D
from . import _lib
from .exceptions import DataError, DivergenceError, NumericError, ShapeError

__all__ = [
    "shard_range",
    "ShardedMatrix",
    "DeviceBackend",
    "build_pkfk",
    "build_star",
    "lmm",
    "tmm",
    "rmm",
    "row_sums",
    "col_sums",
    "sum_all",
    "crossprod",
    "logistic_gd",
    "linreg_gd",
    "linreg_normal",
    "kmeans",
    "gnmf",
]


def shard_range(n, rank, world):
    """Contiguous block [r0, r1) of n rows owned by `rank` (sizes differ by at most one)."""
    return n * rank // world, n * (rank + 1) // world


def _world(group):
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def _rank(group):
    return dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0


def _allreduce(t, group=None, op=None):
    """In-place sum (default) over the group; a no-op on one process."""
    if _world(group) > 1:
        if t.is_cuda and dist.get_backend(group) != "nccl":  # gloo: reduce a host copy
            h = t.cpu()
            dist.all_reduce(h, op=op or dist.ReduceOp.SUM, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op or dist.ReduceOp.SUM, group=group)
    return t


def _nccl(group):
    return _world(group) > 1 and dist.get_backend(group) == "nccl"


def _allgather_rows(buf, chunk, group):
    """buf: (world·chunk, cols); this rank filled rows [rank·chunk, (rank+1)·chunk)."""
    world, rank = _world(group), _rank(group)
    if world == 1:
        return buf
    mine = buf[rank * chunk:(rank + 1) * chunk]
    if _nccl(group):
        dist.all_gather_into_tensor(buf, mine.contiguous(), group=group)
    else:  # gloo (functional checks; its all-gather is host-only): list all-gather on host copies
        host = mine.cpu()
        parts = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(parts, host, group=group)
        for g, t in enumerate(parts):
            buf[g * chunk:(g + 1) * chunk] = t.to(buf.device)
    return buf


def _reduce_scatter_rows(buf, chunk, group):
    """buf: (world·chunk, cols) partial sums on every rank -> this rank's summed row chunk."""
    world, rank = _world(group), _rank(group)
    if world == 1:
        return buf[:chunk]
    if _nccl(group):
        out = torch.empty((chunk,) + tuple(buf.shape[1:]), dtype=buf.dtype, device=buf.device)
        dist.reduce_scatter_tensor(out, buf, group=group)
        return out
    _allreduce(buf, group)  # gloo has no reduce-scatter: same sums, more traffic
    return buf[rank * chunk:(rank + 1) * chunk]


class ShardedMatrix:
    """This rank's row block of a normalized matrix plus its place in the global one.

    ``gcounts[i]``: global key counts (f64) of part i's kept R rows — colSums(K_i) of the whole
    matrix, all-reduced at build time. ``r_slice(i)`` is this rank's R-row slice of part i.
    """

    def __init__(self, local, n_global, row0, group=None, backend=None, gcounts=None):
        self.local = local
        self.n_global = int(n_global)
        self.row0 = int(row0)
        self.group = group
        self.backend = backend or DeviceBackend()
        self.gcounts = gcounts or []

    def r_chunk(self, i):
        n_r = self.backend.part_rows(self.local, i)
        return -(-n_r // _world(self.group)), n_r

    def r_slice(self, i):
        chunk, n_r = self.r_chunk(i)
        lo = min(n_r, _rank(self.group) * chunk)
        return lo, min(n_r, lo + chunk)

    @property
    def n_local(self):
        return self.backend.rows(self.local)

    @property
    def shape(self):
        return (self.n_global, self.backend.cols(self.local))


# ---------------------------------------------------------------------------
# the device backend: local shards on this rank's GPU


class DeviceBackend:
    """Local arithmetic on this rank's GPU (the package's C-ABI kernels)."""

    def tensor(self, a, dtype=torch.float64):
        return torch.as_tensor(a, dtype=dtype, device=D.device())

    def key_counts(self, key, n_r):
        """Histogram of 1-based keys over n_r rows (int32), plus the first bad row (-1 if none)."""
        so = _lib.lib()
        k = D.as_vector_i64(key).to(torch.int64).contiguous()
        counts = torch.empty(max(n_r, 1), dtype=torch.int32, device=k.device)
        bad = torch.empty(1, dtype=torch.int64, device=k.device)
        _lib.check(so.fb_key_check(D.ptr(k), k.numel(), n_r, counts.data_ptr(), bad.data_ptr(), D.stream_handle()))
        return counts, int(bad.item())

    def build(self, s, parts, global_counts):
        """Local NormalizedMatrix whose kept R rows follow the global key histogram."""
        from .normmat import STAR, PKFK, IndicatorMatrix, NormalizedMatrix

        so = _lib.lib()
        st = D.stream_handle()
        host = D.is_host(s)
        s = D.as_matrix(s)
        blocks, source = [(None, s)], [None]
        for (key, r), counts_full in zip(parts, global_counts):
            r = D.as_matrix(r)
            n_r = r.shape[0]
            k = D.as_vector_i64(key).to(torch.int64).contiguous()
            n = k.numel()
            lookup = torch.empty(n_r, dtype=torch.int32, device=r.device)
            n_used_t = torch.empty(1, dtype=torch.int32, device=r.device)
            target = torch.empty(n, dtype=torch.int32, device=r.device)
            used = torch.empty(n_r, dtype=torch.int64, device=r.device)
            kept = torch.empty(n_r, dtype=torch.int32, device=r.device)
            ws = D.workspace(so.fb_key_remap_workspace_bytes(n_r))
            gc = counts_full.to(device=r.device, dtype=torch.int32).contiguous()
            _lib.check(so.fb_key_remap(D.ptr(k), n, n_r, gc.data_ptr(), lookup.data_ptr(), n_used_t.data_ptr(),
                                       D.ptr(target), used.data_ptr(), kept.data_ptr(), ws.data_ptr(), ws.numel(), st))
            n_used = int(n_used_t.item())
            used = used[:n_used]
            if n_used == n_r:
                r_kept = r
            else:
                r_kept = torch.empty((n_used, r.shape[1]), dtype=torch.float64, device=r.device)
                _lib.check(so.fb_gather_rows(D.ptr(r), r.shape[1], used.data_ptr(), n_used, r.shape[1], D.ptr(r_kept),
                                             r.shape[1], st))
            # local counts: this shard's histogram over the kept rows (colSums of the local K)
            blocks.append((IndicatorMatrix(target, n_used), r_kept))
            source.append(used)
        return NormalizedMatrix(PKFK if len(parts) == 1 else STAR, blocks, source_rows=source, host_io=host).device_view()

    def rows(self, nm):
        return nm.base_rows

    def cols(self, nm):
        return nm.base_cols

    def nparts(self, nm):
        return len(nm.indicator_blocks)

    def part_rows(self, nm, i):
        return nm.indicator_blocks[i][1].shape[0]

    def part_cols(self, nm, i):
        return nm.indicator_blocks[i][1].shape[1]

    def source_rows(self, nm, i):
        return nm.source_rows[i + 1]

    def splittable(self, nm):
        return nm.blocks[0][0] is None  # PK-FK / star (M:N matrices keep the replicated path)

    def zeros(self, *shape):
        return torch.zeros(shape, dtype=torch.float64, device=D.device())

    def z_cols(self, d_x):
        return int(_lib.lib().fb_z_stride(d_x))

    def lmm_zpass(self, nm, x, i, lo, hi, z):
        xd = self.tensor(x).contiguous()
        _lib.check(_lib.lib().fb_lmm_zpass(nm.c_struct(), D.ptr(xd), xd.shape[1], i, lo, hi, D.ptr(z),
                                           D.stream_handle()))

    def lmm_spass(self, nm, x, zs):
        import ctypes

        xd = self.tensor(x).contiguous()
        out = torch.empty((nm.base_rows, xd.shape[1]), dtype=torch.float64, device=D.device())
        arr = (ctypes.c_void_p * max(1, len(zs)))(*[z.data_ptr() for z in zs])
        _lib.check(_lib.lib().fb_lmm_spass(nm.c_struct(), D.ptr(xd), xd.shape[1], arr, D.ptr(out),
                                           D.stream_handle()))
        return out

    def wt_spass(self, nm, w, n_w, w_rs, w_cs, bins):
        """(n_w × d) with this rank's SᵀW in the S columns (rest zero); bins[i][:n_r] = WᵀK_i."""
        import ctypes

        so = _lib.lib()
        cs = nm.c_struct()
        if any(b is not None for b in bins) and any(e.skewed for e, _ in nm.indicator_blocks):
            nm.ensure_sorted()  # skewed keys scatter as segmented sums over the sorted order
        out = torch.zeros((n_w, nm.base_cols), dtype=torch.float64, device=D.device())
        ws = D.workspace(so.fb_wt_spass_workspace_bytes(cs, n_w))
        arr = (ctypes.c_void_p * 4)(*[(b.data_ptr() if b is not None else None) for b in bins] + [None] * (4 - len(bins)))
        _lib.check(so.fb_wt_spass(cs, D.ptr(w) if w is not None else None, n_w, w_rs, w_cs, D.ptr(out),
                                  nm.base_cols, 1, arr if w is not None else None, ws.data_ptr(), ws.numel(),
                                  D.stream_handle()))
        return out

    def rows_wt(self, nm, i, lo, hi, wts):
        """(n_w × d_r) = wtsᵀ · R_i[lo:hi] (wts: (hi-lo) × n_w)."""
        so = _lib.lib()
        r = nm.indicator_blocks[i][1]
        d_r = r.shape[1]
        n_w = wts.shape[1]
        out = torch.empty((n_w, d_r), dtype=torch.float64, device=D.device())
        ws = D.workspace(so.fb_rows_wt_workspace_bytes(d_r, n_w))
        wts = wts.contiguous()
        _lib.check(so.fb_rows_wt(r.data_ptr() + 8 * lo * d_r, hi - lo, d_r, D.ptr(wts), n_w, n_w, 1, D.ptr(out), d_r,
                                 1, ws.data_ptr(), ws.numel(), D.stream_handle()))
        return out

    def crossprod_spass(self, nm, kts):
        so = _lib.lib()
        cs = nm.c_struct()
        perm, fks = nm.k.sorted_order()
        d = nm.base_cols
        out = torch.empty((d, d), dtype=torch.float64, device=D.device())
        ws = D.workspace(so.fb_crossprod_workspace_bytes(cs))
        _lib.check(so.fb_crossprod_spass(cs, D.ptr(perm), D.ptr(fks), D.ptr(out), D.ptr(kts), ws.data_ptr(),
                                         ws.numel(), D.stream_handle()))
        return out

    def crossprod_rpass(self, nm, lo, hi, kts_slice, counts_slice):
        so = _lib.lib()
        d = nm.base_cols
        out = torch.zeros((d, d), dtype=torch.float64, device=D.device())
        if hi <= lo:
            return out
        r = nm.r
        st = _lib.FbNormalized()
        st.s, st.n_s, st.d_s, st.q = D.ptr(nm.blocks[0][1]), nm.base_rows, nm.blocks[0][1].shape[1], 1
        p = st.part[0]
        p.fk = D.ptr(nm.k.target)
        p.r = r.data_ptr() + 8 * lo * r.shape[1]
        p.n_r, p.d_r = hi - lo, r.shape[1]
        cnt = counts_slice.contiguous()
        p.counts = D.ptr(cnt)
        kts_slice = kts_slice.contiguous()
        import ctypes

        ws = D.workspace(so.fb_crossprod_workspace_bytes(ctypes.byref(st)))
        _lib.check(so.fb_crossprod_rpass(ctypes.byref(st), D.ptr(kts_slice), D.ptr(out), ws.data_ptr(), ws.numel(),
                                         D.stream_handle()))
        return out

    def lmm(self, nm, x):
        from .rewrite import lmm

        return lmm(nm, self.tensor(x))

    def tmm(self, nm, p):
        from .rewrite import lmm

        return lmm(nm.T, self.tensor(p))

    def rmm(self, x, nm):
        from .rewrite import rmm

        return rmm(self.tensor(x), nm)

    def row_sums(self, nm):
        from .rewrite import row_sums

        return row_sums(nm)

    def col_sums(self, nm):
        from .rewrite import col_sums

        return col_sums(nm)

    def sum_all(self, nm):
        from .rewrite import sum_all

        return self.tensor([sum_all(nm)])

    def crossprod(self, nm):
        from .crossprod_impl import crossprod

        return crossprod(nm)

    def glm_eval(self, nm, y, w, mode):
        so = _lib.lib()
        d = nm.base_cols
        g = torch.empty(d + 1, dtype=torch.float64, device=D.device())
        yd = self.tensor(y).reshape(-1, 1).contiguous()
        wd = self.tensor(w).reshape(-1).contiguous()
        cs = nm.c_struct()
        ws = D.workspace(so.fb_glm_workspace_bytes(cs))
        _lib.check(so.fb_glm_eval(cs, D.ptr(yd), D.ptr(wd), mode, D.ptr(g), g.data_ptr() + 8 * d, ws.data_ptr(),
                                  ws.numel(), D.stream_handle()))
        return g  # [g_0..g_{d-1}, loss]

    def glm_update(self, w, gl, alpha, trace, it, diverged):
        """w += alpha·g (g = gl[:d]), trace[it] = gl[d], first non-finite iteration."""
        so = _lib.lib()
        d = w.numel()
        _lib.check(so.fb_glm_update(D.ptr(w), D.ptr(gl), d, float(alpha), gl.data_ptr() + 8 * d, D.ptr(trace), it,
                                    D.ptr(diverged), D.stream_handle()))

    def col_sq_sums(self, c):
        from .ml import _col_sq_sums

        return _col_sq_sums(c)

    def take_rows(self, nm, idx):
        from .ml import _take_rows

        return _take_rows(nm, idx)

    def square_row_sums(self, nm):
        from .rewrite import row_sums, scalar_fn

        return row_sums(scalar_fn(nm, np.square)).reshape(-1).contiguous()

    def square_sum(self, nm):
        from .rewrite import scalar_fn, sum_all

        return self.tensor([sum_all(scalar_fn(nm, np.square))])

    def kmeans_partial(self, nm, d_t, c, cc, k, it, trace, assign, nan_row):
        so = _lib.lib()
        d = nm.base_cols
        tta = torch.empty((d, k), dtype=torch.float64, device=D.device())
        sizes = torch.empty(k, dtype=torch.int32, device=D.device())
        cs = nm.c_struct()
        ws = D.workspace(so.fb_kmeans_workspace_bytes(cs, k))
        _lib.check(so.fb_kmeans_partial(cs, D.ptr(d_t), D.ptr(c), D.ptr(cc), k, it, D.ptr(trace), D.ptr(assign),
                                        D.ptr(nan_row), D.ptr(tta), D.ptr(sizes), ws.data_ptr(), ws.numel(),
                                        D.stream_handle()))
        return tta, sizes

    def kmeans_update(self, c, tta, sizes, cc):
        so = _lib.lib()
        d, k = c.shape
        _lib.check(so.fb_kmeans_update(D.ptr(c), D.ptr(tta), D.ptr(sizes), d, k, D.ptr(cc), D.stream_handle()))

    def nmf_update(self, f, num, g):
        so = _lib.lib()
        _lib.check(so.fb_nmf_update(D.ptr(f), D.ptr(num), D.ptr(g), f.shape[0], f.shape[1], D.stream_handle()))

    def small_gram(self, f):
        so = _lib.lib()
        g = torch.empty((f.shape[1], f.shape[1]), dtype=torch.float64, device=D.device())
        _lib.check(so.fb_small_gram(D.ptr(f), f.shape[0], f.shape[1], D.ptr(g), D.stream_handle()))
        return g

    def dense_crossprod(self, w):
        from .crossprod_impl import crossprod
        from .normmat import as_normalized

        return crossprod(as_normalized(w))

    def nmf_objective(self, sum_t2, ttw, h, cpw, cph, trace, it):
        so = _lib.lib()
        _lib.check(so.fb_nmf_objective(D.ptr(sum_t2), D.ptr(ttw), D.ptr(h), h.numel(), D.ptr(cpw), D.ptr(cph),
                                       cpw.numel(), D.ptr(trace), it, D.stream_handle()))

    def pinv(self, g):
        from .ml import _pinv_dense

        return _pinv_dense(g.detach().cpu().numpy())

    def to_numpy(self, t):
        return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


# ---------------------------------------------------------------------------
# construction


def build_star(s_local, parts, n_global, group=None, backend=None):
    """Sharded star schema: this rank's rows of S and of every key column, R_i replicated.

    Keys are 1-based (normmat.py:182-198). The key histograms are all-reduced before the
    remap so every rank keeps the same R rows (the reference drops rows unreferenced by
    the *whole* key column).
    """
    be = backend or DeviceBackend()
    world, rank = _world(group), _rank(group)
    r0, r1 = shard_range(n_global, rank, world)
    global_counts = []
    for idx, (key, r) in enumerate(parts):
        n_r = int(np.asarray(r.shape)[0])
        counts, bad = be.key_counts(key, n_r)
        flag = be.tensor([1 if bad != -1 else 0], dtype=torch.int64)
        _allreduce(flag, group)
        if bad != -1:
            raise DataError(f"key (part {idx}) references a nonexistent attribute row at entity row {r0 + bad}")
        if int(flag.item()) > 0:
            raise DataError(f"key (part {idx}) references a nonexistent attribute row on another rank")
        _allreduce(counts, group)
        global_counts.append(counts)
    local = be.build(s_local, parts, global_counts)
    if be.rows(local) != r1 - r0:
        raise ShapeError(f"rank {rank} holds {be.rows(local)} rows, expected {r1 - r0} of {n_global}")
    # global colSums(K_i) of the kept rows: the weights of colSums' R-slice pass
    gcounts = [be.tensor(be.to_numpy(gc)[be.to_numpy(be.source_rows(local, i))].astype(np.float64))
               for i, gc in enumerate(global_counts)]
    return ShardedMatrix(local, n_global, r0, group, be, gcounts)


def build_pkfk(s_local, key_local, r, n_global, group=None, backend=None):
    """Sharded PK-FK matrix (normmat.py:201-214 semantics over the global key column)."""
    return build_star(s_local, [(key_local, r)], n_global, group, backend)


# ---------------------------------------------------------------------------
# operators


def _split(sm, width=1):
    """The R-row-sliced composition applies (multi-rank, PK-FK / star, <= 16 columns per pass)."""
    return _world(sm.group) > 1 and width <= 16 and sm.backend.splittable(sm.local)


def lmm(sm, x):
    """T·X for this rank's rows: z slices (R_slice·X_R) all-gathered, then the S pass."""
    be = sm.backend
    x = be.tensor(x)
    if x.dim() == 1:
        x = x.reshape(-1, 1)
    if not _split(sm, x.shape[1]):
        return be.lmm(sm.local, x)
    zc = be.z_cols(x.shape[1])
    zs = []
    for i in range(be.nparts(sm.local)):
        chunk, n_r = sm.r_chunk(i)
        lo, hi = sm.r_slice(i)
        z = be.zeros(chunk * _world(sm.group), zc)
        if hi > lo:
            be.lmm_zpass(sm.local, x, i, lo, hi, z)
        zs.append(_allgather_rows(z, chunk, sm.group))
    return be.lmm_spass(sm.local, x, zs)


def _wt(sm, w, n_w, w_rs, w_cs):
    """out (n_w × d) = Σ_i w(i, ·)ᵀ T(i, ·) over all ranks' rows (w: this rank's rows)."""
    be = sm.backend
    nparts = be.nparts(sm.local)
    world = _world(sm.group)
    bins = []
    for i in range(nparts):
        chunk, n_r = sm.r_chunk(i)
        bins.append(be.zeros(chunk * world, n_w))
    out = be.wt_spass(sm.local, w, n_w, w_rs, w_cs, [b[:sm.r_chunk(i)[1]] for i, b in enumerate(bins)])
    off = be.cols(sm.local) - sum(be.part_cols(sm.local, i) for i in range(nparts))
    for i in range(nparts):
        chunk, _ = sm.r_chunk(i)
        lo, hi = sm.r_slice(i)
        mine = _reduce_scatter_rows(bins[i], chunk, sm.group)  # summed X·K_i of my R slice
        d_r = be.part_cols(sm.local, i)
        if hi > lo and d_r:
            out[:, off:off + d_r] = be.rows_wt(sm.local, i, lo, hi, mine[:hi - lo])
        off += d_r
    return _allreduce(out, sm.group)


def tmm(sm, p_local):
    """Tᵀ·P (d × m) from this rank's rows of P, summed over ranks."""
    be = sm.backend
    p = be.tensor(p_local)
    if p.dim() == 1:
        p = p.reshape(-1, 1)
    if not _split(sm, p.shape[1]):
        return _allreduce(be.tmm(sm.local, p), sm.group)
    p = p.contiguous()
    m = p.shape[1]
    return _wt(sm, p, m, m, 1).t().contiguous()


def rmm(x_local, sm):
    """X·T (n_x × d) from this rank's columns of X, summed over ranks."""
    be = sm.backend
    x = be.tensor(x_local)
    if not _split(sm, x.shape[0]):
        return _allreduce(be.rmm(x, sm.local), sm.group)
    x = x.contiguous()
    return _wt(sm, x, x.shape[0], 1, x.shape[1])


def row_sums(sm):
    """rowSums(T) for this rank's rows (the LMM composition with X = 1, rewrite.py:118-128)."""
    if not _split(sm):
        return sm.backend.row_sums(sm.local)
    return lmm(sm, np.ones((sm.shape[1], 1)))


def col_sums(sm):
    """colSums(T) = [1ᵀS summed over ranks, global counts_i · R_i by R slice] (rewrite.py:131-149)."""
    be = sm.backend
    if not _split(sm):
        return _allreduce(be.col_sums(sm.local), sm.group)
    out = be.wt_spass(sm.local, None, 1, 1, 1, [None] * be.nparts(sm.local))
    nparts = be.nparts(sm.local)
    off = be.cols(sm.local) - sum(be.part_cols(sm.local, i) for i in range(nparts))
    for i in range(nparts):
        lo, hi = sm.r_slice(i)
        d_r = be.part_cols(sm.local, i)
        if hi > lo and d_r:
            out[:, off:off + d_r] = be.rows_wt(sm.local, i, lo, hi, sm.gcounts[i][lo:hi].reshape(-1, 1))
        off += d_r
    return _allreduce(out, sm.group)


def sum_all(sm):
    if not _split(sm):
        return float(_allreduce(sm.backend.sum_all(sm.local), sm.group)[0])
    return float(col_sums(sm).sum())


def crossprod(sm):
    """TᵀT: this rank's SᵀS + KᵀS; KᵀS reduce-scattered by R slice; (KᵀS)ᵀR and Rᵀdiag(c)R on
    the slice; one all-reduce of the d × d sum, then the upper triangle mirrored
    (rewrite.py:298): an all-reduce may sum element (i, j) and its mirror (j, i) in different
    orders (NCCL rings chunk the buffer), so symmetry is restored explicitly."""
    be = sm.backend
    if _split(sm) and be.nparts(sm.local) == 1:
        chunk, n_r = sm.r_chunk(0)
        d_s = be.cols(sm.local) - be.part_cols(sm.local, 0)
        kts = be.zeros(chunk * _world(sm.group), max(d_s, 1))
        g = be.crossprod_spass(sm.local, kts[:n_r])
        mine = _reduce_scatter_rows(kts, chunk, sm.group)
        lo, hi = sm.r_slice(0)
        g = g + be.crossprod_rpass(sm.local, lo, hi, mine[:hi - lo], sm.gcounts[0][lo:hi])
        g = _allreduce(g, sm.group)
    else:
        g = _allreduce(be.crossprod(sm.local), sm.group)
    if _world(sm.group) > 1:
        g = torch.triu(g) + torch.triu(g, 1).t()
    return g


# ---------------------------------------------------------------------------
# drivers (ml.py semantics; model state replicated, per-row data sharded)


def _glm(sm, y_local, cfg, mode, name):
    from .ml import ModelOutput

    be = sm.backend
    n, d = sm.shape
    w = be.tensor(np.zeros(d))
    trace = be.tensor(np.zeros(cfg.iterations))
    diverged = be.tensor([-1], dtype=torch.int32)
    alpha = cfg.step_size if mode == 0 else -cfg.step_size  # ml.py:212 / ml.py:251
    for it in range(cfg.iterations):
        gl = _allreduce(be.glm_eval(sm.local, y_local, w, mode), sm.group)  # [Tᵀp, loss]
        be.glm_update(w, gl, alpha, trace, it, diverged)  # identical on every rank
    bad = int(diverged[0])
    if bad >= 0:
        raise DivergenceError(bad)
    return ModelOutput(name, (n, d), cfg, be.to_numpy(trace).tolist(), weights=be.to_numpy(w).reshape(d, 1))


def logistic_gd(sm, y_local, cfg):
    """logistic_gd (ml.py:199-215) over sharded rows: one all-reduce of [g, loss] per iteration."""
    return _glm(sm, y_local, cfg, 0, "logistic_gd")


def linreg_gd(sm, y_local, cfg):
    """linreg_gd (ml.py:239-254) over sharded rows."""
    return _glm(sm, y_local, cfg, 1, "linreg_gd")


def linreg_normal(sm, y_local):
    """linreg_normal (ml.py:218-236): all-reduced TᵀT and Tᵀy, host pinv, all-reduced residual."""
    from .ml import ModelOutput

    be = sm.backend
    n, d = sm.shape
    g = crossprod(sm)
    gl = _allreduce(be.glm_eval(sm.local, y_local, np.zeros(d), 1), sm.group)
    tty = -be.to_numpy(gl[:d]).reshape(d, 1)
    w = be.pinv(g) @ tty
    res = _allreduce(be.glm_eval(sm.local, y_local, w.ravel(), 1), sm.group)
    return ModelOutput("linreg_normal", (n, d), None, [float(res[d])], weights=w)


def kmeans(sm, cfg):
    """kmeans (ml.py:257-285): seeds drawn with the reference's RNG call on every rank; each
    iteration all-reduces TᵀA, the integer cluster sizes and the objective."""
    from .ml import ModelOutput

    be = sm.backend
    n, d = sm.shape
    k = cfg.k
    if k > n:
        raise DataError(f"k={k} exceeds the number of data rows ({n})")
    rng = np.random.default_rng(cfg.rng_seed)
    seeds = rng.choice(n, size=k, replace=False)
    mine = [(j, i - sm.row0) for j, i in enumerate(seeds) if sm.row0 <= i < sm.row0 + sm.n_local]
    c0 = be.tensor(np.zeros((k, d)))
    if mine:
        rows = be.take_rows(sm.local, [i for _, i in mine])
        for (j, _), row in zip(mine, rows):
            c0[j] = row
    _allreduce(c0, sm.group)  # every seed row comes from exactly one rank
    c = c0.t().contiguous()
    cc = be.col_sq_sums(c)
    d_t = be.square_row_sums(sm.local)
    trace = be.tensor(np.zeros(cfg.iterations))
    assign = torch.empty(sm.n_local, dtype=torch.int32, device=c.device)
    nan_row = torch.full((1,), -1, dtype=torch.int64, device=c.device)
    for it in range(cfg.iterations):
        tta, sizes = be.kmeans_partial(sm.local, d_t, c, cc, k, it, trace, assign, nan_row)
        _allreduce(tta, sm.group)
        _allreduce(sizes, sm.group)
        be.kmeans_update(c, tta, sizes, cc)
    # every rank takes the same path: the trace and the first NaN row (global index, MIN over
    # ranks) are all-reduced before anyone raises, so no rank is left waiting in a collective
    _allreduce(trace, sm.group)
    bad = int(nan_row[0])  # (iteration << 40) | local row, or -1
    none = np.iinfo(np.int64).max
    low = (1 << 40) - 1
    first = be.tensor([((bad >> 40) << 40) | (sm.row0 + (bad & low)) if bad != -1 else none], dtype=torch.int64)
    _allreduce(first, sm.group, op=dist.ReduceOp.MIN if _world(sm.group) > 1 else None)
    if int(first[0]) != none:
        raise NumericError(f"row_min_mask: NaN in row {int(first[0]) & low}")
    return ModelOutput("kmeans", (n, d), cfg, be.to_numpy(trace).tolist(), centroids=be.to_numpy(c))


def gnmf(sm, cfg):
    """gnmf (ml.py:288-317) with W row-sharded and H replicated: Tᵀ·W, WᵀW and ΣT² are
    all-reduced; the H update is replicated, the W update row-local."""
    from .ml import ModelOutput

    be = sm.backend
    n, d = sm.shape
    r = cfg.r
    rng = np.random.default_rng(cfg.rng_seed)
    w_full = 1.0 - rng.random((n, r))  # the reference's draw order: W then H (ml.py:300-301)
    h = be.tensor(1.0 - rng.random((d, r)))
    w = be.tensor(np.ascontiguousarray(w_full[sm.row0:sm.row0 + sm.n_local]))
    del w_full
    sum_t2 = _allreduce(be.square_sum(sm.local), sm.group)
    cpw = _allreduce(be.dense_crossprod(w), sm.group)
    ttw = tmm(sm, w)
    trace = be.tensor(np.zeros(cfg.iterations))
    for it in range(cfg.iterations):
        be.nmf_update(h, ttw, cpw)            # h = h ∘ TᵀW / (h·WᵀW + eps) (replicated)
        cph = be.small_gram(h)
        th = lmm(sm, h)                       # row-local S pass, R-sliced z
        be.nmf_update(w, th, cph)             # w = w ∘ T·h / (w·hᵀh + eps) (row-local)
        ttw = tmm(sm, w)                      # R-sliced Tᵀ·W
        cpw = _allreduce(be.dense_crossprod(w), sm.group)
        be.nmf_objective(sum_t2, ttw, h, cpw, cph, trace, it)
    return ModelOutput("gnmf", (n, d), cfg, be.to_numpy(trace).tolist(), factors=(be.to_numpy(w), be.to_numpy(h)))

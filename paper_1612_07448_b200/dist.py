"""Row-sharded factorized LA over 1..N GPUs (one process per GPU, ``torch.distributed``).

Partitioning (BASELINE.json north star): the rows of S, of every FK
column and of every per-row vector (y, W, assignments) are split into contiguous blocks,
one per rank; the attribute tables R_i are replicated. Consequences:

* row-local results — LMM T·X, rowSums, the K-Means argmin, the GNMF W update — need no
  communication and stay sharded;
* every Tᵀ-side result — Tᵀ·P, X·T, colSums, sum, crossprod, GLM gradients and losses,
  K-Means cluster sums/sizes, GNMF Tᵀ·W and WᵀW — is a sum over rows: each rank computes its
  shard's partial with the single-GPU kernels and one all-reduce (NCCL over NVLink /
  NVSwitch) combines them. Integer partials (key histograms, cluster sizes) are reduced as
  integers, so they stay bit-exact.
* construction keeps the reference's global semantics (normmat.py:168-198): the key
  histogram is all-reduced first, so every rank drops the same unreferenced R rows and
  remaps keys identically.

The local arithmetic goes through a *backend* (``DeviceBackend``: the sm_100a kernels of
this package). The collective composition is backend-independent, which is what the
world-size-2 ``gloo`` tests exercise on CPU with an oracle-backed backend.
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
        dist.all_reduce(t, op=op or dist.ReduceOp.SUM, group=group)
    return t


class ShardedMatrix:
    """This rank's row block of a normalized matrix plus its place in the global one."""

    def __init__(self, local, n_global, row0, group=None, backend=None):
        self.local = local
        self.n_global = int(n_global)
        self.row0 = int(row0)
        self.group = group
        self.backend = backend or DeviceBackend()

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
    return ShardedMatrix(local, n_global, r0, group, be)


def build_pkfk(s_local, key_local, r, n_global, group=None, backend=None):
    """Sharded PK-FK matrix (normmat.py:201-214 semantics over the global key column)."""
    return build_star(s_local, [(key_local, r)], n_global, group, backend)


# ---------------------------------------------------------------------------
# operators


def lmm(sm, x):
    """T·X for this rank's rows (row-local: no communication)."""
    return sm.backend.lmm(sm.local, x)


def tmm(sm, p_local):
    """Tᵀ·P (d × m) from this rank's rows of P, summed over ranks."""
    return _allreduce(sm.backend.tmm(sm.local, p_local), sm.group)


def rmm(x_local, sm):
    """X·T (n_x × d) from this rank's columns of X, summed over ranks."""
    return _allreduce(sm.backend.rmm(x_local, sm.local), sm.group)


def row_sums(sm):
    return sm.backend.row_sums(sm.local)


def col_sums(sm):
    return _allreduce(sm.backend.col_sums(sm.local), sm.group)


def sum_all(sm):
    return float(_allreduce(sm.backend.sum_all(sm.local), sm.group)[0])


def crossprod(sm):
    """TᵀT: per-rank factorized crossprod partials summed over ranks, then the upper triangle
    mirrored (rewrite.py:298): an all-reduce may sum element (i, j) and its mirror (j, i) in
    different orders (NCCL rings chunk the buffer), so symmetry is restored explicitly."""
    g = _allreduce(sm.backend.crossprod(sm.local), sm.group)
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
    bad = int(nan_row[0])
    none = np.iinfo(np.int64).max
    first = be.tensor([sm.row0 + bad if bad != -1 else none], dtype=torch.int64)
    _allreduce(first, sm.group, op=dist.ReduceOp.MIN if _world(sm.group) > 1 else None)
    if int(first[0]) != none:
        raise NumericError(f"row_min_mask: NaN in row {int(first[0])}")
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
    ttw = _allreduce(be.tmm(sm.local, w), sm.group)
    trace = be.tensor(np.zeros(cfg.iterations))
    for it in range(cfg.iterations):
        be.nmf_update(h, ttw, cpw)            # h = h ∘ TᵀW / (h·WᵀW + eps) (replicated)
        cph = be.small_gram(h)
        th = be.lmm(sm.local, h)              # row-local
        be.nmf_update(w, th, cph)             # w = w ∘ T·h / (w·hᵀh + eps) (row-local)
        ttw = _allreduce(be.tmm(sm.local, w), sm.group)
        cpw = _allreduce(be.dense_crossprod(w), sm.group)
        be.nmf_objective(sum_t2, ttw, h, cpw, cph, trace, it)
    return ModelOutput("gnmf", (n, d), cfg, be.to_numpy(trace).tolist(), factors=(be.to_numpy(w), be.to_numpy(h)))

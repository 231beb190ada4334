"""World-size-2 gloo tests of the row-sharded path (paper_1612_07448_b200.dist) on CPU.

The collective composition (global key histogram before the remap, which results are
row-local, which are all-reduced, replicated model updates) is backend-independent; here
each rank's local arithmetic runs on an oracle-backed backend, and every sharded result
is compared with the unsharded oracle. The device backend runs the same composition on
NCCL (bench.py under torchrun).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-10


class OracleBackend:
    """Local arithmetic with the CPU oracle; tensors are CPU float64 (gloo)."""

    def __init__(self):
        import collections

        import factorla_oracle as O

        self.O = O
        self.calls = collections.Counter()

    def __getattribute__(self, name):
        if name in ("lmm_zpass", "wt_spass", "crossprod_rpass", "rows_wt"):
            object.__getattribute__(self, "calls")[name] += 1
        return object.__getattribute__(self, name)

    def tensor(self, a, dtype=torch.float64):
        return torch.as_tensor(np.asarray(a), dtype=dtype).clone()

    def key_counts(self, key, n_r):
        key = np.asarray(key, dtype=np.int64)
        bad = np.flatnonzero((key < 1) | (key > n_r))
        counts = np.bincount(np.clip(key - 1, 0, n_r - 1), minlength=n_r).astype(np.int32)
        return torch.from_numpy(counts), int(bad[0]) if bad.size else -1

    def build(self, s, parts, global_counts):
        O = self.O
        out, src = [], [None]
        for (key, r), gc in zip(parts, global_counts):
            used = np.flatnonzero(gc.numpy() > 0)
            lut = np.full(len(gc), -1, dtype=np.int64)
            lut[used] = np.arange(used.size)
            out.append((lut[np.asarray(key, dtype=np.int64) - 1], np.asarray(r)[used]))
            src.append(used)
        return O.NM(O.as_matrix(s), out, source_rows=src)

    def rows(self, nm):
        return nm.n

    def cols(self, nm):
        return nm.d

    # ---- the R-row-sliced split passes (same contract as DeviceBackend)
    def nparts(self, nm):
        return len(nm.parts)

    def part_rows(self, nm, i):
        return nm.parts[i][1].shape[0]

    def part_cols(self, nm, i):
        return nm.parts[i][1].shape[1]

    def source_rows(self, nm, i):
        return nm.source_rows[i + 1]

    def splittable(self, nm):
        return True

    def zeros(self, *shape):
        return torch.zeros(shape, dtype=torch.float64)

    def z_cols(self, d_x):
        return d_x

    def _off(self, nm, i):
        return nm.s.shape[1] + sum(r.shape[1] for _, r in nm.parts[:i])

    def lmm_zpass(self, nm, x, i, lo, hi, z):
        r = nm.parts[i][1]
        off = self._off(nm, i)
        z[lo:hi] = self._t(r[lo:hi] @ x.numpy()[off:off + r.shape[1]])

    def lmm_spass(self, nm, x, zs):
        xn = x.numpy()
        out = nm.s @ xn[:nm.s.shape[1]]
        for (t, _), z in zip(nm.parts, zs):
            out = out + z.numpy()[t]
        return self._t(out)

    def wt_spass(self, nm, w, n_w, w_rs, w_cs, bins):
        n, d_s = nm.s.shape
        wm = np.ones((n, 1)) if w is None else torch.as_strided(w, (n, n_w), (w_rs, w_cs)).numpy()
        out = np.zeros((wm.shape[1], nm.d))
        out[:, :d_s] = wm.T @ nm.s
        for (t, r), b in zip(nm.parts, bins):
            if b is not None:
                acc = np.zeros((r.shape[0], wm.shape[1]))
                np.add.at(acc, t, wm)
                b.copy_(self._t(acc))
        return self._t(out)

    def rows_wt(self, nm, i, lo, hi, wts):
        return self._t(wts.numpy().T @ nm.parts[i][1][lo:hi])

    def crossprod_spass(self, nm, kts):
        t, _ = nm.parts[0]
        d_s = nm.s.shape[1]
        g = np.zeros((nm.d, nm.d))
        g[:d_s, :d_s] = nm.s.T @ nm.s
        acc = np.zeros(tuple(kts.shape))
        np.add.at(acc, t, nm.s)
        kts.copy_(self._t(acc))
        return self._t(g)

    def crossprod_rpass(self, nm, lo, hi, kts_slice, counts_slice):
        d_s = nm.s.shape[1]
        g = np.zeros((nm.d, nm.d))
        r = nm.parts[0][1][lo:hi]
        p = r.T @ kts_slice.numpy()
        g[d_s:, :d_s] = p
        g[:d_s, d_s:] = p.T
        g[d_s:, d_s:] = (r * counts_slice.numpy()[:, None]).T @ r
        return self._t(g)

    def _t(self, a):
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))

    def lmm(self, nm, x):
        return self._t(self.O.lmm(nm, np.asarray(x)))

    def tmm(self, nm, p):
        return self._t(self.O.lmm(nm.T, np.asarray(p)))

    def rmm(self, x, nm):
        return self._t(self.O.rmm(np.asarray(x), nm))

    def row_sums(self, nm):
        return self._t(self.O.row_sums(nm))

    def col_sums(self, nm):
        return self._t(self.O.col_sums(nm))

    def sum_all(self, nm):
        return self._t([self.O.sum_all(nm)])

    def crossprod(self, nm):
        return self._t(self.O.crossprod(nm))

    def glm_eval(self, nm, y, w, mode):
        O = self.O
        y = np.asarray(y, dtype=np.float64).reshape(-1, 1)
        tw = O.lmm(nm, np.asarray(w, dtype=np.float64).reshape(-1, 1))
        with np.errstate(over="ignore"):
            if mode == 0:
                p = y / (1.0 + np.exp(tw))
                loss = float(np.sum(np.log1p(np.exp(-np.abs(y * tw))) + np.maximum(-y * tw, 0.0)))
            else:
                p = tw - y
                loss = float(np.sum(p**2))
        g = O.lmm(nm.T, p).ravel()
        return self._t(np.concatenate([g, [loss]]))

    def glm_update(self, w, gl, alpha, trace, it, diverged):
        d = w.numel()
        w += alpha * gl[:d]
        trace[it] = gl[d]
        if not bool(torch.isfinite(w).all()) and int(diverged[0]) < 0:
            diverged[0] = it

    def col_sq_sums(self, c):
        return (c * c).sum(dim=0)

    def take_rows(self, nm, idx):
        return self._t(self.O.take_rows(nm, idx))

    def square_row_sums(self, nm):
        return self._t(self.O.row_sums(self.O.scalar_fn(nm, np.square)).ravel())

    def square_sum(self, nm):
        return self._t([self.O.sum_all(self.O.scalar_fn(nm, np.square))])

    def kmeans_partial(self, nm, d_t, c, cc, k, it, trace, assign, nan_row):
        O = self.O
        dist_ = d_t.numpy()[:, None] + cc.numpy()[None, :] - O.lmm(O.scalar_op(nm, 2.0, "mul"), c.numpy())
        a = np.argmin(dist_, axis=1)
        trace[it] = float(dist_[np.arange(len(a)), a].sum())
        mask = np.zeros_like(dist_)
        mask[np.arange(len(a)), a] = 1.0
        return self._t(O.lmm(nm.T, mask)), torch.from_numpy(np.bincount(a, minlength=k).astype(np.int32))

    def kmeans_update(self, c, tta, sizes, cc):
        ne = sizes.numpy() > 0
        cn = c.numpy()
        cn[:, ne] = tta.numpy()[:, ne] / sizes.numpy()[ne]
        cc.copy_((c * c).sum(dim=0))

    def nmf_update(self, f, num, g):
        fn = f.numpy()
        fn[:] = fn * num.numpy() / (fn @ g.numpy() + 1e-12)

    def small_gram(self, f):
        return self._t(self.O._syrk(f.numpy()))

    def dense_crossprod(self, w):
        return self._t(self.O._syrk(np.asarray(w)))

    def nmf_objective(self, sum_t2, ttw, h, cpw, cph, trace, it):
        sq = float(sum_t2[0]) - 2.0 * float((ttw * h).sum()) + float((cpw * cph).sum())
        trace[it] = float(np.sqrt(max(sq, 0.0)))

    def pinv(self, g):
        return self.O.pinv(g.numpy())

    def to_numpy(self, t):
        return t.numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _data(seed=3):
    rng = np.random.default_rng(seed)
    n, n_r1, n_r2 = 3001, 97, 40
    s = rng.random((n, 6))
    k1 = rng.integers(1, n_r1 + 1, size=n)
    k1[: n // 2][k1[: n // 2] == 5] = 6   # row 5 of R1 referenced only by the second half
    k1[n // 2:][k1[n // 2:] == 7] = 8     # row 7 of R1 referenced only by the first half
    k1[k1 == 11] = 12                     # row 11 never referenced: dropped everywhere
    k2 = rng.integers(1, n_r2 + 1, size=n)
    return s, [(k1, rng.random((n_r1, 4))), (k2, rng.random((n_r2, 3)))], rng


def _worker(rank, world, port, q):
    try:
        sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
        import factorla_oracle as O

        from paper_1612_07448_b200 import dist as D
        from paper_1612_07448_b200.ml import TrainConfig

        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        be = OracleBackend()
        s, parts, rng = _data()
        n = s.shape[0]
        r0, r1 = D.shard_range(n, rank, world)
        sm = D.build_star(s[r0:r1], [(k[r0:r1], r) for k, r in parts], n, backend=be)
        ref = O.build_star(s, parts)
        # same kept rows and remap as the unsharded build
        for i, (t, rk) in enumerate(sm.local.parts):
            np.testing.assert_array_equal(t, ref.parts[i][0][r0:r1])
            np.testing.assert_array_equal(rk, ref.parts[i][1])
        d = ref.d

        def close(a, b, tol=TOL):
            a = np.asarray(a.numpy() if isinstance(a, torch.Tensor) else a, dtype=np.float64)
            b = np.asarray(b, dtype=np.float64)
            assert a.shape == b.shape, (a.shape, b.shape)
            assert O.max_rel_deviation(a, b) <= tol, O.max_rel_deviation(a, b)

        x = rng.standard_normal((d, 3))
        close(D.lmm(sm, x), O.lmm(ref, x)[r0:r1])
        p = rng.standard_normal((n, 2))
        close(D.tmm(sm, p[r0:r1]), O.lmm(ref.T, p))
        close(D.rmm(p[r0:r1].T.copy(), sm), O.rmm(p.T, ref))
        close(D.row_sums(sm), O.row_sums(ref)[r0:r1])
        close(D.col_sums(sm), O.col_sums(ref))
        assert abs(D.sum_all(sm) - O.sum_all(ref)) <= TOL * abs(O.sum_all(ref))
        cp = D.crossprod(sm)
        close(cp, O.crossprod(ref))
        assert torch.equal(cp, cp.t())
        y = np.where(O.lmm(ref, rng.standard_normal((d, 1))) >= 0, 1.0, -1.0)
        out = D.logistic_gd(sm, y[r0:r1], TrainConfig(iterations=4, step_size=1e-3))
        w, obj = O.logistic_gd(ref, y, 4, 1e-3)
        close(out.weights, w)
        close(out.objective, obj)
        yl = O.lmm(ref, rng.standard_normal((d, 1))) + 0.01 * rng.standard_normal((n, 1))
        out = D.linreg_gd(sm, yl[r0:r1], TrainConfig(iterations=3, step_size=1e-5))
        w, obj = O.linreg_gd(ref, yl, 3, 1e-5)
        close(out.weights, w)
        out = D.linreg_normal(sm, yl[r0:r1])
        w, obj = O.linreg_normal(ref, yl)
        close(out.weights, w, 1e-8)
        out = D.kmeans(sm, TrainConfig(iterations=4, k=5, rng_seed=2))
        c, obj, _ = O.kmeans(ref, 5, 4, 2)
        close(out.centroids, c)
        close(out.objective, obj)
        out = D.gnmf(sm, TrainConfig(iterations=3, r=2, rng_seed=4))
        w, h, obj = O.gnmf(ref, 2, 3, 4)
        close(out.factors[0], w[r0:r1])
        close(out.factors[1], h)
        close(out.objective, obj)
        # a PK-FK matrix: the R-sliced crossprod (KᵀS reduce-scatter + R-slice pass)
        pk = D.build_pkfk(s[r0:r1], parts[0][0][r0:r1], parts[0][1], n, backend=be)
        rpk = O.build_pkfk(s, parts[0][0], parts[0][1])
        cp = D.crossprod(pk)
        close(cp, O.crossprod(rpk))
        assert torch.equal(cp, cp.t())
        close(D.col_sums(pk), O.col_sums(rpk))
        close(D.lmm(pk, x[:rpk.d]), O.lmm(rpk, x[:rpk.d])[r0:r1])
        # the split passes really ran (not the replicated fallback)
        assert be.calls["lmm_zpass"] > 0 and be.calls["wt_spass"] > 0 and be.calls["crossprod_rpass"] > 0, be.calls
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc()))


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def test_shard_range_partitions_rows():
    from paper_1612_07448_b200.dist import shard_range

    for n in (0, 1, 7, 1000, 20_000_000):
        for world in (1, 2, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_match_unsharded_oracle(world):
    """world 3: R slices of unequal length (97 and 40 kept rows over 3 ranks)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=280) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert res == {r: "ok" for r in range(world)}, res

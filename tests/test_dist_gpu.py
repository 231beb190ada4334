"""World-size-2 run of the DEVICE backend (paper_1612_07448_b200.dist.DeviceBackend) on one GPU.

Two ranks share cuda:0 over ``gloo`` (the driver's GPU box has one GPU): every local step runs
the sm_100a kernels — including the R-row-sliced split passes (fb_lmm_zpass / fb_lmm_spass,
fb_wt_spass + fb_rows_wt, fb_crossprod_spass / fb_crossprod_rpass) — and the collectives
(all-gather of z, reduce-scatter of the bins and KᵀS, all-reduce of small results) are the
same calls the NCCL path makes. Each sharded result is compared with the unsharded oracle.
The ranks' kernels never wait on one another (gloo collectives are host-side), so sharing a
GPU is a functional test, not a stand-in for NVLink timing.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-9


def _worker(rank, world, port, q):
    try:
        sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
        import torch
        import torch.distributed as dist

        import factorla_oracle as O
        import paper_1612_07448_b200 as fb
        from paper_1612_07448_b200 import dist as D

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        rng = np.random.default_rng(17)
        n, n_r1, n_r2 = 60_001, 1_001, 97
        s = rng.standard_normal((n, 20))
        k1 = rng.integers(1, n_r1 + 1, size=n)
        k1[k1 == 7] = 8  # an unreferenced row: dropped on every rank
        k2 = rng.integers(1, n_r2 + 1, size=n)
        r1, r2 = rng.standard_normal((n_r1, 40)), rng.standard_normal((n_r2, 6))
        r0_, r1_ = D.shard_range(n, rank, world)

        def close(a, b, tol=TOL, what=""):
            a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
            assert a.shape == np.asarray(b).shape, (what, a.shape, np.asarray(b).shape)
            dev = O.max_rel_deviation(a, b)
            assert dev <= tol, (what, dev)

        launches0 = fb.launch_count()
        # PK-FK: every operator through the R-sliced composition
        pk = D.build_pkfk(s[r0_:r1_], k1[r0_:r1_], r1, n)
        ref = O.build_pkfk(s, k1, r1)
        d = ref.d
        for dx in (1, 5, 16):
            x = rng.standard_normal((d, dx))
            close(D.lmm(pk, x), O.lmm(ref, x)[r0_:r1_], what=f"lmm{dx}")
        p = rng.standard_normal((n, 3))
        close(D.tmm(pk, p[r0_:r1_]), O.lmm(ref.T, p), what="tmm")
        close(D.rmm(np.ascontiguousarray(p[r0_:r1_].T), pk), O.rmm(p.T, ref), what="rmm")
        close(D.row_sums(pk), O.row_sums(ref)[r0_:r1_], what="row_sums")
        close(D.col_sums(pk), O.col_sums(ref), what="col_sums")
        assert abs(D.sum_all(pk) - O.sum_all(ref)) <= TOL * abs(O.sum_all(ref))
        cp = D.crossprod(pk)
        close(cp, O.crossprod(ref), what="crossprod")
        assert bool((cp == cp.t()).all())
        out = D.gnmf(D.build_pkfk(np.abs(s[r0_:r1_]), k1[r0_:r1_], np.abs(r1), n), fb.TrainConfig(iterations=3, r=4))
        w, h, obj = O.gnmf(O.build_pkfk(np.abs(s), k1, np.abs(r1)), 4, 3, 0)
        close(out.factors[0], w[r0_:r1_], what="gnmf W")
        close(out.factors[1], h, what="gnmf H")
        # star: LMM / Tᵀ·P split, crossprod replicated, drivers
        st = D.build_star(s[r0_:r1_], [(k1[r0_:r1_], r1), (k2[r0_:r1_], r2)], n)
        rs = O.build_star(s, [(k1, r1), (k2, r2)])
        x = rng.standard_normal((rs.d, 4))
        close(D.lmm(st, x), O.lmm(rs, x)[r0_:r1_], what="star lmm")
        close(D.tmm(st, p[r0_:r1_]), O.lmm(rs.T, p), what="star tmm")
        close(D.crossprod(st), O.crossprod(rs), what="star crossprod")
        y = np.where(O.lmm(rs, rng.standard_normal((rs.d, 1))) >= 0, 1.0, -1.0)
        out = D.logistic_gd(st, y[r0_:r1_], fb.TrainConfig(iterations=4, step_size=1e-4))
        w, obj = O.logistic_gd(rs, y, 4, 1e-4)
        close(out.weights, w, what="logreg")
        out = D.kmeans(st, fb.TrainConfig(iterations=3, k=5, rng_seed=1))
        c, obj, _ = O.kmeans(rs, 5, 3, 1)
        close(out.centroids, c, what="kmeans")
        assert fb.launch_count() > launches0
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc()))


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


@pytest.mark.timeout(600)
def test_device_backend_two_ranks_one_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=580) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert res == {0: "ok", 1: "ok"}, res

"""Benchmark of the factorized-LA hot path (BASELINE.json configs[1], "c2").

One step = the c2 memory-bound operator suite over the device-resident normalized matrix
T = [S, K·R] (S 20,000,000×20, R 1,000,000×80 float64 ~N(0,1), FK int32 uniform):
LMM with X 100×1, LMM with X 100×16, RMM with X 1×n_S, rowSums, colSums.
``value`` = algorithmic bytes of the suite (every input and output byte once)
÷ device time, summed over ranks (GB/s). S is 3.2 GB per rank, far larger than the 126 MB
L2, so no flush is needed between steps.

``--impl reference`` times the CPU restatement of the reference (oracle/factorla_oracle.py,
same NumPy/SciPy/OpenBLAS primitives as factorla) on a bounded sample of the same workload.

Multi-GPU (torchrun): S/FK rows are sharded (each rank holds its own 20M-row shard: weak
scaling), R is replicated; RMM and colSums partials are combined with an NCCL all-reduce.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2 = dict(n_s=20_000_000, d_s=20, n_r=1_000_000, d_r=80)
HBM_PEAK_FALLBACK = 6650.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback"


def op_bytes(n_s, d_s, n_r, d_r):
    """Algorithmic bytes per operator (inputs + outputs once; z/bins intermediates excluded)."""
    d = d_s + d_r
    fac = 8 * (n_s * d_s + n_r * d_r)
    fk = 4 * n_s
    return {
        "lmm_x1": fac + fk + 8 * (d + n_s),
        "lmm_x16": fac + fk + 8 * (16 * d + 16 * n_s),
        "rmm_x1": fac + fk + 8 * (n_s + d),
        "row_sums": fac + fk + 8 * n_s,
        "col_sums": fac + 8 * (n_r + d),  # cached counts (indicator.py:61-66) replace the FK read
    }


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                rows.append((float(f[0]), float(f[1]), f[3:7], float(f[7]) if f[7] not in ("[N/A]", "") else 0.0))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        loaded = [r for r in rows if r[3] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in loaded])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded)}


# ----------------------------------------------------------------------------- CPU arms
def _cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_suite(frac=0.25, reps=1, seed=0):
    """Time the oracle port (the reference's algorithm on NumPy/SciPy/OpenBLAS) on a c2 sample.

    The sample keeps c2's widths and tuple ratio: n_S = frac·20M, n_R = frac·1M.
    Returns (GB/s over the suite, seconds per suite, sample description, per-op ms).
    """
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import factorla_oracle as O
    from threadpoolctl import threadpool_limits

    n_s, n_r = int(C2["n_s"] * frac), int(C2["n_r"] * frac)
    d_s, d_r = C2["d_s"], C2["d_r"]
    rng = np.random.default_rng(seed)
    s = rng.standard_normal((n_s, d_s))
    r = rng.standard_normal((n_r, d_r))
    key = rng.integers(1, n_r + 1, size=n_s, dtype=np.int64)
    threads = _cpu_threads()
    with threadpool_limits(threads):
        nm = O.build_pkfk(s, key, r)
        d = d_s + d_r
        x1 = rng.standard_normal((d, 1))
        x16 = rng.standard_normal((d, 16))
        xr = rng.standard_normal((1, n_s))
        cnt = O.counts(nm.parts[0][0], nm.parts[0][1].shape[0])  # cached like IndicatorMatrix.counts
        nm.k_csr(0)  # CSR cache built once, as the reference caches it (indicator.py:71-76)
        ops = {
            "lmm_x1": lambda: O.lmm(nm, x1),
            "lmm_x16": lambda: O.lmm(nm, x16),
            "rmm_x1": lambda: O.rmm(xr, nm),
            "row_sums": lambda: O.row_sums(nm),
            "col_sums": lambda: O.col_sums(nm),
        }
        del cnt
        for fn in ops.values():  # warm-up (bench._timed, bench.py:46-54)
            fn()
        per = {k: [] for k in ops}
        for _ in range(reps):
            for k, fn in ops.items():
                t0 = time.perf_counter()
                fn()
                per[k].append(time.perf_counter() - t0)
    nb = op_bytes(n_s, d_s, nm.parts[0][1].shape[0], d_r)
    ms = {k: 1e3 * float(np.median(v)) for k, v in per.items()}
    sec = sum(ms.values()) / 1e3
    gbs = sum(nb.values()) / sec / 1e9
    sample = f"c2 sample n_S={n_s:,} d_S={d_s}, n_R={n_r:,} d_R={d_r} (1/{int(1/frac)} of rows, same widths and tuple ratio)"
    return gbs, sec, sample, threads, {k: round(v, 3) for k, v in ms.items()}


def run_reference(args, rank, world):
    if rank != 0:
        return
    steps = []
    sample = threads = ms = None
    for i in range(args.warmup + args.steps):
        gbs, sec, sample, threads, ms = cpu_suite(frac=args.cpu_frac, reps=1, seed=i)
        if i >= args.warmup:
            steps.append((gbs, sec))
    gbs = float(np.median([g for g, _ in steps]))
    sec = float(np.median([s for _, s in steps]))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sec, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c2 memory-bound operator suite (LMM X100x1, LMM X100x16, RMM X1xn, rowSums, colSums)",
                   "sample": sample, "parallelism": "host BLAS threads"},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ops_ms": ms,
    }
    print(json.dumps(line), flush=True)


METRIC = "factorized c2 operator-suite algorithmic HBM throughput (LMM x1/x16, RMM, rowSums, colSums)"


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1612_07448_b200 as fb
    from paper_1612_07448_b200 import dist as fbd

    ngpu = max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank % ngpu)
    dev = torch.device("cuda", local_rank % ngpu)
    cfg = dict(C2)
    if args.small:
        cfg.update(n_s=cfg["n_s"] // 20, n_r=cfg["n_r"] // 20)
    n_s, d_s, n_r, d_r = cfg["n_s"], cfg["d_s"], cfg["n_r"], cfg["d_r"]
    d = d_s + d_r
    # synthetic c2 inputs, seeded: S shard per rank, R identical on every rank
    g_r = torch.Generator(device=dev).manual_seed(1234)
    g_s = torch.Generator(device=dev).manual_seed(1000 + rank)
    r = torch.randn(n_r, d_r, dtype=torch.float64, device=dev, generator=g_r)
    s = torch.randn(n_s, d_s, dtype=torch.float64, device=dev, generator=g_s)
    key = torch.randint(1, n_r + 1, (n_s,), dtype=torch.int64, device=dev, generator=g_s)
    # row-sharded build with the global key histogram (every rank keeps the same R rows)
    sm = fbd.build_pkfk(s, key, r, n_s * world)
    nm = sm.local
    del key
    n_r_kept = nm.r.shape[0]
    x1 = torch.randn(d, 1, dtype=torch.float64, device=dev, generator=g_r)
    x16 = torch.randn(d, 16, dtype=torch.float64, device=dev, generator=g_r)
    xr = torch.randn(1, n_s, dtype=torch.float64, device=dev, generator=g_s)
    nm.k.counts  # cache the counts (indicator.py:61-66) outside the timed region
    torch.cuda.synchronize()

    def allreduce(t):
        if world > 1:
            dist.all_reduce(t)
        return t

    # LMM / rowSums are row-local; RMM and colSums all-reduce a 1 × 100 partial (dist.py)
    ops = {
        "lmm_x1": lambda: fbd.lmm(sm, x1),
        "lmm_x16": lambda: fbd.lmm(sm, x16),
        "rmm_x1": lambda: fbd.rmm(xr, sm),
        "row_sums": lambda: fbd.row_sums(sm),
        "col_sums": lambda: fbd.col_sums(sm),
    }
    nb = op_bytes(n_s, d_s, n_r_kept, d_r)
    step_bytes = sum(nb.values())
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        for fn in ops.values():
            fn()
    barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    ev = {k: [] for k in ops}
    launches0 = fb.launch_count()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    barrier()
    start.record(stream)
    for _ in range(args.steps):
        for k, fn in ops.items():
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            ev[k].append((a, b))
    stop.record(stream)
    barrier()
    launches = fb.launch_count() - launches0
    clocks = sampler.stop()
    total_ms = start.elapsed_time(stop)
    op_ms = {k: float(np.mean([a.elapsed_time(b) for a, b in v])) for k, v in ev.items()}
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = world * step_bytes / (ms_step * 1e-3) / 1e9

    # e2e: the public API with host operands (pinned), result read back to host each step
    pin = lambda a: a.cpu().pin_memory()
    hx1, hx16, hxr = pin(x1), pin(x16), pin(xr)
    # rowSums of a device-resident T returns a device vector: read it back into page-locked
    # memory (a pageable .cpu() of 160 MB costs ~75 ms of first-touch faults, not PCIe time)
    hrs = torch.empty((n_s, 1), dtype=torch.float64, pin_memory=True)
    e2e_ops = {
        "lmm_x1": lambda: fb.lmm(nm, hx1),
        "lmm_x16": lambda: fb.lmm(nm, hx16),
        "rmm_x1": lambda: _host_allreduce(fb.rmm(hxr, nm), world, dev),
        "row_sums": lambda: (hrs.copy_(fb.row_sums(nm).reshape(n_s, 1), non_blocking=True),
                             torch.cuda.current_stream().synchronize()),
        "col_sums": lambda: _host_allreduce(fb.col_sums(nm).cpu(), world, dev),
    }
    h2d = 8 * (x1.numel() + x16.numel() + xr.numel())
    d2h = 8 * (n_s * 1 + n_s * 16 + d + n_s + d)
    for fn in e2e_ops.values():
        fn()
    barrier()
    e2e_steps = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        for fn in e2e_ops.values():
            fn()
    barrier()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = world * step_bytes / float(te.item()) / 1e9

    peak, peak_kind = _peaks()
    top = max(op_ms, key=op_ms.get)
    achieved = nb[top] / (op_ms[top] * 1e-3) / 1e9
    traffic = _traffic_from_profile(top)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gbs, sec, sample, threads, ms = cpu_suite(frac=args.cpu_frac, reps=1)
        cpu = {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample,
               "ops_ms": ms}
    extras = None
    if rank == 0 and world == 1 and not args.no_extras:
        extras = run_extras(dev, cpu=not args.no_cpu)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded torch RNG on device: N(0,1) S and R, uniform FK)",
            "config": {"workload": "c2 memory-bound operator suite (BASELINE.json configs[1]): LMM X100x1, LMM X100x16, "
                                   "RMM X1xn_S, rowSums, colSums",
                       "n_s_per_gpu": n_s, "d_s": d_s, "n_r": n_r_kept, "d_r": d_r,
                       "parallelism": f"row-sharded S/FK over {world} GPU(s), R replicated",
                       "l2": "no flush: S alone is 3.2 GB per GPU (> 126 MB L2)",
                       "bytes_per_step": step_bytes},
            "ops": {k: {"ms": round(op_ms[k], 4), "GBps": round(nb[k] / op_ms[k] / 1e6, 1),
                        "frac": round(nb[k] / op_ms[k] / 1e6 / peak, 3)} for k in ops},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": f"fb_{top} (op-level: R-side z/bins pass + fused S pass)",
                         "peak_kind": peak_kind, "algorithmic_bytes": nb[top]},
            "e2e": {"value": round(e2e_val, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "note": "public API with pinned host X, results returned to host"},
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clocks,
            "extras": extras,
        }
        print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- secondary workloads
def _events_ms(fn, reps, stream=None):
    import torch

    st = stream or torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def dgemm_peak_tflops():
    """cuBLAS DGEMM 8192³ (best of 5) — the FP64 tensor roofline denominator for crossprod."""
    import torch

    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.mm(a, b)
    torch.cuda.synchronize()
    best = min(_events_ms(lambda: torch.mm(a, b), 1) for _ in range(5))
    del a, b
    return 2 * n**3 / (best * 1e-3) / 1e12


def zipf_keys_dev(n, n_r, s, gen, dev):
    import torch

    p = torch.arange(1, n_r + 1, dtype=torch.float64, device=dev) ** (-s)
    cdf = torch.cumsum(p / p.sum(), 0)
    u = torch.rand(n, dtype=torch.float64, device=dev, generator=gen)
    return torch.clamp(torch.searchsorted(cdf, u, right=True), max=n_r - 1) + 1


def _slope(run, trials=3):
    """Per-iteration wall time of a driver: median over trials of (wall(20) - wall(1)) / 19."""
    pers, last = [], None
    for _ in range(trials):
        r1 = run(1)
        last = run(20)
        pers.append((last.wall_time_s - r1.wall_time_s) / 19)
    pers.sort()
    return pers[len(pers) // 2], last


def run_extras(dev, cpu=True):
    """c3 crossprod + LinReg normal, c1 LogReg iter/s, c4 K-Means, c5 GNMF (BASELINE.json configs)."""
    import torch

    import paper_1612_07448_b200 as fb

    out = {}
    g = torch.Generator(device=dev).manual_seed(7)
    peak_fp64 = dgemm_peak_tflops()
    out["fp64_dgemm_peak_tflops"] = round(peak_fp64, 2)
    # ---- c3: crossprod + linreg_normal (S 10M×60, R 500k×120 U[0,1))
    n_s, d_s, n_r, d_r = 10_000_000, 60, 500_000, 120
    s = torch.rand(n_s, d_s, dtype=torch.float64, device=dev, generator=g)
    r = torch.rand(n_r, d_r, dtype=torch.float64, device=dev, generator=g)
    key = torch.randint(1, n_r + 1, (n_s,), device=dev, generator=g)
    nm = fb.build_pkfk(s, key, r)
    del key
    from paper_1612_07448_b200.crossprod_impl import fk_sorted_order

    fk_sorted_order(nm.k)  # one-time cache (the reference caches _csr_t the same way)
    flops = 2 * (0.5 * n_s * d_s * d_s + 0.5 * n_r * d_r * d_r + d_s * d_r * n_r)  # costmodel.py:85-88
    nbytes = 8 * (n_s * d_s + n_r * d_r) + 4 * n_s + 8 * (d_s + d_r) ** 2
    for _ in range(2):
        fb.crossprod(nm)
    ms = _events_ms(lambda: fb.crossprod(nm), 5)
    out["c3_crossprod"] = {"ms": round(ms, 3), "TFLOPs": round(flops / ms / 1e9, 2),
                           "frac_fp64_peak": round(flops / ms / 1e9 / peak_fp64, 3),
                           "GBps": round(nbytes / ms / 1e6, 1), "algorithmic_gflop": round(flops / 1e9, 2)}
    w = torch.randn(d_s + d_r, 1, dtype=torch.float64, device=dev, generator=g)
    y = fb.lmm(nm, w) + 0.01 * torch.randn(n_s, 1, dtype=torch.float64, device=dev, generator=g)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = fb.linreg_normal(nm, y)
    out["c3_linreg_normal"] = {"s": round(time.perf_counter() - t0, 4), "objective": res.objective[0],
                               "note": "noise N(0, 0.01^2) (σ = 0.01)"}
    del nm, s, r, y
    torch.cuda.empty_cache()
    # ---- c1: LogReg GD, 20 iterations (S 100k×20, R 10k×40 N(0,1)), step 1e-3
    n_s, d_s, n_r, d_r = 100_000, 20, 10_000, 40
    rng = np.random.default_rng(1)
    s1 = rng.standard_normal((n_s, d_s))
    r1 = rng.standard_normal((n_r, d_r))
    k1 = rng.integers(1, n_r + 1, size=n_s)
    nm = fb.build_pkfk(torch.from_numpy(s1).to(dev), torch.from_numpy(k1).to(dev), torch.from_numpy(r1).to(dev))
    wt = rng.standard_normal((d_s + d_r, 1))
    y1 = torch.from_numpy(np.where(fb.lmm(nm, torch.from_numpy(wt).to(dev)).cpu().numpy() >= 0, 1.0, -1.0)).to(dev)
    cfg = fb.TrainConfig(iterations=20, step_size=1e-3)
    fb.logistic_gd(nm, y1, cfg)
    walls = [fb.logistic_gd(nm, y1, cfg).wall_time_s for _ in range(5)]
    out["c1_logreg"] = {"iter_per_s": round(20 / float(np.median(walls)), 1), "ms_per_iter": round(1e3 * float(np.median(walls)) / 20, 4),
                        "timing": "wall clock over 20 iterations incl. the final device->host read"}
    if cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import factorla_oracle as O
        from threadpoolctl import threadpool_limits

        with threadpool_limits(_cpu_threads()):
            ref = O.build_pkfk(s1, k1, r1)
            y1h = y1.cpu().numpy()
            O.logistic_gd(ref, y1h, 2, 1e-3)
            t0 = time.perf_counter()
            O.logistic_gd(ref, y1h, 20, 1e-3)
            out["c1_logreg"]["cpu_iter_per_s"] = round(20 / (time.perf_counter() - t0), 1)
            out["c1_logreg"]["cpu_cores"] = _cpu_threads()
    # ---- c4: K-Means k=10, 20 iterations, star schema (S 10M×20, R1 1M×40, R2 100k×60)
    n_s = 10_000_000
    s = torch.randn(n_s, 20, dtype=torch.float64, device=dev, generator=g)
    r1t = torch.randn(1_000_000, 40, dtype=torch.float64, device=dev, generator=g)
    r2t = torch.randn(100_000, 60, dtype=torch.float64, device=dev, generator=g)
    k1t = torch.randint(1, 1_000_001, (n_s,), device=dev, generator=g)
    k2t = torch.randint(1, 100_001, (n_s,), device=dev, generator=g)
    nm = fb.build_star(s, [(k1t, r1t), (k2t, r2t)])
    del k1t, k2t
    fb.kmeans(nm, fb.TrainConfig(iterations=2, k=10, rng_seed=0))  # warm: workspaces, kernel attributes
    per, res = _slope(lambda it: fb.kmeans(nm, fb.TrainConfig(iterations=it, k=10, rng_seed=0)))
    out["c4_kmeans"] = {"iter_per_s": round(1 / per, 1), "ms_per_iter": round(1e3 * per, 3),
                        "s_total_20_iters": round(res.wall_time_s, 4),
                        "timing": "per iteration = median over 3 trials of (wall(20 iters) - wall(1 iter)) / 19; total incl. seeding and rowSums(T²)"}
    del nm, s, r1t, r2t
    torch.cuda.empty_cache()
    # ---- c5: GNMF r=5, 20 iterations, Zipf(1.2) FK (S 5M×10, R 50k×40 U[0,1))
    n_s, n_r = 5_000_000, 50_000
    s = torch.rand(n_s, 10, dtype=torch.float64, device=dev, generator=g)
    r = torch.rand(n_r, 40, dtype=torch.float64, device=dev, generator=g)
    key = zipf_keys_dev(n_s, n_r, 1.2, g, dev)
    nm = fb.build_pkfk(s, key, r)
    fb.gnmf(nm, fb.TrainConfig(iterations=2, r=5, rng_seed=0))  # warm: workspaces, sorted order, attributes
    per, res = _slope(lambda it: fb.gnmf(nm, fb.TrainConfig(iterations=it, r=5, rng_seed=0)))
    out["c5_gnmf"] = {"iter_per_s": round(1 / per, 1), "ms_per_iter": round(1e3 * per, 3),
                      "s_total_20_iters": round(res.wall_time_s, 4), "kept_r_rows": int(nm.r.shape[0]),
                      "timing": "per iteration = median over 3 trials of (wall(20 iters) - wall(1 iter)) / 19; total incl. the host "
                                "RNG draw of W (5M×5, the reference's default_rng call) and its upload"}
    del nm, s, r, key
    torch.cuda.empty_cache()
    return out


def _host_allreduce(t, world, dev):
    if world > 1:
        import torch
        import torch.distributed as dist

        d = torch.as_tensor(t).to(dev)
        dist.all_reduce(d)
        return d.cpu().numpy()
    return t


def _traffic_from_profile(op):
    """dram bytes per launch from the committed ncu --set full summary, if present."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(op)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-frac", type=float, default=0.25)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--small", action="store_true", help="1/20 of c2 (development only)")
    ap.add_argument("--no-extras", action="store_true", help="skip the c1/c3/c4/c5 secondary workloads")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = os.environ.get("FB_DIST_BACKEND", "nccl")  # gloo: functional check with ranks sharing a GPU
        ngpu = max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank % ngpu)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank % ngpu))
        else:
            dist.init_process_group(backend)
    try:
        run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()

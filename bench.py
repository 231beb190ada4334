"""Benchmark of the factorized-LA hot path (BASELINE.json configs[1], "c2").

One step = the c2 memory-bound operator suite over the device-resident normalized matrix
T = [S, K·R] (S 20,000,000×20, R 1,000,000×80 float64 ~N(0,1), FK int32 uniform):
LMM with X 100×1, LMM with X 100×16, RMM with X 1×n_S, rowSums, colSums.
``value`` = algorithmic bytes of the suite (every input and output byte once)
÷ device time (GB/s), for the whole job. Inputs are the seeded NumPy draws of
``workloads.py``, generated on the host and uploaded before timing. S is
3.2 GB (> the 126 MB L2), so no flush is needed between steps.

Multi-GPU (``--gpus N``: torchrun, or spawned by this script when WORLD_SIZE is unset):
strong scaling — the fixed 20M-row S and its FK column are row-sharded N ways (each rank
draws only its own rows, ``workloads.generate(lo, hi)``), R is replicated; the R-side work
is split by R-row slice with NCCL all-gather / reduce-scatter (paper_1612_07448_b200/dist.py).

``--impl reference`` times the reference's own CPU implementation of the same suite on the
same full c2 inputs: stock ``factorla`` (installed into baseline/_ref) when importable,
else the pinned oracle port (oracle/factorla_oracle.py), on all host cores.

The default (N=1) run also reports, in ``parity``, the deviation of every GPU result from
the CPU reference on the same inputs (c2 suite, and c1/c3/c4/c5 in ``extras``), and the
CPU reference's own timings in ``cpu_baseline`` / ``extras``.
"""
import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

C2 = W.SHAPES["c2"]
HBM_PEAK_FALLBACK = 6650.0
TOL = 1e-9
METRIC = "factorized c2 operator-suite algorithmic HBM throughput (LMM x1/x16, RMM, rowSums, colSums)"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback (B200_PROFILING.md)"


def c2_config(world, n_r_kept):
    """The ``config`` object both arms print (identical for the same N)."""
    return {"workload": "c2 memory-bound operator suite (BASELINE.json configs[1]): LMM X100x1, LMM X100x16, "
                        "RMM X1xn_S, rowSums, colSums",
            "n_s": C2["n_s"], "d_s": C2["d_s"], "n_r": n_r_kept, "d_r": C2["parts"][0][1],
            "inputs": f"workloads.py seeded NumPy draws (seed {W.SEEDS['c2']}): S, R ~N(0,1), FK uniform int32",
            "parallelism": f"dp{world}: S/FK rows sharded {world} way(s), R replicated, R-side work split by R-row slice",
            "l2": "no flush: S alone is 3.2 GB (> 126 MB L2)"}


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


# ----------------------------------------------------------------------------- the CPU reference
def _cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class CpuReference:
    """The reference's CPU path: stock ``factorla`` from baseline/_ref when it imports (kind
    "reference"), else the pinned oracle port (kind "port"). Same calls either way."""

    def __init__(self):
        self.kind, self.fl, self.O = "port", None, None
        ref_dir = os.path.join(ROOT, "baseline", "_ref")
        if os.path.isdir(os.path.join(ref_dir, "factorla")):
            sys.path.insert(0, ref_dir)
            try:
                import factorla

                if os.path.abspath(factorla.__file__).startswith(os.path.abspath(ref_dir)):
                    self.fl, self.kind = factorla, "reference"
            except Exception:
                self.fl = None
        if self.fl is None:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import factorla_oracle as O

            self.O = O
        self.cores = _cpu_threads()
        from threadpoolctl import threadpool_limits

        self._limits = threadpool_limits(self.cores)  # all host cores for the BLAS calls

    @property
    def name(self):
        if self.fl is not None:
            return f"stock factorla {getattr(self.fl, '__version__', '?')} (baseline/_ref, pip-installed /root/reference/pkg)"
        return "oracle/factorla_oracle.py (CPU restatement of factorla, pinned to its golden vectors)"

    def build(self, g):
        parts = W.keys_1based(g["parts"])
        if self.fl is not None:
            if len(parts) == 1:
                return self.fl.build_pkfk(g["s"], parts[0][0], parts[0][1])
            return self.fl.build_star(g["s"], parts)
        if len(parts) == 1:
            return self.O.build_pkfk(g["s"], parts[0][0], parts[0][1])
        return self.O.build_star(g["s"], parts)

    def prepare(self, nm):
        """One-time caches the reference builds on first use (counts, CSR of K: indicator.py:61-86)."""
        if self.fl is not None:
            for ind, _ in nm.blocks[1:]:
                ind.counts
                ind._csr
                ind._csr_t
        else:
            for i, (t, r) in enumerate(nm.parts):
                self.O.counts(t, r.shape[0])
                nm.k_csr(i)

    def op(self, name, nm, *a):
        m = self.fl if self.fl is not None else self.O
        return getattr(m, name)(*a) if name in ("rmm",) else getattr(m, name)(nm, *a)

    def logistic_gd(self, nm, y, iters, step):
        if self.fl is not None:
            out = self.fl.logistic_gd(nm, y, self.fl.TrainConfig(iterations=iters, step_size=step))
            return out.weights, out.objective
        return self.O.logistic_gd(nm, y, iters, step)

    def linreg_normal(self, nm, y):
        if self.fl is not None:
            out = self.fl.linreg_normal(nm, y)
            return out.weights, out.objective
        return self.O.linreg_normal(nm, y)

    def kmeans(self, nm, k, iters, seed):
        if self.fl is not None:
            out = self.fl.kmeans(nm, self.fl.TrainConfig(iterations=iters, k=k, rng_seed=seed))
            return out.centroids, out.objective
        c, tr, _ = self.O.kmeans(nm, k, iters, seed)
        return c, tr

    def gnmf(self, nm, r, iters, seed):
        if self.fl is not None:
            out = self.fl.gnmf(nm, self.fl.TrainConfig(iterations=iters, r=r, rng_seed=seed))
            return out.factors[0], out.factors[1], out.objective
        return self.O.gnmf(nm, r, iters, seed)


def max_rel_deviation(a, b):
    """Normwise max|a−b| / max|b| (reference bench.py:38-43)."""
    a = np.asarray(a.cpu().numpy() if hasattr(a, "cpu") else a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return float("inf")
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-30)
    return float(np.max(np.abs(a - b)) / scale) if a.size else 0.0


def _c2_ops_cpu(ref, nm, g):
    return {
        "lmm_x1": lambda: ref.op("lmm", nm, g["x1"]),
        "lmm_x16": lambda: ref.op("lmm", nm, g["x16"]),
        "rmm_x1": lambda: ref.op("rmm", None, g["xr"], nm),
        "row_sums": lambda: ref.op("row_sums", nm),
        "col_sums": lambda: ref.op("col_sums", nm),
    }


def cpu_suite(ref, g, reps=1, keep=False):
    """Time the c2 suite on the CPU reference (warm-up suite, then median of ``reps``)."""
    nm = ref.build(g)
    ref.prepare(nm)
    ops = _c2_ops_cpu(ref, nm, g)
    outs = {}
    for k, fn in ops.items():  # warm-up (bench._timed, reference bench.py:46-54)
        r = fn()
        if keep:
            outs[k] = r
    per = {k: [] for k in ops}
    for _ in range(reps):
        for k, fn in ops.items():
            t0 = time.perf_counter()
            fn()
            per[k].append(time.perf_counter() - t0)
    n_r = nm.blocks[1][1].shape[0] if ref.fl is not None else nm.parts[0][1].shape[0]
    return {k: float(np.median(v)) for k, v in per.items()}, outs, n_r


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU suite on the full c2 inputs (rank 0 only)."""
    if rank != 0:
        return
    ref = CpuReference()
    g = W.generate("c2")
    nm = ref.build(g)
    ref.prepare(nm)
    n_r = nm.blocks[1][1].shape[0] if ref.fl is not None else nm.parts[0][1].shape[0]
    nb = W.algorithmic_bytes_c2(C2["n_s"], C2["d_s"], n_r, C2["parts"][0][1])
    ops = _c2_ops_cpu(ref, nm, g)
    secs, per = [], {k: [] for k in ops}
    for i in range(args.warmup + args.steps):
        tot = 0.0
        for k, fn in ops.items():
            t0 = time.perf_counter()
            fn()
            dt = time.perf_counter() - t0
            tot += dt
            if i >= args.warmup:
                per[k].append(dt)
        if i >= args.warmup:
            secs.append(tot)
    sec = float(np.median(secs))
    gbs = sum(nb.values()) / sec / 1e9
    sample = f"full c2 (n_S={C2['n_s']:,}, n_R={n_r:,}), every step the whole suite; {ref.name}"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sec, 3),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (workloads.py seeded NumPy draws, SURVEY.md §8(d))",
        "config": c2_config(world, n_r),
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": ref.cores, "kind": ref.kind,
                         "sample": sample},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ops_ms": {k: round(1e3 * float(np.median(v)), 3) for k, v in per.items()},
        "note": "host BLAS threads = all cores; SciPy sparse products, take and ufuncs are single-threaded "
                "in the reference",
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
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


def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1612_07448_b200 as fb
    from paper_1612_07448_b200 import dist as fbd

    ngpu = max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank % ngpu)
    dev = torch.device("cuda", local_rank % ngpu)
    n_global = C2["n_s"]
    lo, hi = fbd.shard_range(n_global, rank, world)
    g = W.generate("c2", lo, hi)  # this rank's rows; R and X are the same draws on every rank
    (fk, r_h), = g["parts"]
    s = torch.from_numpy(g["s"]).to(dev)
    key = torch.from_numpy(fk).to(dev).to(torch.int64) + 1
    r = torch.from_numpy(r_h).to(dev)
    torch.cuda.synchronize()
    t_b = time.perf_counter()
    sm = fbd.build_pkfk(s, key, r, n_global)
    torch.cuda.synchronize()
    one_time = {"build_pkfk_ms": round((time.perf_counter() - t_b) * 1e3, 2)}
    del key
    nm = sm.local
    t_b = time.perf_counter()
    nm.ensure_sorted()
    torch.cuda.synchronize()
    one_time["fk_sort_ms"] = round((time.perf_counter() - t_b) * 1e3, 2)
    one_time["note"] = ("wall clock, device-resident inputs, paid once per matrix: key check + used-row scan + remap + R "
                        "gather + counts (normmat.py:168-214), then the cached stable FK sort the Tᵀ-side operators "
                        "use (the reference's cached _csr_t, indicator.py:78-86)")
    n_r_kept = nm.r.shape[0]
    d_s, d_r = C2["d_s"], C2["parts"][0][1]
    x1 = torch.from_numpy(g["x1"]).to(dev)
    x16 = torch.from_numpy(g["x16"]).to(dev)
    xr = torch.from_numpy(g["xr"]).to(dev)
    nm.k.counts  # cache the counts (indicator.py:61-66) outside the timed region
    torch.cuda.synchronize()

    ops = {
        "lmm_x1": lambda: fbd.lmm(sm, x1),
        "lmm_x16": lambda: fbd.lmm(sm, x16),
        "rmm_x1": lambda: fbd.rmm(xr, sm),
        "row_sums": lambda: fbd.row_sums(sm),
        "col_sums": lambda: fbd.col_sums(sm),
    }
    nb = W.algorithmic_bytes_c2(n_global, d_s, n_r_kept, d_r)
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
    sampler = ClockSampler(local_rank % ngpu)
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
    t = torch.tensor([total_ms] + [op_ms[k] for k in ops], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t[0].item()) / args.steps
    op_ms = {k: float(t[i + 1].item()) for i, k in enumerate(ops)}
    value = step_bytes / (ms_step * 1e-3) / 1e9

    # parity of this run's results against the CPU reference on the same inputs (N = 1)
    parity, cpu = None, None
    ref = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ref = CpuReference()
        gpu_out = {k: _to_host(fn()) for k, fn in ops.items()}
        ms_cpu, outs, _ = cpu_suite(ref, g, reps=2, keep=True)
        parity = {"c2": {k: max_rel_deviation(gpu_out[k], outs[k]) for k in ops}}
        del gpu_out, outs
        sec = sum(ms_cpu.values())
        cpu = {"value": round(step_bytes / sec / 1e9, 3), "unit": "GB/s", "cores": ref.cores, "kind": ref.kind,
               "sample": f"full c2 suite, median of 2 after a warm-up suite; {ref.name}",
               "ops_ms": {k: round(1e3 * v, 3) for k, v in ms_cpu.items()}}

    # e2e: the public API with host operands (pinned), results read back to host each step
    pin = lambda a: a.cpu().pin_memory()
    hx1, hx16, hxr = pin(x1), pin(x16), pin(xr)
    # rowSums of a device-resident T returns a device vector: read it back into page-locked
    # memory (a pageable .cpu() of 160 MB costs ~75 ms of first-touch faults, not PCIe time)
    n_loc = hi - lo
    hrs = torch.empty((n_loc, 1), dtype=torch.float64, pin_memory=True)
    e2e_ops = {
        "lmm_x1": lambda: fb.lmm(nm, hx1),
        "lmm_x16": lambda: fb.lmm(nm, hx16),
        "rmm_x1": lambda: _to_host(fbd.rmm(hxr, sm)),
        "row_sums": lambda: (hrs.copy_(fb.row_sums(nm).reshape(n_loc, 1), non_blocking=True),
                             torch.cuda.current_stream().synchronize()),
        "col_sums": lambda: _to_host(fbd.col_sums(sm)),
    }
    d = d_s + d_r
    h2d = 8 * (x1.numel() + x16.numel() + xr.numel())
    d2h = 8 * (n_loc * 1 + n_loc * 16 + d + n_loc + d)
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
    e2e_val = step_bytes / float(te.item()) / 1e9

    peak, peak_kind = _peaks()
    top = max(op_ms, key=op_ms.get)
    achieved = nb[top] / (op_ms[top] * 1e-3) / 1e9
    traffic, traffic_src = _traffic_from_profile(top)
    del s, r, sm, nm, x16
    torch.cuda.empty_cache()
    extras = None
    if rank == 0 and world == 1 and not args.no_extras:
        extras = run_extras(dev, ref, parity)
    if rank == 0:
        if parity is not None:
            worst = max(v for c in parity.values() for v in c.values() if isinstance(v, float))
            parity["tol"] = TOL
            parity["reference"] = ref.name if ref else None
            parity["pass"] = bool(worst <= TOL) and all(
                c.get("assignments_equal", True) for c in parity.values() if isinstance(c, dict))
            parity["worst"] = worst
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (workloads.py seeded NumPy draws, SURVEY.md §8(d)), uploaded before timing",
            "config": c2_config(world, n_r_kept),
            "ops": {k: {"ms": round(op_ms[k], 4), "GBps": round(nb[k] / op_ms[k] / 1e6, 1),
                        "frac": round(nb[k] / op_ms[k] / 1e6 / peak, 3)} for k in ops},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak / world, 4), "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": f"fb_{top} (op-level: R-side z/bins pass + fused S pass)",
                         "peak_kind": peak_kind, "algorithmic_bytes": nb[top]},
            "e2e": {"value": round(e2e_val, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "note": "public API with pinned host X, results returned to host"},
            "cpu_baseline": cpu,
            "one_time": one_time,
            "parity": parity,
            "gpu_launches": launches,
            "clocks": clocks,
            "extras": extras,
        }
        print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- secondary workloads
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


def _loop_ms_per_iter(run, iters=20, trials=3):
    """Per-iteration device time of a driver's iteration loop: median over trials of the CUDA-event span the
    driver records around its loop (`ModelOutput.loop_ms`) / iterations. (Until the last session of round 2 this was
    a wall-clock slope, (wall(20) - wall(1)) / 19, whose two ~0.1 s host-side seeding / RNG terms made it jitter by
    +-0.2 ms per iteration between boxes.)"""
    pers, last = [], None
    for _ in range(trials):
        last = run(iters)
        pers.append(last.loop_ms * 1e-3 / iters)
    pers.sort()
    return pers[len(pers) // 2], last


def _build_gpu(fb, g, dev):
    import torch

    parts = [(torch.from_numpy(k).to(dev), torch.from_numpy(r).to(dev)) for k, r in W.keys_1based(g["parts"])]
    s = torch.from_numpy(g["s"]).to(dev)
    if len(parts) == 1:
        return fb.build_pkfk(s, parts[0][0], parts[0][1])
    return fb.build_star(s, parts)


def run_extras(dev, ref, parity):
    """c3 crossprod + LinReg normal, c1 LogReg, c4 K-Means, c5 GNMF (BASELINE.json configs):
    GPU timings, the CPU reference's timings on the same inputs, and parity."""
    import torch

    import paper_1612_07448_b200 as fb

    out = {}
    peak_fp64 = dgemm_peak_tflops()
    out["fp64_dgemm_peak_tflops"] = round(peak_fp64, 2)
    cpu = ref is not None

    def timed(fn):
        t0 = time.perf_counter()
        r = fn()
        return r, time.perf_counter() - t0

    # ---- c3: crossprod + linreg_normal (S 10M×60, R 500k×120 U[0,1))
    g = W.generate("c3")
    n_s, d_s = g["s"].shape
    n_r, d_r = g["parts"][0][1].shape
    nm = _build_gpu(fb, g, dev)
    nm.ensure_sorted()  # one-time FK-sorted order (the reference caches _csr_t the same way)
    flops = 2 * (0.5 * n_s * d_s * d_s + 0.5 * n_r * d_r * d_r + d_s * d_r * n_r)  # costmodel.py:85-88
    nbytes = 8 * (n_s * d_s + n_r * d_r) + 4 * n_s + 8 * (d_s + d_r) ** 2
    for _ in range(2):
        fb.crossprod(nm)
    ms = _events_ms(lambda: fb.crossprod(nm), 5)
    cp_gpu = fb.crossprod(nm).cpu().numpy()
    yd = torch.from_numpy(g["y"]).to(dev)
    fb.linreg_normal(nm, yd)
    lr = fb.linreg_normal(nm, yd)
    out["c3_crossprod"] = {"ms": round(ms, 3), "TFLOPs": round(flops / ms / 1e9, 2),
                           "frac_fp64_peak": round(flops / ms / 1e9 / peak_fp64, 3),
                           "GBps": round(nbytes / ms / 1e6, 1), "algorithmic_gflop": round(flops / 1e9, 2)}
    out["c3_linreg_normal"] = {"s": round(lr.wall_time_s, 4), "objective": lr.objective[0],
                               "note": "noise N(0, 0.01^2) (σ = 0.01)"}
    del nm, yd
    torch.cuda.empty_cache()
    if cpu:
        rn = ref.build(g)
        ref.prepare(rn)
        ref.op("crossprod", rn)  # warm-up
        cp_ref, t_cp = timed(lambda: ref.op("crossprod", rn))
        (w_ref, obj_ref), t_lr = timed(lambda: ref.linreg_normal(rn, g["y"]))
        out["c3_crossprod"]["cpu_ms"] = round(1e3 * t_cp, 1)
        out["c3_linreg_normal"]["cpu_s"] = round(t_lr, 3)
        parity["c3"] = {"crossprod": max_rel_deviation(cp_gpu, cp_ref),
                        "crossprod_symmetric": bool(np.array_equal(cp_gpu, cp_gpu.T)),
                        "linreg_w": max_rel_deviation(lr.weights, w_ref),
                        "linreg_objective": max_rel_deviation(lr.objective, obj_ref)}
        del rn
    del g
    # ---- c1: LogReg GD, 20 iterations (S 100k×20, R 10k×40 N(0,1)), step 1e-3
    g = W.generate("c1")
    nm = _build_gpu(fb, g, dev)
    y1 = torch.from_numpy(g["y"]).to(dev)
    cfg = fb.TrainConfig(iterations=g["iterations"], step_size=g["step"])
    fb.logistic_gd(nm, y1, cfg)
    runs = [fb.logistic_gd(nm, y1, cfg) for _ in range(5)]
    wall = float(np.median([r.wall_time_s for r in runs]))
    out["c1_logreg"] = {"iter_per_s": round(20 / wall, 1), "ms_per_iter": round(1e3 * wall / 20, 4),
                        "timing": "wall clock over 20 iterations incl. the final device->host read"}
    if cpu:
        rn = ref.build(g)
        ref.prepare(rn)
        ref.logistic_gd(rn, g["y"], 2, g["step"])
        (w_ref, tr_ref), t = timed(lambda: ref.logistic_gd(rn, g["y"], g["iterations"], g["step"]))
        out["c1_logreg"]["cpu_iter_per_s"] = round(g["iterations"] / t, 1)
        out["c1_logreg"]["cpu_cores"] = ref.cores
        parity["c1"] = {"logreg_w": max_rel_deviation(runs[-1].weights, w_ref),
                        "logreg_objective": max_rel_deviation(runs[-1].objective, tr_ref)}
    del nm, y1
    # ---- c4: K-Means k=10, star schema (S 10M×20, R1 1M×40, R2 100k×60)
    g = W.generate("c4")
    nm = _build_gpu(fb, g, dev)
    k, seed = g["k"], g["kmeans_seed"]
    fb.kmeans(nm, fb.TrainConfig(iterations=2, k=k, rng_seed=seed))  # warm: workspaces, kernel attributes
    per, res = _loop_ms_per_iter(lambda it: fb.kmeans(nm, fb.TrainConfig(iterations=it, k=k, rng_seed=seed)))
    out["c4_kmeans"] = {"iter_per_s": round(1 / per, 1), "ms_per_iter": round(1e3 * per, 3),
                        "s_total_20_iters": round(res.wall_time_s, 4),
                        "timing": "per iteration = median over 3 trials of the 20-iteration loop's CUDA-event span "
                                  "/ 20 (ModelOutput.loop_ms); total = wall clock incl. seeding and rowSums(T²)"}
    # the same star schema's crossprod (d = 120): per-part fused passes + pair-count cross blocks
    for _ in range(2):
        fb.crossprod(nm)
    ms_cp4 = _events_ms(lambda: fb.crossprod(nm), 5)
    cp4 = fb.crossprod(nm).cpu().numpy()
    out["c4_star_crossprod"] = {"ms": round(ms_cp4, 3), "d": int(cp4.shape[0])}
    if cpu:
        it_c = 3
        gpu3 = fb.kmeans(nm, fb.TrainConfig(iterations=it_c, k=k, rng_seed=seed))
        rn = ref.build(g)
        ref.prepare(rn)
        _, t1 = timed(lambda: ref.kmeans(rn, k, 1, seed))
        (c_ref, tr_ref), t3 = timed(lambda: ref.kmeans(rn, k, it_c, seed))
        out["c4_kmeans"]["cpu_ms_per_iter"] = round(1e3 * (t3 - t1) / (it_c - 1), 1)
        out["c4_kmeans"]["cpu_timing"] = f"(wall({it_c} iters) - wall(1 iter)) / {it_c - 1}"
        parity["c4"] = {f"centroids_{it_c}_iters": max_rel_deviation(gpu3.centroids, c_ref),
                        f"objective_{it_c}_iters": max_rel_deviation(gpu3.objective, tr_ref)}
        cp4_ref, t_cp4 = timed(lambda: ref.op("crossprod", rn))
        out["c4_star_crossprod"]["cpu_ms"] = round(1e3 * t_cp4, 1)
        parity["c4"]["star_crossprod"] = max_rel_deviation(cp4, cp4_ref)
        parity["c4"]["star_crossprod_symmetric"] = bool(np.array_equal(cp4, cp4.T))
        del rn
    del nm, g
    torch.cuda.empty_cache()
    # ---- c5: GNMF r=5, Zipf(1.2) FK (S 5M×10, R 50k×40 U[0,1))
    g = W.generate("c5")
    nm = _build_gpu(fb, g, dev)
    rr, seed = g["r"], g["gnmf_seed"]
    fb.gnmf(nm, fb.TrainConfig(iterations=2, r=rr, rng_seed=seed))  # warm: workspaces, sorted order, attributes
    per, res = _loop_ms_per_iter(lambda it: fb.gnmf(nm, fb.TrainConfig(iterations=it, r=rr, rng_seed=seed)))
    out["c5_gnmf"] = {"iter_per_s": round(1 / per, 1), "ms_per_iter": round(1e3 * per, 3),
                      "s_total_20_iters": round(res.wall_time_s, 4), "kept_r_rows": int(nm.r.shape[0]),
                      "timing": "per iteration = median over 3 trials of the 20-iteration loop's CUDA-event span / 20 "
                                "(ModelOutput.loop_ms); total = wall clock incl. the host RNG draw of W (5M×5, the "
                                "reference's default_rng call) and its upload"}
    if cpu:
        rn = ref.build(g)
        ref.prepare(rn)
        _, t1 = timed(lambda: ref.gnmf(rn, rr, 1, seed))
        (w_ref, h_ref, tr_ref), t20 = timed(lambda: ref.gnmf(rn, rr, g["iterations"], seed))
        out["c5_gnmf"]["cpu_ms_per_iter"] = round(1e3 * (t20 - t1) / (g["iterations"] - 1), 1)
        parity["c5"] = {"W": max_rel_deviation(res.factors[0], w_ref), "H": max_rel_deviation(res.factors[1], h_ref),
                        "objective": max_rel_deviation(res.objective, tr_ref)}
        del rn
    del nm, g
    torch.cuda.empty_cache()
    return out


def _to_host(t):
    return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


def _traffic_from_profile(op):
    """DRAM bytes per launch of the op's kernels from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        return t.get(op), t.get("_source")
    except Exception:
        return None, None


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU reference legs and parity")
    ap.add_argument("--no-extras", action="store_true", help="skip the c1/c3/c4/c5 secondary workloads")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this script under torchrun on 127.0.0.1
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
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

"""Calibrate the factorize-or-materialize thresholds on this GPU (costmodel.B200_THRESHOLDS).

For a grid of tuple ratios (n_S / n_R) and feature ratios (d_R / d_S) it times LMM (d_x = 1),
colSums and RMM (n_x = 1) on the factorized plan (the gather / scatter kernels over S, FK, R)
and on the materialized plan (the same kernels over T expanded once into HBM), median of CUDA-
event timings, and writes gpurun_out/dispatch_calibration.json.
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_07448_b200 as fb
from paper_1612_07448_b200.normmat import as_normalized

dev = torch.device("cuda", 0)


def t_ms(fn, reps=7):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))


n_s, d_s = 4_000_000, 16
rows = []
for tr in (1, 2, 4, 8, 16):
    for fr in (0.25, 0.5, 1, 2, 4):
        d_r, n_r = int(d_s * fr), n_s // tr
        g = torch.Generator(device=dev).manual_seed(tr * 100 + int(fr * 4))
        s = torch.randn(n_s, d_s, dtype=torch.float64, device=dev, generator=g)
        r = torch.randn(n_r, d_r, dtype=torch.float64, device=dev, generator=g)
        k = torch.randint(1, n_r + 1, (n_s,), device=dev, generator=g)
        nm = fb.build_pkfk(s, k, r)
        t = as_normalized(fb.materialize(nm))
        x = torch.randn(d_s + d_r, 1, dtype=torch.float64, device=dev)
        xr = torch.randn(1, n_s, dtype=torch.float64, device=dev)
        rec = {"tuple_ratio": tr, "feature_ratio": fr, "n_s": n_s, "d_s": d_s, "n_r": n_r, "d_r": d_r}
        for op, ff, fm in (("lmm", lambda: fb.lmm(nm, x), lambda: fb.lmm(t, x)),
                           ("colsums", lambda: fb.col_sums(nm), lambda: fb.col_sums(t)),
                           ("rmm", lambda: fb.rmm(xr, nm), lambda: fb.rmm(xr, t))):
            rec[op + "_fact_ms"] = round(t_ms(ff), 4)
            rec[op + "_mat_ms"] = round(t_ms(fm), 4)
        rows.append(rec)
        print(json.dumps(rec), flush=True)
        del nm, t, s, r, k
        torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"device": torch.cuda.get_device_name(0), "grid": rows}, open("gpurun_out/dispatch_calibration.json", "w"), indent=1)

"""Quick GPU timing of the c2 operator suite (development aid, not the bench)."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1612_07448_b200 as fb

n_s, d_s, n_r, d_r = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (20_000_000, 20, 1_000_000, 80)))
only = sys.argv[5].split(",") if len(sys.argv) > 5 else None
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 10
g = torch.Generator(device="cuda").manual_seed(0)
s = torch.randn(n_s, d_s, dtype=torch.float64, device="cuda", generator=g)
r = torch.randn(n_r, d_r, dtype=torch.float64, device="cuda", generator=g)
k = torch.randint(1, n_r + 1, (n_s,), device="cuda", generator=g)
t0 = time.time(); nm = fb.build_pkfk(s, k, r); torch.cuda.synchronize(); print("build s", time.time() - t0)
d = d_s + d_r
x1 = torch.randn(d, 1, dtype=torch.float64, device="cuda"); x16 = torch.randn(d, 16, dtype=torch.float64, device="cuda")
xr = torch.randn(1, n_s, dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
ops = {
    "lmm_x1": (lambda: fb.lmm(nm, x1), 8 * (n_s * d_s + n_r * d_r + d + n_s) + 4 * n_s),
    "lmm_x16": (lambda: fb.lmm(nm, x16), 8 * (n_s * d_s + n_r * d_r + 16 * d + 16 * n_s) + 4 * n_s),
    "rmm_x1": (lambda: fb.rmm(xr, nm), 8 * (n_s * d_s + n_r * d_r + n_s + d) + 4 * n_s),
    "row_sums": (lambda: fb.row_sums(nm), 8 * (n_s * d_s + n_r * d_r + n_s) + 4 * n_s),
    "col_sums": (lambda: fb.col_sums(nm), 8 * (n_s * d_s + n_r * d_r + d)),
}
res = {}
for name, (fn, nbytes) in ops.items():
    if only and name not in only: continue
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    res[name] = {"ms": round(ms, 4), "GBps": round(nbytes / ms / 1e6, 1), "frac": round(nbytes / ms / 1e6 / 6534.5, 3)}
print(json.dumps(res, indent=1))

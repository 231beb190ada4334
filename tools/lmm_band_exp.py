"""c2 LMM X100xDX with and without the FK-band layout (fb_lmm_banded), CUDA events, median of 10.

env: NR, DX, FB_LMM_BAND_MB (z bytes per band), FB_LMM_BAND_MIN_MB (0 = storage-order pass only).
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
g = torch.Generator(device="cuda").manual_seed(0)
n_s, n_r, dx = 20_000_000, int(os.environ.get("NR", "1000000")), int(os.environ.get("DX", "16"))
s = torch.randn(n_s, 20, dtype=torch.float64, device="cuda", generator=g)
r = torch.randn(n_r, 80, dtype=torch.float64, device="cuda", generator=g)
k = torch.randint(1, n_r + 1, (n_s,), device="cuda", generator=g)
nm = fb.build_pkfk(s, k, r)
x = torch.randn(100, dx, dtype=torch.float64, device="cuda", generator=g)
torch.cuda.synchronize()
t0 = time.perf_counter()
band = nm.band_layout(dx)
torch.cuda.synchronize()
build_ms = (time.perf_counter() - t0) * 1e3
for _ in range(3):
    fb.lmm(nm, x)
ts = []
for _ in range(10):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out = fb.lmm(nm, x); e.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(e))
ts.sort()
nb = 8 * (n_s * 20 + n_r * 80) + 4 * n_s + 8 * (100 * dx + n_s * dx)
nbands = nm._cache["band"][0].n_bands if band is not None else 0
print(f"NR={n_r} DX={dx} bands={nbands} build_ms={build_ms:.1f} ms={ts[5]:.4f} GBps={nb / ts[5] / 1e6:.0f} "
      f"frac={nb / ts[5] / 1e6 / 6542.1:.3f}", flush=True)

"""c2 LMM X100xDX op time (CUDA events, median of 10) under env knobs, for S-pass decomposition.

env: NR (R rows, default 1M), DX (default 16), KEYS = uniform | bandB (keys grouped into B FK
bands in storage order: emulates a band-ordered S), FB_LMM_DEBUG (1 skip stores, 2 no gathers).
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
g = torch.Generator(device="cuda").manual_seed(0)
n_s, n_r, dx = 20_000_000, int(os.environ.get("NR", "1000000")), int(os.environ.get("DX", "16"))
s = torch.randn(n_s, 20, dtype=torch.float64, device="cuda", generator=g)
r = torch.randn(n_r, 80, dtype=torch.float64, device="cuda", generator=g)
mode = os.environ.get("KEYS", "uniform")
if mode.startswith("band"):
    b = int(mode[4:])
    band = torch.arange(n_s, device="cuda") * b // n_s
    k = band * (n_r // b) + torch.randint(0, n_r // b, (n_s,), device="cuda", generator=g) + 1
else:
    k = torch.randint(1, n_r + 1, (n_s,), device="cuda", generator=g)
nm = fb.build_pkfk(s, k, r)
x = torch.randn(100, dx, dtype=torch.float64, device="cuda", generator=g)
for _ in range(3):
    fb.lmm(nm, x)
ts = []
for _ in range(10):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out = fb.lmm(nm, x); e.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(e))
ts.sort()
nb = 8 * (n_s * 20 + n_r * 80) + 4 * n_s + 8 * (100 * dx + n_s * dx)
print(f"NR={n_r} DX={dx} KEYS={mode} DEBUG={os.environ.get('FB_LMM_DEBUG', '0')} "
      f"ms={ts[5]:.4f} GBps={nb / ts[5] / 1e6:.0f}", flush=True)

"""Time c2 LMM X100x1 / X100x16 with CUDA events (median of 10). usage: python tools/time_lmm.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
g = torch.Generator(device="cuda").manual_seed(0)
n_s, n_r = 20_000_000, int(os.environ.get("NR", "1000000"))
s = torch.randn(n_s, 20, dtype=torch.float64, device="cuda", generator=g)
r = torch.randn(n_r, 80, dtype=torch.float64, device="cuda", generator=g)
k = torch.randint(1, n_r + 1, (n_s,), device="cuda", generator=g)
nm = fb.build_pkfk(s, k, r)
res = {}
for dx in (1, 16):
    x = torch.randn(100, dx, dtype=torch.float64, device="cuda", generator=g)
    ref = fb.lmm(nm, x)
    for _ in range(3):
        fb.lmm(nm, x)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); out = fb.lmm(nm, x); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    nb = 8 * (n_s * 20 + n_r * 80) + 4 * n_s + 8 * (100 * dx + n_s * dx)
    res[dx] = (round(ts[5], 4), round(nb / ts[5] / 1e6 / 6532.5, 3), float((out - ref).abs().max()))
print(os.environ.get("FB_ZSTORE_FRAC", "-"), os.environ.get("FB_ZGATHER_FRAC", "-"), res, flush=True)

"""Time the c2 RMM (X1x20M · T) with CUDA events. usage: python tools/time_rmm.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
g = torch.Generator(device="cuda").manual_seed(0)
n_s, n_r = 20_000_000, 1_000_000
s = torch.randn(n_s, 20, dtype=torch.float64, device="cuda", generator=g)
r = torch.randn(n_r, 80, dtype=torch.float64, device="cuda", generator=g)
k = torch.randint(1, n_r + 1, (n_s,), device="cuda", generator=g)
nm = fb.build_pkfk(s, k, r)
xr = torch.randn(1, n_s, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = fb.rmm(xr, nm)
for _ in range(3):
    fb.rmm(xr, nm)
ts = []
for _ in range(20):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out = fb.rmm(xr, nm); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(os.environ.get("FB_SEG_CTAS", "8"), "median ms", round(ts[len(ts) // 2], 4), "min", round(ts[0], 4),
      "maxdiff", float((out - ref).abs().max()))
